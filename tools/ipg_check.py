"""Device vs host iP-GVIMP pieces: errors and timings (debug aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2411_03416_b200 as P
from conftest import golden, rel_err

g = golden("slr")
for N, dt in [(20, 0.25), (50, 0.1), (100, 0.05), (300, 1.0 / 60)]:
    x0, goal = np.zeros(6), np.array([10.0, 5.0, 0, 0, 0, 0])
    a = np.linspace(0, 1, N + 1)[:, None]
    nom = P.NominalTrajectory(means=(1 - a) * x0 + a * goal, covs=np.repeat(0.05 * np.eye(6)[None], N + 1, 0))
    rule = P.smolyak_rule(3, 6)
    t0 = time.perf_counter(); h = P.slr_linearize(P.planar_quadrotor(), nom, dt, rule); th = time.perf_counter() - t0
    P.slr_linearize(P.planar_quadrotor(), nom, dt, rule, device=True)
    t0 = time.perf_counter(); d = P.slr_linearize(P.planar_quadrotor(), nom, dt, rule, device=True); td = time.perf_counter() - t0
    ea = rel_err(np.stack([s.A for s in d.steps]), np.stack([s.A for s in h.steps]))
    msg = f"N={N} slr host {th*1e3:.1f} ms dev {td*1e3:.2f} ms errA {ea:.1e}"
    try:
        t0 = time.perf_counter(); ph = P.assemble_prior(h, x0, goal, 0.5, 1e-3); tph = time.perf_counter() - t0
        t0 = time.perf_counter(); pd = P.assemble_prior_device(h, x0, goal, 0.5, 1e-3); tpd = time.perf_counter() - t0
        msg += (f" | prior host {tph*1e3:.1f} ms dev {tpd*1e3:.2f} ms phi {rel_err(np.stack(pd.phis), np.stack(ph.phis)):.1e}"
                f" gram {rel_err(np.stack(pd.grammians), np.stack(ph.grammians)):.1e} diag {rel_err(pd.prec.diag_stack, ph.prec.diag_stack):.1e}"
                f" info {rel_err(pd.info, ph.info):.1e} mean {rel_err(pd.mean, ph.mean):.1e}")
    except Exception as e:
        msg += f" | prior: {type(e).__name__}: {e}"
    print(msg)
