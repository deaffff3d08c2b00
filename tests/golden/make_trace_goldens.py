"""Per-probe reference traces for the long-horizon parity tests (C5 sample, C2).

Run in the dev container (oracle/_ref built by oracle/build_ref.sh):

    python tests/golden/make_trace_goldens.py            # c5_sample.npz + c2_trace.npz (~15 min, 8 cores)

Every number written is produced by the UNMODIFIED reference package
(`gvplan` from oracle/_ref) or, for the arbiters, by LAPACK on the
reference's own matrices:

* the reference's run_pgvimp on each plan, with every probe of every
  select_step_size logged as (beta, spd, KL) (optimizer.py:188-231);
* per probe, KL_dense: the same KL(next || cur) from banded Cholesky factors
  of the reference's own candidate and current precisions (refkl.py — a sum of
  squares, no trace_product cancellation), the arbiter for probes where the
  reference's KL sits within its own error of the bound;
* per near-bound probe (|KL - eps| < 1e-2), KL_np: the reference's KL with the
  gradients of its pure-numpy kernel backend (_kernels_py) at the same state
  and beta — the reference's own backend spread;
* per iteration, the record the numpy backend would have produced from the
  same state at the same beta (record spread), and the iterate's mean at every
  50th knot.

C5 sample: plans 0, 128, ..., 3968 of bench.c5_goals(4096) on the bench's own
problem construction (shared prior precision of the base goal, per-plan info
= base info + anchor dg at the last knot, bench.build_problem), 10
iterations each. C2: SURVEY §8d C2 (N = 500, k_q = 5), 4 iterations.
"""

from __future__ import annotations

import dataclasses
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(1, HERE)

import gvplan  # noqa: E402
from gvplan import optimizer as ro  # noqa: E402
from gvplan import _kernels_py  # noqa: E402
from gvplan.factors import assemble_joint_gradients, evaluate_all_factors, interior_collision_maps  # noqa: E402
from gvplan.sdf import Box  # noqa: E402

from refkl import kl_banded  # noqa: E402

assert gvplan.HAVE_EXTENSION or os.environ.get("GVPLAN_PURE_PYTHON"), \
    "build the reference extension first (oracle/build_ref.sh)"

_COST_BREAKDOWN = ro.cost_breakdown  # unwrapped (the runs below wrap the module attribute)

KEYS = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
        "mean_shift"]
NEAR = 1e-2          # |KL - eps| below which the numpy-backend KL is also computed
KNOT_STRIDE = 50     # iterate means stored at knots 0, 50, 100, ...
C5_SAMPLE = np.arange(0, 4096, 128)
C5_ITERS = 10
SEED = 2411_03416


def c2_map():
    return gvplan.rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                             Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                            bounds=[[-2, 12], [-2, 12]], cell_size=0.05)


def c5_goals(total):  # bench.c5_goals
    rng = np.random.default_rng(SEED)
    g = np.tile(np.array([10.0, 10.0, 0.0, 0.0]), (total, 1))
    g[:, :2] += rng.uniform(-0.5, 0.5, size=(total, 2))
    return g


def c5_base_prior():
    sys_ltv = gvplan.point_robot_lti(2)(1000, 10.0 / 1000)
    return sys_ltv, gvplan.assemble_prior(sys_ltv, np.zeros(4), np.array([10.0, 10.0, 0.0, 0.0]), 1.0, 1e-3)


def c5_plan_prior(base, goal):
    """bench.build_problem for one plan: shared precision, info with the goal
    anchor moved (anchor = I / sigma_b^2 is diagonal: the product is exact),
    the anchored mean from the reference's own gbp_mean_solve."""
    K, n = base.nsteps + 1, base.n
    anchor = np.eye(n) / 1e-3 ** 2
    info = base.info.reshape(K, n).copy()
    info[-1] += (goal - base.goal) @ anchor.T
    info = info.reshape(-1)
    return dataclasses.replace(base, info=info, mean=gvplan.gbp_mean_solve(base.prec, info), goal=goal)


def trace_run(sys_ltv, prior, env, cfg):
    """run_pgvimp with every select_step_size instrumented (see module doc)."""
    rule = gvplan.smolyak_rule(cfg.k_q, prior.n)
    orig_sel = ro.select_step_size
    iters = []

    def sel(cur, prior_, g_mu, g_sigma, cfg_, temp):
        log = []
        o_prox, o_kl, o_marg = ro.proximal_update, ro.kl_joint, ro.gbp_marginals
        st = {}

        def prox(c, p, gm, gs, beta, t):
            st["beta"] = beta
            return o_prox(c, p, gm, gs, beta, t)

        def marg(prec):
            try:
                return o_marg(prec)
            except Exception:
                log.append([st["beta"], 0.0, np.inf, None])
                raise

        def kl(nxt, c, m=None):
            v = o_kl(nxt, c, m)
            log.append([st["beta"], 1.0, v, nxt])
            return v

        ro.proximal_update, ro.kl_joint, ro.gbp_marginals = prox, kl, marg
        try:
            out = orig_sel(cur, prior_, g_mu, g_sigma, cfg_, temp)
        finally:
            ro.proximal_update, ro.kl_joint, ro.gbp_marginals = o_prox, o_kl, o_marg
        nb, n = cur.prec.nblocks, cur.prec.block_size
        m_cur = o_marg(cur.prec)
        fv_np = evaluate_all_factors(cur.mean, cur.prec, env.sdf, env.model, rule, marginals=m_cur,
                                     backend=_kernels_py)
        gm_np, gs_np = assemble_joint_gradients(fv_np, interior_collision_maps(nb), nb, n)
        cd, co = np.stack(cur.prec.diag), np.stack(cur.prec.off)
        rows = []
        for beta, spd, k, nxt in log:
            if not spd:
                rows.append((beta, 0.0, np.inf, np.nan, np.nan))
                continue
            kd = kl_banded(nxt.mean, np.stack(nxt.prec.diag), np.stack(nxt.prec.off), cur.mean, cd, co)
            knp = np.nan
            if abs(k - cfg_.kl_bound) < NEAR:
                c2 = o_prox(cur, prior_, gm_np, gs_np, beta, temp)
                try:
                    knp = o_kl(c2, cur, o_marg(c2.prec))
                except Exception:
                    knp = np.inf
            rows.append((beta, 1.0, k, knp, kd))
        # the numpy backend's record at the same beta from the same state
        nxt_np = o_prox(cur, prior_, gm_np, gs_np, out.beta, temp)
        m_np = o_marg(nxt_np.prec)
        f_np = evaluate_all_factors(nxt_np.mean, nxt_np.prec, env.sdf, env.model, rule, marginals=m_np,
                                    backend=_kernels_py)
        c_np = _COST_BREAKDOWN(nxt_np, prior_, temp, marginals=m_np, factor_values=f_np)
        rec_np = [out.beta, temp, c_np.prior_cost, c_np.collision_cost, c_np.entropy_cost, c_np.total,
                  o_kl(nxt_np, cur, m_np), float(np.linalg.norm(nxt_np.mean - cur.mean))]
        iters.append({"probes": np.array(rows), "rec_np": np.array(rec_np),
                      "mean_np": nxt_np.mean.reshape(nb, n)[::KNOT_STRIDE].copy(),
                      "mean_np_full": nxt_np.mean.reshape(nb, n).copy()})
        return out

    ro.select_step_size = sel
    try:
        t0 = time.time()
        res = gvplan.run_pgvimp(sys_ltv, env, cfg, prior.x0, prior.goal, 1.0, 1e-3, prior=prior)
        dt = time.time() - t0
    finally:
        ro.select_step_size = orig_sel
    return res, iters, dt


def pack(res, iters, K, n, means):
    """Fixed-shape arrays: probes padded to 40 rows with NaN."""
    it = len(iters)
    pr = np.full((it, 40, 5), np.nan)
    cnt = np.zeros(it, dtype=np.int32)
    for k, d in enumerate(iters):
        p = d["probes"]
        pr[k, :len(p)] = p
        cnt[k] = len(p)
    return {"probes": pr, "nprobes": cnt,
            "records": np.array([[r[k] for k in KEYS] for r in res.records]),
            "records_np": np.stack([d["rec_np"] for d in iters]),
            "means": np.stack(means),  # (it, K // stride + 1, n) after each iteration
            "means_np": np.stack([d["mean_np"] for d in iters]),
            "final_mean": res.final.mean.reshape(K, n),
            "final_mean_np": iters[-1]["mean_np_full"]}


def c5_worker(b):
    sys_ltv, base = c5_base_prior()
    goal = c5_goals(4096)[b]
    prior = c5_plan_prior(base, goal)
    env = ro.Environment(sdf=c2_map(), model=gvplan.CollisionModel(0.2, 8.0))
    cfg = gvplan.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=C5_ITERS, threads=1)
    means = []
    orig_step = ro.select_step_size

    # the iterate after each iteration: wrap cost_breakdown (called once per iteration with nxt)
    o_cost = ro.cost_breakdown

    def cost(nxt, *a, **kw):
        means.append(nxt.mean.reshape(1001, 4)[::KNOT_STRIDE].copy())
        return o_cost(nxt, *a, **kw)

    ro.cost_breakdown = cost
    try:
        res, iters, dt = trace_run(sys_ltv, prior, env, cfg)
    finally:
        ro.cost_breakdown = o_cost
        ro.select_step_size = orig_step
    out = pack(res, iters, 1001, 4, means)
    out["pmean"] = prior.mean.reshape(1001, 4)
    print(f"plan {b}: {len(res.records)} iterations in {dt:.1f} s", flush=True)
    return b, out


def c5_sample(procs=8):
    import multiprocessing as mp

    sys_ltv, base = c5_base_prior()
    with mp.get_context("fork").Pool(procs) as pool:
        outs = dict(pool.map(c5_worker, list(C5_SAMPLE)))
    K, n = 1001, 4
    data = {"plans": C5_SAMPLE.astype(np.int32), "kdiag": np.stack(base.prec.diag),
            "koff": np.stack(base.prec.off), "info0": base.info.reshape(K, n), "goal0": base.goal,
            "knot_stride": np.int32(KNOT_STRIDE)}
    for key in outs[C5_SAMPLE[0]]:
        data[key] = np.stack([outs[b][key] for b in C5_SAMPLE])
    np.savez_compressed(os.path.join(HERE, "c5_sample.npz"), **data)


def c2_trace():
    sys_ltv = gvplan.point_robot_lti(2)(500, 10.0 / 500)
    prior = gvplan.assemble_prior(sys_ltv, np.zeros(4), np.array([10.0, 10.0, 0, 0]), 1.0, 1e-3)
    env = ro.Environment(sdf=c2_map(), model=gvplan.CollisionModel(0.2, 8.0))
    cfg = gvplan.OptimizerConfig(k_q=5, kl_bound=10.0, beta_max=0.5, max_iters=4, threads=1)
    means = []
    o_cost = ro.cost_breakdown

    def cost(nxt, *a, **kw):
        means.append(nxt.mean.reshape(501, 4)[::KNOT_STRIDE].copy())
        return o_cost(nxt, *a, **kw)

    ro.cost_breakdown = cost
    try:
        res, iters, dt = trace_run(sys_ltv, prior, env, cfg)
    finally:
        ro.cost_breakdown = o_cost
    out = pack(res, iters, 501, 4, means)
    out.update(kdiag=np.stack(prior.prec.diag), koff=np.stack(prior.prec.off), info=prior.info.reshape(501, 4),
               pmean=prior.mean.reshape(501, 4), knot_stride=np.int32(KNOT_STRIDE))
    np.savez_compressed(os.path.join(HERE, "c2_trace.npz"), **out)
    print(f"c2: {len(res.records)} iterations in {dt:.1f} s", flush=True)


def c4_run():
    """SURVEY §8d C4 parity variant: planar quadrotor via iP-GVIMP (slr.py:95-149),
    N = 50, dt = 0.1, q_c = 0.5, sigma_b = 1e-3, Disc((5, 4.5), 0.8), r + eps = 1.5,
    sigma = 6, OptimizerConfig(k_q=3, kl_bound=10, temp_low=1, temp_high=5,
    max_iters=100), OuterConfig(max_outer=3). Returns arrays of one run with the
    backend selected at import (Cython, or numpy under GVPLAN_PURE_PYTHON=1)."""
    from gvplan import OuterConfig, planar_quadrotor, run_ipgvimp
    from gvplan.sdf import Disc

    sdf = gvplan.rasterize([Disc(center=np.array([5.0, 4.5]), radius=0.8)], bounds=[[-5, 15], [-5, 10]],
                           cell_size=0.05)
    env = ro.Environment(sdf=sdf, model=gvplan.CollisionModel(radius_eps=1.5, sigma_obs=6.0))
    cfg = gvplan.OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0, temp_high=5.0, max_iters=100, threads=1)
    import gvplan.slr as rslr

    inner = []  # records of every inner run (one per outer iteration)
    o_run = rslr.run_pgvimp

    def run(*a, **kw):
        r = o_run(*a, **kw)
        inner.append(np.array([[rec[k] for k in KEYS] for rec in r.records]))
        return r

    rslr.run_pgvimp = run
    try:
        t0 = time.time()
        res, log = run_ipgvimp(planar_quadrotor(), env, cfg, OuterConfig(max_outer=3), np.zeros(6),
                               np.array([10.0, 5.0, 0, 0, 0, 0]), dt=0.1, num_steps=50, q_c=0.5, sigma_b=1e-3)
        dt = time.time() - t0
    finally:
        rslr.run_pgvimp = o_run
    out = {"records": np.array([[r[k] for k in KEYS] for r in res.records]),
           "final_mean": res.final.mean.reshape(51, 6),
           "final_covs": np.stack(res.marginals.covs),
           "iterations": np.int32(res.iterations), "converged": np.int32(res.converged),
           "seconds": np.float64(dt),
           "inner_records": np.stack([np.pad(x, ((0, 100 - len(x)), (0, 0)), constant_values=np.nan)
                                      for x in inner])}
    for key in log[0]:
        vals = [r[key] for r in log]
        try:
            out["outer_" + key] = np.array(vals, dtype=float)
        except (TypeError, ValueError):
            pass
    return out


def c4():
    """The C4 run with the reference's Cython backend and, in a fresh
    interpreter, with its pure-numpy backend: the second is the reference's
    own spread on this ill-conditioned run (the parity tolerance scale)."""
    import pickle
    import subprocess

    a = c4_run()
    env = dict(os.environ, GVPLAN_PURE_PYTHON="1")
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "c4py"], capture_output=True, env=env,
                         timeout=7200)
    assert out.returncode == 0, out.stderr[-2000:]
    b = pickle.loads(out.stdout)
    data = dict(a)
    data.update({"py_" + k: v for k, v in b.items()})
    np.savez_compressed(os.path.join(HERE, "c4_parity.npz"), **data)
    print(f"c4: {a['iterations']} inner iterations, {a['seconds']:.1f} s (numpy backend {b['seconds']:.1f} s)")


C4_STEPS = (1, 2, 50, 100)  # inner iterations (1-based) whose full state is stored per outer iteration


def c4_stages():
    """C4 parity variant stage by stage (the full run is chaotic: the reference's
    own two backends part after 2 inner iterations). Per outer iteration of the
    reference's run_ipgvimp: the nominal it linearises about, its SLR output
    (A, a per step), its assembled prior, and at inner iterations C4_STEPS the
    full state (mean, precision, temperature), the accepted beta, the record,
    the probe log with KL_dense per probe, the next mean and the exact solution
    of the reference's own mean system (oracle/ref_bench.exact_solve)."""
    import gvplan.slr as rslr
    from gvplan import OuterConfig, planar_quadrotor, run_ipgvimp
    from gvplan.sdf import Disc

    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import ref_bench

    sdf = gvplan.rasterize([Disc(center=np.array([5.0, 4.5]), radius=0.8)], bounds=[[-5, 15], [-5, 10]],
                           cell_size=0.05)
    env = ro.Environment(sdf=sdf, model=gvplan.CollisionModel(radius_eps=1.5, sigma_obs=6.0))
    cfg = gvplan.OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0, temp_high=5.0, max_iters=100, threads=1)
    st = {"outer": -1, "iter": 0}
    out = {"nominal_means": [], "nominal_covs": [], "lin_A": [], "lin_a": [], "prior_diag": [], "prior_off": [],
           "prior_info": [], "prior_mean": [], "steps": []}
    o_lin, o_prior, o_sel, o_solve = rslr.slr_linearize, ro.assemble_prior, ro.select_step_size, ro.gbp_mean_solve

    def lin(sys_nl, nominal, dt, rule):
        ltv = o_lin(sys_nl, nominal, dt, rule)
        st["outer"] += 1
        st["iter"] = 0
        out["nominal_means"].append(np.array(nominal.means))
        out["nominal_covs"].append(np.array(nominal.covs))
        out["lin_A"].append(np.stack([x.A for x in ltv.steps]))
        out["lin_a"].append(np.stack([x.a for x in ltv.steps]))
        return ltv

    def prior_fn(*a, **kw):
        pr = o_prior(*a, **kw)
        out["prior_diag"].append(np.stack(pr.prec.diag))
        out["prior_off"].append(np.stack(pr.prec.off))
        out["prior_info"].append(pr.info.copy())
        out["prior_mean"].append(pr.mean.copy())
        return pr

    def sel(cur, prior_, g_mu, g_sigma, cfg_, temp):
        st["iter"] += 1
        if st["iter"] not in C4_STEPS:
            return o_sel(cur, prior_, g_mu, g_sigma, cfg_, temp)
        log, cap = [], []
        o_prox, o_kl, o_marg = ro.proximal_update, ro.kl_joint, ro.gbp_marginals
        bs = {}

        def prox(c, p, gm, gs, beta, t):
            bs["beta"] = beta
            return o_prox(c, p, gm, gs, beta, t)

        def marg(prec):
            try:
                return o_marg(prec)
            except Exception:
                log.append([bs["beta"], 0.0, np.inf, None])
                raise

        def kl(nxt, c, m=None):
            v = o_kl(nxt, c, m)
            log.append([bs["beta"], 1.0, v, nxt])
            return v

        def solve(S, rhs):
            x = o_solve(S, rhs)
            cap.append((S, np.array(rhs), x))
            return x

        ro.proximal_update, ro.kl_joint, ro.gbp_marginals, ro.gbp_mean_solve = prox, kl, marg, solve
        try:
            res = o_sel(cur, prior_, g_mu, g_sigma, cfg_, temp)
        finally:
            ro.proximal_update, ro.kl_joint, ro.gbp_marginals, ro.gbp_mean_solve = o_prox, o_kl, o_marg, o_solve
        cd, co = np.stack(cur.prec.diag), np.stack(cur.prec.off)
        rows = []
        for beta, spd, k, nxt in log:
            kd = np.nan if not spd else kl_banded(nxt.mean, np.stack(nxt.prec.diag), np.stack(nxt.prec.off),
                                                  cur.mean, cd, co)
            rows.append((beta, spd, k, np.nan, kd))
        S, rhs, x = next(v for v in cap if np.array_equal(v[2], res.next_state.mean))
        nb, n = cur.prec.nblocks, cur.prec.block_size
        out["steps"].append({"outer": st["outer"], "iter": st["iter"], "temp": temp, "beta": res.beta,
                             "mean": cur.mean.reshape(nb, n).copy(), "diag": cd, "off": co,
                             "probes": np.array(rows), "next_mean": res.next_state.mean.reshape(nb, n).copy(),
                             "next_exact": ref_bench.exact_solve(S, rhs, x).reshape(nb, n), "kl": res.kl})
        return res

    rslr.slr_linearize, ro.assemble_prior, ro.select_step_size = lin, prior_fn, sel
    try:
        res, log = run_ipgvimp(planar_quadrotor(), env, cfg, OuterConfig(max_outer=3), np.zeros(6),
                               np.array([10.0, 5.0, 0, 0, 0, 0]), dt=0.1, num_steps=50, q_c=0.5, sigma_b=1e-3)
    finally:
        rslr.slr_linearize, ro.assemble_prior, ro.select_step_size = o_lin, o_prior, o_sel
    data = {k: np.stack(v) for k, v in out.items() if k != "steps"}
    stp = out["steps"]
    data["step_outer"] = np.array([d["outer"] for d in stp], dtype=np.int32)
    data["step_iter"] = np.array([d["iter"] for d in stp], dtype=np.int32)
    for key in ("temp", "beta", "kl"):
        data["step_" + key] = np.array([d[key] for d in stp])
    for key in ("mean", "diag", "off", "next_mean", "next_exact"):
        data["step_" + key] = np.stack([d[key] for d in stp])
    pr = np.full((len(stp), 40, 5), np.nan)
    npb = np.zeros(len(stp), dtype=np.int32)
    for i, d in enumerate(stp):
        pr[i, :len(d["probes"])] = d["probes"]
        npb[i] = len(d["probes"])
    data["step_probes"], data["step_nprobes"] = pr, npb
    np.savez_compressed(os.path.join(HERE, "c4_stages.npz"), **data)
    print("c4 stages:", len(stp), "stored steps, outer norm diffs", [r["norm_diff"] for r in log])


def sqrt_cases():
    """gaussian_sqrt's fallbacks (quadrature.py:164-181) inside the factor stage:
    C1 scene (N = 50, k_q = 3) at its initial state, with knot covariances made
    indefinite by eigenvalue shifts: -5e-11 (Cholesky fails, the 1e-10 jitter
    retry succeeds) on knots 9-12 (clouds on the obstacle), and -1e-6 on knot 20
    (eigh root with a clipped eigenvalue: the reference's _moment_gradients
    np.linalg.solve raises LinAlgError)."""
    from gvplan.factors import evaluate_all_factors
    from gvplan.gbp import ChainMarginals
    from gvplan.sdf import Disc

    sdf = gvplan.rasterize([Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                           cell_size=0.05)
    model = gvplan.CollisionModel(0.2, 8.0)
    sys_ltv = gvplan.point_robot_lti(2)(50, 3.0 / 50)
    prior = gvplan.assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
    cfg = gvplan.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5)
    cur = ro.initial_state(prior, cfg)
    marg = gvplan.gbp_marginals(cur.prec)
    covs = [c.copy() for c in marg.covs]

    def shift(c, lam):
        w, v = np.linalg.eigh(c)
        w[0] = lam
        return 0.5 * ((v * w) @ v.T + ((v * w) @ v.T).T)

    for k in (9, 10, 11, 12):
        covs[k] = shift(covs[k], -5e-11)
    jit = ChainMarginals(covs=covs, crosses=list(marg.crosses))
    for k in (9, 10, 11, 12):  # the intended branch is the jitter retry
        try:
            np.linalg.cholesky(covs[k])
            raise AssertionError("cholesky should fail")
        except np.linalg.LinAlgError:
            np.linalg.cholesky(covs[k] + 1e-10 * np.eye(4))
    rule = gvplan.smolyak_rule(3, 4)
    fv = evaluate_all_factors(cur.mean, cur.prec, sdf, model, rule, marginals=jit)
    fp = evaluate_all_factors(cur.mean, cur.prec, sdf, model, rule, marginals=jit, backend=_kernels_py)
    out = {"mean": cur.mean.reshape(51, 4), "covs_jitter": np.stack(covs),
           "e_psi": np.array([f.e_psi for f in fv]), "g_mu": np.stack([f.g_mu for f in fv]),
           "g_sigma": np.stack([f.g_sigma for f in fv]),
           # the reference's numpy kernel backend on the same inputs: its own spread
           "py_e_psi": np.array([f.e_psi for f in fp]), "py_g_mu": np.stack([f.g_mu for f in fp]),
           "py_g_sigma": np.stack([f.g_sigma for f in fp])}
    covs2 = list(covs)
    covs2[20] = shift(covs2[20], -1e-6)
    try:
        evaluate_all_factors(cur.mean, cur.prec, sdf, model, rule,
                             marginals=ChainMarginals(covs=covs2, crosses=list(marg.crosses)))
        raised = ""
    except np.linalg.LinAlgError as exc:
        raised = type(exc).__name__ + ": " + str(exc)
    out["covs_eigh"] = np.stack(covs2)
    out["eigh_raises"] = np.array(raised)
    assert raised, "the eigh case should raise in the reference"
    np.savez_compressed(os.path.join(HERE, "sqrt_cases.npz"), **out)
    print("sqrt cases:", raised)


if __name__ == "__main__":
    what = sys.argv[1:] or ["c2", "c5", "c4", "c4s", "sqrt"]
    if "c4s" in what:
        c4_stages()
    if "sqrt" in what:
        sqrt_cases()
    if "c4py" in what:
        import pickle

        sys.stdout.buffer.write(pickle.dumps(c4_run()))
        sys.exit(0)
    if "c2" in what:
        c2_trace()
    if "c5" in what:
        c5_sample()
    if "c4" in what:
        c4()
