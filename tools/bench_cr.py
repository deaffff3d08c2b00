"""Latency of gbp_marginals (cyclic reduction) for one chain vs the oracle (debug/measurement aid)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import gvp_oracle as O
import paper_2411_03416_b200 as P
from conftest import rel_err

for N in (50, 500, 1000):
    sys_ltv = P.point_robot_lti(2)(N, 10.0 / N)
    A, a, B = O.point_robot_triples(2)
    pr = O.assemble_prior([A] * (N + 1), [a] * (N + 1), [B] * (N + 1), 10.0 / N, np.zeros(4), np.array([10.0, 10, 0, 0]), 1.0, 1e-3)
    d, o = pr["diag"] * 10.0, pr["off"] * 10.0
    prec = P.BlockTridiagonalMatrix(d, o)
    m = P.gbp_marginals(prec)
    t0 = time.perf_counter()
    for _ in range(20):
        m = P.gbp_marginals(prec)
    dt = (time.perf_counter() - t0) / 20
    cv, cr = O.marginals(d, o)
    print(f"N={N}: gbp_marginals {dt*1e3:.3f} ms/call (host<->device incl.); rel covs {rel_err(np.stack(m.covs), cv):.2e} "
          f"crosses {rel_err(np.stack(m.crosses), cr):.2e}")
