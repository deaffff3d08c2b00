"""Per-kernel device time of one C2 / C1 planner iteration (single plan) on
the engine (gvp_engine_step_profiled_ex), after a few warm iterations."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_2411_03416_b200 as P


def run(tag, N, k_q, sdf, model, goal, T):
    sys_ltv = P.point_robot_lti(2)(N, T / N)
    pr = P.assemble_prior(sys_ltv, np.zeros(4), goal, 1.0, 1e-3)
    cfg = P.OptimizerConfig(k_q=k_q, kl_bound=10.0, beta_max=0.5, max_iters=60)
    K = N + 1
    eng = P.PlanBatch(1, K, 4, sdf, model, P.smolyak_rule(k_q, 4), cfg, shared_prior=True)
    init = np.linspace(0, 1, K)[None, :, None] * goal[None, None, :]
    eng.load(pr.prec.diag_stack, pr.prec.off_stack, pr.info.reshape(1, K, 4), pr.mean.reshape(1, K, 4), init)
    eng.step(5, sync=True)
    ms = np.zeros(6)
    for _ in range(20):
        ms += eng.step_profiled_ex(1)
    out = dict(zip(eng.PROFILE_BUCKETS, (ms / 20).round(4).tolist()))
    out["lanes"] = eng.lanes()
    print(tag, json.dumps(out))
    eng.close()


run("C2", 500, 5, bench.c2_map(P), P.CollisionModel(0.2, 8.0), np.array([10.0, 10.0, 0, 0]), 10.0)
sdf1 = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], [[-2, 4], [-2, 4]], 0.05)
run("C1", 50, 3, sdf1, P.CollisionModel(0.2, 8.0), np.array([2.0, 1.5, 0, 0]), 3.0)
