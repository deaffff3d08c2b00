"""C4 at N = 300 (GPU-only throughput config; the reference
cannot produce a plan there, §8c). Runs iP-GVIMP with SLR + prior assembly on
the device and reports where/how it fails or its timings, for several T."""
import json
import os
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03416_b200 as P  # noqa: E402


def run(T, q_c=0.5, sigma_b=1e-3, N=300, max_iters=100, max_outer=3, robust=False):
    sdf = P.rasterize([P.sdf.Disc(center=np.array([5.0, 4.5]), radius=0.8)], bounds=[[-5, 15], [-5, 10]],
                      cell_size=0.05)
    env = P.Environment(sdf=sdf, model=P.CollisionModel(radius_eps=1.5, sigma_obs=6.0))
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0, temp_high=5.0, max_iters=max_iters)
    t0 = time.perf_counter()
    out = {"T": T, "N": N, "q_c": q_c, "sigma_b": sigma_b, "robust": robust}
    try:
        kw = {"robust": True} if robust else {}
        res, log = P.run_ipgvimp(P.planar_quadrotor(), env, cfg, P.OuterConfig(max_outer=max_outer), np.zeros(6),
                                 np.array([10.0, 5.0, 0, 0, 0, 0]), dt=T / N, num_steps=N, q_c=q_c,
                                 sigma_b=sigma_b, device=True, **kw)
        out.update(ok=True, ms=(time.perf_counter() - t0) * 1e3, inner_iterations=res.iterations,
                   norm_diff=[r["norm_diff"] for r in log],
                   final_total=res.records[-1]["total_cost"], final_collision=res.records[-1]["collision_cost"])
    except Exception as exc:  # report, this is an exploration
        out.update(ok=False, ms=(time.perf_counter() - t0) * 1e3, error=repr(exc),
                   cause=repr(exc.__cause__) if exc.__cause__ else None,
                   tb=traceback.format_exc()[-600:])
    return out


if __name__ == "__main__":
    for robust in (False, True):
        for T in (5.0, 15.0, 30.0):
            print(json.dumps(run(T, robust=robust)), flush=True)
