"""Per-kernel device times of the C1 plan (B=1) on the engine (debugging aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03416_b200 as P

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 0
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sdf = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
sys_ltv = P.point_robot_lti(2)(50, 3.0 / 50)
cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=iters + 1)
pr = P.assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
eng = P.PlanBatch(1, 51, 4, sdf, P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4), cfg, spec_lanes=lanes)
eng.load(pr.prec.diag_stack, pr.prec.off_stack, pr.info.reshape(1, 51, 4), pr.mean.reshape(1, 51, 4),
         np.linspace(0, 1, 51)[None, :, None] * np.array([2.0, 1.5, 0, 0])[None, None, :])
eng.step(1, sync=True)
ms = eng.step_profiled(iters)
t0 = time.perf_counter(); eng.load(pr.prec.diag_stack, pr.prec.off_stack, pr.info.reshape(1, 51, 4), pr.mean.reshape(1, 51, 4),
         np.linspace(0, 1, 51)[None, :, None] * np.array([2.0, 1.5, 0, 0])[None, None, :]); eng.step(iters, sync=True)
wall = (time.perf_counter() - t0) * 1e3
print(f"C1 lanes={eng.lanes()} per-iter bisect={ms[0]/iters:.3f} commit={ms[1]/iters:.3f} factor={ms[2]/iters:.3f} control={ms[3]/iters:.3f} ms; graph wall {wall/iters:.3f} ms/iter")
