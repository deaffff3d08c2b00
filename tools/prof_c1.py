"""Small C1 run for profiling (ncu) the single-plan path."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03416_b200 as P

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sdf = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
env = P.Environment(sdf, P.CollisionModel(0.2, 8.0))
sys_ltv = P.point_robot_lti(2)(50, 3.0 / 50)
cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=iters)
pr = P.assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
t0 = time.perf_counter()
r = P.run_pgvimp(sys_ltv, env, cfg, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3, prior=pr, spec_lanes=lanes)
print(f"lanes={lanes} iters={r.iterations} ms={(time.perf_counter()-t0)*1e3:.1f}")
