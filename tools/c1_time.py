"""Wall time of the pinned C1 run_pgvimp (3 runs after a warm-up)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03416_b200 as P
sdf1 = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
env1 = P.Environment(sdf1, P.CollisionModel(0.2, 8.0))
sys1 = P.point_robot_lti(2)(50, 3.0 / 50)
cfg1 = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=600)
pr1 = P.assemble_prior(sys1, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
P.run_pgvimp(sys1, env1, cfg1, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3, prior=pr1)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    r = P.run_pgvimp(sys1, env1, cfg1, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3, prior=pr1)
    ts.append((time.perf_counter() - t0) * 1e3)
print(os.environ.get("GVP_B200_LIB", "current"), r.iterations, [round(t, 2) for t in ts])
