"""Engine smoke at a given batch size / lane count (debugging aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03416_b200 as P

B = int(sys.argv[1]); lanes = int(sys.argv[2]); iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sdf = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
env = P.Environment(sdf, P.CollisionModel(0.2, 8.0))
sys_ltv = P.point_robot_lti(2)(50, 3.0 / 50)
cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=iters)
goals = np.tile(np.array([2.0, 1.5, 0, 0]), (B, 1))
try:
    r = P.run_pgvimp_batch(sys_ltv, env, cfg, np.zeros(4), goals, 1.0, 1e-3, spec_lanes=lanes)
    print(f"B={B} lanes={lanes} ok iters={r.iterations[:4]} status={set(r.status.tolist())}")
except Exception as e:
    print(f"B={B} lanes={lanes} FAIL {str(e)[:120]}")
