"""Wall-time breakdown of one C1 run_pgvimp call (engine create / load / run / fetch)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03416_b200 as P
from paper_2411_03416_b200.optimizer import initial_mean

sdf = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
env = P.Environment(sdf, P.CollisionModel(0.2, 8.0))
sys1 = P.point_robot_lti(2)(50, 3.0 / 50)
cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=600)
pr = P.assemble_prior(sys1, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
P.run_pgvimp(sys1, env, cfg, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3, prior=pr)
for rep in range(3):
    T = {}
    t = time.perf_counter()
    rule = P.smolyak_rule(3, 4); T["rule"] = time.perf_counter() - t; t = time.perf_counter()
    eng = P.PlanBatch(1, 51, 4, env.sdf, env.model, rule, cfg)
    T["create"] = time.perf_counter() - t; t = time.perf_counter()
    eng.load(pr.prec.diag_stack, pr.prec.off_stack, pr.info.reshape(1, 51, 4), pr.mean.reshape(1, 51, 4),
             initial_mean(pr, cfg).reshape(1, 51, 4)); eng.sync()
    T["load"] = time.perf_counter() - t; t = time.perf_counter()
    it = eng.run(); T["run"] = time.perf_counter() - t; t = time.perf_counter()
    st = eng.state(); sm = eng.summary(); rec = eng.records(); T["fetch"] = time.perf_counter() - t; t = time.perf_counter()
    eng.close(); T["close"] = time.perf_counter() - t
    t = time.perf_counter()
    P.run_pgvimp(sys1, env, cfg, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3, prior=pr)
    T["run_pgvimp_total"] = time.perf_counter() - t
    print({k: round(v * 1e3, 2) for k, v in T.items()}, "iters", sm["iterations"][0])
