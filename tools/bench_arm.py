"""Throughput of the sphere-arm factor kernel (SURVEY C3 scale: n = 14,
k_q = 3 -> 421 points / 113 projections, 128^3 map) (measurement aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2411_03416_b200 as P

F = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
sdf = P.rasterize([P.sdf.Disc(center=np.array([0.45, 0.0, 0.55]), radius=0.15),
                   P.sdf.Box(center=np.array([0.4, 0.35, 0.3]), halfextents=np.array([0.1, 0.1, 0.25]))],
                  bounds=[[-1.27, 1.27], [-1.27, 1.27], [-0.5, 2.04]], cell_size=0.02)
print("grid", sdf.values.shape)
rng = np.random.default_rng(0)
means = np.concatenate([rng.uniform(-1.2, 1.2, size=(F, 7)), rng.normal(0, 0.3, size=(F, 7))], axis=1)
chols = np.repeat((np.linalg.cholesky(0.01 * np.eye(14)))[None], F, 0)
rule = P.smolyak_rule(3, 14)
tab = P.arm_projection_tables(rule)
arm = P.panda_like()
m = P.CollisionModel(0.05, 10.0)
P.arm_factor_expectations(means[:1000], chols[:1000], rule, sdf, arm, m, tab)
t0 = time.perf_counter()
out = P.arm_factor_expectations(means, chols, rule, sdf, arm, m, tab)
dt = time.perf_counter() - t0
print(f"{F} factors in {dt*1e3:.1f} ms incl. transfers+map upload -> {F/dt:.3e} factor-evals/s, "
      f"{F*rule.npoints/dt:.3e} sigma-pt/s; nonzero {np.count_nonzero(out[0])}")
