"""First select_step of C5 plan 0: device probes vs the oracle's (debug aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import gvp_oracle as O
import paper_2411_03416_b200 as P
from paper_2411_03416_b200.sdf import Box

g = np.load(os.path.join(ROOT, "tests/golden/configs.npz"))
goal = g["c5p_goal"]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
sdf = P.rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                   Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))], bounds=[[-2, 12], [-2, 12]],
                  cell_size=0.05)
A, a, B = O.point_robot_triples(2)
pr = O.assemble_prior([A] * (N + 1), [a] * (N + 1), [B] * (N + 1), 10.0 / N, np.zeros(4), goal, 1.0, 1e-3)
pts, wts = O.smolyak(3, 4)
K, n = N + 1, 4
al = np.linspace(0.0, 1.0, K).reshape(-1, 1)
mean = (1.0 - al) * np.zeros(4) + al * goal
diag, off = pr["diag"] * 10.0, pr["off"] * 10.0
covs, crosses = O.marginals(diag, off)
e_psi, gm, gs, _ = O.evaluate_factors(mean, covs, pts, wts, sdf.values, sdf.origin, 0.05, 0.2, 8.0)
g_mu, g_diag = O.joint_gradients(gm, gs, K)
tr = []
O.select_step(mean, diag, off, pr["diag"], pr["off"], pr["info"], g_mu, g_diag, np.zeros_like(off), 1.0, 10.0,
              1e-4, 0.5, trace=tr)
cur = P.JointGaussian(mean.reshape(-1), P.BlockTridiagonalMatrix(diag, off))
prior = P.DiscretePrior(phis=(), offsets=(), grammians=(), flow_mean=None, mean=pr["mean"].reshape(-1),
                        info=pr["info"].reshape(-1), prec=P.BlockTridiagonalMatrix(pr["diag"], pr["off"]),
                        x0=np.zeros(4), goal=goal, sigma_b=1e-3)
sel = P.select_step_size(cur, prior, g_mu.reshape(-1), P.BlockTridiagonalMatrix(g_diag, np.zeros((K - 1, n, n))),
                         P.OptimizerConfig(kl_bound=10.0, beta_max=0.5), 1.0)
print("device beta", sel.beta, "oracle", [t for t in tr if t[1]][-1][0])
for (b, f, k), (b2, f2, k2) in zip(tr, sel.probes):
    print(f"{b:.10g} {b2:.10g} ref {k:.12g} dev {k2:.12g} rel {abs(k - k2) / max(abs(k), 1e-300):.2e}")
