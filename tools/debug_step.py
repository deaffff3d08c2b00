"""Run one drop-in select_step_size (golden case s1/s2) at a given lane count."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2411_03416_b200 as P
from paper_2411_03416_b200 import _native

s = sys.argv[1]; lanes = int(sys.argv[2])
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "steps.npz"))
K, n = g[f"{s}_mean"].shape
cur = P.JointGaussian(g[f"{s}_mean"].reshape(-1), P.BlockTridiagonalMatrix(g[f"{s}_diag"], g[f"{s}_off"]))
prior = P.DiscretePrior(phis=(), offsets=(), grammians=(), flow_mean=None, mean=g[f"{s}_pmean"].reshape(-1),
                        info=g[f"{s}_info"].reshape(-1), prec=P.BlockTridiagonalMatrix(g[f"{s}_kdiag"], g[f"{s}_koff"]),
                        x0=np.zeros(n), goal=np.zeros(n), sigma_b=1e-3)
gs = P.BlockTridiagonalMatrix(g[f"{s}_gdiag"], np.zeros((K - 1, n, n)))
kl_bound, bmin, bmax, temp = g[f"{s}_cfg"]
assert _native.load().gvp_set_step_lanes(lanes) == 0
sel = P.select_step_size(cur, prior, g[f"{s}_gmu"].reshape(-1), gs,
                         P.OptimizerConfig(kl_bound=kl_bound, beta_min=bmin, beta_max=bmax), temp)
print(s, lanes, "beta", sel.beta, "ref", float(g[f"{s}_beta"]), "kl", sel.kl, "nprobes", len(sel.probes))
