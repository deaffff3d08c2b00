"""Which path the factor kernel takes on the C5 bench state (host replica of
its tests, csrc/factor_kernels.cu:685-783): provably clear (one lookup), a
full quadrature with no hit, or a hit; and the warp-level mix."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_2411_03416_b200 as P

B, K = 4096, 1001
goals = bench.c5_goals(B)
prior, info, pmean, init = bench.build_problem(P, goals)
sdf = bench.c2_map(P)
rule = P.smolyak_rule(3, 4)
eng = P.PlanBatch(B, K, 4, sdf, P.CollisionModel(0.2, 8.0), rule, bench.c5_cfg(P, 40), shared_prior=True)
eng.load(prior.prec.diag_stack, prior.prec.off_stack, info, pmean, init)
g = np.asarray(sdf.values, dtype=np.float64)  # (ny, nx)
ny, nx = g.shape
cell, ox, oy = float(sdf.cell_size), float(sdf.origin[0]), float(sdf.origin[1])
mx = np.abs(np.diff(g, axis=1))
my = np.abs(np.diff(g, axis=0))
cx = np.maximum(mx[:-1, :], mx[1:, :])
cy = np.maximum(my[:, :-1], my[:, 1:])
lip = np.sqrt((cx ** 2 + cy ** 2).max()) / cell * (1 + 1e-12)
proj = np.unique(np.round(rule.points[:, :2], 12), axis=0)
prad = np.sqrt((proj ** 2).sum(1)).max() * (1 + 1e-12)


def interp(px, py):
    u = np.clip((px - ox) / cell, 0, nx - 1)
    v = np.clip((py - oy) / cell, 0, ny - 1)
    ix = np.minimum(u.astype(np.int64), nx - 2)
    iy = np.minimum(v.astype(np.int64), ny - 2)
    fx, fy = u - ix, v - iy
    top = g[iy, ix] + fx * (g[iy, ix + 1] - g[iy, ix])
    bot = g[iy + 1, ix] + fx * (g[iy + 1, ix + 1] - g[iy + 1, ix])
    return top + fy * (bot - top)


for it in (1, 5, 20, 40):
    while eng.summary()["iterations"].max() < it:
        eng.step(1, sync=True)
    mean = np.empty((K, 4, B))
    covs = np.empty((K, 10, B))
    eng.packed_into(mean=mean, covs=covs)
    mu = mean[1:K - 1]  # interior knots (K-2, 4, B)
    S = covs[1:K - 1]
    a, c, b01 = S[:, 0], S[:, 2], S[:, 1]  # packed lower: (0,0), (1,0), (1,1)
    h = 0.5 * (a - c)
    fr = (0.5 * (a + c) + np.sqrt(h * h + b01 * b01)) * (1 + 1e-12)
    rad = np.sqrt(fr) * prad
    d = interp(mu[:, 0], mu[:, 1])
    clear = d - lip * rad - 0.2 > 1e-9
    # warps: 32 consecutive plans at one knot
    w = clear.reshape(K - 2, B // 32, 32)
    allc = w.all(-1).mean()
    print(f"iteration {it}: clear {clear.mean():.3f} of factors; warps all-clear {allc:.3f}, "
          f"mixed {(~w.all(-1) & w.any(-1)).mean():.3f}, none-clear {(~w.any(-1)).mean():.3f}; lip {lip:.3f}")
eng.close()
