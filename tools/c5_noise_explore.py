"""Exploration: per-probe KL noise of the reference on a C5 plan (bench prior).
For each probe of each iteration: KL with the Cython factor backend (the run),
KL with the numpy backend's gradients at the same state/beta, and a banded
dense-Cholesky KL (no trace cancellation)."""
import os
import sys
import time

import numpy as np
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(1, ROOT)
import gvplan  # noqa: E402
from gvplan import optimizer as ro  # noqa: E402
from gvplan import _kernels_py  # noqa: E402
from gvplan.factors import evaluate_all_factors, assemble_joint_gradients, interior_collision_maps  # noqa: E402
import bench  # noqa: E402


def banded(diag, off):
    K, n, _ = diag.shape
    dim = K * n
    bw = 2 * n - 1
    ab = np.zeros((bw + 1, dim))  # lower form: ab[i-j, j] = A[i, j]
    A = np.zeros((dim, dim)) if False else None
    for i in range(K):
        for r in range(n):
            for c in range(r + 1):
                ab[r - c, i * n + c] = diag[i, r, c]
        if i < K - 1:
            for r in range(n):  # block (i+1, i) = off[i]^T  (off = block (i, i+1))
                for c in range(n):
                    row, col = (i + 1) * n + r, i * n + c
                    ab[row - col, col] = off[i, c, r]
    return ab


def kl_dense(nxt_mean, nd, no, cur_mean, cd, co):
    abn = banded(nd, no)
    abc = banded(cd, co)
    Ln = sl.cholesky_banded(abn, lower=True)
    Lc = sl.cholesky_banded(abc, lower=True)
    n = nd.shape[1]
    dim = nd.shape[0] * n
    # tr(Lc Lc^T Ln^-T Ln^-1) = ||Ln^-1 Lc||_F^2 ; Lc dense from banded
    bw = Lc.shape[0] - 1
    Lcd = np.zeros((dim, dim))
    for k in range(bw + 1):
        idx = np.arange(dim - k)
        Lcd[idx + k, idx] = Lc[k, :dim - k]
    X = sl.solve_triangular(_dense_lower(Ln), Lcd, lower=True)
    tr = float(np.sum(X * X))
    d = cur_mean - nxt_mean
    y = sl.solve_triangular(_dense_lower(Lc).T, d, lower=False, trans=0) if False else None
    mah = float(np.sum((_dense_lower(Lc).T @ d) ** 2))
    ldn = 2 * np.sum(np.log(Ln[0]))
    ldc = 2 * np.sum(np.log(Lc[0]))
    return 0.5 * (tr + mah - dim + ldn - ldc)


def _dense_lower(L):
    dim = L.shape[1]
    out = np.zeros((dim, dim))
    for k in range(L.shape[0]):
        idx = np.arange(dim - k)
        out[idx + k, idx] = L[k, :dim - k]
    return out


def main(b=0, iters=3, dense=True):
    P = gvplan
    goals = bench.c5_goals(4096)
    # the bench's prior for plan b (shared precision, affine info/mean)
    base = np.array([10.0, 10.0, 0.0, 0.0])
    sys0 = P.point_robot_lti(2)(1000, 0.01)
    p0 = P.assemble_prior(sys0, np.zeros(4), base, 1.0, 1e-3)
    info = p0.info.reshape(1001, 4).copy()
    info[-1] += (goals[b] - base) @ (np.eye(4) / 1e-3 ** 2).T
    info = info.reshape(-1)
    import dataclasses
    prior = dataclasses.replace(p0, mean=P.gbp_mean_solve(p0.prec, info), info=info, goal=goals[b])
    sdf = bench.c2_map(P)
    env = ro.Environment(sdf=sdf, model=P.CollisionModel(0.2, 8.0))
    rule = P.smolyak_rule(3, 4)
    orig_sel = ro.select_step_size
    rows = []

    def sel(cur, prior_, g_mu, g_sigma, cfg, temp):
        log = []
        orig_prox, orig_kl, orig_marg = ro.proximal_update, ro.kl_joint, ro.gbp_marginals
        st = {}

        def prox(c, p, gm, gs, beta, t):
            st["beta"] = beta
            return orig_prox(c, p, gm, gs, beta, t)

        def marg(prec):
            try:
                return orig_marg(prec)
            except Exception:
                log.append((st["beta"], 0.0, np.inf))
                raise

        def kl(nxt, c, m=None):
            v = orig_kl(nxt, c, m)
            log.append((st["beta"], 1.0, v, nxt))
            return v
        ro.proximal_update, ro.kl_joint, ro.gbp_marginals = prox, kl, marg
        try:
            out = orig_sel(cur, prior_, g_mu, g_sigma, cfg, temp)
        finally:
            ro.proximal_update, ro.kl_joint, ro.gbp_marginals = orig_prox, orig_kl, orig_marg
        m = orig_marg(cur.prec)
        fv = evaluate_all_factors(cur.mean, cur.prec, sdf, env.model, rule, marginals=m, backend=_kernels_py)
        gm2, gs2 = assemble_joint_gradients(fv, interior_collision_maps(cur.prec.nblocks), cur.prec.nblocks, 4)
        for ent in log:
            beta = ent[0]
            if ent[1] == 0.0:
                rows.append((beta, 0, np.inf, np.nan, np.nan))
                continue
            c2 = ro.proximal_update(cur, prior_, gm2, gs2, beta, temp)
            try:
                k2 = orig_kl(c2, cur, orig_marg(c2.prec))
            except Exception:
                k2 = np.inf
            kd = np.nan
            if dense:
                nx = ent[3]
                kd = kl_dense(nx.mean, np.stack(nx.prec.diag), np.stack(nx.prec.off), cur.mean,
                              np.stack(cur.prec.diag), np.stack(cur.prec.off))
            rows.append((beta, 1, ent[2], k2, kd))
        rows.append(None)
        return out

    ro.select_step_size = sel
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=iters, threads=1)
    sys_ltv = P.point_robot_lti(2)(1000, 0.01)
    t0 = time.time()
    res = P.run_pgvimp(sys_ltv, env, cfg, np.zeros(4), goals[b], 1.0, 1e-3, prior=prior)
    print("time", time.time() - t0)
    it = 1
    for r in rows:
        if r is None:
            it += 1
            continue
        beta, f, k, k2, kd = r
        print(f"it{it} beta={beta:.12g} f={f} kl={k:.10f} np-cy={k2 - k:+.2e} dense-cy={kd - k:+.2e} margin={k - 10:+.2e}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 0, int(sys.argv[2]) if len(sys.argv) > 2 else 2,
         dense=len(sys.argv) <= 3)
