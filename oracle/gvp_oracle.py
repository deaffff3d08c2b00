"""CPU oracle for the P-GVIMP hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker the parity tests, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg compare the CUDA engine against. It is never
imported by the product package (``paper_2411_03416_b200``); the product
path has no CPU fallback.

It restates, in batched numpy, the algorithm of the reference package
``gvplan`` (``/root/reference/pkg/src/gvplan``). Every function names the
reference file:line it follows. Arrays are *stacked* rather than the
reference's lists of blocks:

    block-tridiagonal matrix  -> (diag (K, n, n), off (K-1, n, n))
    joint mean / vectors      -> (K, n)

with K = N + 1 knots. Linear algebra calls the same LAPACK routines the
reference calls (``np.linalg.cholesky`` / ``np.linalg.solve``) block by block
in the same order, so the restatement agrees with the reference to roundoff
(pinned by ``tests/test_oracle_golden.py`` against fixtures generated from
the reference itself, ``tests/golden/make_goldens.py``).
"""

from __future__ import annotations

from math import comb

import numpy as np
from numpy.polynomial.hermite_e import hermegauss

PIVOT_FLOOR = 1e-300          # blocktri.py:17
BISECTION_RTOL = 1e-3         # optimizer.py:39
LOG_2PI = float(np.log(2.0 * np.pi))  # optimizer.py:38
SQRT_JITTER = 1e-10           # quadrature.py:27


class OracleNotSPD(np.linalg.LinAlgError):
    """Mirror of gvplan.blocktri.NotPositiveDefiniteError (blocktri.py:20)."""


# --------------------------------------------------------------------------
# small dense helpers
# --------------------------------------------------------------------------

def sym(a):
    """0.5 (A + A^T) on the last two axes (blocktri.py:43-45)."""
    return 0.5 * (a + np.swapaxes(a, -1, -2))


def chol_checked(mat, what):
    """Lower Cholesky with the reference SPD predicate (blocktri.py:24-32):
    LAPACK failure or any pivot <= 1e-300 is 'not positive definite'."""
    try:
        low = np.linalg.cholesky(mat)
    except np.linalg.LinAlgError as exc:
        raise OracleNotSPD(f"{what} is not positive definite") from exc
    if np.any(np.diag(low) <= PIVOT_FLOOR):
        raise OracleNotSPD(f"{what} has a non-positive pivot")
    return low


def chol_solve(low, rhs):
    """L^{-T} L^{-1} rhs with two dense solves (gbp.py:39-40)."""
    return np.linalg.solve(low.T, np.linalg.solve(low, rhs))


def gaussian_sqrt(cov):
    """Cholesky, then +1e-10 I retry, then clipped eigh root
    (quadrature.py:164-181)."""
    cov = np.asarray(cov, dtype=float)
    for jitter in (0.0, SQRT_JITTER):
        try:
            return np.linalg.cholesky(cov + jitter * np.eye(cov.shape[0]))
        except np.linalg.LinAlgError:
            pass
    vals, vecs = np.linalg.eigh(0.5 * (cov + cov.T))
    return vecs * np.sqrt(np.clip(vals, 0.0, None))


# --------------------------------------------------------------------------
# quadrature (quadrature.py)
# --------------------------------------------------------------------------

def gauss_hermite_1d(p):
    """Probabilists' GH nodes, weights normalised to N(0,1)
    (quadrature.py:55-66)."""
    x, w = hermegauss(p)
    return x, w / np.sqrt(2.0 * np.pi)


def smolyak(k_q, d):
    """Smolyak combination of 1D GH rules (quadrature.py:89-129): level
    vectors with surplus <= k_q-1, coefficient (-1)^(q-|l|) C(d-1, q-|l|),
    points merged on round(., 12), lexicographic key order, |w| <= 1e-15
    dropped."""
    q = d + k_q - 1
    rules = {lev: gauss_hermite_1d(lev) for lev in range(1, k_q + 1)}
    acc = {}

    def levels(slots, budget):
        # same enumeration order as quadrature.py:132-146
        if slots == 1:
            for s in range(budget + 1):
                yield (s + 1,)
            return
        for s in range(budget + 1):
            for rest in levels(slots - 1, budget - s):
                yield (s + 1,) + rest

    for lv in levels(d, k_q - 1):
        coeff = (-1) ** (q - sum(lv)) * comb(d - 1, q - sum(lv))
        if coeff == 0:
            continue
        axes = [rules[v][0] for v in lv]
        grids = np.meshgrid(*axes, indexing="ij")
        pts = np.stack([g.reshape(-1) for g in grids], axis=1)
        wts = rules[lv[0]][1]
        for v in lv[1:]:
            wts = np.multiply.outer(wts, rules[v][1]).reshape(-1)
        wts = coeff * wts
        for key_row, pt, wt in zip(np.round(pts, 12), pts, wts):
            key = tuple(key_row)
            if key in acc:
                acc[key] = (acc[key][0], acc[key][1] + wt)
            else:
                acc[key] = (pt, wt)
    items = sorted(acc.items(), key=lambda kv: kv[0])
    pts = np.array([v[0] for _, v in items])
    wts = np.array([v[1] for _, v in items])
    keep = np.abs(wts) > 1e-15
    return np.ascontiguousarray(pts[keep]), np.ascontiguousarray(wts[keep])


def tensor(p, d):
    """Full tensor GH rule (quadrature.py:69-86)."""
    x, w = gauss_hermite_1d(p)
    grids = np.meshgrid(*([x] * d), indexing="ij")
    pts = np.stack([g.reshape(-1) for g in grids], axis=1)
    wts = w
    for _ in range(d - 1):
        wts = np.multiply.outer(wts, w).reshape(-1)
    return pts, wts


# --------------------------------------------------------------------------
# kernel (a): factor expectations (_kernels.pyx:93-177, _kernels_py.py:16-85)
# --------------------------------------------------------------------------

def interp(grid, origin, cell, pts):
    """Border-clamped bi/trilinear interpolation + OOB count
    (_kernels.pyx:18-90; sdf.py:80-122). Grid axes are (y, x) / (z, y, x)."""
    dim = grid.ndim
    u = (pts[:, :dim] - np.asarray(origin, float)[:dim]) / cell
    top = np.array(grid.shape[::-1], dtype=float) - 1.0
    oob = int(np.count_nonzero(np.any((u < 0.0) | (u > top), axis=1)))
    u = np.clip(u, 0.0, top)
    base = np.clip(np.floor(u), 0.0, top - 1.0).astype(np.int64)
    f = u - base
    if dim == 2:
        ix, iy = base[:, 0], base[:, 1]
        fx, fy = f[:, 0], f[:, 1]
        val = (grid[iy, ix] * (1 - fx) * (1 - fy) + grid[iy, ix + 1] * fx * (1 - fy)
               + grid[iy + 1, ix] * (1 - fx) * fy + grid[iy + 1, ix + 1] * fx * fy)
    else:
        ix, iy, iz = base[:, 0], base[:, 1], base[:, 2]
        fx, fy, fz = f[:, 0], f[:, 1], f[:, 2]

        def plane(k):
            return (grid[k, iy, ix] * (1 - fx) * (1 - fy)
                    + grid[k, iy, ix + 1] * fx * (1 - fy)
                    + grid[k, iy + 1, ix] * (1 - fx) * fy
                    + grid[k, iy + 1, ix + 1] * fx * fy)
        # combine order of the compiled kernel (_kernels.pyx:86-90)
        val = plane(iz) * (1 - fz) + plane(iz + 1) * fz
    return val, oob


def factor_expectations(means, chols, points, weights, grid, origin, cell,
                        radius_eps, sigma_obs, pos_dim=None):
    """e0/e1/e2 hinge moments per factor + total OOB count
    (_kernels.pyx:93-129 per factor; contract _kernels_py.py:16-53).

    Sequential ascending-point accumulation like the compiled kernel; points
    with gap <= 0 are skipped (_kernels.pyx:121-122)."""
    grid = np.ascontiguousarray(grid, dtype=float)
    means = np.asarray(means, float)
    chols = np.asarray(chols, float)
    nfac, n = means.shape
    dim = grid.ndim
    e0 = np.zeros(nfac)
    e1 = np.zeros((nfac, n))
    e2 = np.zeros((nfac, n, n))
    oob = 0
    for f in range(nfac):
        dx = points @ chols[f].T                       # (Q, n), x_l - mu
        d, o = interp(grid, origin, cell, means[f] + dx)
        oob += o
        gap = radius_eps - d
        hit = gap > 0.0
        wc = weights[hit] * sigma_obs * gap[hit] * gap[hit]
        dxh = dx[hit]
        e0[f] = np.sum(wc)
        e1[f] = wc @ dxh
        e2[f] = dxh.T @ (dxh * wc[:, None])
    return e0, e1, e2, oob


def moment_gradients(e0, e1, e2, cov):
    """g_mu = P^{-1} e1, g_S = sym(-1/2 P^{-1} e0 + 1/2 P^{-1} e2 P^{-1})
    with P^{-1} built from the Cholesky root (factors.py:95-104)."""
    low = gaussian_sqrt(cov)
    inv_low = np.linalg.solve(low, np.eye(cov.shape[0]))
    prec = inv_low.T @ inv_low
    g_mu = prec @ e1
    g_s = sym(-0.5 * prec * e0 + 0.5 * prec @ e2 @ prec)
    return g_mu, g_s


def evaluate_factors(mean, covs, points, weights, grid, origin, cell,
                     radius_eps, sigma_obs):
    """Interior-knot collision factors of one plan (factors.py:167-225).

    mean (K, n), covs (K, n, n) -> e_psi (K-2,), g_mu (K-2, n),
    g_sigma (K-2, n, n), oob. e_psi is clamped at 0, gradients use raw e0
    (factors.py:218-224). Raises FloatingPointError on non-finite moments
    (factors.py:212-217)."""
    K, n = mean.shape
    idx = np.arange(1, K - 1)
    chols = np.stack([gaussian_sqrt(covs[i]) for i in idx]) if len(idx) else np.zeros((0, n, n))
    e0, e1, e2, oob = factor_expectations(mean[idx], chols, points, weights,
                                          grid, origin, cell, radius_eps, sigma_obs)
    e_psi = np.zeros(len(idx))
    g_mu = np.zeros((len(idx), n))
    g_s = np.zeros((len(idx), n, n))
    for k, i in enumerate(idx):
        if not (np.isfinite(e0[k]) and np.all(np.isfinite(e1[k])) and np.all(np.isfinite(e2[k]))):
            raise FloatingPointError(f"factor {i}: non-finite expectation")
        g_mu[k], g_s[k] = moment_gradients(e0[k], e1[k], e2[k], covs[i])
        e_psi[k] = max(float(e0[k]), 0.0)
    return e_psi, g_mu, g_s, oob


def joint_gradients(g_mu_f, g_s_f, K):
    """Scatter interior unary factors to knots 1..K-2 (factors.py:228-255)."""
    n = g_mu_f.shape[1] if g_mu_f.ndim == 2 else 0
    g_mu = np.zeros((K, n))
    g_diag = np.zeros((K, n, n))
    g_mu[1:K - 1] += g_mu_f
    g_diag[1:K - 1] += g_s_f
    return g_mu, g_diag


# --------------------------------------------------------------------------
# block-tridiagonal algebra (blocktri.py) and GBP (gbp.py)
# --------------------------------------------------------------------------

def bt_dense(diag, off):
    K, n, _ = diag.shape
    out = np.zeros((K * n, K * n))
    for i in range(K):
        out[i * n:(i + 1) * n, i * n:(i + 1) * n] = diag[i]
    for i in range(K - 1):
        out[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] = off[i]
        out[(i + 1) * n:(i + 2) * n, i * n:(i + 1) * n] = off[i].T
    return out


def bt_matvec(diag, off, x):
    """blocktri.py:117-127."""
    out = np.einsum("kij,kj->ki", diag, x)
    out[:-1] += np.einsum("kij,kj->ki", off, x[1:])
    out[1:] += np.einsum("kji,kj->ki", off, x[:-1])
    return out


def bt_quad(diag, off, x):
    """blocktri.py:129-131."""
    return float(x.reshape(-1) @ bt_matvec(diag, off, x).reshape(-1))


def forward_schur_chols(diag, off):
    """S_0 = D_0, S_i = D_i - W^T W, W = L_{i-1}^{-1} U_{i-1}
    (blocktri.py:151-165); no symmetrisation."""
    chols = []
    for i in range(diag.shape[0]):
        s = diag[i]
        if i > 0:
            w = np.linalg.solve(chols[i - 1], off[i - 1])
            s = diag[i] - w.T @ w
        chols.append(chol_checked(s, f"pivot block {i}"))
    return chols


def logdet(diag, off):
    """2 sum log diag of the forward Schur pivots (blocktri.py:168-174)."""
    return 2.0 * float(sum(np.sum(np.log(np.diag(c))) for c in forward_schur_chols(diag, off)))


def marginals(diag, off):
    """Exact chain GBP (gbp.py:43-80): backward Schur sweep with an SPD
    check per knot, then forward covariance sweep. Returns covs (K,n,n),
    crosses (K-1,n,n)."""
    K, n, _ = diag.shape
    eye = np.eye(n)
    back = [None] * K
    back[K - 1] = chol_checked(diag[K - 1], f"belief precision at knot {K - 1}")
    for i in range(K - 2, -1, -1):
        w = chol_solve(back[i + 1], off[i].T)
        back[i] = chol_checked(sym(diag[i] - off[i] @ w), f"belief precision at knot {i}")
    covs = np.zeros((K, n, n))
    crosses = np.zeros((max(K - 1, 0), n, n))
    covs[0] = sym(chol_solve(back[0], eye))
    for i in range(K - 1):
        phi_inv = chol_solve(back[i + 1], eye)
        crosses[i] = -covs[i] @ off[i] @ phi_inv
        covs[i + 1] = sym(phi_inv + phi_inv @ off[i].T @ covs[i] @ off[i] @ phi_inv)
    return covs, crosses


def mean_solve(diag, off, eta):
    """Block Thomas: forward elimination with SPD pivots, back
    substitution (gbp.py:83-106)."""
    K, n, _ = diag.shape
    piv, rhs = [], []
    for i in range(K):
        d = diag[i]
        r = eta[i].copy()
        if i > 0:
            u = off[i - 1]
            d = d - u.T @ chol_solve(piv[i - 1], u)
            r = r - u.T @ chol_solve(piv[i - 1], rhs[i - 1])
        piv.append(chol_checked(sym(d), f"pivot block {i}"))
        rhs.append(r)
    out = np.zeros((K, n))
    out[K - 1] = chol_solve(piv[K - 1], rhs[K - 1])
    for i in range(K - 2, -1, -1):
        out[i] = chol_solve(piv[i], rhs[i] - off[i] @ out[i + 1])
    return out


def trace_product(a_diag, a_off, covs, crosses):
    """tr(A Sigma) over A's sparsity (gbp.py:109-120)."""
    t = 0.0
    for a, s in zip(a_diag, covs):
        t += float(np.sum(a * s.T))
    for a, s in zip(a_off, crosses):
        t += 2.0 * float(np.sum(a * s))
    return t


# --------------------------------------------------------------------------
# proximal step and bisection (optimizer.py)
# --------------------------------------------------------------------------

def proximal_update(mean, diag, off, k_diag, k_off, info, g_mu, g_diag, g_off, beta, temp):
    """Theorem-1 update with the reference's operation order
    (optimizer.py:129-161): matrices scaled by reciprocals, rhs divided."""
    if beta <= 0:
        raise ValueError("beta must be positive")
    ki_d, ki_o = k_diag * (1.0 / temp), k_off * (1.0 / temp)
    lb_d, lb_o = diag * (1.0 / beta), off * (1.0 / beta)
    c = beta / (beta + 1.0)
    nd = sym((g_diag * (2.0 / temp) + ki_d + lb_d) * c)
    no = (g_off * (2.0 / temp) + ki_o + lb_o) * c
    rhs = -g_mu / temp + info / temp + bt_matvec(lb_d, lb_o, mean)
    nm = mean_solve(ki_d + lb_d, ki_o + lb_o, rhs)
    return nm, nd, no


def kl_joint(n_mean, n_diag, n_off, n_covs, n_crosses, mean, diag, off, logdet_cur=None):
    """KL(next || cur), clipped at 0 (optimizer.py:164-177)."""
    tr = trace_product(diag, off, n_covs, n_crosses)
    delta = mean - n_mean
    mahal = bt_quad(diag, off, delta)
    ld_n = logdet(n_diag, n_off)
    ld_c = logdet(diag, off) if logdet_cur is None else logdet_cur
    return max(0.5 * (tr + mahal - diag.shape[0] * diag.shape[1] + ld_n - ld_c), 0.0)


def select_step(mean, diag, off, k_diag, k_off, info, g_mu, g_diag, g_off, temp,
                kl_bound, beta_min, beta_max, trace=None):
    """Largest feasible beta by bisection (optimizer.py:188-231). Returns
    (beta, mean', diag', off', kl, covs, crosses). ``trace`` (a list) gets
    (beta, feasible, kl) per probe."""

    def probe(beta):
        nm, nd, no = proximal_update(mean, diag, off, k_diag, k_off, info,
                                     g_mu, g_diag, g_off, beta, temp)
        try:
            cv, cr = marginals(nd, no)
        except OracleNotSPD:
            if trace is not None:
                trace.append((beta, False, np.inf))
            return None
        kl = kl_joint(nm, nd, no, cv, cr, mean, diag, off)
        if trace is not None:
            trace.append((beta, kl <= kl_bound, kl))
        if kl > kl_bound:
            return None
        return (beta, nm, nd, no, kl, cv, cr)

    best = probe(beta_max)
    if best is not None:
        return best
    best = probe(beta_min)
    if best is None:
        raise RuntimeError(f"no feasible step size at beta_min={beta_min} (KL bound {kl_bound})")
    lo, hi = beta_min, beta_max
    while (hi - lo) > BISECTION_RTOL * hi:
        mid = 0.5 * (lo + hi)
        cand = probe(mid)
        if cand is None:
            hi = mid
        else:
            lo = mid
            best = cand
    return best


def entropy_of(diag, off):
    """optimizer.py:234-235."""
    return 0.5 * (diag.shape[0] * diag.shape[1] * (LOG_2PI + 1.0) - logdet(diag, off))


def cost_breakdown(mean, diag, off, prior_mean, k_diag, k_off, covs, crosses, e_psi, temp):
    """(prior, collision, entropy) costs (optimizer.py:238-277)."""
    delta = mean - prior_mean
    prior_cost = 0.5 * bt_quad(k_diag, k_off, delta) + 0.5 * trace_product(k_diag, k_off, covs, crosses)
    collision = float(sum(float(v) for v in e_psi))
    ent = -temp * entropy_of(diag, off)
    return prior_cost, collision, ent


# --------------------------------------------------------------------------
# prior (prior.py) — host setup, used by the oracle driver
# --------------------------------------------------------------------------

def point_robot_triples(dim):
    """dynamics.py:66-85: A=[[0,I],[0,0]], a=0, B=[0;I]."""
    n = 2 * dim
    A = np.zeros((n, n))
    A[:dim, dim:] = np.eye(dim)
    B = np.zeros((n, dim))
    B[dim:] = np.eye(dim)
    return A, np.zeros(n), B


def assemble_prior(As, avs, Bs, dt, x0, goal, q_c, sigma_b):
    """Anchored lifted prior (prior.py:56-170). As/avs/Bs are per-step
    (N+1 entries; the last is unused like the reference). Returns dict with
    diag, off, info, mean."""
    from numpy.polynomial.legendre import leggauss
    from scipy.linalg import expm
    N = len(As) - 1
    n = As[0].shape[0]
    nodes, w = leggauss(10)
    s_vals, w_vals = 0.5 * dt * (nodes + 1.0), 0.5 * dt * w
    diag = np.zeros((N + 1, n, n))
    off = np.zeros((N, n, n))
    info = np.zeros((N + 1, n))
    anchor = np.eye(n) / sigma_b ** 2
    diag[0] += anchor
    info[0] += anchor @ x0
    diag[N] += anchor
    info[N] += anchor @ goal
    for i in range(N):
        aug = np.zeros((n + 1, n + 1))
        aug[:n, :n] = As[i]
        aug[:n, n] = avs[i]
        big = expm(aug * dt)
        phi, off_vec = big[:n, :n], big[:n, n]
        bqb = q_c * (Bs[i] @ Bs[i].T)
        g = np.zeros((n, n))
        for s, ws in zip(s_vals, w_vals):
            tr = expm(As[i] * (dt - s))
            g += ws * (tr @ bqb @ tr.T)
        g = sym(g)
        try:
            chol_checked(g, "grammian")
        except OracleNotSPD:
            g = g + 1e-10 * np.eye(n)
        ql = chol_checked(g, f"grammian {i}")
        qi = sym(np.linalg.solve(ql.T, np.linalg.solve(ql, np.eye(n))))
        diag[i] += phi.T @ qi @ phi
        diag[i + 1] += qi
        off[i] += -phi.T @ qi
        info[i] += -phi.T @ (qi @ off_vec)
        info[i + 1] += qi @ off_vec
    diag = sym(diag)
    mean = mean_solve(diag, off, info)
    return {"diag": diag, "off": off, "info": info, "mean": mean}


# --------------------------------------------------------------------------
# Algorithm 1 driver (optimizer.py:280-401)
# --------------------------------------------------------------------------

def run_pgvimp(prior, grid, origin, cell, radius_eps, sigma_obs, points, weights,
               kl_bound=0.1, beta_min=1e-4, beta_max=0.9, temp_low=1.0, temp_high=10.0,
               collision_tol=None, max_iters=200, tol_mean=1e-5, tol_cost=1e-6,
               init_cov_scale=0.1, x0=None, goal=None, init_mean=None, trace=None, factor_fn=None):
    """Device-free restatement of run_pgvimp (optimizer.py:299-401) for one
    plan with an environment. Returns dict(mean, diag, off, covs, crosses,
    records, converged, iterations, switch_iteration). factor_fn(mean, covs) ->
    (e_psi, g_mu, g_sigma, oob) replaces the point-robot factor stage (the
    7-DOF arm oracle, arm_oracle.arm_evaluate_factors)."""
    k_diag, k_off, info, pmean = prior["diag"], prior["off"], prior["info"], prior["mean"]
    K, n = pmean.shape
    N = K - 1
    ctol = collision_tol if collision_tol is not None else 1e-4 * N
    if init_mean is not None:
        mean = np.asarray(init_mean, float).reshape(K, n).copy()
    else:
        al = np.linspace(0.0, 1.0, K).reshape(-1, 1)
        mean = (1.0 - al) * x0 + al * goal            # optimizer.py:292-294
    diag = k_diag * (1.0 / init_cov_scale)
    off = k_off * (1.0 / init_cov_scale)
    covs, crosses = marginals(diag, off)
    temp = temp_low
    prev_total = prev_temp = None
    switched = False
    switch_it = None
    cached = None
    records = []
    converged = False
    it = 0
    g_off = np.zeros_like(k_off)
    for it in range(1, max_iters + 1):
        if cached is None:
            e_psi, gm, gs, _ = (factor_fn(mean, covs) if factor_fn else
                                evaluate_factors(mean, covs, points, weights, grid, origin, cell, radius_eps,
                                                 sigma_obs))
            cached = (e_psi, gm, gs)
        g_mu, g_diag = joint_gradients(cached[1], cached[2], K)
        beta, nm, nd, no, kl, cv, cr = select_step(mean, diag, off, k_diag, k_off, info,
                                                   g_mu, g_diag, g_off, temp, kl_bound,
                                                   beta_min, beta_max, trace=trace)
        e_psi, gm, gs, _ = (factor_fn(nm, cv) if factor_fn else
                            evaluate_factors(nm, cv, points, weights, grid, origin, cell, radius_eps, sigma_obs))
        cached = (e_psi, gm, gs)
        pc, cc, ec = cost_breakdown(nm, nd, no, pmean, k_diag, k_off, cv, cr, e_psi, temp)
        total = pc + cc + ec
        shift = float(np.linalg.norm(nm - mean))
        records.append({"iter": it, "beta": beta, "temperature": temp, "prior_cost": pc,
                        "collision_cost": cc, "entropy_cost": ec, "total_cost": total,
                        "kl_step": kl, "mean_shift": shift})
        mean, diag, off, covs, crosses = nm, nd, no, cv, cr
        same = prev_temp is not None and prev_temp == temp
        change = abs(total - prev_total) if prev_total is not None else np.inf
        if same and shift < tol_mean and change < tol_cost:
            converged = True
            break
        prev_total = total if same or prev_temp is None else None
        prev_temp = temp
        if not switched and cc < ctol and temp != temp_high:
            temp = temp_high
            switched = True
            switch_it = it
            prev_total = None
    return {"mean": mean, "diag": diag, "off": off, "covs": covs, "crosses": crosses,
            "records": records, "converged": converged, "iterations": it,
            "switch_iteration": switch_it}
