"""Independent KL(next || cur) for the golden generators (test infrastructure).

The reference's kl_joint (optimizer.py:164-177) evaluates tr(Lambda_cur
Sigma_next) through trace_product (gbp.py:109-120) over the backward-sweep
marginals; at N = 1000 with sigma_b = 1e-3 anchors those marginals carry
~1e-8 relative error against large precision entries, so the reference's KL
is only good to ~1e-4 absolute (tools/c5_noise_explore.py). This module
computes the same quantity WITHOUT the selected inversion:

    tr(Lc Lc^T Ln^-T Ln^-1) = || Ln^-1 Lc ||_F^2      (sum of squares)
    delta^T Lambda_cur delta = || Lc^T delta ||^2
    log det = 2 sum log diag(L)

with Ln, Lc the banded Cholesky factors (LAPACK dpbtrf via
scipy.linalg.cholesky_banded) and Ln^-1 Lc by a banded triangular solve
(LAPACK dtbtrs) — every term a sum of non-negative numbers, accurate to
~1e-12 relative. It is the arbiter for probes where the reference's own KL
lies within its noise of the bound.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sl
import scipy.linalg.lapack as lapack


def banded_lower(diag: np.ndarray, off: np.ndarray) -> np.ndarray:
    """Stacked blocks (K,n,n) diag / (K-1,n,n) off (block (i,i+1)) -> LAPACK
    lower band storage ab[i-j, j] = A[i, j], bandwidth 2n-1."""
    K, n, _ = diag.shape
    dim = K * n
    ab = np.zeros((2 * n, dim))
    for r in range(n):
        for c in range(r + 1):
            ab[r - c, c::n][:K] = diag[:, r, c]
    # block (i+1, i) = off[i]^T: A[(i+1)n + r, i n + c] = off[i, c, r]
    for r in range(n):
        for c in range(n):
            k = n + r - c
            ab[k, c::n][:K - 1] = off[:, c, r]
    return ab


def band_to_dense_lower(L: np.ndarray) -> np.ndarray:
    dim = L.shape[1]
    out = np.zeros((dim, dim))
    for k in range(L.shape[0]):
        idx = np.arange(dim - k)
        out[idx + k, idx] = L[k, :dim - k]
    return out


def kl_banded(nxt_mean, nxt_diag, nxt_off, cur_mean, cur_diag, cur_off) -> float:
    """0.5 [tr(Lc Sigma_n) + d^T Lc d - dim + logdet Ln - logdet Lc] (unclipped)."""
    Ln = sl.cholesky_banded(banded_lower(np.asarray(nxt_diag), np.asarray(nxt_off)), lower=True)
    Lc = sl.cholesky_banded(banded_lower(np.asarray(cur_diag), np.asarray(cur_off)), lower=True)
    dim = Ln.shape[1]
    X, info = lapack.dtbtrs(Ln, band_to_dense_lower(Lc), uplo=b"L")
    if info != 0:
        raise np.linalg.LinAlgError(f"dtbtrs info={info}")
    tr = float(np.sum(X * X))
    d = np.asarray(cur_mean, dtype=float).reshape(-1) - np.asarray(nxt_mean, dtype=float).reshape(-1)
    # Lc^T d through the band: (Lc^T d)_j = sum_k Lc[k, j] d[j + k]
    y = np.zeros(dim)
    for k in range(Lc.shape[0]):
        y[:dim - k] += Lc[k, :dim - k] * d[k:]
    mah = float(np.sum(y * y))
    ldn = 2.0 * float(np.sum(np.log(Ln[0])))
    ldc = 2.0 * float(np.sum(np.log(Lc[0])))
    return 0.5 * (tr + mah - dim + ldn - ldc)
