"""Gaussian belief propagation on the chain factor graph (API of gvplan/gbp.py).

``gbp_marginals`` and ``gbp_mean_solve`` run on the GPU through
libgvp_b200 (chain_kernels.cu: marginals_kernel, mean_solve_kernel); the
chain recursion stays exact (two sweeps, O(N n^3)), with every n x n block
held in registers of the thread that owns the plan.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .blocktri import BlockTridiagonalMatrix, NotPositiveDefiniteError


@dataclass(frozen=True)
class GaussianMessage:
    """Canonical-form message (gbp.py:20-25)."""

    info: np.ndarray
    prec: np.ndarray


@dataclass(frozen=True)
class ChainMarginals:
    """Per-knot covariance blocks and adjacent cross blocks of Lambda^{-1}
    (gbp.py:28-36). ``covs``/``crosses`` are sequences of (n, n) arrays; the
    stacked arrays are kept for zero-copy handoff to the kernels."""

    covs: tuple
    crosses: tuple

    def __len__(self) -> int:
        return len(self.covs)

    @classmethod
    def from_stacks(cls, covs: np.ndarray, crosses: np.ndarray) -> "ChainMarginals":
        m = cls(covs=tuple(covs), crosses=tuple(crosses))
        object.__setattr__(m, "_stacks", (covs, crosses))  # the kernels' arrays, reused as is
        return m

    @property
    def covs_stack(self) -> np.ndarray:
        st = getattr(self, "_stacks", None)
        return st[0] if st is not None else np.stack(self.covs)

    @property
    def crosses_stack(self) -> np.ndarray:
        st = getattr(self, "_stacks", None)
        if st is not None:
            return st[1]
        n = self.covs[0].shape[0]
        return np.stack(self.crosses) if len(self.crosses) else np.zeros((0, n, n))


def gbp_marginals(prec: BlockTridiagonalMatrix) -> ChainMarginals:
    """Marginal covariance blocks of an SPD block-tridiagonal precision
    (gbp.py:43-80), on the GPU. Raises NotPositiveDefiniteError when a belief
    precision fails its Cholesky."""
    lib = N.load()
    K, n = prec.nblocks, prec.block_size
    d, o = N.f64(prec.diag_stack), N.f64(prec.off_stack)
    covs = np.empty((K, n, n))
    crosses = np.empty((max(K - 1, 0), n, n))
    where = np.zeros(1, dtype=np.int64)
    code = N.check(lib.gvp_gbp_marginals(N.ptr(d), N.ptr(o), K, n, N.ptr(covs), N.ptr(crosses),
                                         N.ptr(where)), "gbp_marginals")
    if code == N.GVP_ERR_NOT_SPD:
        raise NotPositiveDefiniteError(
            f"belief precision at knot {int(where[0])} is not positive definite")
    return ChainMarginals.from_stacks(covs, crosses)


def gbp_mean_solve(prec: BlockTridiagonalMatrix, info: np.ndarray) -> np.ndarray:
    """Solve Lambda mu = eta by block elimination (gbp.py:83-106), on the GPU."""
    lib = N.load()
    K, n = prec.nblocks, prec.block_size
    d, o = N.f64(prec.diag_stack), N.f64(prec.off_stack)
    eta = N.f64(info).reshape(K, n)
    out = np.empty((K, n))
    where = np.zeros(1, dtype=np.int64)
    code = N.check(lib.gvp_gbp_mean_solve(N.ptr(d), N.ptr(o), N.ptr(eta), K, n, N.ptr(out),
                                          N.ptr(where)), "gbp_mean_solve")
    if code == N.GVP_ERR_NOT_SPD:
        raise NotPositiveDefiniteError(f"pivot block {int(where[0])} is not positive definite")
    return out.reshape(-1)


def trace_product(a: BlockTridiagonalMatrix, marg: ChainMarginals) -> float:
    """tr(A Sigma) over A's block-tridiagonal sparsity (gbp.py:109-120)."""
    covs = marg.covs_stack
    total = float(np.einsum("kij,kji->", a.diag_stack, covs))
    if a.nblocks > 1:
        total += 2.0 * float(np.einsum("kij,kij->", a.off_stack, marg.crosses_stack))
    return total
