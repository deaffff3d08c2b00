"""Symmetric block-tridiagonal matrices (API of gvplan/blocktri.py).

Storage is two stacked float64 arrays — ``diag_stack`` (K, n, n) and
``off_stack`` (K-1, n, n) — which is the layout the CUDA chain kernels take
(include/gvp_b200.h, family 1). ``diag`` / ``off`` expose per-block views
so code written against the reference's lists of blocks keeps working.

Log-determinants and SPD tests run on the GPU (libgvp_b200); the small
host helpers (matvec, quad_form, dense) are data-model utilities.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

PIVOT_FLOOR = 1e-300  # blocktri.py:17


class NotPositiveDefiniteError(np.linalg.LinAlgError):
    """A matrix required to be SPD failed its Cholesky factorization
    (blocktri.py:20)."""


def chol_spd(mat: np.ndarray, what: str = "matrix") -> np.ndarray:
    """Lower Cholesky with the reference SPD predicate (blocktri.py:24-32).
    Small single-block helper used by host-side setup code."""
    try:
        low = np.linalg.cholesky(mat)
    except np.linalg.LinAlgError as exc:
        raise NotPositiveDefiniteError(f"{what} is not positive definite") from exc
    if np.any(np.diag(low) <= PIVOT_FLOOR):
        raise NotPositiveDefiniteError(f"{what} has a non-positive pivot")
    return low


def is_spd(mat: np.ndarray) -> bool:
    try:
        chol_spd(mat)
        return True
    except NotPositiveDefiniteError:
        return False


def symmetrize(mat: np.ndarray) -> np.ndarray:
    """0.5 (M + M^T) over the last two axes (blocktri.py:43-45)."""
    return 0.5 * (mat + np.swapaxes(mat, -1, -2))


class _BlockList:
    """List-like per-block view of a stacked array; item assignment writes
    through to the stack."""

    __slots__ = ("_a",)

    def __init__(self, arr):
        self._a = arr

    def __len__(self):
        return self._a.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._a[j] for j in range(*i.indices(len(self)))]
        return self._a[i]

    def __setitem__(self, i, val):
        self._a[i] = val

    def __iter__(self):
        return (self._a[i] for i in range(self._a.shape[0]))

    def __add__(self, other):
        return list(self) + list(other)


class BlockTridiagonalMatrix:
    """Symmetric block matrix: K diagonal blocks, K-1 super-diagonal blocks
    (block ``off[i]`` at block position (i, i+1)); the sub-diagonal is implied
    by symmetry (blocktri.py:48-66)."""

    __slots__ = ("diag_stack", "off_stack")

    def __init__(self, diag, off):
        d = np.array(diag if not isinstance(diag, _BlockList) else diag._a, dtype=np.float64)
        if d.ndim != 3 or d.shape[1] != d.shape[2]:
            blocks = [np.asarray(b, dtype=np.float64) for b in diag]
            n = blocks[0].shape[0]
            for blk in blocks:
                if blk.shape != (n, n):
                    raise ValueError(f"inconsistent block shape {blk.shape}, expected {(n, n)}")
            d = np.stack(blocks)
        n = d.shape[1]
        off_list = off._a if isinstance(off, _BlockList) else off
        if len(off_list) == 0:
            o = np.zeros((0, n, n))
        else:
            try:
                o = np.array(off_list, dtype=np.float64)
            except ValueError:
                o = None
            if o is None or o.ndim != 3:
                blocks = [np.asarray(b, dtype=np.float64) for b in off_list]
                for blk in blocks:
                    if blk.shape != (n, n):
                        raise ValueError(f"inconsistent block shape {blk.shape}, expected {(n, n)}")
                o = np.stack(blocks)
        if o.shape[0] != d.shape[0] - 1:
            raise ValueError(f"expected {d.shape[0] - 1} off blocks, got {o.shape[0]}")
        if o.shape[1:] != (n, n):
            raise ValueError(f"inconsistent block shape {o.shape[1:]}, expected {(n, n)}")
        self.diag_stack = np.ascontiguousarray(d)
        self.off_stack = np.ascontiguousarray(o)

    # ---- list-of-blocks compatibility
    @property
    def diag(self):
        return _BlockList(self.diag_stack)

    @property
    def off(self):
        return _BlockList(self.off_stack)

    @property
    def nblocks(self) -> int:
        return self.diag_stack.shape[0]

    @property
    def block_size(self) -> int:
        return self.diag_stack.shape[1]

    @property
    def dim(self) -> int:
        return self.nblocks * self.block_size

    @classmethod
    def zeros(cls, nblocks: int, block_size: int) -> "BlockTridiagonalMatrix":
        return cls(np.zeros((nblocks, block_size, block_size)),
                   np.zeros((max(nblocks - 1, 0), block_size, block_size)))

    @classmethod
    def from_stacks(cls, diag: np.ndarray, off: np.ndarray) -> "BlockTridiagonalMatrix":
        return cls(diag, off)

    @classmethod
    def from_dense(cls, dense: np.ndarray, block_size: int) -> "BlockTridiagonalMatrix":
        n = block_size
        K = dense.shape[0] // n
        d = np.stack([dense[i * n:(i + 1) * n, i * n:(i + 1) * n] for i in range(K)])
        if K > 1:
            o = np.stack([dense[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] for i in range(K - 1)])
        else:
            o = np.zeros((0, n, n))
        return cls(d, o)

    def dense(self) -> np.ndarray:
        n, K = self.block_size, self.nblocks
        out = np.zeros((K * n, K * n))
        for i in range(K):
            out[i * n:(i + 1) * n, i * n:(i + 1) * n] = self.diag_stack[i]
        for i in range(K - 1):
            out[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] = self.off_stack[i]
            out[(i + 1) * n:(i + 2) * n, i * n:(i + 1) * n] = self.off_stack[i].T
        return out

    def copy(self) -> "BlockTridiagonalMatrix":
        return BlockTridiagonalMatrix(self.diag_stack.copy(), self.off_stack.copy())

    def symmetrized(self) -> "BlockTridiagonalMatrix":
        """Diagonal blocks averaged with their transpose (blocktri.py:112-115)."""
        return BlockTridiagonalMatrix(symmetrize(self.diag_stack), self.off_stack.copy())

    def matvec(self, x: np.ndarray) -> np.ndarray:
        """Same accumulation order as blocktri.py:117-127 (diag, then the
        transposed previous off block, then the next off block)."""
        K, n = self.nblocks, self.block_size
        xb = np.asarray(x, dtype=np.float64).reshape(K, n)
        out = np.einsum("kij,kj->ki", self.diag_stack, xb)
        if K > 1:
            out[1:] += np.einsum("kji,kj->ki", self.off_stack, xb[:-1])
            out[:-1] += np.einsum("kij,kj->ki", self.off_stack, xb[1:])
        return out.reshape(-1)

    def quad_form(self, x: np.ndarray) -> float:
        x = np.asarray(x, dtype=np.float64).reshape(-1)
        return float(x @ self.matvec(x))

    def __add__(self, other: "BlockTridiagonalMatrix") -> "BlockTridiagonalMatrix":
        return BlockTridiagonalMatrix(self.diag_stack + other.diag_stack,
                                      self.off_stack + other.off_stack)

    def scaled(self, alpha: float) -> "BlockTridiagonalMatrix":
        return BlockTridiagonalMatrix(alpha * self.diag_stack, alpha * self.off_stack)

    def add_to_diag_block(self, i: int, blk: np.ndarray) -> None:
        self.diag_stack[i] = self.diag_stack[i] + blk

    def add_to_off_block(self, i: int, blk: np.ndarray) -> None:
        self.off_stack[i] = self.off_stack[i] + blk

    def __repr__(self) -> str:
        return f"BlockTridiagonalMatrix(nblocks={self.nblocks}, block_size={self.block_size})"


def _stacks(mat: BlockTridiagonalMatrix):
    return N.f64(mat.diag_stack), N.f64(mat.off_stack)


def logdet_block_tridiag(mat: BlockTridiagonalMatrix) -> float:
    """log det via forward Schur pivots, on the GPU (blocktri.py:151-174).
    Raises NotPositiveDefiniteError naming the failing pivot block."""
    lib = N.load()
    d, o = _stacks(mat)
    out = np.zeros(1)
    where = np.zeros(1, dtype=np.int64)
    code = N.check(lib.gvp_logdet_block_tridiag(N.ptr(d), N.ptr(o), mat.nblocks, mat.block_size,
                                                N.ptr(out), N.ptr(where)), "logdet_block_tridiag")
    if code == N.GVP_ERR_NOT_SPD:
        raise NotPositiveDefiniteError(f"pivot block {int(where[0])} is not positive definite")
    return float(out[0])


def forward_schur_chols(mat: BlockTridiagonalMatrix) -> list:
    """Cholesky factors of the forward Schur pivots S_0 = D_0, S_i = D_i -
    U_{i-1}' S_{i-1}^-1 U_{i-1}, on the GPU (blocktri.py:151-165)."""
    lib = N.load()
    d, o = _stacks(mat)
    n, K = mat.block_size, mat.nblocks
    out = np.zeros((K, n, n))
    where = np.zeros(1, dtype=np.int64)
    code = N.check(lib.gvp_forward_schur_chols(N.ptr(d), N.ptr(o), K, n, N.ptr(out), N.ptr(where)),
                   "forward_schur_chols")
    if code == N.GVP_ERR_NOT_SPD:
        raise NotPositiveDefiniteError(f"pivot block {int(where[0])} is not positive definite")
    return list(out)


def is_spd_block_tridiag(mat: BlockTridiagonalMatrix) -> bool:
    try:
        logdet_block_tridiag(mat)
        return True
    except NotPositiveDefiniteError:
        return False
