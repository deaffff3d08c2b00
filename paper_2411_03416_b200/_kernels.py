"""Drop-in replacement of the reference's ``kernels`` module object.

The reference selects its factor kernel module in backend.py:14-20 and calls
``kernels.factor_expectations(...)`` (factors.py:195-207, bench.py:82-93); any
module exposing ``IS_COMPILED`` and this function can be injected through
``evaluate_all_factors(..., backend=...)``. This module forwards to the
sm_100a kernel ``factor_moments_kernel`` (csrc/factor_kernels.cu) through the
C ABI ``gvp_factor_expectations`` — same arguments, same outputs, and the
same bits as the compiled reference kernel.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

IS_COMPILED = True


def factor_expectations(means, chols, points, weights, grid_arr, origin_arr, cell_size,
                        radius_eps, sigma_obs, pos_dim, num_threads=1):
    """Hinge-potential quadrature moments for every factor
    (_kernels.pyx:132-177). Returns (e0 (F,), e1 (F, n), e2 (F, n, n), oob).

    ``num_threads`` is accepted for interface parity; the GPU evaluates all
    factors concurrently and the per-factor reduction order is fixed, so the
    result is identical for any value (the reference's serial == parallel
    contract, test_factors.py:235-243)."""
    if num_threads < 0:
        raise ValueError("thread count must be >= 0")
    lib = N.load()
    means = np.asarray(means)
    chols = np.asarray(chols)
    if means.dtype != np.float64 or chols.dtype != np.float64:
        raise ValueError("Buffer dtype mismatch, expected 'double'")  # memoryview contract
    if not (means.flags.c_contiguous and chols.flags.c_contiguous):
        raise ValueError("ndarray is not C-contiguous")
    points = N.f64(points)
    weights = N.f64(weights).reshape(-1)
    grid = N.f64(grid_arr)
    origin = N.f64(origin_arr).reshape(-1)
    nfac, n = means.shape
    if chols.shape != (nfac, n, n) or points.shape[1] != n or weights.shape[0] != points.shape[0]:
        raise ValueError("inconsistent factor/rule shapes")
    e0 = np.empty(nfac)
    e1 = np.empty((nfac, n))
    e2 = np.empty((nfac, n, n))
    oob = np.zeros(1, dtype=np.int64)
    shape = np.asarray(grid.shape, dtype=np.int64)
    N.check(lib.gvp_factor_expectations(
        N.ptr(means), N.ptr(chols), nfac, n, N.ptr(points), N.ptr(weights), points.shape[0],
        N.ptr(grid), grid.ndim, N.ptr(shape), N.ptr(origin), float(cell_size), float(radius_eps),
        float(sigma_obs), int(pos_dim), N.ptr(e0), N.ptr(e1), N.ptr(e2), N.ptr(oob)),
        "factor_expectations")
    return e0, e1, e2, int(oob[0])
