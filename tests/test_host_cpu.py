"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, and the host-side setup code (rules, maps, block-tridiagonal data
model, layouts) matches the reference's golden fixtures."""

import os
import re

import numpy as np
import pytest

from conftest import REPO, golden, rel_err


def declared_symbols():
    hdr = open(os.path.join(REPO, "include", "gvp_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(gvp_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2411_03416_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    missing = [s for s in names if not hasattr(lib, s)]
    assert not missing, missing
    # the python binding declares a signature for each of them
    assert set(names) <= set(_native.exported_symbols())


def test_library_reports_no_device_without_gpu():
    import torch

    from paper_2411_03416_b200 import _native

    lib = _native.load()
    assert lib.gvp_version().decode().startswith("gvp_b200")
    if not torch.cuda.is_available():
        assert lib.gvp_device_count() == 0


def test_gpu_entry_points_fail_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2411_03416_b200 as P
    from paper_2411_03416_b200._native import NativeLibraryError

    assert not P.HAVE_EXTENSION
    prec = P.BlockTridiagonalMatrix.zeros(3, 2)
    with pytest.raises(NativeLibraryError):
        P.gbp_marginals(prec)


def test_smolyak_rules_match_reference():
    from paper_2411_03416_b200 import smolyak_rule, tensor_rule

    g = golden("rules")
    for k, d in [(2, 4), (3, 4), (5, 4), (3, 6), (3, 3), (3, 14)]:
        r = smolyak_rule(k, d)
        assert np.array_equal(r.points, g[f"smolyak_{k}_{d}_points"])
        assert np.array_equal(r.weights, g[f"smolyak_{k}_{d}_weights"])
    for p, d in [(3, 4), (2, 4), (3, 1)]:
        r = tensor_rule(p, d)
        assert np.array_equal(r.points, g[f"tensor_{p}_{d}_points"])
        assert np.array_equal(r.weights, g[f"tensor_{p}_{d}_weights"])


def test_rasterized_maps_match_reference():
    from paper_2411_03416_b200.sdf import Box, Disc, rasterize

    g = golden("maps")
    s = rasterize([Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
    assert np.array_equal(s.values, g["c1"])
    s = rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                   Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                  bounds=[[-2, 12], [-2, 12]], cell_size=0.05)
    assert np.array_equal(s.values, g["c2"])
    assert np.array_equal(rasterize([], bounds=[[0, 1], [0, 2]], cell_size=0.25).values, g["empty"])


def test_host_interpolation_matches_oracle():
    import gvp_oracle as O

    from paper_2411_03416_b200.sdf import SignedDistanceField, distance_batch

    f = golden("factors")
    sdf = SignedDistanceField(origin=f["scene_origin"], cell_size=float(f["scene_cell"]), values=f["scene_grid"])
    pts = np.random.default_rng(0).uniform(-5, 5, size=(500, 2))
    v, o = distance_batch(sdf, pts)
    vo, oo = O.interp(f["scene_grid"], f["scene_origin"], float(f["scene_cell"]), pts)
    assert np.array_equal(v, vo) and o == oo


def test_block_tridiagonal_data_model():
    import gvp_oracle as O

    from paper_2411_03416_b200 import BlockTridiagonalMatrix

    g = golden("chain")
    d, o = g["a_diag"], g["a_off"]
    m = BlockTridiagonalMatrix(list(d), list(o))
    assert m.nblocks == 51 and m.block_size == 4 and m.dim == 204
    dense = m.dense()
    assert np.array_equal(dense, O.bt_dense(d, o))
    assert np.array_equal(BlockTridiagonalMatrix.from_dense(dense, 4).diag_stack, d)
    x = np.random.default_rng(1).normal(size=204)
    assert rel_err(m.matvec(x), dense @ x) <= 1e-13
    assert abs(m.quad_form(x) - x @ dense @ x) <= 1e-10 * abs(x @ dense @ x)
    m2 = m.copy()
    m2.add_to_diag_block(3, np.eye(4))
    assert np.array_equal(m2.diag[3], d[3] + np.eye(4)) and np.array_equal(m.diag[3], d[3])
    with pytest.raises(ValueError):
        BlockTridiagonalMatrix(list(d), list(o[:-1]))


def test_plan_minor_layout_roundtrip():
    from paper_2411_03416_b200.engine import from_plan_minor, to_plan_minor

    x = np.random.default_rng(2).normal(size=(5, 7, 4, 4))
    pm = to_plan_minor(x)
    assert pm.shape == (7, 4, 4, 5) and pm.flags.c_contiguous
    # element (b, i, r, c) at ((i*16 + r*4 + c) * B + b)
    assert pm.reshape(-1)[((3 * 16 + 2 * 4 + 1) * 5) + 4] == x[4, 3, 2, 1]
    assert np.array_equal(from_plan_minor(pm), x)


def test_optimizer_config_validation():
    from paper_2411_03416_b200 import OptimizerConfig

    OptimizerConfig().validate()
    for bad in (dict(kl_bound=0.0), dict(beta_min=1.0, beta_max=0.5), dict(temp_low=0.0),
                dict(max_iters=0), dict(init="nope")):
        with pytest.raises(ValueError):
            OptimizerConfig(**bad).validate()
