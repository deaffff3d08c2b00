"""Signed-distance maps on the device: rasterisation
bit-identical to the reference's rasterize, and the per-plan map bank of the
engine (batched plans on different maps == independent single-map runs)."""

import os
import sys

import numpy as np
import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
pytestmark = pytest.mark.gpu


def _ref_sdf():
    if not os.path.isdir(os.path.join(REF, "gvplan")):
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, REF)
    try:
        from gvplan import sdf as R
    finally:
        sys.path.remove(REF)
    return R


SCENES = [
    ("c2", [("box", (5, 1.2), (0.3, 3.4)), ("box", (5, 8.8), (0.3, 3.4))], [[-2, 12], [-2, 12]], 0.05),
    ("mixed", [("disc", (1.1, 0.55), 0.45), ("box", (2.0, -0.5), (0.7, 0.2)), ("disc", (-1.0, 2.0), 1.3)],
     [[-2, 4], [-2, 4]], 0.05),
    ("empty", [], [[0, 1], [0, 2]], 0.25),
    ("3d", [("disc", (0.5, 0.5, 0.5), 0.3), ("box", (1.5, 1.0, 0.2), (0.2, 0.4, 0.3))],
     [[0, 2], [0, 1.5], [0, 1]], 0.05),
]


def _prims(mod, spec):
    out = []
    for kind, c, r in spec:
        out.append(mod.Disc(center=np.array(c, float), radius=r) if kind == "disc"
                   else mod.Box(center=np.array(c, float), halfextents=np.array(r, float)))
    return out


@pytest.mark.parametrize("name,spec,bounds,cell", SCENES, ids=[s[0] for s in SCENES])
def test_rasterize_device_bitwise(gpu, name, spec, bounds, cell):
    import paper_2411_03416_b200 as P

    R = _ref_sdf()
    ref = R.rasterize(_prims(R, spec), bounds, cell)
    got = P.rasterize_device(_prims(P.sdf, spec), bounds, cell)
    assert got.values.shape == ref.values.shape
    assert np.array_equal(got.values, ref.values)
    assert np.array_equal(got.origin, ref.origin) and got.cell_size == ref.cell_size


def _scene(P):
    sys_ltv = P.point_robot_lti(2)(15, 0.2)
    prior = P.assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
    K = 16
    maps_spec = [[P.sdf.Disc(center=np.array([1.0, 0.75]), radius=0.45)],
                 [P.sdf.Disc(center=np.array([0.8, 0.9]), radius=0.35),
                  P.sdf.Box(center=np.array([1.6, 0.4]), halfextents=np.array([0.2, 0.3]))]]
    maps = [P.rasterize(m, [[-2, 4], [-2, 4]], 0.05) for m in maps_spec]
    init = np.linspace(0, 1, K)[None, :, None] * np.array([2.0, 1.5, 0, 0])[None, None, :]
    return prior, K, maps_spec, maps, init


def _run(P, prior, K, sdf, nplans, iters, bank=None, raster=None):
    cfg = P.OptimizerConfig(max_iters=iters)
    eng = P.PlanBatch(nplans, K, 4, sdf, P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4), cfg)
    if bank is not None:
        eng.set_map_bank(*bank)
    if raster is not None:
        eng.raster_map_bank(*raster)
    info = np.repeat(prior.info.reshape(1, K, 4), nplans, 0)
    pm = np.repeat(prior.mean.reshape(1, K, 4), nplans, 0)
    init = np.repeat((np.linspace(0, 1, K)[:, None] * np.array([2.0, 1.5, 0, 0]))[None], nplans, 0)
    eng.load(prior.prec.diag_stack, prior.prec.off_stack, info, pm, init)
    eng.run()
    st, rec = eng.state(), eng.records()
    eng.close()
    return st, rec


def test_map_bank_plans_match_single_map_runs(gpu):
    import paper_2411_03416_b200 as P

    prior, K, maps_spec, maps, _ = _scene(P)
    plan_map = np.array([0, 1, 1, 0, 1])
    st, rec = _run(P, prior, K, maps[0], 5, 12, bank=(maps, plan_map))
    singles = [_run(P, prior, K, maps[m], 1, 12) for m in range(2)]
    for b, m in enumerate(plan_map):
        s1, r1 = singles[m]
        assert np.array_equal(st["mean"][b], s1["mean"][0])
        assert np.array_equal(np.nan_to_num(rec[b]), np.nan_to_num(r1[0]))
    assert not np.array_equal(st["mean"][0], st["mean"][1])  # the two maps really differ


def test_raster_bank_equals_host_bank(gpu):
    import paper_2411_03416_b200 as P

    prior, K, maps_spec, maps, _ = _scene(P)
    plan_map = np.array([1, 0, 1])
    a = _run(P, prior, K, maps[0], 3, 8, bank=(maps, plan_map))
    b = _run(P, prior, K, maps[0], 3, 8, raster=(maps_spec, plan_map))
    assert np.array_equal(a[0]["mean"], b[0]["mean"])
    with pytest.raises(ValueError):
        _run(P, prior, K, maps[0], 3, 2, bank=(maps, np.array([0, 2, 1])))
