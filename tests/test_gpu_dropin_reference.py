"""The drop-in proven through the REFERENCE's own code.

The unmodified reference (`gvplan`, built by oracle/build_ref.sh into
oracle/_ref) is imported as the caller; our `_kernels` module is handed to it
at its one native seam — per call (`evaluate_all_factors(..., backend=...)`,
factors.py:175,184) and as the module-level selection the maintainer's
backend.py switch makes (`factors.kernels`, backend.py:14-20). Because the
device factor_expectations reproduces the Cython kernel bit for bit, the
reference's whole run must be bit-identical with either kernel."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


@pytest.fixture(scope="module")
def gv(gpu):
    if not os.path.isdir(os.path.join(REF, "gvplan")):
        pytest.skip("oracle/_ref not built (oracle/build_ref.sh)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gvplan

    assert gvplan.HAVE_EXTENSION, "reference built without its Cython kernel"
    return gvplan


@pytest.fixture(scope="module")
def ours(gpu):
    from paper_2411_03416_b200 import _kernels

    assert _kernels.IS_COMPILED
    return _kernels


def c1_env(gv):
    from gvplan.sdf import Disc

    sdf = gv.rasterize([Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                       cell_size=0.05)
    return gv.Environment(sdf=sdf, model=gv.CollisionModel(0.2, 8.0))


def _factor_arrays(fv):
    return (np.array([f.e_psi for f in fv]), np.stack([f.g_mu for f in fv]), np.stack([f.g_sigma for f in fv]))


@pytest.mark.parametrize("k_q", [3, 5])
def test_reference_factor_stage_with_our_kernel(gv, ours, k_q):
    """gvplan.factors.evaluate_all_factors with backend=ours == with the
    reference's Cython kernel, bitwise (C1 map, N = 50, initial state and a
    perturbed state whose clouds reach the obstacle)."""
    from gvplan import optimizer as ro
    from gvplan.backend import kernels as cython_kernels
    from gvplan.factors import evaluate_all_factors

    env = c1_env(gv)
    sys_ltv = gv.point_robot_lti(2)(50, 3.0 / 50)
    prior = gv.assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
    cfg = gv.OptimizerConfig(k_q=k_q, kl_bound=10.0, beta_max=0.5)
    rule = gv.smolyak_rule(k_q, 4)
    cur = ro.initial_state(prior, cfg)
    rng = np.random.default_rng(7)
    for mean in (cur.mean, cur.mean + 0.3 * rng.normal(size=cur.mean.shape)):
        a = _factor_arrays(evaluate_all_factors(mean, cur.prec, env.sdf, env.model, rule, backend=cython_kernels))
        b = _factor_arrays(evaluate_all_factors(mean, cur.prec, env.sdf, env.model, rule, backend=ours))
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        assert np.max(a[0]) > 0.0  # the obstacle is actually hit


def test_reference_run_pgvimp_with_backend_switch(gv, ours):
    """The reference's run_pgvimp (C1, 10 iterations) with the backend switch
    of INTEGRATION.md §2 (factors.kernels -> ours): records and final state
    bit-identical to the stock reference run."""
    import gvplan.factors as rf

    env = c1_env(gv)
    sys_ltv = gv.point_robot_lti(2)(50, 3.0 / 50)
    goal = np.array([2.0, 1.5, 0, 0])
    cfg = gv.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=10)
    stock = gv.run_pgvimp(sys_ltv, env, cfg, np.zeros(4), goal, 1.0, 1e-3)
    saved = rf.kernels
    rf.kernels = ours
    try:
        swapped = gv.run_pgvimp(sys_ltv, env, cfg, np.zeros(4), goal, 1.0, 1e-3)
    finally:
        rf.kernels = saved
    keys = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
            "mean_shift"]
    a = np.array([[r[k] for k in keys] for r in stock.records])
    b = np.array([[r[k] for k in keys] for r in swapped.records])
    assert a.shape == (10, 8)
    assert np.array_equal(a, b)
    assert np.array_equal(stock.final.mean, swapped.final.mean)
    assert env.sdf.oob_count >= 0
