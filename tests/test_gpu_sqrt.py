"""gaussian_sqrt's fallbacks (quadrature.py:164-181) inside the device factor
stage, against the reference (tests/golden/sqrt_cases.npz,
make_trace_goldens.py sqrt): the 1e-10 jitter retry when Cholesky fails, and
the eigendecomposition root (Jacobi on device) whose clipped eigenvalue makes
the reference's _moment_gradients raise numpy.linalg.LinAlgError."""

import numpy as np
import pytest

from conftest import golden, rel_err

pytestmark = pytest.mark.gpu


def _scene(P):
    sdf = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                      cell_size=0.05)
    prior = P.assemble_prior(P.point_robot_lti(2)(50, 3.0 / 50), np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
    return sdf, P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4), prior.prec


def test_jitter_retry_matches_reference(gpu):
    import paper_2411_03416_b200 as P

    g = golden("sqrt_cases")
    sdf, model, rule, prec = _scene(P)
    marg = P.gbp.ChainMarginals.from_stacks(g["covs_jitter"], np.zeros((50, 4, 4)))
    fv = P.evaluate_all_factors(g["mean"].reshape(-1), prec, sdf, model, rule, marginals=marg)
    e = np.array([f.e_psi for f in fv])
    assert np.all(e[[10, 11]] > 0)  # the jittered knots' clouds reach the obstacle
    # the jittered covariances have an eigenvalue ~5e-11, so P^-1 ~ 2e10 and the
    # moment-form g_sigma cancels -e0 P^-1 / 2 against P^-1 E2 P^-1 / 2: bounded
    # by 1e-9 or 4x the reference's own Cython-vs-numpy spread on these inputs
    for key, got in (("e_psi", e), ("g_mu", np.stack([f.g_mu for f in fv])),
                     ("g_sigma", np.stack([f.g_sigma for f in fv]))):
        spread = rel_err(g["py_" + key], g[key])
        assert rel_err(got, g[key]) <= max(1e-9, 4 * spread), (key, rel_err(got, g[key]), spread)


def test_eigh_root_singular_raises_like_reference(gpu):
    import paper_2411_03416_b200 as P

    g = golden("sqrt_cases")
    assert str(g["eigh_raises"]).startswith("LinAlgError")
    sdf, model, rule, prec = _scene(P)
    marg = P.gbp.ChainMarginals.from_stacks(g["covs_eigh"], np.zeros((50, 4, 4)))
    with pytest.raises(np.linalg.LinAlgError, match="Singular matrix"):
        P.evaluate_all_factors(g["mean"].reshape(-1), prec, sdf, model, rule, marginals=marg)

