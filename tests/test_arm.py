"""7-DOF sphere-arm collision factor: the CPU oracle's
self-consistency (no reference model exists — parity unpinned by a reference)
and the CUDA kernel against the oracle."""

import numpy as np
import pytest

import arm_oracle as AO
from conftest import rel_err


def _scene(P):
    sdf = P.rasterize([P.sdf.Disc(center=np.array([0.45, 0.0, 0.55]), radius=0.15),
                       P.sdf.Box(center=np.array([0.4, 0.35, 0.3]), halfextents=np.array([0.1, 0.1, 0.25]))],
                      bounds=[[-1.0, 1.0], [-1.0, 1.0], [0.0, 1.2]], cell_size=0.04)
    return sdf, P.CollisionModel(radius_eps=0.05, sigma_obs=10.0)


def _factors(F, seed):
    rng = np.random.default_rng(seed)
    means = np.concatenate([rng.uniform(-1.2, 1.2, size=(F, 7)), rng.normal(0, 0.3, size=(F, 7))], axis=1)
    chols = []
    for f in range(F):
        a = rng.normal(size=(14, 14))
        cov = (a @ a.T / 14 + np.eye(14)) * (0.002 if f % 2 else 0.02)
        chols.append(np.linalg.cholesky(cov))
    return means, np.stack(chols)


def test_projection_tables_reproduce_rule_moments():
    import paper_2411_03416_b200 as P

    rule = P.smolyak_rule(3, 14)
    t = P.arm_projection_tables(rule)
    assert len(t.proj) == 113 and t.cnt.sum() == rule.npoints          # Q = 421, Q_p = 113
    assert np.isclose(t.mom[:, 0].sum(), rule.weights.sum(), rtol=0, atol=1e-12)
    assert np.allclose(t.mom[:, 1:15].sum(0), rule.weights @ rule.points, atol=1e-12)
    r, c = np.tril_indices(14)
    full = (rule.points.T * rule.weights) @ rule.points
    assert np.allclose(t.mom[:, 15:].sum(0), full[r, c], atol=1e-12)


def test_oracle_kinematics_consistency():
    import paper_2411_03416_b200 as P

    arm = P.panda_like()
    rng = np.random.default_rng(0)
    reach = np.sum(np.abs(arm.dh[:, 0])) + np.sum(np.abs(arm.dh[:, 1])) + 0.1
    for _ in range(20):
        q = rng.uniform(-np.pi, np.pi, 7)
        fr = AO.link_frames(arm.dh, arm.base, q)
        for F in fr:
            assert np.allclose(F[:3, :3] @ F[:3, :3].T, np.eye(3), atol=1e-12)
        c = AO.sphere_centers(arm.dh, arm.base, arm.sphere_link, arm.geom, q)
        assert np.all(np.linalg.norm(c - arm.base, axis=1) <= reach)
    # joint 1 rotates the whole arm about the base z axis
    q = rng.uniform(-1, 1, 7)
    q2 = q.copy()
    q2[0] += 0.7
    c1 = AO.sphere_centers(arm.dh, arm.base, arm.sphere_link, arm.geom, q)
    c2 = AO.sphere_centers(arm.dh, arm.base, arm.sphere_link, arm.geom, q2)
    Rz = np.array([[np.cos(0.7), -np.sin(0.7), 0], [np.sin(0.7), np.cos(0.7), 0], [0, 0, 1]])
    assert np.allclose(c2, c1 @ Rz.T, atol=1e-12)


def test_oracle_degenerate_covariance_is_point_cost():
    import paper_2411_03416_b200 as P

    sdf, model = _scene(P)
    arm = P.panda_like()
    rule = P.smolyak_rule(3, 14)
    means, _ = _factors(3, 1)
    zeros = np.zeros((3, 14, 14))
    e0, e1, e2, _ = AO.arm_factor_expectations(means, zeros, rule.points, rule.weights, sdf.values, sdf.origin,
                                               sdf.cell_size, arm.dh, arm.base, arm.sphere_link, arm.geom,
                                               model.radius_eps, model.sigma_obs)
    for f in range(3):
        psi, _ = AO.arm_cost(arm.dh, arm.base, arm.sphere_link, arm.geom, sdf.values, sdf.origin, sdf.cell_size,
                             model.radius_eps, model.sigma_obs, means[f, :7])
        assert np.isclose(e0[f], psi * rule.weights.sum(), rtol=1e-12, atol=0)
        assert np.all(e1[f] == 0) and np.all(e2[f] == 0)


@pytest.mark.gpu
def test_arm_kernel_matches_oracle(gpu):
    import paper_2411_03416_b200 as P

    sdf, model = _scene(P)
    arm = P.panda_like()
    rule = P.smolyak_rule(3, 14)
    means, chols = _factors(6, 2)
    ref = AO.arm_factor_expectations(means, chols, rule.points, rule.weights, sdf.values, sdf.origin,
                                     sdf.cell_size, arm.dh, arm.base, arm.sphere_link, arm.geom,
                                     model.radius_eps, model.sigma_obs)
    got = P.arm_factor_expectations(means, chols, rule, sdf, arm, model)
    assert np.any(ref[0] > 0)  # the scene touches the arm
    for g, r in zip(got[:3], ref[:3]):
        assert rel_err(g, r) <= 1e-11
    assert got[3] == ref[3]


@pytest.mark.gpu
def test_arm_kernel_clear_of_obstacles_is_zero(gpu):
    import paper_2411_03416_b200 as P

    sdf = P.rasterize([], bounds=[[-1.0, 1.0], [-1.0, 1.0], [0.0, 1.2]], cell_size=0.1)
    arm = P.panda_like()
    means, chols = _factors(5, 3)
    e0, e1, e2, oob = P.arm_factor_expectations(means, chols, P.smolyak_rule(3, 14), sdf, arm,
                                                P.CollisionModel(0.05, 10.0))
    assert np.all(e0 == 0) and np.all(e1 == 0) and np.all(e2 == 0)
