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


def _joint_factors(F, seed):
    means, chols = _factors(F, seed)
    K = F + 2
    joint = np.zeros((K, 14))
    joint[1:K - 1] = means
    covs = np.stack([np.eye(14)] + [L @ L.T for L in chols] + [np.eye(14)])
    return joint, covs


@pytest.mark.gpu
def test_arm_factor_gradients_match_oracle(gpu):
    """gvp_arm_factor_grads (gaussian_sqrt -> moments -> _moment_gradients on
    the device) against the oracle's factor stage."""
    import paper_2411_03416_b200 as P

    sdf, model = _scene(P)
    arm = P.panda_like()
    rule = P.smolyak_rule(3, 14)
    env = P.ArmEnvironment(sdf, model, arm)
    joint, covs = _joint_factors(6, 4)
    e_psi, g_mu, g_s = env.factor_gradients(joint, covs, rule)
    r_e, r_gm, r_gs, _ = AO.arm_evaluate_factors(joint, covs, rule.points, rule.weights, sdf.values, sdf.origin,
                                                 sdf.cell_size, arm.dh, arm.base, arm.sphere_link, arm.geom,
                                                 model.radius_eps, model.sigma_obs)
    assert np.any(r_e > 0)
    assert rel_err(e_psi, r_e) <= 1e-10
    assert rel_err(g_mu, r_gm) <= 1e-9
    assert rel_err(g_s, r_gs) <= 1e-9
    env.close()


@pytest.mark.gpu
def test_arm_run_pgvimp_matches_oracle(gpu):
    """C3 shape at a test size: the 7-DOF arm (n = 14) planned end to end on
    the GPU (wide-block chain kernels + the arm factor stage) against the
    oracle's run_pgvimp with the arm factor stage: identical beta sequence,
    records within 1e-8 relative."""
    import gvp_oracle as O
    import paper_2411_03416_b200 as P

    sdf, model = _scene(P)
    arm = P.panda_like()
    N, dt = 10, 0.1
    x0 = np.zeros(14)
    goal = np.concatenate([[0.9, 0.6, 0.0, -0.8, 0.0, 1.0, 0.0], np.zeros(7)])
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=5)
    env = P.ArmEnvironment(sdf, model, arm)
    res = P.run_pgvimp(P.joint_double_integrator(N, dt), env, cfg, x0, goal, 1.0, 1e-3)
    env.close()
    rule = P.smolyak_rule(3, 14)
    A = np.zeros((14, 14))
    A[:7, 7:] = np.eye(7)
    B = np.zeros((14, 7))
    B[7:, :] = np.eye(7)
    prior = O.assemble_prior([A] * (N + 1), [np.zeros(14)] * (N + 1), [B] * (N + 1), dt, x0, goal, 1.0, 1e-3)
    fn = lambda m, c: AO.arm_evaluate_factors(m, c, rule.points, rule.weights, sdf.values, sdf.origin,  # noqa: E731
                                              sdf.cell_size, arm.dh, arm.base, arm.sphere_link, arm.geom,
                                              model.radius_eps, model.sigma_obs)
    ref = O.run_pgvimp(prior, None, None, None, None, None, rule.points, rule.weights, kl_bound=cfg.kl_bound,
                       beta_min=cfg.beta_min, beta_max=cfg.beta_max, temp_low=cfg.temp_low,
                       temp_high=cfg.temp_high, collision_tol=cfg.collision_tol, max_iters=cfg.max_iters,
                       tol_mean=cfg.tol_mean, tol_cost=cfg.tol_cost, init_cov_scale=cfg.init_cov_scale, x0=x0,
                       goal=goal, factor_fn=fn)
    assert res.iterations == ref["iterations"]
    assert any(r["collision_cost"] > 0 for r in ref["records"])
    for got, exp in zip(res.records, ref["records"]):
        assert got["beta"] == exp["beta"]
        for k in ("prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step", "mean_shift"):
            assert abs(got[k] - exp[k]) <= 1e-8 * max(1.0, abs(exp[k])), k
    assert rel_err(res.final.mean, ref["mean"].reshape(-1)) <= 1e-8
