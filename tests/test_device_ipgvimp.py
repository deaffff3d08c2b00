"""iP-GVIMP on the device (csrc/slr_prior.cu): SLR and LTV
prior assembly against the reference's outputs / the host (scipy) path."""

import numpy as np
import pytest

from conftest import golden, rel_err

pytestmark = pytest.mark.gpu


def _quad_ltv(P, N=20, dt=0.25):
    x0, goal = np.zeros(6), np.array([10.0, 5.0, 0, 0, 0, 0])
    a = np.linspace(0, 1, N + 1)[:, None]
    nom = P.NominalTrajectory(means=(1 - a) * x0 + a * goal, covs=np.repeat(0.05 * np.eye(6)[None], N + 1, 0))
    return P.slr_linearize(P.planar_quadrotor(), nom, dt, P.smolyak_rule(3, 6)), x0, goal, nom


def test_device_slr_matches_reference(gpu):
    import paper_2411_03416_b200 as P

    g = golden("slr")
    nom = P.NominalTrajectory(g["lin_means"], g["lin_covs"])
    ltv = P.slr_linearize(P.planar_quadrotor(), nom, 0.1, P.smolyak_rule(3, 6), device=True)
    assert rel_err(np.stack([s.A for s in ltv.steps]), g["lin_A"]) <= 1e-12
    assert rel_err(np.stack([s.a for s in ltv.steps]), g["lin_a"]) <= 1e-12


def test_device_slr_equals_host_on_straight_line(gpu):
    import paper_2411_03416_b200 as P

    host, _, _, nom = _quad_ltv(P)
    dev = P.slr_linearize(P.planar_quadrotor(), nom, 0.25, P.smolyak_rule(3, 6), device=True)
    assert rel_err(np.stack([s.A for s in dev.steps]), np.stack([s.A for s in host.steps])) <= 1e-12
    assert rel_err(np.stack([s.a for s in dev.steps]), np.stack([s.a for s in host.steps])) <= 1e-12


def test_device_prior_matches_host_scipy_path(gpu):
    """Transition kernels and Grammians to ~1e-13; the assembled blocks carry
    the Grammian inverse's conditioning (cond Q ~ 5e6 here); the anchored
    mean is an ill-conditioned solve (a 1e-15 perturbation of expm moves it
    by ~1e-8, /tmp study in DESIGN §5), bounded accordingly."""
    import paper_2411_03416_b200 as P

    ltv, x0, goal, _ = _quad_ltv(P)
    host = P.assemble_prior(ltv, x0, goal, 0.5, 1e-3)
    dev = P.assemble_prior_device(ltv, x0, goal, 0.5, 1e-3)
    assert rel_err(np.stack(dev.phis), np.stack(host.phis)) <= 1e-14         # measured 1.9e-16
    assert rel_err(np.stack(dev.offsets), np.stack(host.offsets)) <= 1e-14
    assert rel_err(np.stack(dev.grammians), np.stack(host.grammians)) <= 1e-14  # 3.3e-16
    assert rel_err(dev.prec.diag_stack, host.prec.diag_stack) <= 1e-11  # 4.4e-13 (Q^-1, cond Q 5e6)
    assert rel_err(dev.prec.off_stack, host.prec.off_stack) <= 1e-11
    assert rel_err(dev.info, host.info) <= 1e-12
    assert rel_err(dev.flow_mean, host.flow_mean) <= 1e-12
    assert rel_err(dev.mean, host.mean) <= 1e-6  # 8.7e-9: ill-conditioned anchored solve


def test_device_prior_point_robot_rejected(gpu):
    import paper_2411_03416_b200 as P

    with pytest.raises(NotImplementedError):
        P.assemble_prior_device(P.point_robot_lti(2)(10, 0.1), np.zeros(4), np.ones(4), 1.0, 1e-3)


def test_device_ipgvimp_close_to_reference(gpu):
    """Whole Algorithm 2 with SLR + prior on the device vs the reference run
    (tests/golden slr.npz); tolerance = the reference's own backend spread
    scaled for the device expm."""
    import paper_2411_03416_b200 as P

    g, gp = golden("slr"), golden("slr_py")
    sdf = P.rasterize([P.sdf.Disc(center=np.array([5.0, 4.5]), radius=0.8)], bounds=[[-5, 15], [-5, 10]],
                      cell_size=0.05)
    env = P.Environment(sdf=sdf, model=P.CollisionModel(radius_eps=1.5, sigma_obs=6.0))
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0, temp_high=5.0, max_iters=15)
    res, log = P.run_ipgvimp(P.planar_quadrotor(), env, cfg, P.OuterConfig(max_outer=2), np.zeros(6),
                             np.array([10.0, 5.0, 0, 0, 0, 0]), dt=0.25, num_steps=20, q_c=0.5, sigma_b=1e-3,
                             device=True)
    nd = np.array([r["norm_diff"] for r in log])
    spread = rel_err(gp["ip_norm_diff"], g["ip_norm_diff"])
    assert rel_err(nd, g["ip_norm_diff"]) <= 10 * spread
    got = np.array([r["beta"] for r in res.records])
    assert np.array_equal(got, g["ip_records"][:, 0])
    assert rel_err(res.final.mean.reshape(21, 6), g["ip_final_mean"]) <= 1e-5
