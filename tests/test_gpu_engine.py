"""GPU engine (csrc/engine.cu): whole Algorithm-1 runs vs the reference's
recorded runs, and batch == independent single runs."""

import numpy as np
import pytest

import gvp_oracle as O
from conftest import golden, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-9
MEAN_TOL_LONG = 2e-6  # iterate of an N >= 500 chain after several ill-conditioned mean solves


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2411_03416_b200 as P

    assert P.HAVE_EXTENSION
    return P


def c1_env(P):
    sdf = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                      cell_size=0.05)
    return P.Environment(sdf=sdf, model=P.CollisionModel(radius_eps=0.2, sigma_obs=8.0))


def test_short_run_matches_reference_records(P):
    """Reference test scene (test_optimizer.py:158-163), N=15, default config,
    25 iterations (tests/golden runs.npz t15)."""
    g = golden("runs")
    sdf = P.rasterize([P.sdf.Disc(center=np.array([1.0, 0.75]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                      cell_size=0.05)
    env = P.Environment(sdf=sdf, model=P.CollisionModel(radius_eps=0.2, sigma_obs=8.0))
    res = P.run_pgvimp(P.point_robot_lti(2)(15, 0.2), env, P.OptimizerConfig(max_iters=25), np.zeros(4),
                       np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
    keys = list(g["record_keys"])
    got = np.array([[r[k] for k in keys] for r in res.records])
    ref = g["t15_records"]
    assert got.shape == ref.shape
    assert np.array_equal(got[:, 0], ref[:, 0])  # identical beta sequence
    assert np.array_equal(got[:, 1], ref[:, 1])  # identical temperature schedule
    assert rel_err(got[:, 2:6], ref[:, 2:6]) <= TOL
    assert rel_err(res.final.mean.reshape(16, 4), g["t15_final_mean"]) <= TOL
    assert rel_err(np.stack(res.marginals.covs), g["t15_final_covs"]) <= TOL
    assert res.converged == bool(g["t15_meta"][0]) and res.iterations == int(g["t15_meta"][1])


@pytest.mark.slow
def test_c1_converges_like_reference(P):
    """C1 pinned: reference converges in 94 iterations."""
    g = golden("runs")
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=600)
    res = P.run_pgvimp(P.point_robot_lti(2)(50, 3.0 / 50), c1_env(P), cfg, np.zeros(4),
                       np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
    ref = g["c1_records"]
    keys = list(g["record_keys"])
    got = np.array([[r[k] for k in keys] for r in res.records])
    assert res.converged and res.iterations == int(g["c1_meta"][1])
    assert np.array_equal(got[:, 0], ref[:, 0])
    assert rel_err(got[:, 5], ref[:, 5]) <= TOL
    assert rel_err(res.final.mean.reshape(51, 4), g["c1_final_mean"]) <= TOL
    assert rel_err(np.stack(res.marginals.covs), g["c1_final_covs"]) <= TOL


def test_obstacle_free_converges_to_prior(P):
    """test_optimizer.py:167-175 on the engine (env=None)."""
    sys_ltv = P.point_robot_lti(2)(20, 0.2)
    prior = P.assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
    cfg = P.OptimizerConfig(temp_low=1.0, temp_high=1.0, max_iters=300, kl_bound=10.0)
    res = P.run_pgvimp(sys_ltv, None, cfg, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
    assert res.converged
    assert np.linalg.norm(res.final.mean - prior.mean) <= 1e-5 * np.linalg.norm(prior.mean)


def test_batch_equals_single_runs(P):
    """B plans in one engine give bit-identical results to B=1 runs."""
    env = c1_env(P)
    sys_ltv = P.point_robot_lti(2)(30, 0.1)
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=12)
    rng = np.random.default_rng(5)
    goals = np.tile(np.array([2.0, 1.5, 0.0, 0.0]), (6, 1))
    goals[:, :2] += rng.uniform(-0.3, 0.3, size=(6, 2))
    batch = P.run_pgvimp_batch(sys_ltv, env, cfg, np.zeros(4), goals, 1.0, 1e-3)
    assert np.all(batch.status == 0)
    # the batch's own per-plan priors (optimizer.batch_problem); each plan alone
    from dataclasses import replace

    from paper_2411_03416_b200.optimizer import batch_problem

    base, info, pmean, _ = batch_problem(sys_ltv, np.zeros(4), goals, 1.0, 1e-3, cfg)
    own = P.assemble_prior(sys_ltv, np.zeros(4), goals[3], 1.0, 1e-3)  # vs a separate assembly
    assert np.abs(info[3].reshape(-1) - own.info).max() <= 1e-15 * np.abs(own.info).max()
    assert np.abs(pmean[3].reshape(-1) - own.mean).max() <= 1e-6 * np.abs(own.mean).max()
    for b in range(6):
        prior_b = replace(base, info=info[b].reshape(-1), mean=pmean[b].reshape(-1), goal=goals[b])
        single = P.run_pgvimp(sys_ltv, env, cfg, np.zeros(4), goals[b], 1.0, 1e-3, prior=prior_b)
        assert batch.iterations[b] == single.iterations
        assert np.array_equal(batch.mean[b].reshape(-1), single.final.mean)
        assert np.array_equal(batch.covs[b], np.stack(single.marginals.covs))


def test_engine_matches_oracle_driver(P):
    """A few C1 iterations: engine records vs the oracle's restated driver."""
    env = c1_env(P)
    sys_ltv = P.point_robot_lti(2)(50, 3.0 / 50)
    prior = P.assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=6)
    res = P.run_pgvimp(sys_ltv, env, cfg, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3, prior=prior)
    rule = P.smolyak_rule(3, 4)
    pr = {"diag": prior.prec.diag_stack, "off": prior.prec.off_stack, "info": prior.info.reshape(51, 4),
          "mean": prior.mean.reshape(51, 4)}
    ref = O.run_pgvimp(pr, env.sdf.values, env.sdf.origin, 0.05, 0.2, 8.0, rule.points, rule.weights,
                       kl_bound=10.0, beta_max=0.5, max_iters=6, x0=np.zeros(4), goal=np.array([2.0, 1.5, 0, 0]))
    assert [r["beta"] for r in res.records] == [r["beta"] for r in ref["records"]]
    for a, b in zip(res.records, ref["records"]):
        for k in ("prior_cost", "collision_cost", "entropy_cost", "total_cost"):
            assert abs(a[k] - b[k]) <= TOL * max(1.0, abs(b[k])), (k, a[k], b[k])


def _c2_env(P):
    from paper_2411_03416_b200.sdf import Box
    sdf = P.rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                       Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                      bounds=[[-2, 12], [-2, 12]], cell_size=0.05)
    return P.Environment(sdf=sdf, model=P.CollisionModel(radius_eps=0.2, sigma_obs=8.0))


def test_c2_config_matches_reference(P):
    """C2: N=500, k_q=5 (57-projection factor kernel), 4 iterations."""
    g = golden("configs")
    cfg = P.OptimizerConfig(k_q=5, kl_bound=10.0, beta_max=0.5, max_iters=4)
    res = P.run_pgvimp(P.point_robot_lti(2)(500, 10.0 / 500), _c2_env(P), cfg, np.zeros(4),
                       np.array([10.0, 10.0, 0, 0]), 1.0, 1e-3)
    keys = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
            "mean_shift"]
    got = np.array([[r[k] for k in keys] for r in res.records])
    assert np.array_equal(got[:, 0], g["c2_records"][:, 0])
    assert rel_err(got[:, 2:7], g["c2_records"][:, 2:7]) <= TOL
    # the mean solve S mu' = rhs has cond ~1e10 at N = 500 (sigma_b = 1e-3 anchors): two correct fp64
    # solvers agree to ~cond * eps on the iterate (the p500 prior-mean test shows the reference itself
    # 1.3e-9 from the exact solve after ONE solve); the records above stay within 1e-9
    assert rel_err(res.final.mean.reshape(501, 4), g["c2_final_mean"]) <= MEAN_TOL_LONG


def test_c5_bench_plan_matches_reference(P):
    """Plan 0 of the bench workload (C5: N=1000, k_q=3, C2 map): the first
    iteration's probe log against the reference's own (tests/golden configs).

    At N=1000 the reference's KL is itself only good to ~1e-5 relative: its
    trace_product (gbp.py:109-120) cancels terms ~1e4 down to ~4e3, so two
    implementations of the same marginals sweep differ by 1e-4 in KL (and the
    reference's Cython and numpy factor backends differ by 8e-6 on this very
    probe). Decisions must agree outside that band; the probe right at the
    bound (margin 3e-6) is the reference's coin flip. DESIGN.md §5."""
    g = golden("configs")
    ref = g["c5p_probes1"]
    noise = 2e-4  # absolute KL noise of the reference here (2x its backend spread)
    env = _c2_env(P)
    sys_ltv = P.point_robot_lti(2)(1000, 10.0 / 1000)
    prior = P.assemble_prior(sys_ltv, np.zeros(4), g["c5p_goal"], 1.0, 1e-3)
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=2)
    K = 1001
    eng = P.PlanBatch(1, K, 4, env.sdf, env.model, P.smolyak_rule(3, 4), cfg)
    eng.trace_probes(64)
    init = np.linspace(0, 1, K)[None, :, None] * g["c5p_goal"][None, None, :]
    eng.load(prior.prec.diag_stack, prior.prec.off_stack, prior.info.reshape(1, K, 4), prior.mean.reshape(1, K, 4),
             init)
    eng.step(1, sync=True)
    got = eng.probes()[0]
    eng.close()
    for j, (rb, rs, rk) in enumerate(ref):
        assert j < len(got)
        gb, gs, gk = got[j]
        assert gb == rb and gs == rs, j
        if np.isfinite(rk):
            assert abs(gk - rk) <= noise + 1e-5 * abs(rk), (j, gk, rk)
            if abs(rk - 10.0) <= noise:
                break  # inside the reference's own noise band: the searches may part here
    else:
        assert len(got) == len(ref)


def test_profiled_iterations_match_graphed_ones(P):
    """gvp_engine_step_profiled_ex (the bench's per-kernel timing) runs the
    same iteration kernel by kernel: records identical to the CUDA-graph
    path's, six non-negative buckets, and the 4-bucket form folds them."""
    env = c1_env(P)
    sys_ltv = P.point_robot_lti(2)(50, 3.0 / 50)
    goal = np.array([2.0, 1.5, 0.0, 0.0])
    prior = P.assemble_prior(sys_ltv, np.zeros(4), goal, 1.0, 1e-3)
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=12)
    K = 51
    init = np.linspace(0, 1, K)[None, :, None] * goal[None, None, :]
    recs = []
    for mode in ("graph", "ex", "four"):
        eng = P.PlanBatch(1, K, 4, env.sdf, env.model, P.smolyak_rule(3, 4), cfg)
        eng.load(prior.prec.diag_stack, prior.prec.off_stack, prior.info.reshape(1, K, 4),
                 prior.mean.reshape(1, K, 4), init)
        if mode == "graph":
            eng.step(6, sync=True)
        elif mode == "ex":
            ms = np.zeros(6)
            for _ in range(6):
                ms += eng.step_profiled_ex(1)
            assert ms.shape == (6,) and np.all(ms >= 0.0) and ms[1] > 0.0 and ms[2] > 0.0
        else:
            ms4 = np.zeros(4)
            for _ in range(6):
                ms4 += eng.step_profiled(1)
            assert np.all(ms4 >= 0.0) and ms4[0] > 0.0
        recs.append(eng.records()[0][:6])
        eng.close()
    assert np.array_equal(recs[0], recs[1], equal_nan=True)
    assert np.array_equal(recs[0], recs[2], equal_nan=True)


def test_boundary_load_matches_host_batch_problem(P):
    """gvp_engine_load_boundary (the per-plan info / prior mean / initial mean
    expanded on the device from the boundary states) solves the same batch
    as gvp_engine_load of optimizer.batch_problem's host arrays."""
    from paper_2411_03416_b200.optimizer import batch_parts, batch_problem

    env = c1_env(P)
    sys_ltv = P.point_robot_lti(2)(50, 3.0 / 50)
    rng = np.random.default_rng(7)
    B = 9  # odd: the engine pads a copy of plan 0
    x0s = np.zeros((B, 4))
    x0s[:, :2] = rng.uniform(-0.2, 0.2, (B, 2))
    goals = np.tile(np.array([2.0, 1.5, 0.0, 0.0]), (B, 1))
    goals[:, :2] += rng.uniform(-0.3, 0.3, (B, 2))
    cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=8)
    K = 51
    base, info, pmean, init = batch_problem(sys_ltv, x0s, goals, 1.0, 1e-3, cfg)
    parts = batch_parts(sys_ltv, x0s, goals, 1.0, 1e-3)
    out = []
    for mode in ("host", "boundary"):
        eng = P.PlanBatch(B, K, 4, env.sdf, env.model, P.smolyak_rule(3, 4), cfg, shared_prior=True)
        if mode == "host":
            eng.load(base.prec.diag_stack, base.prec.off_stack, info, pmean, init)
        else:
            b0, r0, rg, an, xa, ga = parts
            eng.load_boundary(b0.prec.diag_stack, b0.prec.off_stack, b0.info, b0.mean, r0, rg, an, xa, ga)
        m0 = eng.mean().copy()
        eng.step(8, sync=True)
        out.append((m0, eng.records(), eng.mean()))
        eng.close()
    assert rel_err(out[1][0], out[0][0]) <= 1e-14  # the straight-line initial means
    assert np.array_equal(out[1][1][:, :, 0], out[0][1][:, :, 0], equal_nan=True)  # beta sequences
    fin = np.isfinite(out[0][1][:, :, 2])
    assert rel_err(out[1][1][:, :, 2:6][fin], out[0][1][:, :, 2:6][fin]) <= 1e-9
    assert rel_err(out[1][2], out[0][2]) <= 1e-9
