"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the dev container (where /root/reference exists):

    oracle/build_ref.sh                 # builds gvplan (+ Cython kernel) into oracle/_ref
    python tests/golden/make_goldens.py

Every array written here is an output of the unmodified reference package
(`gvplan`, /root/reference/pkg) on seeded inputs; the tests compare both the
CPU oracle (oracle/gvp_oracle.py) and the CUDA engine against them. The
fixtures are committed; this script (and /root/reference) is never needed on
the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

import gvplan  # noqa: E402
from gvplan import (  # noqa: E402
    BlockTridiagonalMatrix, CollisionModel, Environment, JointGaussian,
    OptimizerConfig, assemble_prior, gbp_marginals, gbp_mean_solve,
    logdet_block_tridiag, point_robot_lti, rasterize, run_pgvimp,
    select_step_size, smolyak_rule, tensor_rule,
)
from gvplan import optimizer as ref_opt  # noqa: E402
from gvplan.factors import assemble_joint_gradients, evaluate_all_factors, interior_collision_maps  # noqa: E402
from gvplan.quadrature import gaussian_sqrt  # noqa: E402
from gvplan.sdf import Box, Disc  # noqa: E402
from gvplan.backend import kernels  # noqa: E402

assert gvplan.HAVE_EXTENSION or os.environ.get("GVPLAN_PURE_PYTHON"), \
    "build the reference extension first (oracle/build_ref.sh)"


def stack_bt(m):
    return np.stack(m.diag), (np.stack(m.off) if m.off else np.zeros((0,) + m.diag[0].shape))


def random_spd_bt(rng, nblocks, n):
    """Same construction as the reference test helper (tests/helpers.py:13-23)."""
    dim = nblocks * n
    g = np.zeros((dim, dim))
    for i in range(nblocks):
        sl = slice(i * n, (i + 1) * n)
        g[sl, sl] = rng.normal(size=(n, n)) + 2.0 * np.eye(n)
        if i > 0:
            g[sl, slice((i - 1) * n, i * n)] = 0.4 * rng.normal(size=(n, n))
    return BlockTridiagonalMatrix.from_dense(g @ g.T + np.eye(dim), n)


def rules():
    out = {}
    for k, d in [(2, 4), (3, 4), (5, 4), (3, 6), (3, 3), (3, 14)]:
        r = smolyak_rule(k, d)
        out[f"smolyak_{k}_{d}_points"] = r.points
        out[f"smolyak_{k}_{d}_weights"] = r.weights
    for p, d in [(3, 4), (2, 4), (3, 1)]:
        r = tensor_rule(p, d)
        out[f"tensor_{p}_{d}_points"] = r.points
        out[f"tensor_{p}_{d}_weights"] = r.weights
    np.savez_compressed(os.path.join(HERE, "rules.npz"), **out)


def factor_scene(nblocks, spread=2.0):
    """The reference's factor test scene (tests/test_factors.py:213-225)."""
    rng = np.random.default_rng(123)
    sdf = rasterize([Disc(center=np.array([0.0, 0.0]), radius=0.8),
                     Disc(center=np.array([1.5, 1.0]), radius=0.5)],
                    bounds=[[-4, 4], [-4, 4]], cell_size=0.05)
    model = CollisionModel(radius_eps=0.2, sigma_obs=5.0)
    prec = random_spd_bt(rng, nblocks, 4)
    mean = np.zeros(nblocks * 4)
    mean[0::4] = np.linspace(-spread, spread, nblocks)
    mean[1::4] = np.linspace(-spread, spread, nblocks)
    return sdf, model, mean, prec


def factors():
    out = {}
    sdf, model, mean, prec = factor_scene(40)
    out["scene_grid"] = sdf.values
    out["scene_origin"] = sdf.origin
    out["scene_cell"] = np.array(sdf.cell_size)
    out["scene_model"] = np.array([model.radius_eps, model.sigma_obs])
    out["scene_mean"] = mean
    d, o = stack_bt(prec)
    out["scene_diag"], out["scene_off"] = d, o
    marg = gbp_marginals(prec)
    covs = np.stack(marg.covs)
    out["scene_covs"] = covs
    K, n = 40, 4
    for tag, rule in [("t34", tensor_rule(3, 4)), ("s34", smolyak_rule(3, 4)), ("s54", smolyak_rule(5, 4))]:
        for scale_tag, scale in [("", 1.0), ("_wide", 400.0)]:
            cv = covs * scale
            means = np.ascontiguousarray(mean.reshape(K, n)[1:K - 1])
            chols = np.stack([gaussian_sqrt(cv[i]) for i in range(1, K - 1)])
            e0, e1, e2, oob = kernels.factor_expectations(
                means, chols, rule.points, rule.weights, sdf.values, sdf.origin,
                sdf.cell_size, model.radius_eps, model.sigma_obs, pos_dim=2, num_threads=1)
            key = tag + scale_tag
            out[f"{key}_chols"] = chols
            out[f"{key}_e0"], out[f"{key}_e1"], out[f"{key}_e2"] = e0, e1, e2
            out[f"{key}_oob"] = np.array(oob)
            if scale == 1.0:
                # full factor stage (moment gradients, clamp) with the compiled kernel
                fg = evaluate_all_factors(mean, prec, sdf, model, rule, threads=1, marginals=marg)
                out[f"{key}_epsi"] = np.array([f.e_psi for f in fg])
                out[f"{key}_gmu"] = np.stack([f.g_mu for f in fg])
                out[f"{key}_gsigma"] = np.stack([f.g_sigma for f in fg])
    # 3D field, point3d state (n = 6)
    rng = np.random.default_rng(7)
    sdf3 = rasterize([Disc(center=np.array([0.5, 0.2, 0.1]), radius=0.6),
                      Box(center=np.array([-0.8, 0.6, -0.4]), halfextents=np.array([0.3, 0.5, 0.2]))],
                     bounds=[[-2, 2], [-1.5, 2], [-1.5, 1.5]], cell_size=0.1)
    rule = smolyak_rule(3, 6)
    F = 24
    means3 = np.zeros((F, 6))
    means3[:, 0] = np.linspace(-1.8, 1.8, F)
    means3[:, 1] = np.linspace(-1.2, 1.6, F)
    means3[:, 2] = np.linspace(-1.0, 1.0, F)
    means3[:, 3:] = rng.normal(size=(F, 3))
    chols3 = []
    for _ in range(F):
        a = rng.normal(size=(6, 6))
        chols3.append(np.linalg.cholesky(0.05 * (a @ a.T + 6 * np.eye(6)) / 6))
    chols3 = np.stack(chols3)
    e0, e1, e2, oob = kernels.factor_expectations(
        means3, chols3, rule.points, rule.weights, sdf3.values, sdf3.origin, sdf3.cell_size,
        0.3, 4.0, pos_dim=3, num_threads=1)
    out.update({"g3_grid": sdf3.values, "g3_origin": sdf3.origin, "g3_cell": np.array(sdf3.cell_size),
                "g3_means": means3, "g3_chols": chols3, "g3_e0": e0, "g3_e1": e1, "g3_e2": e2,
                "g3_oob": np.array(oob)})
    np.savez_compressed(os.path.join(HERE, "factors.npz"), **out)


def chain():
    out = {}
    for tag, seed, K, n in [("a", 17, 51, 4), ("b", 23, 20, 3), ("c", 5, 30, 6), ("d", 8, 12, 1), ("e", 31, 50, 4)]:
        rng = np.random.default_rng(seed)
        prec = random_spd_bt(rng, K, n)
        eta = rng.normal(size=K * n)
        d, o = stack_bt(prec)
        marg = gbp_marginals(prec)
        out[f"{tag}_diag"], out[f"{tag}_off"] = d, o
        out[f"{tag}_eta"] = eta.reshape(K, n)
        out[f"{tag}_covs"] = np.stack(marg.covs)
        out[f"{tag}_crosses"] = np.stack(marg.crosses)
        out[f"{tag}_mean"] = gbp_mean_solve(prec, eta).reshape(K, n)
        out[f"{tag}_logdet"] = np.array(logdet_block_tridiag(prec))
    np.savez_compressed(os.path.join(HERE, "chain.npz"), **out)


def probe_log():
    """Wrap the reference's probe internals to record (beta, feasible, kl)."""
    log = []
    orig_prox, orig_kl, orig_marg = ref_opt.proximal_update, ref_opt.kl_joint, ref_opt.gbp_marginals
    state = {}

    def prox(cur, prior, g_mu, g_sigma, beta, temp):
        state["beta"] = beta
        return orig_prox(cur, prior, g_mu, g_sigma, beta, temp)

    def marg(prec):
        try:
            return orig_marg(prec)
        except Exception:
            log.append((state["beta"], 0.0, np.inf))
            raise

    def kl(nxt, cur, m=None):
        v = orig_kl(nxt, cur, m)
        log.append((state["beta"], 1.0, v))
        return v

    ref_opt.proximal_update, ref_opt.kl_joint, ref_opt.gbp_marginals = prox, kl, marg
    return log, lambda: setattr(ref_opt, "proximal_update", orig_prox) or setattr(ref_opt, "kl_joint", orig_kl) or setattr(ref_opt, "gbp_marginals", orig_marg)


def c1_env():
    """Disc((1.1, 0.55), 0.45) on [-2,4]^2, cell 0.05."""
    sdf = rasterize([Disc(center=np.array([1.1, 0.55]), radius=0.45)],
                    bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
    return Environment(sdf=sdf, model=CollisionModel(radius_eps=0.2, sigma_obs=8.0))


def steps():
    out = {}
    # (1) the reference bisection test case (test_optimizer.py:98-113)
    sys_ltv = point_robot_lti(2)(10, 0.25)
    prior = assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
    cfg = OptimizerConfig(kl_bound=5e-3)
    state = ref_opt.initial_state(prior, cfg)
    g_mu = np.full(prior.mean.shape, 3.0)
    zs = BlockTridiagonalMatrix.zeros(prior.nsteps + 1, prior.n)
    log, restore = probe_log()
    sel = select_step_size(state, prior, g_mu, zs, cfg, temp=1.0)
    restore()
    K, n = prior.nsteps + 1, prior.n
    pd, po = stack_bt(prior.prec)
    cd, co = stack_bt(state.prec)
    nd, no = stack_bt(sel.next_state.prec)
    out.update({"s1_kdiag": pd, "s1_koff": po, "s1_info": prior.info.reshape(K, n),
                "s1_pmean": prior.mean.reshape(K, n), "s1_mean": state.mean.reshape(K, n),
                "s1_diag": cd, "s1_off": co, "s1_gmu": g_mu.reshape(K, n), "s1_gdiag": np.zeros((K, n, n)),
                "s1_cfg": np.array([cfg.kl_bound, cfg.beta_min, cfg.beta_max, 1.0]),
                "s1_beta": np.array(sel.beta), "s1_kl": np.array(sel.kl),
                "s1_nmean": sel.next_state.mean.reshape(K, n), "s1_ndiag": nd, "s1_noff": no,
                "s1_ncovs": np.stack(sel.marginals.covs), "s1_ncrosses": np.stack(sel.marginals.crosses),
                "s1_probes": np.array(log)})
    # (2) a real first iteration of C1 (collision gradients from the compiled kernel)
    env = c1_env()
    sys_ltv = point_robot_lti(2)(50, 3.0 / 50)
    prior = assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
    cfg = OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=600)
    state = ref_opt.initial_state(prior, cfg)
    marg = gbp_marginals(state.prec)
    rule = smolyak_rule(3, 4)
    fv = evaluate_all_factors(state.mean, state.prec, env.sdf, env.model, rule, marginals=marg)
    maps = interior_collision_maps(51)
    gm, gs = assemble_joint_gradients(fv, maps, 51, 4)
    log, restore = probe_log()
    sel = select_step_size(state, prior, gm, gs, cfg, temp=1.0)
    restore()
    K, n = 51, 4
    pd, po = stack_bt(prior.prec)
    cd, co = stack_bt(state.prec)
    gd, _ = stack_bt(gs)
    nd, no = stack_bt(sel.next_state.prec)
    out.update({"s2_kdiag": pd, "s2_koff": po, "s2_info": prior.info.reshape(K, n),
                "s2_pmean": prior.mean.reshape(K, n), "s2_mean": state.mean.reshape(K, n),
                "s2_diag": cd, "s2_off": co, "s2_gmu": gm.reshape(K, n), "s2_gdiag": gd,
                "s2_covs": np.stack(marg.covs), "s2_crosses": np.stack(marg.crosses),
                "s2_epsi": np.array([f.e_psi for f in fv]),
                "s2_cfg": np.array([cfg.kl_bound, cfg.beta_min, cfg.beta_max, 1.0]),
                "s2_beta": np.array(sel.beta), "s2_kl": np.array(sel.kl),
                "s2_nmean": sel.next_state.mean.reshape(K, n), "s2_ndiag": nd, "s2_noff": no,
                "s2_ncovs": np.stack(sel.marginals.covs), "s2_ncrosses": np.stack(sel.marginals.crosses),
                "s2_probes": np.array(log), "c1_grid": env.sdf.values, "c1_origin": env.sdf.origin,
                "c1_cell": np.array(env.sdf.cell_size)})
    np.savez_compressed(os.path.join(HERE, "steps.npz"), **out)


def runs():
    """Full run_pgvimp records: C1 pinned to convergence and the reference's
    short obstacle run (test_optimizer.py:158-187)."""
    out = {}
    keys = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost",
            "total_cost", "kl_step", "mean_shift"]
    env = c1_env()
    sys_ltv = point_robot_lti(2)(50, 3.0 / 50)
    cfg = OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=600)
    res = run_pgvimp(sys_ltv, env, cfg, np.zeros(4), np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
    out["c1_records"] = np.array([[r[k] for k in keys] for r in res.records])
    out["c1_final_mean"] = res.final.mean.reshape(51, 4)
    out["c1_final_covs"] = np.stack(res.marginals.covs)
    out["c1_meta"] = np.array([res.converged, res.iterations,
                               -1 if res.switch_iteration is None else res.switch_iteration])
    # short default-config run on the reference test scene, N=15
    sdf = rasterize([Disc(center=np.array([1.0, 0.75]), radius=0.45)],
                    bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
    env2 = Environment(sdf=sdf, model=CollisionModel(radius_eps=0.2, sigma_obs=8.0))
    sys2 = point_robot_lti(2)(15, 0.2)
    cfg2 = OptimizerConfig(max_iters=25)
    res2 = run_pgvimp(sys2, env2, cfg2, np.zeros(4), np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
    out["t15_records"] = np.array([[r[k] for k in keys] for r in res2.records])
    out["t15_final_mean"] = res2.final.mean.reshape(16, 4)
    out["t15_final_covs"] = np.stack(res2.marginals.covs)
    out["t15_meta"] = np.array([res2.converged, res2.iterations,
                                -1 if res2.switch_iteration is None else res2.switch_iteration])
    out["t15_grid"] = sdf.values
    out["record_keys"] = np.array(keys)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)


def priors():
    out = {}
    for tag, N, T in [("p50", 50, 3.0), ("p10", 10, 2.5), ("p500", 500, 10.0)]:
        sys_ltv = point_robot_lti(2)(N, T / N)
        pr = assemble_prior(sys_ltv, np.zeros(4), np.array([2.0, 1.5, 0.0, 0.0]), 1.0, 1e-3)
        d, o = stack_bt(pr.prec)
        out[f"{tag}_diag"], out[f"{tag}_off"] = d, o
        out[f"{tag}_info"] = pr.info.reshape(N + 1, 4)
        out[f"{tag}_mean"] = pr.mean.reshape(N + 1, 4)
    sys3 = point_robot_lti(3)(20, 0.1)
    pr = assemble_prior(sys3, np.zeros(6), np.array([1.0, 2.0, 0.5, 0, 0, 0]), 0.5, 1e-2)
    d, o = stack_bt(pr.prec)
    out["p3d_diag"], out["p3d_off"], out["p3d_info"], out["p3d_mean"] = d, o, pr.info.reshape(21, 6), pr.mean.reshape(21, 6)
    np.savez_compressed(os.path.join(HERE, "priors.npz"), **out)


def maps():
    out = {}
    s = rasterize([Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]], cell_size=0.05)
    out["c1"] = s.values
    s = rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                   Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                  bounds=[[-2, 12], [-2, 12]], cell_size=0.05)
    out["c2"] = s.values
    s = rasterize([], bounds=[[0, 1], [0, 2]], cell_size=0.25)
    out["empty"] = s.values
    np.savez_compressed(os.path.join(HERE, "maps.npz"), **out)


def slr():
    """iP-GVIMP (slr.py): one SLR linearisation of the quadrotor and a short
    outer loop on a C4-like scene (SURVEY §8d C4 parity variant, shortened)."""
    from gvplan import NominalTrajectory, OuterConfig, planar_quadrotor, run_ipgvimp, slr_linearize
    out = {}
    rng = np.random.default_rng(11)
    sys_nl = planar_quadrotor()
    means = rng.normal(size=(8, 6)) * np.array([2, 2, 0.3, 1, 1, 0.5])
    covs = []
    for _ in range(8):
        a = rng.normal(size=(6, 6))
        covs.append(0.05 * (a @ a.T + 6 * np.eye(6)) / 6)
    covs = np.stack(covs)
    ltv = slr_linearize(sys_nl, NominalTrajectory(means=means, covs=covs), 0.1, smolyak_rule(3, 6))
    out["lin_means"], out["lin_covs"] = means, covs
    out["lin_A"] = np.stack([s.A for s in ltv.steps])
    out["lin_a"] = np.stack([s.a for s in ltv.steps])
    sdf = rasterize([Disc(center=np.array([5.0, 4.5]), radius=0.8)], bounds=[[-5, 15], [-5, 10]], cell_size=0.05)
    env = Environment(sdf=sdf, model=CollisionModel(radius_eps=1.5, sigma_obs=6.0))
    cfg = OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0, temp_high=5.0, max_iters=15)
    res, log = run_ipgvimp(sys_nl, env, cfg, OuterConfig(max_outer=2), np.zeros(6),
                           np.array([10.0, 5.0, 0, 0, 0, 0]), dt=0.25, num_steps=20, q_c=0.5, sigma_b=1e-3)
    keys = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
            "mean_shift"]
    out["ip_norm_diff"] = np.array([r["norm_diff"] for r in log])
    out["ip_records"] = np.array([[r[k] for k in keys] for r in res.records])
    out["ip_final_mean"] = res.final.mean.reshape(21, 6)
    np.savez_compressed(os.path.join(HERE, "slr.npz"), **out)


def configs():
    """SURVEY §8d configurations the bench/engine specialise for, a few
    iterations each: C2 (N=500, k_q=5: the 57-projection factor kernel) and
    plan 0 of the C5 bench workload (N=1000, k_q=3, C2 map)."""
    from gvplan.sdf import Box
    out = {}
    keys = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
            "mean_shift"]
    c2map = rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                       Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                      bounds=[[-2, 12], [-2, 12]], cell_size=0.05)
    env = Environment(sdf=c2map, model=CollisionModel(radius_eps=0.2, sigma_obs=8.0))
    # C2: point2d N=500, T=10, k_q=5
    cfg = OptimizerConfig(k_q=5, kl_bound=10.0, beta_max=0.5, max_iters=4)
    res = run_pgvimp(point_robot_lti(2)(500, 10.0 / 500), env, cfg, np.zeros(4), np.array([10.0, 10.0, 0, 0]),
                     1.0, 1e-3)
    out["c2_records"] = np.array([[r[k] for k in keys] for r in res.records])
    out["c2_final_mean"] = res.final.mean.reshape(501, 4)
    # C5 plan 0: goal from the bench's generator (bench.c5_goals)
    rng = np.random.default_rng(2411_03416)
    goal = np.array([10.0, 10.0, 0.0, 0.0])
    goal[:2] += rng.uniform(-0.5, 0.5, size=(1, 2))[0]
    cfg = OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=3)
    res = run_pgvimp(point_robot_lti(2)(1000, 10.0 / 1000), env, cfg, np.zeros(4), goal, 1.0, 1e-3)
    out["c5p_goal"] = goal
    out["c5p_records"] = np.array([[r[k] for k in keys] for r in res.records])
    out["c5p_final_mean"] = res.final.mean.reshape(1001, 4)
    # the reference's own probe log of the first iteration (beta, spd, KL)
    log, restore = probe_log()
    run_pgvimp(point_robot_lti(2)(1000, 10.0 / 1000), env, OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5,
                                                                          max_iters=1), np.zeros(4), goal, 1.0, 1e-3)
    restore()
    out["c5p_probes1"] = np.array(log)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **out)


def slr_py():
    """The same iP-GVIMP run through the reference's pure-numpy kernel backend
    (GVPLAN_PURE_PYTHON=1, backend.py:14). The quadrotor run is ill-conditioned
    (sigma_b = 1e-3, 15 unconverged inner iterations): the reference's two
    backends already disagree at ~1e-5, which is the honest tolerance scale
    for any non-bitwise implementation of the run."""
    assert os.environ.get("GVPLAN_PURE_PYTHON") and not gvplan.HAVE_EXTENSION
    from gvplan import OuterConfig, planar_quadrotor, run_ipgvimp
    sdf = rasterize([Disc(center=np.array([5.0, 4.5]), radius=0.8)], bounds=[[-5, 15], [-5, 10]], cell_size=0.05)
    env = Environment(sdf=sdf, model=CollisionModel(radius_eps=1.5, sigma_obs=6.0))
    cfg = OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0, temp_high=5.0, max_iters=15)
    res, log = run_ipgvimp(planar_quadrotor(), env, cfg, OuterConfig(max_outer=2), np.zeros(6),
                           np.array([10.0, 5.0, 0, 0, 0, 0]), dt=0.25, num_steps=20, q_c=0.5, sigma_b=1e-3)
    keys = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
            "mean_shift"]
    out = {"ip_norm_diff": np.array([r["norm_diff"] for r in log]),
           "ip_records": np.array([[r[k] for k in keys] for r in res.records]),
           "ip_final_mean": res.final.mean.reshape(21, 6)}
    np.savez_compressed(os.path.join(HERE, "slr_py.npz"), **out)


def wide():
    """Wide blocks (SURVEY.md §8c golden (2): n = 14, the 7-DOF arm state; plus
    n = 10 and n = 20): chain drop-ins and one select_step_size on a 7-DOF
    double-integrator prior."""
    out = {}
    for tag, seed, K, n in [("w14", 41, 51, 14), ("w10", 43, 30, 10), ("w20", 47, 12, 20)]:
        rng = np.random.default_rng(seed)
        prec = random_spd_bt(rng, K, n)
        eta = rng.normal(size=K * n)
        d, o = stack_bt(prec)
        marg = gbp_marginals(prec)
        out[f"{tag}_diag"], out[f"{tag}_off"] = d, o
        out[f"{tag}_eta"] = eta.reshape(K, n)
        out[f"{tag}_covs"] = np.stack(marg.covs)
        out[f"{tag}_crosses"] = np.stack(marg.crosses)
        out[f"{tag}_mean"] = gbp_mean_solve(prec, eta).reshape(K, n)
        out[f"{tag}_logdet"] = np.array(logdet_block_tridiag(prec))
    # select_step_size at n = 14 (7-DOF double integrator, N = 30)
    from gvplan.dynamics import LTVStep, LTVSystem
    A = np.zeros((14, 14))
    A[:7, 7:] = np.eye(7)
    B = np.zeros((14, 7))
    B[7:, :] = np.eye(7)
    sys_ltv = LTVSystem(steps=tuple([LTVStep(A=A, a=np.zeros(14), B=B)] * 31), dt=0.1, n=14, m=7)
    goal = np.concatenate([np.linspace(0.5, 1.5, 7), np.zeros(7)])
    prior = assemble_prior(sys_ltv, np.zeros(14), goal, 1.0, 1e-3)
    cfg = OptimizerConfig(kl_bound=5e-2)
    state = ref_opt.initial_state(prior, cfg)
    rng = np.random.default_rng(53)
    K, n = prior.nsteps + 1, prior.n
    g_mu = 3.0 * rng.normal(size=K * n)
    gs = BlockTridiagonalMatrix.zeros(K, n)
    for i in range(1, K - 1):
        a = 0.1 * rng.normal(size=(n, n))
        gs.diag[i] = a @ a.T
    log, restore = probe_log()
    sel = select_step_size(state, prior, g_mu, gs, cfg, temp=1.0)
    restore()
    pd, po = stack_bt(prior.prec)
    cd, co = stack_bt(state.prec)
    gd, _ = stack_bt(gs)
    nd, no = stack_bt(sel.next_state.prec)
    prox = ref_opt.proximal_update(state, prior, g_mu, gs, 0.05, 1.0)
    xd, xo = stack_bt(prox.prec)
    out.update({"s14_kdiag": pd, "s14_koff": po, "s14_info": prior.info.reshape(K, n),
                "s14_mean": state.mean.reshape(K, n), "s14_diag": cd, "s14_off": co,
                "s14_gmu": g_mu.reshape(K, n), "s14_gdiag": gd,
                "s14_cfg": np.array([cfg.kl_bound, cfg.beta_min, cfg.beta_max, 1.0]),
                "s14_beta": np.array(sel.beta), "s14_kl": np.array(sel.kl),
                "s14_nmean": sel.next_state.mean.reshape(K, n), "s14_ndiag": nd, "s14_noff": no,
                "s14_ncovs": np.stack(sel.marginals.covs), "s14_ncrosses": np.stack(sel.marginals.crosses),
                "s14_probes": np.array(log),
                "s14_prox_mean": prox.mean.reshape(K, n), "s14_prox_diag": xd, "s14_prox_off": xo})
    np.savez_compressed(os.path.join(HERE, "wide.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rules", "factors", "chain", "steps", "priors", "maps", "runs", "slr"]
    for name in which:
        globals()[name]()
        print("wrote", name)
