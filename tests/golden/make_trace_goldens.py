"""Per-probe reference traces for the long-horizon parity tests (C5 sample, C2).

Run in the dev container (oracle/_ref built by oracle/build_ref.sh):

    python tests/golden/make_trace_goldens.py            # c5_sample.npz + c2_trace.npz (~15 min, 8 cores)

Every number written is produced by the UNMODIFIED reference package
(`gvplan` from oracle/_ref) or, for the arbiters, by LAPACK on the
reference's own matrices:

* the reference's run_pgvimp on each plan, with every probe of every
  select_step_size logged as (beta, spd, KL) (optimizer.py:188-231);
* per probe, KL_dense: the same KL(next || cur) from banded Cholesky factors
  of the reference's own candidate and current precisions (refkl.py — a sum of
  squares, no trace_product cancellation), the arbiter for probes where the
  reference's KL sits within its own error of the bound;
* per near-bound probe (|KL - eps| < 1e-2), KL_np: the reference's KL with the
  gradients of its pure-numpy kernel backend (_kernels_py) at the same state
  and beta — the reference's own backend spread;
* per iteration, the record the numpy backend would have produced from the
  same state at the same beta (record spread), and the iterate's mean at every
  50th knot.

C5 sample: plans 0, 128, ..., 3968 of bench.c5_goals(4096) on the bench's own
problem construction (shared prior precision of the base goal, per-plan info
= base info + anchor dg at the last knot, bench.build_problem), 10
iterations each. C2: SURVEY §8d C2 (N = 500, k_q = 5), 4 iterations.
"""

from __future__ import annotations

import dataclasses
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(1, HERE)

import gvplan  # noqa: E402
from gvplan import optimizer as ro  # noqa: E402
from gvplan import _kernels_py  # noqa: E402
from gvplan.factors import assemble_joint_gradients, evaluate_all_factors, interior_collision_maps  # noqa: E402
from gvplan.sdf import Box  # noqa: E402

from refkl import kl_banded  # noqa: E402

assert gvplan.HAVE_EXTENSION, "build the reference extension first (oracle/build_ref.sh)"

_COST_BREAKDOWN = ro.cost_breakdown  # unwrapped (the runs below wrap the module attribute)

KEYS = ["beta", "temperature", "prior_cost", "collision_cost", "entropy_cost", "total_cost", "kl_step",
        "mean_shift"]
NEAR = 1e-2          # |KL - eps| below which the numpy-backend KL is also computed
KNOT_STRIDE = 50     # iterate means stored at knots 0, 50, 100, ...
C5_SAMPLE = np.arange(0, 4096, 128)
C5_ITERS = 10
SEED = 2411_03416


def c2_map():
    return gvplan.rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                             Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                            bounds=[[-2, 12], [-2, 12]], cell_size=0.05)


def c5_goals(total):  # bench.c5_goals
    rng = np.random.default_rng(SEED)
    g = np.tile(np.array([10.0, 10.0, 0.0, 0.0]), (total, 1))
    g[:, :2] += rng.uniform(-0.5, 0.5, size=(total, 2))
    return g


def c5_base_prior():
    sys_ltv = gvplan.point_robot_lti(2)(1000, 10.0 / 1000)
    return sys_ltv, gvplan.assemble_prior(sys_ltv, np.zeros(4), np.array([10.0, 10.0, 0.0, 0.0]), 1.0, 1e-3)


def c5_plan_prior(base, goal):
    """bench.build_problem for one plan: shared precision, info with the goal
    anchor moved (anchor = I / sigma_b^2 is diagonal: the product is exact),
    the anchored mean from the reference's own gbp_mean_solve."""
    K, n = base.nsteps + 1, base.n
    anchor = np.eye(n) / 1e-3 ** 2
    info = base.info.reshape(K, n).copy()
    info[-1] += (goal - base.goal) @ anchor.T
    info = info.reshape(-1)
    return dataclasses.replace(base, info=info, mean=gvplan.gbp_mean_solve(base.prec, info), goal=goal)


def trace_run(sys_ltv, prior, env, cfg):
    """run_pgvimp with every select_step_size instrumented (see module doc)."""
    rule = gvplan.smolyak_rule(cfg.k_q, prior.n)
    orig_sel = ro.select_step_size
    iters = []

    def sel(cur, prior_, g_mu, g_sigma, cfg_, temp):
        log = []
        o_prox, o_kl, o_marg = ro.proximal_update, ro.kl_joint, ro.gbp_marginals
        st = {}

        def prox(c, p, gm, gs, beta, t):
            st["beta"] = beta
            return o_prox(c, p, gm, gs, beta, t)

        def marg(prec):
            try:
                return o_marg(prec)
            except Exception:
                log.append([st["beta"], 0.0, np.inf, None])
                raise

        def kl(nxt, c, m=None):
            v = o_kl(nxt, c, m)
            log.append([st["beta"], 1.0, v, nxt])
            return v

        ro.proximal_update, ro.kl_joint, ro.gbp_marginals = prox, kl, marg
        try:
            out = orig_sel(cur, prior_, g_mu, g_sigma, cfg_, temp)
        finally:
            ro.proximal_update, ro.kl_joint, ro.gbp_marginals = o_prox, o_kl, o_marg
        nb, n = cur.prec.nblocks, cur.prec.block_size
        m_cur = o_marg(cur.prec)
        fv_np = evaluate_all_factors(cur.mean, cur.prec, env.sdf, env.model, rule, marginals=m_cur,
                                     backend=_kernels_py)
        gm_np, gs_np = assemble_joint_gradients(fv_np, interior_collision_maps(nb), nb, n)
        cd, co = np.stack(cur.prec.diag), np.stack(cur.prec.off)
        rows = []
        for beta, spd, k, nxt in log:
            if not spd:
                rows.append((beta, 0.0, np.inf, np.nan, np.nan))
                continue
            kd = kl_banded(nxt.mean, np.stack(nxt.prec.diag), np.stack(nxt.prec.off), cur.mean, cd, co)
            knp = np.nan
            if abs(k - cfg_.kl_bound) < NEAR:
                c2 = o_prox(cur, prior_, gm_np, gs_np, beta, temp)
                try:
                    knp = o_kl(c2, cur, o_marg(c2.prec))
                except Exception:
                    knp = np.inf
            rows.append((beta, 1.0, k, knp, kd))
        # the numpy backend's record at the same beta from the same state
        nxt_np = o_prox(cur, prior_, gm_np, gs_np, out.beta, temp)
        m_np = o_marg(nxt_np.prec)
        f_np = evaluate_all_factors(nxt_np.mean, nxt_np.prec, env.sdf, env.model, rule, marginals=m_np,
                                    backend=_kernels_py)
        c_np = _COST_BREAKDOWN(nxt_np, prior_, temp, marginals=m_np, factor_values=f_np)
        rec_np = [out.beta, temp, c_np.prior_cost, c_np.collision_cost, c_np.entropy_cost, c_np.total,
                  o_kl(nxt_np, cur, m_np), float(np.linalg.norm(nxt_np.mean - cur.mean))]
        iters.append({"probes": np.array(rows), "rec_np": np.array(rec_np),
                      "mean_np": nxt_np.mean.reshape(nb, n)[::KNOT_STRIDE].copy(),
                      "mean_np_full": nxt_np.mean.reshape(nb, n).copy()})
        return out

    ro.select_step_size = sel
    try:
        t0 = time.time()
        res = gvplan.run_pgvimp(sys_ltv, env, cfg, prior.x0, prior.goal, 1.0, 1e-3, prior=prior)
        dt = time.time() - t0
    finally:
        ro.select_step_size = orig_sel
    return res, iters, dt


def pack(res, iters, K, n, means):
    """Fixed-shape arrays: probes padded to 40 rows with NaN."""
    it = len(iters)
    pr = np.full((it, 40, 5), np.nan)
    cnt = np.zeros(it, dtype=np.int32)
    for k, d in enumerate(iters):
        p = d["probes"]
        pr[k, :len(p)] = p
        cnt[k] = len(p)
    return {"probes": pr, "nprobes": cnt,
            "records": np.array([[r[k] for k in KEYS] for r in res.records]),
            "records_np": np.stack([d["rec_np"] for d in iters]),
            "means": np.stack(means),  # (it, K // stride + 1, n) after each iteration
            "means_np": np.stack([d["mean_np"] for d in iters]),
            "final_mean": res.final.mean.reshape(K, n),
            "final_mean_np": iters[-1]["mean_np_full"]}


def c5_worker(b):
    sys_ltv, base = c5_base_prior()
    goal = c5_goals(4096)[b]
    prior = c5_plan_prior(base, goal)
    env = ro.Environment(sdf=c2_map(), model=gvplan.CollisionModel(0.2, 8.0))
    cfg = gvplan.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=C5_ITERS, threads=1)
    means = []
    orig_step = ro.select_step_size

    # the iterate after each iteration: wrap cost_breakdown (called once per iteration with nxt)
    o_cost = ro.cost_breakdown

    def cost(nxt, *a, **kw):
        means.append(nxt.mean.reshape(1001, 4)[::KNOT_STRIDE].copy())
        return o_cost(nxt, *a, **kw)

    ro.cost_breakdown = cost
    try:
        res, iters, dt = trace_run(sys_ltv, prior, env, cfg)
    finally:
        ro.cost_breakdown = o_cost
        ro.select_step_size = orig_step
    out = pack(res, iters, 1001, 4, means)
    out["pmean"] = prior.mean.reshape(1001, 4)
    print(f"plan {b}: {len(res.records)} iterations in {dt:.1f} s", flush=True)
    return b, out


def c5_sample(procs=8):
    import multiprocessing as mp

    sys_ltv, base = c5_base_prior()
    with mp.get_context("fork").Pool(procs) as pool:
        outs = dict(pool.map(c5_worker, list(C5_SAMPLE)))
    K, n = 1001, 4
    data = {"plans": C5_SAMPLE.astype(np.int32), "kdiag": np.stack(base.prec.diag),
            "koff": np.stack(base.prec.off), "info0": base.info.reshape(K, n), "goal0": base.goal,
            "knot_stride": np.int32(KNOT_STRIDE)}
    for key in outs[C5_SAMPLE[0]]:
        data[key] = np.stack([outs[b][key] for b in C5_SAMPLE])
    np.savez_compressed(os.path.join(HERE, "c5_sample.npz"), **data)


def c2_trace():
    sys_ltv = gvplan.point_robot_lti(2)(500, 10.0 / 500)
    prior = gvplan.assemble_prior(sys_ltv, np.zeros(4), np.array([10.0, 10.0, 0, 0]), 1.0, 1e-3)
    env = ro.Environment(sdf=c2_map(), model=gvplan.CollisionModel(0.2, 8.0))
    cfg = gvplan.OptimizerConfig(k_q=5, kl_bound=10.0, beta_max=0.5, max_iters=4, threads=1)
    means = []
    o_cost = ro.cost_breakdown

    def cost(nxt, *a, **kw):
        means.append(nxt.mean.reshape(501, 4)[::KNOT_STRIDE].copy())
        return o_cost(nxt, *a, **kw)

    ro.cost_breakdown = cost
    try:
        res, iters, dt = trace_run(sys_ltv, prior, env, cfg)
    finally:
        ro.cost_breakdown = o_cost
    out = pack(res, iters, 501, 4, means)
    out.update(kdiag=np.stack(prior.prec.diag), koff=np.stack(prior.prec.off), info=prior.info.reshape(501, 4),
               pmean=prior.mean.reshape(501, 4), knot_stride=np.int32(KNOT_STRIDE))
    np.savez_compressed(os.path.join(HERE, "c2_trace.npz"), **out)
    print(f"c2: {len(res.records)} iterations in {dt:.1f} s", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["c2", "c5"]
    if "c2" in what:
        c2_trace()
    if "c5" in what:
        c5_sample()
