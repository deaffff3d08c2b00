"""Reference-side legs of bench.py — TEST INFRASTRUCTURE.

Only bench.py's `cpu_baseline` leg, `bench.py --impl reference` and tests
use this module; it is never on the product path. It drives the UNMODIFIED
reference (`gvplan`, built from /root/reference by oracle/build_ref.sh into
oracle/_ref) through its own public functions:

* `RefPlan` — one C5 plan of the bench workload, set up exactly as
  bench.build_problem does (shared prior precision of the base goal, per-plan
  info with the goal anchor moved, the anchored mean from the reference's
  gbp_mean_solve), then stepped in STEADY STATE: each `iterate()` is one
  iteration of the reference's own loop body (optimizer.py:338-398:
  assemble_joint_gradients -> select_step_size -> evaluate_all_factors at the
  accepted state -> cost_breakdown -> temperature switch), the state carried
  over between calls. One iteration = F = N - 1 factor-expectation evals, the
  same counting rule as the GPU arm (one plan-iteration = F evals).
* `run_parallel` — one worker process per host core, each owning one plan
  (a process per plan); a step = one iteration of every plan.
* `c1_full` — the reference's run_pgvimp on the pinned C1 plan to convergence
  (time-to-converge on the box's host).
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")

N_INTERVALS = 1000
T_TOTAL = 10.0
SEED = 2411_03416


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "gvplan"))


def _gv():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gvplan

    return gvplan


def c5_goal(b: int, total: int = 4096) -> np.ndarray:
    rng = np.random.default_rng(SEED)  # bench.c5_goals
    g = np.tile(np.array([10.0, 10.0, 0.0, 0.0]), (total, 1))
    g[:, :2] += rng.uniform(-0.5, 0.5, size=(total, 2))
    return g[b]


def c2_map(gv):
    from gvplan.sdf import Box

    return gv.rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                         Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                        bounds=[[-2, 12], [-2, 12]], cell_size=0.05)


class RefPlan:
    """One C5 plan on the reference, iterated in steady state (module doc)."""

    def __init__(self, b: int, threads: int = 1):
        gv = self.gv = _gv()
        from gvplan import optimizer as O
        from gvplan.factors import interior_collision_maps

        self.O = O
        n = 4
        self.sys = gv.point_robot_lti(2)(N_INTERVALS, T_TOTAL / N_INTERVALS)
        base = gv.assemble_prior(self.sys, np.zeros(n), np.array([10.0, 10.0, 0.0, 0.0]), 1.0, 1e-3)
        goal = c5_goal(b)
        info = base.info.reshape(N_INTERVALS + 1, n).copy()
        info[-1] += (goal - base.goal) @ (np.eye(n) / 1e-3 ** 2).T
        info = info.reshape(-1)
        self.prior = dataclasses.replace(base, info=info, mean=gv.gbp_mean_solve(base.prec, info), goal=goal)
        self.env = O.Environment(sdf=c2_map(gv), model=gv.CollisionModel(0.2, 8.0))
        self.cfg = gv.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=10 ** 6, threads=threads)
        self.rule = gv.smolyak_rule(3, n)
        self.nblocks, self.n = N_INTERVALS + 1, n
        self.maps = interior_collision_maps(self.nblocks)
        self.collision_tol = 1e-4 * N_INTERVALS
        # optimizer.py:326-344
        self.cur = O.initial_state(self.prior, self.cfg)
        self.temp = self.cfg.temp_low
        self.switched = False
        marg = gv.gbp_marginals(self.cur.prec)
        self.factors = self._factors(self.cur, marg)
        self.iterations = 0

    def _factors(self, state, marg):
        from gvplan.factors import evaluate_all_factors

        return evaluate_all_factors(state.mean, state.prec, self.env.sdf, self.env.model, self.rule,
                                    threads=self.cfg.threads, marginals=marg)

    def iterate(self) -> int:
        """One iteration of the reference's loop body; returns the factor evals done."""
        from gvplan.factors import assemble_joint_gradients

        O = self.O
        g_mu, g_sigma = assemble_joint_gradients(self.factors, self.maps, self.nblocks, self.n)
        step = O.select_step_size(self.cur, self.prior, g_mu, g_sigma, self.cfg, self.temp)
        nxt = step.next_state
        nxt_f = self._factors(nxt, step.marginals)
        costs = O.cost_breakdown(nxt, self.prior, self.temp, marginals=step.marginals, factor_values=nxt_f)
        self.cur, self.factors = nxt, nxt_f
        self.iterations += 1
        if not self.switched and costs.collision_cost < self.collision_tol and self.temp != self.cfg.temp_high:
            self.temp, self.switched = self.cfg.temp_high, True
        return len(self.maps)


def _worker(conn, b, threads):
    plan = RefPlan(b, threads)
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg == "stop":
            break
        t0 = time.perf_counter()
        evals = plan.iterate()
        conn.send((evals, time.perf_counter() - t0))
    conn.close()


def run_parallel(lanes: int, steps: int, warmup: int) -> dict:
    """`lanes` worker processes, one C5 plan each (plans 0..lanes-1); a step =
    one steady-state iteration of every plan. Wall time per step measured
    around the whole step (send -> all replies)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in saved:
        os.environ[k] = "1"
    procs, conns = [], []
    try:
        for w in range(lanes):
            a, c = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(c, w, 1), daemon=True)
            p.start()
            procs.append(p)
            conns.append(a)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for a in conns:
        assert a.recv() == "ready"
    times, evals = [], 0
    for step in range(warmup + steps):
        t0 = time.perf_counter()
        for a in conns:
            a.send("step")
        got = [a.recv() for a in conns]
        dt = time.perf_counter() - t0
        if step >= warmup:
            times.append(dt)
            evals += sum(e for e, _ in got)
    for a in conns:
        a.send("stop")
    for p in procs:
        p.join(timeout=30)
    return {"times": times, "evals": evals, "lanes": lanes}


def cpu_baseline(iters: int = 2, warm: int = 1) -> dict:
    """One C5 plan, one core (threads=1, single-threaded BLAS), steady-state
    iterations; run in a fresh interpreter so the thread limits hold."""
    code = (f"import sys, json; sys.path.insert(0, {HERE!r}); import ref_bench as R; "
            f"print(json.dumps(R._cpu_baseline_inproc({iters}, {warm})))")
    import subprocess

    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=1200)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-800:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def _cpu_baseline_inproc(iters, warm):
    gv = _gv()
    plan = RefPlan(0, threads=1)
    for _ in range(warm):
        plan.iterate()
    t0 = time.perf_counter()
    evals = sum(plan.iterate() for _ in range(iters))
    dt = time.perf_counter() - t0
    return {"evals": evals, "seconds": dt, "iterations": iters, "ext": bool(gv.HAVE_EXTENSION)}


def c1_full(threads: int = 1) -> dict:
    """The reference's run_pgvimp on the pinned C1 plan to its
    own termination, in a fresh interpreter (threads=1: single-threaded BLAS)."""
    code = (f"import sys, json; sys.path.insert(0, {HERE!r}); import ref_bench as R; "
            f"print(json.dumps(R._c1_inproc({threads})))")
    import subprocess

    env = dict(os.environ)
    if threads == 1:
        env.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=1200)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-800:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def _c1_inproc(threads):
    gv = _gv()
    from gvplan.sdf import Disc

    sdf = gv.rasterize([Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                       cell_size=0.05)
    env = gv.Environment(sdf=sdf, model=gv.CollisionModel(0.2, 8.0))
    sys_ltv = gv.point_robot_lti(2)(50, 3.0 / 50)
    goal = np.array([2.0, 1.5, 0, 0])
    cfg = gv.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=600, threads=threads)
    t0 = time.perf_counter()
    res = gv.run_pgvimp(sys_ltv, env, cfg, np.zeros(4), goal, 1.0, 1e-3)
    ms = (time.perf_counter() - t0) * 1e3
    # factor stage alone at C1 (bench_factors-style median of 10, bench.py:73-94) and GBP vs dense (:97-105)
    from gvplan import optimizer as O
    from gvplan.factors import evaluate_all_factors

    prior = gv.assemble_prior(sys_ltv, np.zeros(4), goal, 1.0, 1e-3)
    st = O.initial_state(prior, cfg)
    marg = gv.gbp_marginals(st.prec)
    rule = gv.smolyak_rule(3, 4)

    def med(fn, reps):
        fn()
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t) * 1e3)
        return float(np.median(ts))

    fac_ms = med(lambda: evaluate_all_factors(st.mean, st.prec, env.sdf, env.model, rule, threads=threads,
                                              marginals=marg), 10)
    gbp_ms = med(lambda: gv.gbp_marginals(prior.prec), 3)
    dense = prior.prec.dense()
    dense_ms = med(lambda: np.linalg.inv(dense), 3)
    return {"ms": ms, "iterations": res.iterations, "converged": bool(res.converged), "threads": threads,
            "factor_stage_ms": fac_ms, "gbp_ms": gbp_ms, "dense_inverse_ms": dense_ms,
            "records_beta": [r["beta"] for r in res.records][:5]}


def exact_solve(S, rhs, x0, sweeps: int = 3):
    """Iterative refinement of S x = rhs (the reference's own double-precision
    S and rhs, block tridiagonal) with residuals in 80-bit long double: the
    exact solution of the reference's system to ~1e-12 relative, the arbiter for
    the ill-conditioned mean solve (cond ~1e10 at N = 1000)."""
    gv = _gv()
    D = np.stack(S.diag).astype(np.longdouble)
    U = np.stack(S.off).astype(np.longdouble)
    K, n = D.shape[0], D.shape[1]
    b = np.asarray(rhs, dtype=np.longdouble).reshape(K, n)
    x = np.asarray(x0, dtype=np.longdouble).reshape(K, n)
    for _ in range(sweeps):
        y = np.einsum("kij,kj->ki", D, x)
        y[:-1] += np.einsum("kij,kj->ki", U, x[1:])
        y[1:] += np.einsum("kji,kj->ki", U, x[:-1])
        r = b - y
        dx = gv.gbp_mean_solve(S, np.asarray(r, dtype=np.float64).reshape(-1)).reshape(K, n)
        x = x + dx.astype(np.longdouble)
    return np.asarray(x, dtype=np.float64)


def trace_states(b: int, iters: int) -> list:
    """The reference's own trajectory of C5 plan b (bench construction, RefPlan),
    per iteration: the state it starts from, the accepted beta, the record, the
    next mean and the exact solution of the reference's own mean system at that
    beta (exact_solve). For the one-step parity test."""
    plan = RefPlan(b, threads=1)
    O = plan.O
    o_solve = O.gbp_mean_solve
    captured = {}

    def solve(S, rhs):
        x = o_solve(S, rhs)
        captured[len(captured)] = (S, np.array(rhs), x)
        return x

    out = []
    for _ in range(iters):
        from gvplan.factors import assemble_joint_gradients

        cur, temp = plan.cur, plan.temp
        captured.clear()
        O.gbp_mean_solve = solve
        try:
            g_mu, g_sigma = assemble_joint_gradients(plan.factors, plan.maps, plan.nblocks, plan.n)
            step = O.select_step_size(cur, plan.prior, g_mu, g_sigma, plan.cfg, temp)
        finally:
            O.gbp_mean_solve = o_solve
        # the accepted probe's mean system (bitwise: its solution is step.next_state.mean)
        S, rhs, x = next(v for v in captured.values() if np.array_equal(v[2], step.next_state.mean))
        exact = exact_solve(S, rhs, x)
        nxt = step.next_state
        nxt_f = plan._factors(nxt, step.marginals)
        costs = O.cost_breakdown(nxt, plan.prior, temp, marginals=step.marginals, factor_values=nxt_f)
        rec = [step.beta, temp, costs.prior_cost, costs.collision_cost, costs.entropy_cost, costs.total, step.kl,
               float(np.linalg.norm(nxt.mean - cur.mean))]
        out.append({"beta": step.beta, "temp": temp, "mean": cur.mean.reshape(plan.nblocks, plan.n),
                    "diag": np.stack(cur.prec.diag), "off": np.stack(cur.prec.off),
                    "next_mean": nxt.mean.reshape(plan.nblocks, plan.n),
                    "next_exact": exact.reshape(plan.nblocks, plan.n), "record": np.array(rec)})
        plan.cur, plan.factors = nxt, nxt_f
        if not plan.switched and costs.collision_cost < plan.collision_tol and plan.temp != plan.cfg.temp_high:
            plan.temp, plan.switched = plan.cfg.temp_high, True
    return out


def _trace_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    return args[0], trace_states(*args)


def trace_states_many(plans, iters: int, procs: int | None = None) -> dict:
    """trace_states for several plans, one process each (spawned: single-threaded BLAS)."""
    import multiprocessing as mp

    procs = procs or min(len(plans), len(os.sched_getaffinity(0)))
    saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in saved:
        os.environ[k] = "1"
    try:
        with mp.get_context("spawn").Pool(procs) as pool:
            res = pool.map(_trace_worker, [(int(b), iters) for b in plans], chunksize=1)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return dict(res)
