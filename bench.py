#!/usr/bin/env python
"""Benchmark: batched P-GVIMP on B200 (BASELINE.json metric
"factor-expectation evals/s and time-to-converge per plan").

Workload (BASELINE configs[4], "C5"): independent point2d plans, N=1000
intervals (1001 knots), T=10 s, Smolyak k_q=3 (41 sigma points), the C2
narrow-gap map (two boxes, 281 x 281 cells at 0.05), start 0, goal
(10,10,0,0) + U(-0.5,0.5)^2 on position from default_rng(2411_03416),
collision r=0.2 sigma=8, q_c=1, sigma_b=1e-3, the C1 optimizer settings
(kl_bound=10, beta_max=0.5). --plans plans per GPU (weak scaling: each rank
runs its own shard of independent plans, no data-path collective).

One step = one Algorithm-1 iteration of every plan on the rank: the whole
bisection step-size search (GBP marginals + proximal update + KL per probe),
the factor stage at the accepted state, and cost/convergence control.
value = factor-expectation evaluations (plan x interior knot, Q sigma points
each) completed per second, all ranks. Inputs are resident in HBM; the
working set (~4 GB at 4096 plans) is far larger than L2, so no L2 flush is
needed between steps.

Also reported: e2e (the same through the C ABI from pinned host buffers),
time-to-converge of the C1 plan, roofline of the dominant kernel, a CPU
baseline of the reference on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_INTERVALS = 1000
T_TOTAL = 10.0
K_Q = 3
SEED = 2411_03416


def c2_map(P):
    from paper_2411_03416_b200.sdf import Box
    return P.rasterize([Box(center=np.array([5.0, 1.2]), halfextents=np.array([0.3, 3.4])),
                        Box(center=np.array([5.0, 8.8]), halfextents=np.array([0.3, 3.4]))],
                       bounds=[[-2, 12], [-2, 12]], cell_size=0.05)


def c5_goals(total: int) -> np.ndarray:
    rng = np.random.default_rng(SEED)
    g = np.tile(np.array([10.0, 10.0, 0.0, 0.0]), (total, 1))
    g[:, :2] += rng.uniform(-0.5, 0.5, size=(total, 2))
    return g


def c5_cfg(P, max_iters):
    return P.OptimizerConfig(k_q=K_Q, kl_bound=10.0, beta_max=0.5, max_iters=max_iters)


def build_problem(P, goals):
    """The C5 problem through the public batch API's builder
    (optimizer.batch_problem, what run_pgvimp_batch loads): one prior (the
    first plan's), per-plan info / anchored mean / initial mean from the
    affine dependence on the goal (setup only, not timed)."""
    sys_ltv = P.point_robot_lti(2)(N_INTERVALS, T_TOTAL / N_INTERVALS)
    from paper_2411_03416_b200.optimizer import batch_problem

    return batch_problem(sys_ltv, np.zeros(4), goals, 1.0, 1e-3, c5_cfg(P, 10))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 20 ms; summary() keeps
    the samples taken inside the timed window (mark_start / mark_end)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None
        self.path = os.path.join(REPO, "gpurun_out", f"clocks_r{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        deadline = time.time() + 5.0  # nvidia-smi start-up: wait for its first sample
        while self.proc is not None and time.time() < deadline:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.02)
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        time.sleep(0.05)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        import datetime
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8 and parts[1].isdigit():
                    try:
                        ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    except ValueError:
                        ts = None
                    rows.append((ts, parts[1:]))
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        inside = [r for ts, r in rows if ts is not None and self.t0 is not None and self.t1 is not None
                  and self.t0 - 0.03 <= ts <= self.t1 + 0.03]
        sel = inside or [r for _, r in rows]
        sm = sorted(int(r[0]) for r in sel)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({nm for r in sel for nm, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(sel[0][1]), "reasons": reasons,
                "samples": len(sel), "window": "timed region" if inside else "whole run (no sample inside)"}


def probe_flops_per_knot(n: int) -> dict:
    """Algorithmic fp64 flops of one bisection probe at one knot (both chains
    of the one-pass probe, csrc/step_probe.cu; FMA = 2, rsqrt = 1), counted
    from its loop nests. Returns {"A", "B", "total"}."""
    T, N2 = n * (n + 1) // 2, n * n
    fma = lambda k: 2 * k  # noqa: E731
    chol = fma(T - n) + n + n + n + sum((n - 1 - j) * (1 + fma(j)) for j in range(n)) \
        + sum(fma(r - c) + 1 for c in range(n) for r in range(c + 1, n))
    common = (4 * N2                      # off block scaled: (K/T + Lambda/beta) (* c)
              + fma(n * T) * 2            # W = Li M_o, G = Li Lambda_o
              + fma(N2 * n)               # Z = Psi W - G
              + fma(T * n) + fma(T * 2 * n)  # Phi -= W'W, Phi' += W'Z - G'W
              + chol
              + fma(n * T) + fma(sum(q + 1 for r in range(n) for q in range(r + 1)))  # Psi = Li Phi' Li'
              + n)                        # trace / accumulate
    a = 6 * T + common + 1
    b = 3 * T + common + n + fma(N2) + n + fma(3 * N2) + fma(2 * T) + fma(N2) + 3 * n
    return {"A": a, "B": b, "total": a + b}


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "fallback": True}


def _ref_bench():
    """oracle/ref_bench.py: the reference-side legs (cpu_baseline, --impl reference)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import ref_bench

    return ref_bench


def fp64_peak():
    """Measured fp64 FMA throughput (profiles/fp64_peak.txt, tools/micro/lat.cu
    on the B200 box: 148 SMs x 64 DFMA/clk x 2 at 1965 MHz); falls back to the
    ncu peak_sustained arithmetic at the recorded max SM clock."""
    path = os.path.join(REPO, "profiles", "fp64_peak.txt")
    try:
        for line in open(path):
            if line.startswith("DFMA throughput:"):
                return float(line.split(":")[1].split()[0]), "measured (profiles/fp64_peak.txt, tools/micro/lat.cu)"
    except OSError:
        pass
    mhz = float(measured_peaks().get("sm_max_mhz", 1965.0))
    return 148 * 64 * 2 * mhz * 1e6 / 1e12, "derived: 148 SMs x 64 DFMA/clk x 2 x sm_max_mhz"


def run_reference_arm(args):
    """--impl reference: the reference's CPU implementation of the path on all
    host cores, rank 0 only. One worker process per core, each owning one C5
    plan; a step = one steady-state iteration of the
    reference's own loop body on every plan (oracle/ref_bench.py), counted as
    F = N - 1 factor-expectation evals per plan-iteration like the GPU arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    R = _ref_bench()
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (run oracle/build_ref.sh)"}))
        return
    lanes = len(os.sched_getaffinity(0))
    out = R.run_parallel(lanes, args.steps, args.warmup)
    wall = sum(out["times"])
    value = out["evals"] / wall
    line = {"metric": "factor-expectation evals/s", "value": value, "unit": "factor-evals/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / len(out["times"]), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5 sample: {lanes} independent point2d plans (one per host core, plans "
                                   f"0..{lanes - 1} of the bench workload), N={N_INTERVALS}, k_q=3, C2 map; step = "
                                   "one steady-state iteration of every plan",
                       "plans_per_step": lanes, "N": N_INTERVALS, "k_q": K_Q},
            "cpu_baseline": {"value": value, "unit": "factor-evals/s", "cores": lanes, "kind": "reference",
                             "sample": f"{lanes} plans x 1 iteration per step, one process per plan, gvplan "
                                       "from oracle/_ref (Cython kernel), steady state"},
            "e2e": {"value": value, "unit": "factor-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _spawn_ranks(args) -> int:
    """--gpus N without a launcher: re-run this script under torch.distributed.run,
    one rank per GPU (NCCL), rendezvous on 127.0.0.1."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    env.setdefault("NCCL_DEBUG_FILE", os.path.join(REPO, "gpurun_out", "nccl.%h.%p.log"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def time_to_converge(P, args, B, goals, prior, info, pmean, init, dev):
    """C5: the whole 4096-plan batch from initial_state until every plan hit the
    reference's termination (optimizer.py:386-392) or max_iters = 600;
    C2: one plan (N = 500, k_q = 5) the same way. Wall clock around the calls,
    inputs already resident / built (setup untimed)."""
    import torch

    from paper_2411_03416_b200.engine import to_plan_minor

    K, n = N_INTERVALS + 1, 4
    out = {}
    eng = P.PlanBatch(B, K, n, c2_map(P), P.CollisionModel(0.2, 8.0), P.smolyak_rule(K_Q, n), c5_cfg(P, 600),
                      shared_prior=True)
    try:
        t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in
             (prior.prec.diag_stack, prior.prec.off_stack, to_plan_minor(info), to_plan_minor(pmean),
              to_plan_minor(init))]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.load_device(*[x.data_ptr() for x in t])
        done = eng.run(check_every=25)
        wall = (time.perf_counter() - t0) * 1e3
        sm = eng.summary()
    finally:
        eng.close()
    its = sm["iterations"].astype(np.int64)
    conv = sm["converged"].astype(bool)
    out["C5"] = {"config": f"C5: {B} plans, N={N_INTERVALS}, k_q=3, max_iters=600", "ms": wall,
                 "iterations_launched": int(done), "converged_fraction": float(conv.mean()),
                 "iterations_median": float(np.median(its)), "iterations_max": int(its.max()),
                 "iterations_median_converged": float(np.median(its[conv])) if conv.any() else None,
                 "failed": int((sm["status"] != 0).sum()),
                 "ms_per_plan_amortized": wall / B}
    sys2 = P.point_robot_lti(2)(500, 10.0 / 500)
    env2 = P.Environment(c2_map(P), P.CollisionModel(0.2, 8.0))
    g2 = np.array([10.0, 10.0, 0, 0])
    pr2 = P.assemble_prior(sys2, np.zeros(4), g2, 1.0, 1e-3)
    cfg2 = P.OptimizerConfig(k_q=5, kl_bound=10.0, beta_max=0.5, max_iters=600)
    P.run_pgvimp(sys2, env2, P.OptimizerConfig(k_q=5, kl_bound=10.0, beta_max=0.5, max_iters=2), np.zeros(4), g2,
                 1.0, 1e-3, prior=pr2)  # warm
    t0 = time.perf_counter()
    r2 = P.run_pgvimp(sys2, env2, cfg2, np.zeros(4), g2, 1.0, 1e-3, prior=pr2)
    w2 = (time.perf_counter() - t0) * 1e3
    # C4 at N = 300 (GPU-only: the reference's arithmetic fails there):
    # iP-GVIMP with SLR + prior on the device, robust-conditioning mode (deviates)
    sdf4 = P.rasterize([P.sdf.Disc(center=np.array([5.0, 4.5]), radius=0.8)], bounds=[[-5, 15], [-5, 10]],
                       cell_size=0.05)
    env4 = P.Environment(sdf4, P.CollisionModel(radius_eps=1.5, sigma_obs=6.0))
    cfg4 = P.OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0, temp_high=5.0, max_iters=100)
    try:  # warm (module loads, rules, device buffers), like the other legs
        P.run_ipgvimp(P.planar_quadrotor(), env4, P.OptimizerConfig(k_q=3, kl_bound=10.0, temp_low=1.0,
                                                                   temp_high=5.0, max_iters=2),
                      P.OuterConfig(max_outer=1), np.zeros(6), np.array([10.0, 5.0, 0, 0, 0, 0]), dt=5.0 / 300,
                      num_steps=300, q_c=0.5, sigma_b=1e-3, device=True, robust=True)
    except Exception:  # noqa: BLE001 (the timed run below reports any failure)
        pass
    t0 = time.perf_counter()
    try:
        r4, log4 = P.run_ipgvimp(P.planar_quadrotor(), env4, cfg4, P.OuterConfig(max_outer=3), np.zeros(6),
                                 np.array([10.0, 5.0, 0, 0, 0, 0]), dt=5.0 / 300, num_steps=300, q_c=0.5,
                                 sigma_b=1e-3, device=True, robust=True)
        out["C4_N300"] = {"config": "C4: planar quadrotor iP-GVIMP, N=300, T=5, k_q=3, 3 outer x 100 inner, device "
                                    "SLR + prior, robust-conditioning mode (Grammian reg 1e-6; deviates from the "
                                    "reference, whose arithmetic fails at N=300)",
                          "ms": (time.perf_counter() - t0) * 1e3, "outer": len(log4),
                          "inner_iterations_last": r4.iterations, "converged": r4.converged,
                          "norm_diff": [x["norm_diff"] for x in log4]}
    except Exception as exc:  # reported, not fatal: the headline is C5
        out["C4_N300"] = {"error": repr(exc)[:300]}
    out["C2"] = {"config": "C2: point2d N=500, k_q=5 (385 points), narrow gap, max_iters=600", "ms": w2,
                 "iterations": r2.iterations, "converged": r2.converged, "ms_per_iteration": w2 / max(r2.iterations, 1),
                 "reference_s_per_iteration_survey": 2.29}
    return out


def c1_legs(P, args, world):
    """C1 pinned plan: GPU run_pgvimp to convergence, the reference's own run on
    this host (rank 0, N = 1 only), and the reference-format CSV rows
    (bench.py:26: serial = reference CPU at 1 thread, parallel = this engine)."""
    from paper_2411_03416_b200 import runio

    sdf1 = P.rasterize([P.sdf.Disc(center=np.array([1.1, 0.55]), radius=0.45)], bounds=[[-2, 4], [-2, 4]],
                       cell_size=0.05)
    env1 = P.Environment(sdf1, P.CollisionModel(0.2, 8.0))
    sys1 = P.point_robot_lti(2)(50, 3.0 / 50)
    g1 = np.array([2.0, 1.5, 0, 0])
    cfg1 = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=600)
    pr1 = P.assemble_prior(sys1, np.zeros(4), g1, 1.0, 1e-3)
    P.run_pgvimp(sys1, env1, cfg1, np.zeros(4), g1, 1.0, 1e-3, prior=pr1)  # warm
    runs = []
    for _ in range(3):  # wall clock of the whole call (engine setup, iterations, fetch)
        t0 = time.perf_counter()
        r1 = P.run_pgvimp(sys1, env1, cfg1, np.zeros(4), g1, 1.0, 1e-3, prior=pr1)
        runs.append((time.perf_counter() - t0) * 1e3)
    ttc = {"config": "C1 pinned: point2d N=50, k_q=3, kl_bound=10, beta_max=0.5", "ms": min(runs), "ms_runs": runs,
           "iterations": r1.iterations, "converged": r1.converged, "reference_iterations": 94,
           "ms_per_iteration": min(runs) / max(r1.iterations, 1)}
    # our factor stage / GBP marginals at C1 (median of 10 / 3, like the reference's bench_factors)
    rule = P.smolyak_rule(3, 4)
    st = P.optimizer.initial_state(pr1, cfg1)
    marg = P.gbp_marginals(st.prec)

    def med(fn, reps):
        fn()
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t) * 1e3)
        return float(np.median(ts))

    fac_ms = med(lambda: P.evaluate_all_factors(st.mean, st.prec, sdf1, env1.model, rule, marginals=marg), 10)
    gbp_ms = med(lambda: P.gbp_marginals(pr1.prec), 3)
    rows = []
    R = _ref_bench()
    if world == 1 and R.available():
        try:
            ref = R.c1_full(threads=1)
        except Exception as exc:  # the reference leg is a reported baseline, not the product
            ttc["reference"] = {"error": str(exc)[-300:]}
        else:
            ttc["reference"] = {"ms": ref["ms"], "iterations": ref["iterations"], "converged": ref["converged"],
                                "threads": 1, "where": "this host, gvplan from oracle/_ref"}
            rows = [runio.bench_row("factors", 50, 4, 3, ref["factor_stage_ms"], fac_ms),
                    runio.bench_row("gbp", 50, 4, 0, ref["dense_inverse_ms"], gbp_ms),
                    runio.bench_row("full", 50, 4, 3, ref["ms"], min(runs))]
            if args.csv:
                os.makedirs(os.path.dirname(os.path.abspath(args.csv)), exist_ok=True)
                with open(args.csv, "w") as fh:
                    fh.write(runio.rows_to_csv(rows))
    return {"ttc": ttc, "rows": rows}


def cpu_baseline_leg():
    """The reference on ONE host core: C5 plan 0 in steady state (oracle/ref_bench.py),
    2 timed iterations after 1 warm-up (~15 s of CPU)."""
    R = _ref_bench()
    if not R.available():
        return {"value": None, "error": "oracle/_ref not built"}
    try:
        r = R.cpu_baseline(iters=2, warm=1)
    except Exception as exc:
        return {"value": None, "error": str(exc)[-300:]}
    return {"value": r["evals"] / r["seconds"], "unit": "factor-evals/s", "cores": 1, "kind": "reference",
            "sample": f"1 C5 plan (N={N_INTERVALS}, k_q=3) x {r['iterations']} steady-state iterations of the "
                      f"reference's loop body, gvplan from oracle/_ref (Cython kernel: {r['ext']}), threads=1, "
                      f"{r['seconds']:.2f} s"}


def timed_steps(eng, steps, F, sync, start, stop, dev=None, marks=None):
    """The contract's timed region: barrier + synchronize on both sides, exactly
    `steps` iterations of every plan on the rank, the rank's time from
    start()/stop() (CUDA events on the engine stream), then the max over ranks
    and the work (plan-iterations x F factor evals) summed over ranks."""
    from paper_2411_03416_b200 import dist as D

    it_before = eng.summary()["iterations"].astype(np.int64)
    D.barrier()
    sync()
    if marks:
        marks[0]()
    start()
    eng.step(steps)
    ms = stop()
    sync()
    if marks:
        marks[1]()
    D.barrier()
    it_after = eng.summary()["iterations"].astype(np.int64)
    evals = float((it_after - it_before).sum() * F)
    return {"ms": ms, "evals": evals, "it_after": it_after, "ms_max": D.reduce_max(ms, device=dev),
            "evals_all": D.reduce_sum(evals, device=dev)}


class StubBatch:
    """--stub-engine: CPU stand-in with PlanBatch's step/summary surface, so the
    launcher, sharding and cross-rank reductions run without a GPU (gloo)."""

    def __init__(self, B):
        self.iters = np.zeros(B, dtype=np.int32)

    def step(self, k, sync=False):
        time.sleep(0.005 * k)
        self.iters += k

    def summary(self):
        return {"iterations": self.iters.copy()}


def run_stub(args):
    import torch.distributed as dist

    from paper_2411_03416_b200.dist import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
    lo, hi = shard(args.plans * world, world, rank)
    eng = StubBatch(hi - lo)
    eng.step(args.warmup)
    t = {}
    tr = timed_steps(eng, args.steps, N_INTERVALS - 1, lambda: None, lambda: t.setdefault("t0", time.perf_counter()),
                     lambda: (time.perf_counter() - t["t0"]) * 1e3)
    if rank == 0:
        print(json.dumps({"metric": "factor-expectation evals/s", "value": tr["evals_all"] / (tr["ms_max"] / 1e3),
                          "unit": "factor-evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": tr["ms_max"] / args.steps, "stub": True,
                          "evals_all": tr["evals_all"], "plans_total": args.plans * world}))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--plans", type=int, default=4096, help="plans per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c1", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--stub-engine", action="store_true", help=argparse.SUPPRESS)  # CPU launcher test
    ap.add_argument("--no-converge", action="store_true", help="skip the C5/C2 time-to-converge runs")
    ap.add_argument("--csv", default=os.path.join(REPO, "gpurun_out", "bench.csv"),
                    help="reference-format bench CSV rows (bench.py:26 header)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    if args.stub_engine:
        return run_stub(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2411_03416_b200 as P
    from paper_2411_03416_b200 import _native

    _native.load().gvp_device_count()
    # the library's runtime follows the device torch made current for this rank
    B = args.plans
    # weak scaling: every rank runs B plans of its own (a contiguous shard of
    # the world's B * world plans), no collective on the data path
    from paper_2411_03416_b200.dist import shard
    lo_p, hi_p = shard(B * world, world, rank)
    goals = c5_goals(B * world)[lo_p:hi_p]
    prior, info, pmean, init = build_problem(P, goals)
    K, n = N_INTERVALS + 1, 4
    F = K - 2
    sdf = c2_map(P)
    model = P.CollisionModel(0.2, 8.0)
    rule = P.smolyak_rule(K_Q, n)
    max_iters = args.warmup + 2 * args.steps + 4
    eng = P.PlanBatch(B, K, n, sdf, model, rule, c5_cfg(P, max_iters), shared_prior=True)
    eng.trace_probes(64)  # per-plan probe counts (the useful work of the bisection)

    # problem resident in HBM (plan-minor torch tensors), loaded device-to-device
    from paper_2411_03416_b200.engine import to_plan_minor
    dev = torch.device("cuda", local)
    t_kd = torch.from_numpy(np.ascontiguousarray(prior.prec.diag_stack)).to(dev)
    t_ko = torch.from_numpy(np.ascontiguousarray(prior.prec.off_stack)).to(dev)
    t_info = torch.from_numpy(to_plan_minor(info)).to(dev)
    t_pm = torch.from_numpy(to_plan_minor(pmean)).to(dev)
    t_m0 = torch.from_numpy(to_plan_minor(init)).to(dev)
    torch.cuda.synchronize()

    def load_device():
        eng.load_device(t_kd.data_ptr(), t_ko.data_ptr(), t_info.data_ptr(), t_pm.data_ptr(), t_m0.data_ptr())

    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=dev)

    from paper_2411_03416_b200 import dist as D

    barrier = D.barrier
    max_over_ranks = lambda x: D.reduce_max(x, device=dev)  # noqa: E731
    sum_over_ranks = lambda x: D.reduce_sum(x, device=dev)  # noqa: E731

    # ---------------- timed region: K steps, inputs resident in HBM
    load_device()
    eng.step(args.warmup, sync=True)
    launches_before = eng.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def ev_stop():
        ev1.record(stream)
        ev1.synchronize()
        return ev0.elapsed_time(ev1)

    with ClockSampler(local) as clk:
        tr = timed_steps(eng, args.steps, F, torch.cuda.synchronize, lambda: ev0.record(stream), ev_stop, dev,
                         marks=(clk.mark_start, clk.mark_end))
    launches = eng.launches() - launches_before
    it_after, ms_max, evals_all = tr["it_after"], tr["ms_max"], tr["evals_all"]
    value = evals_all / (ms_max / 1e3)

    # ---------------- per-kernel device times (events around each kernel) and
    # the bisection's useful work: the reference's probe count of each plan
    kms = np.zeros(len(eng.PROFILE_BUCKETS))
    probes = 0
    it_prev = it_after
    for _ in range(args.steps):
        kms += eng.step_profiled_ex(1)
        it_now = eng.summary()["iterations"].astype(np.int64)
        moved = (it_now - it_prev) > 0
        counts = [len(p) for p in eng.probes()]
        probes += int(sum(c for c, m in zip(counts, moved) if m))
        it_prev = it_now
    # ---------------- e2e: through the C ABI from pinned host buffers
    # the caller's inputs of a shared-system batch: the system's prior blocks and
    # anchored-mean responses (optimizer.batch_parts, once per system) and every
    # plan's start and goal; the per-plan information / prior mean / initial mean
    # are expanded on the device (gvp_engine_load_boundary, run_pgvimp_batch's path)
    from paper_2411_03416_b200.optimizer import batch_parts

    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    base, resp0, respg, anchor, x0a, goala = batch_parts(
        P.point_robot_lti(2)(N_INTERVALS, T_TOTAL / N_INTERVALS), np.zeros(4), goals, 1.0, 1e-3)
    h_in = [pin(a) for a in (base.prec.diag_stack, base.prec.off_stack, base.info, base.mean, resp0, respg,
                             anchor, x0a, goala)]
    h_rec = torch.empty((max_iters, B, 8), dtype=torch.float64).pin_memory().numpy()
    # the results a caller needs: records, final means and marginal covariances (packed)
    h_mean = torch.empty((K, n, B), dtype=torch.float64).pin_memory().numpy()
    h_cov = torch.empty((K, n * (n + 1) // 2, B), dtype=torch.float64).pin_memory().numpy()
    h2d = sum(a.nbytes for a in h_in)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    e0.record(stream)
    eng.lib.gvp_engine_load_boundary(eng.handle, *[_native.ptr(a) for a in h_in])
    eng.step(args.steps)
    eng.lib.gvp_engine_get_records(eng.handle, _native.ptr(h_rec))
    eng.packed_into(mean=h_mean, covs=h_cov)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), (time.perf_counter() - t_wall) * 1e3))
    d2h = h_rec.nbytes + h_mean.nbytes + h_cov.nbytes
    e2e_evals = sum_over_ranks(float(np.isfinite(h_rec[:, :, 0]).sum() * F))
    e2e_value = e2e_evals / (e2e_ms / 1e3)

    result = None
    if rank == 0:
        peaks = measured_peaks()
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        steps_prof = max(args.steps, 1)
        res_ms, probe_ms, com_ms, fac_ms, fix_ms, ctl_ms = (float(x) / steps_prof for x in kms)
        bis_ms = res_ms + probe_ms
        # Dominant kernel: the bisection (one-pass probes), fp64-pipe bound.
        # achieved = useful probes (the reference's own probe sequence, counted
        # on device) x knots x algorithmic flops per probe-knot / kernel time;
        # speculative probes that the reference would not make are not counted.
        fl = probe_flops_per_knot(n)
        fp64_pk, fp64_src = fp64_peak()
        bis_flops = probes / steps_prof * K * fl["total"]
        ach = bis_flops / (probe_ms / 1e3) / 1e12
        # the engine runs the split probe kernel while the grid is below 2 CTAs per SM
        lanes = eng.lanes()
        P_cols = 32 // lanes  # launch_probe: split while ceil(B / P) < 2 x 148 CTAs
        probe_kernel = "probe_split_kernel" if -(-B // P_cols) < 2 * 148 else "probe_fused_kernel"
        traffic = None
        tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
        fac_traffic = None
        if os.path.exists(tpath):
            with open(tpath) as fh:
                tj = json.load(fh)
            traffic, fac_traffic = tj.get(probe_kernel), tj.get("factor_grads_kernel")
        #  factor stage: 8 (n^2 + 3n + 1) = 232 B per factor
        fac_bytes = B * F * 232
        fac_ach = fac_bytes / (fac_ms / 1e3) / 1e9 if fac_ms > 0 else None
        result = {
            "metric": "factor-expectation evals/s",
            "value": value,
            "unit": "factor-evals/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"C5 batched sweep: {B} independent point2d plans per GPU, N={N_INTERVALS} "
                                   f"(1001 knots), k_q=3 (41 sigma points), C2 narrow-gap map 281x281, "
                                   "C1 optimizer settings; step = one full P-GVIMP iteration "
                                   "(bisection step selection + factor stage + control)",
                       "plans_per_gpu": B, "plans_total": B * world, "N": N_INTERVALS, "k_q": K_Q,
                       "sigma_points": int(rule.npoints), "parallelism": f"plan-sharded x{world}",
                       "l2": "working set > L2 (no flush needed)"},
            "sigma_point_evals_per_s": value * rule.npoints,
            "plan_iterations_per_s": value / F,
            "gpu_launches": int(launches),
            "kernel_ms_per_step": {"bisection": bis_ms, "residual": res_ms, "probes": probe_ms,
                                   "commit": com_ms, "factor_grads": fac_ms, "eigh_fixup": fix_ms,
                                   "control": ctl_ms},
            "roofline": {"kernel": probe_kernel, "bound": "fp64", "achieved": ach,
                         "peak": fp64_pk, "unit": "TFLOP/s", "frac": ach / fp64_pk, "traffic": traffic,
                         "traffic_unit": "bytes/launch (ncu dram read+write)",
                         "flops_per_probe_knot": fl["total"], "probes_per_plan_iter": probes / max(1, B * steps_prof),
                         "lanes_per_plan": lanes,
                         "plans_per_cta": (min(P_cols, max(2, -(-(-(-B // 296)) // 2) * 2))
                                           if probe_kernel == "probe_split_kernel" else P_cols),
                         "peak_source": fp64_src,
                         "factor_grads": {"bound": "hbm", "achieved": fac_ach, "peak": hbm, "unit": "GB/s",
                                          "frac": (fac_ach / hbm) if fac_ach else None,
                                          "bytes_per_factor": 232, "traffic": fac_traffic,
                                          "traffic_unit": "bytes/launch (ncu dram read+write, C5 mid-run)"}},
            "e2e": {"value": e2e_value, "unit": "factor-evals/s", "h2d_bytes_per_step": h2d // max(args.steps, 1),
                    "d2h_bytes_per_step": d2h // max(args.steps, 1),
                    "what": "gvp_engine_load_boundary from pinned host (the system's prior blocks and anchored-mean responses, every plan's start and goal; per-plan arrays expanded on the device) + steps + D2H of the records, final means and packed marginal covariances, one C-ABI call chain"},
            "clocks": clk.summary(),
        }
    eng.close()  # release the timed batch
    # ---------------- time-to-converge (optimizer.py:386-392 termination), rank 0
    if rank == 0 and not args.no_converge:
        result["time_to_converge"] = time_to_converge(P, args, B, goals, prior, info, pmean, init, dev)
    if rank == 0 and not args.no_c1:
        c1 = c1_legs(P, args, world)
        result.setdefault("time_to_converge", {})["C1"] = c1["ttc"]
        result["bench_csv"] = c1["rows"]
    # ---------------- C3 (7-DOF sphere arm, n = 14, N = 200): wall time per planner iteration, rank 0
    if rank == 0 and not args.no_c3:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
        from c3_run import c3_scene
        sdf3, model3 = c3_scene()
        env3 = P.ArmEnvironment(sdf3, model3, P.panda_like())
        goal3 = np.concatenate([[0.9, 0.6, 0.0, -0.8, 0.0, 1.0, 0.0], np.zeros(7)])
        sys3 = P.joint_double_integrator(200, 4.0 / 200)
        pr3 = P.assemble_prior(sys3, np.zeros(14), goal3, 1.0, 1e-3)
        cfg3 = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=3)
        P.run_pgvimp(sys3, env3, cfg3, np.zeros(14), goal3, 1.0, 1e-3, prior=pr3)  # warm
        cfg3 = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=20)
        t0 = time.perf_counter()
        r3 = P.run_pgvimp(sys3, env3, cfg3, np.zeros(14), goal3, 1.0, 1e-3, prior=pr3)
        w3 = (time.perf_counter() - t0) * 1e3
        env3.close()
        result["c3"] = {"config": "C3: 7-DOF sphere arm (panda_like, 14 spheres), n=14, N=200, k_q=3 (421 points, "
                                  "113 joint projections), 128^3 map, kl_bound=10, beta_max=0.5",
                        "iterations": r3.iterations, "ms": w3, "ms_per_iteration": w3 / max(r3.iterations, 1),
                        "ms_per_iteration_median": float(np.median([r["wall_time_ms"] for r in r3.records
                                                                    if r.get("type") == "iter"])),
                        "path": "run_pgvimp host loop over the wide-block chain kernels + device arm factor stage"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline_leg()
    if rank == 0:
        print(json.dumps(result))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
