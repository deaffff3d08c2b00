"""ms per iteration across batch sizes and horizons, engine defaults vs forced
probe variants (debug aid for the lane / kernel heuristics)."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "one":
    import bench
    import paper_2411_03416_b200 as P
    B, N, lanes = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    bench.N_INTERVALS = N
    bench.T_TOTAL = 10.0
    goals = bench.c5_goals(B)
    prior, info, pmean, init = bench.build_problem(P, goals)
    K = N + 1
    eng = P.PlanBatch(B, K, 4, bench.c2_map(P), P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4),
                      bench.c5_cfg(P, 12), shared_prior=True, spec_lanes=lanes)
    eng.load(prior.prec.diag_stack, prior.prec.off_stack, info, pmean, init)
    eng.step(2, sync=True)
    ms = eng.step_profiled(4) / 4
    print(json.dumps({"B": B, "N": N, "lanes": eng.lanes(), "probe": os.environ.get("GVP_PROBE", "auto"),
                      "bisect": round(ms[0], 3), "commit": round(ms[1], 3), "total": round(float(ms.sum()), 3),
                      "us_per_plan_iter": round(float(ms.sum()) * 1e3 / B, 3)}))
    sys.exit(0)

for N in (1000, 50):
    for B in (1, 16, 64, 256, 1024, 4096):
        for probe in ("auto", "fused", "split"):
            for lanes in (0,):
                env = dict(os.environ)
                if probe != "auto":
                    env["GVP_PROBE"] = probe
                r = subprocess.run([sys.executable, __file__, "one", str(B), str(N), str(lanes)], env=env,
                                   capture_output=True, text=True, timeout=300)
                print(r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
