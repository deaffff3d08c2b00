"""Dump the reference-order probe sequence of every plan for a few C5
iterations (input to offline speculation-policy studies)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2411_03416_b200 as P

B = int(sys.argv[1]); iters = int(sys.argv[2]); out = sys.argv[3]
goals = bench.c5_goals(B)
prior, info, pmean, init = bench.build_problem(P, goals)
K, n = bench.N_INTERVALS + 1, 4
eng = P.PlanBatch(B, K, n, bench.c2_map(P), P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4),
                  bench.c5_cfg(P, iters + 2), shared_prior=True, spec_lanes=4)
eng.trace_probes(64)
eng.load(prior.prec.diag_stack, prior.prec.off_stack, info, pmean, init)
logs = []
for it in range(iters):
    eng.step(1, sync=True)
    pr = eng.probes()
    arr = np.full((B, 64, 3), np.nan)
    for b, p in enumerate(pr):
        arr[b, :len(p)] = p
    logs.append(arr)
np.savez_compressed(out, probes=np.stack(logs))
cnt = np.isfinite(np.stack(logs)[..., 0]).sum(-1)
print("probes per plan-iteration: mean", cnt.mean(), "max", cnt.max(), "min", cnt.min())
