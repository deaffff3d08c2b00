"""Engine timing at a given batch size / lane count on the C5 problem shape (debugging aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2411_03416_b200 as P

B = int(sys.argv[1]); lanes = int(sys.argv[2]); iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
goals = bench.c5_goals(B)
prior, info, pmean, init = bench.build_problem(P, goals)
K, n = bench.N_INTERVALS + 1, 4
eng = P.PlanBatch(B, K, n, bench.c2_map(P), P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4),
                  bench.c5_cfg(P, iters + 2), shared_prior=True, spec_lanes=lanes)
eng.load(prior.prec.diag_stack, prior.prec.off_stack, info, pmean, init)
eng.step(1, sync=True)
ms = eng.step_profiled(iters)
s = eng.summary()
print(f"B={B} lanes={eng.lanes()} ms/iter bisect={ms[0]/iters:.2f} commit={ms[1]/iters:.2f} factor={ms[2]/iters:.3f} control={ms[3]/iters:.3f} "
      f"status={set(s['status'].tolist())} iters={s['iterations'][:3]}")
