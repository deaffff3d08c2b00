"""Where a C3 iteration's wall time goes (host timers around the loop's calls)."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np

import paper_2411_03416_b200 as P
import paper_2411_03416_b200.optimizer as OPT
from paper_2411_03416_b200 import arm as ARM
from c3_run import c3_scene

acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(mod, name, tag=None):
    f = getattr(mod, name)

    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[tag or name] += time.perf_counter() - t
            cnt[tag or name] += 1
    setattr(mod, name, g)


for nm in ("select_step_size", "cost_breakdown", "gbp_marginals", "initial_state"):
    wrap(OPT, nm)
wrap(ARM.ArmEnvironment, "factor_gradients")
import paper_2411_03416_b200.factors as FAC
wrap(FAC, "assemble_joint_gradients")
import paper_2411_03416_b200.blocktri as BT
wrap(BT, "logdet_block_tridiag")
wrap(OPT, "logdet_block_tridiag", "logdet(opt)")
wrap(OPT, "trace_product")

sdf, model = c3_scene()
env = P.ArmEnvironment(sdf, model, P.panda_like())
goal = np.concatenate([[0.9, 0.6, 0.0, -0.8, 0.0, 1.0, 0.0], np.zeros(7)])
cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 20)
N = 200
t0 = time.perf_counter()
res = P.run_pgvimp(P.joint_double_integrator(N, 4.0 / N), env, cfg, np.zeros(14), goal, 1.0, 1e-3)
wall = time.perf_counter() - t0
print(f"iterations {res.iterations}  wall {wall*1e3:.1f} ms  per-iter {wall*1e3/res.iterations:.2f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:28s} {v*1e3:9.1f} ms  x{cnt[k]}  ({v*1e3/max(cnt[k],1):.2f} ms each)")
