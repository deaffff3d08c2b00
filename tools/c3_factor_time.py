"""Time the C3 arm factor stage call (gvp_arm_factor_grads) at a mid-run state."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np

import paper_2411_03416_b200 as P
from c3_run import c3_scene

sdf, model = c3_scene()
env = P.ArmEnvironment(sdf, model, P.panda_like())
goal = np.concatenate([[0.9, 0.6, 0.0, -0.8, 0.0, 1.0, 0.0], np.zeros(7)])
cfg = P.OptimizerConfig(k_q=3, kl_bound=10.0, beta_max=0.5, max_iters=20)
N = 200
res = P.run_pgvimp(P.joint_double_integrator(N, 4.0 / N), env, cfg, np.zeros(14), goal, 1.0, 1e-3)
covs = np.stack(res.marginals.covs)
mean = res.final.mean
rule = P.smolyak_rule(3, 14)
env.factor_gradients(mean, covs, rule)
for rep in range(3):
    t = time.perf_counter()
    for _ in range(20):
        env.factor_gradients(mean, covs, rule)
    print(f"factor_gradients {1e3 * (time.perf_counter() - t) / 20:.3f} ms")
t = time.perf_counter()
for _ in range(20):
    np.stack(res.marginals.covs)
print(f"np.stack covs {1e3 * (time.perf_counter() - t) / 20:.3f} ms")
t = time.perf_counter()
for _ in range(20):
    P.smolyak_rule(3, 14)
print(f"smolyak_rule {1e3 * (time.perf_counter() - t) / 20:.3f} ms")

# alternate with the optimizer's select_step_size (as in the planner loop)
import paper_2411_03416_b200.optimizer as OPT
from paper_2411_03416_b200.prior import assemble_prior
sys_ltv = P.joint_double_integrator(N, 4.0 / N)
prior = assemble_prior(sys_ltv, np.zeros(14), goal, 1.0, 1e-3)
e_psi, g_mu, g_s = env.factor_gradients(mean, covs, rule)
gmu_full = np.zeros((N + 1, 14))
gmu_full[1:N] = g_mu
gd = np.zeros((N + 1, 14, 14))
gd[1:N] = g_s
gsig = P.BlockTridiagonalMatrix(gd, np.zeros((N, 14, 14)))
tsel = tfac = 0.0
for _ in range(10):
    t = time.perf_counter()
    st = OPT.select_step_size(res.final, prior, gmu_full.reshape(-1), gsig, cfg, 1.0)
    t1 = time.perf_counter()
    env.factor_gradients(st.next_state.mean, np.stack(st.marginals.covs), rule)
    t2 = time.perf_counter()
    tsel += t1 - t
    tfac += t2 - t1
print(f"alternating: select {tsel * 100:.2f} ms  factor {tfac * 100:.2f} ms")
