"""gbp_marginals kernel time: cyclic reduction vs the sequential sweep (measurement aid)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import numpy as np, gvp_oracle as O, paper_2411_03416_b200 as P
    for N in (50, 100, 1000):
        A, a, B = O.point_robot_triples(2)
        pr = O.assemble_prior([A] * (N + 1), [a] * (N + 1), [B] * (N + 1), 3.0 / N, np.zeros(4), np.array([2.0, 1.5, 0, 0]), 1.0, 1e-3)
        prec = P.BlockTridiagonalMatrix(pr["diag"] * 10.0, pr["off"] * 10.0)
        for _ in range(5):
            P.gbp_marginals(prec)
    sys.exit(0)
for mode in ("cr", "seq"):
    env = dict(os.environ, GVP_MARGINALS=mode)
    subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--clock-control", "none", "--csv", "--log-file",
                    f"{ROOT}/gpurun_out/marg_{mode}.csv", sys.executable, __file__, "run"], env=env,
                   capture_output=True)
    print(mode)
    os.system(f"{sys.executable} {ROOT}/tools/ktimes.py {ROOT}/gpurun_out/marg_{mode}.csv")
