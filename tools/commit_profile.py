"""Pass B / pass F cycles of commit_kernel on C5 (diagnostic build:
tools/variant_build.sh commit prof_commit -DGVP_COMMIT_PROFILE)."""
import ctypes as C
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GVP_B200_LIB", os.path.join(REPO, "paper_2411_03416_b200", "prof_commit", "libgvp_b200.so"))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import paper_2411_03416_b200 as P  # noqa: E402
from paper_2411_03416_b200 import _native  # noqa: E402

lib = _native.load()
prof = lib.gvp_commit_profile
prof.argtypes = [C.POINTER(C.c_double)]
B = 4096
goals = bench.c5_goals(B)
prior, info, pmean, init = bench.build_problem(P, goals)
eng = P.PlanBatch(B, 1001, 4, bench.c2_map(P), P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4),
                  bench.c5_cfg(P, 12), shared_prior=True)
eng.load(prior.prec.diag_stack, prior.prec.off_stack, info, pmean, init)
out = np.zeros(19)
eng.step(3, sync=True)
prof(out.ctypes.data_as(C.POINTER(C.c_double)))
eng.step(5, sync=True)
prof(out.ctypes.data_as(C.POINTER(C.c_double)))
ctas = max(out[2], 1)
print(json.dumps({"passB_cycles_per_cta": out[0] / ctas, "passF_cycles_per_cta": out[1] / ctas,
                  "passB_us": out[0] / ctas / 1965.0, "passF_us": out[1] / ctas / 1965.0,
                  "launches_x_ctas": out[2]}))
roles = ["chain Lambda'", "chain mean", "side 0 (stores / traces)", "side 1 (means / prior)"]
for ps, name in ((0, "pass B"), (1, "pass F")):
    for w in range(4):
        wk, wt = out[3 + ps * 8 + w * 2], out[3 + ps * 8 + w * 2 + 1]
        print(f"{name} warp {w} ({roles[w]}): work {wk / ctas / 1965.0:8.1f} us  wait {wt / ctas / 1965.0:8.1f} us "
              f"(work fraction {wk / max(wk + wt, 1):.2f})")
