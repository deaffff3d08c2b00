"""Per-role work / wait cycles of probe_split_kernel on C5 (diagnostic build,
tools/probe_profile.sh): which warp role sets the per-knot step time."""
import ctypes as C
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GVP_B200_LIB", os.path.join(REPO, "paper_2411_03416_b200", "prof", "libgvp_b200.so"))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import paper_2411_03416_b200 as P  # noqa: E402
from paper_2411_03416_b200 import _native  # noqa: E402

lib = _native.load()
prof = lib.gvp_probe_profile
prof.argtypes = [C.POINTER(C.c_double)]
B = 4096
goals = bench.c5_goals(B)
prior, info, pmean, init = bench.build_problem(P, goals)
eng = P.PlanBatch(B, 1001, 4, bench.c2_map(P), P.CollisionModel(0.2, 8.0), P.smolyak_rule(3, 4),
                  bench.c5_cfg(P, 12), shared_prior=True)
eng.load(prior.prec.diag_stack, prior.prec.off_stack, info, pmean, init)
eng.step(3, sync=True)
out = np.zeros(8)
prof(out.ctypes.data_as(C.POINTER(C.c_double)))
eng.step(3, sync=True)
prof(out.ctypes.data_as(C.POINTER(C.c_double)))
names = ["Lambda' Schur", "Lambda' tangent", "S Schur", "S tangent"]
res = {}
for r in range(4):
    w, t = out[2 * r], out[2 * r + 1]
    res[names[r]] = {"work_frac": w / (w + t), "work_cycles": w, "wait_cycles": t}
print(json.dumps(res, indent=1))
