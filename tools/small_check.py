"""k_pcg_small vs the multi-kernel iteration on one small problem: iterations,
history and u side by side, and M r through the test hook (multi-kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402

pr = P.poisson2d(64, 8, 1, 1001)
res = {}
for fused in ("0", "1"):
    os.environ["DDG_SMALL_FUSED"] = fused
    s = Solver.from_problem(pr)
    s.launch_count(reset=True)
    try:
        u, it, hist, rep = s.solve(pr.f, 1e-8)
        res[fused] = (u, it, hist)
        print(fused, "iters", it, "launches", s.launch_count(), "hist", hist[:4], "res_final", rep.res_final)
    except Exception as e:          # noqa: BLE001
        print(fused, "error", e)
    s.close()
if "0" in res and "1" in res:
    u0, i0, h0 = res["0"]
    u1, i1, h1 = res["1"]
    m = min(len(h0), len(h1))
    print("u rel", np.linalg.norm(u1 - u0) / np.linalg.norm(u0), "hist rel", np.max(np.abs(h1[:m] - h0[:m]) / h0[:m]))
