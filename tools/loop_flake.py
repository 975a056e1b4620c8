"""Repeat loopback multi-rank runs (DDG_DEBUG_FILL=255 by default) and report
which operation first deviates from the single-context result."""
import os
import sys
import threading

os.environ.setdefault("DDG_DEBUG_FILL", "255")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402
from paper_1504_00907_b200.ddg import LoopGroup  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 8
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pr = P.biharmonic2d(128, 16, 3, 1005)
r = np.random.default_rng(4).standard_normal(pr.n)
s1 = Solver.from_problem(pr)
ref = {"spmv": s1.spmv(r), "coarse": s1.coarse_correct(r), "precond": s1.apply_precond(r)}
u1, it1, h1, _ = s1.solve(pr.f, 1e-8)
s1.close()
bad = 0
for trial in range(trials):
    g = LoopGroup(nr)
    out = [None] * nr

    def body(k):
        s = Solver.from_problem(pr, comm=g.comm(k))
        res = {}
        for nm, fn in (("spmv", s.spmv), ("coarse", s.coarse_correct), ("precond", s.apply_precond)):
            v = fn(r)
            res[nm] = float(np.linalg.norm(v - ref[nm]) / np.linalg.norm(ref[nm]))
        u, it, hist, rep = s.solve(pr.f, 1e-8)
        res["solve"] = (it, float(np.linalg.norm(u - u1) / np.linalg.norm(u1)),
                        float(np.max(np.abs(hist[:3] - h1[:3]) / h1[:3])))
        s.close()
        out[k] = res

    th = [threading.Thread(target=body, args=(k,)) for k in range(nr)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    g.close()
    worst = {k: max((o[k] if k != "solve" else o[k][1]) for o in out) for k in ("spmv", "coarse", "precond", "solve")}
    flag = any(v > 1e-9 or v != v for v in worst.values())
    bad += flag
    print(trial, "BAD" if flag else "ok", worst, [o["solve"] for o in out] if flag else "", flush=True)
print("bad trials:", bad, "of", trials)
