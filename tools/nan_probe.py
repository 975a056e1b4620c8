"""Which multi-rank operation reads uninitialised device memory: run P
loopback ranks with DDG_DEBUG_FILL=255 (NaN-poisoned allocations) and report
NaNs in each rank's spmv, coarse correction, preconditioner and solve."""
import os
import sys
import threading

os.environ.setdefault("DDG_DEBUG_FILL", "255")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402
from paper_1504_00907_b200.ddg import LoopGroup  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "biharm"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pr = {"biharm": lambda: P.biharmonic2d(128, 16, 3, 1005), "lognormal": lambda: P.lognormal3d(32, 4, 1, 1003),
      "poisson": lambda: P.poisson3d(32, 8, 2, 1002)}[cfg]()
r = np.random.default_rng(4).standard_normal(pr.n)
if os.environ.get("SINGLE_FIRST"):          # a single-GPU context first, as the parity test does
    s1 = Solver.from_problem(pr)
    z1 = s1.apply_precond(r)
    print("single", int(np.isnan(z1).sum()), flush=True)
    s1.close()
g = LoopGroup(nr)
out = [None] * nr


def body(k):
    s = Solver.from_problem(pr, comm=g.comm(k))
    res = {}
    steps = (("precond", s.apply_precond),) if os.environ.get("PRECOND_ONLY") else (
        ("spmv", s.spmv), ("coarse", s.coarse_correct), ("precond", s.apply_precond))
    for nm, fn in steps:
        v = fn(r)
        res[nm] = (int(np.isnan(v).sum()), np.nonzero(np.isnan(v))[0][:8].tolist())
    u, it, hist, rep = s.solve(pr.f, 1e-8)
    res["solve"] = (int(np.isnan(u).sum()), it, bool(rep.converged), hist[:4].tolist())
    s.close()
    out[k] = res


th = [threading.Thread(target=body, args=(k,)) for k in range(nr)]
for t in th:
    t.start()
for t in th:
    t.join()
g.close()
for k in range(nr):
    print(k, out[k], flush=True)
