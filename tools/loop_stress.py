"""Repeat the loopback apply_precond check (tests/test_gpu_loopback.py) and
report every mismatch: which rank, how large, where (rows owned by which rank).

  python tools/loop_stress.py [reps] [nranks] [case]
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402
from paper_1504_00907_b200.ddg import LoopGroup  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 8
case = sys.argv[3] if len(sys.argv) > 3 else "biharm"
pr = {"biharm": lambda: P.biharmonic2d(128, 16, 3, 24), "lognormal": lambda: P.lognormal3d(32, 4, 1, 23)}[case]()
r = np.random.default_rng(4).standard_normal(pr.n)
s1 = Solver.from_problem(pr)
z1 = s1.apply_precond(r)
s1.close()
bad = 0
for rep in range(reps):
    g = LoopGroup(nr)
    out = [None] * nr

    def body(k):
        s = Solver.from_problem(pr, comm=g.comm(k))
        za = s.apply_precond(r)
        zb = s.apply_precond(r)
        out[k] = (za, zb)
        s.close()

    th = [threading.Thread(target=body, args=(k,)) for k in range(nr)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    g.close()
    for k, (za, zb) in enumerate(out):
        ea = np.linalg.norm(za - z1) / np.linalg.norm(z1)
        eb = np.linalg.norm(zb - z1) / np.linalg.norm(z1)
        if ea > 1e-13 or eb > 1e-13:
            bad += 1
            w = np.flatnonzero(np.abs(za - z1) > 1e-10 * np.abs(z1).max())
            print(f"rep {rep} rank {k}: first apply {ea:.2e}, second {eb:.2e}, {len(w)} rows differ, "
                  f"rows {w[:8]} ...", flush=True)
print(f"{bad} mismatching (rank, rep) of {reps * nr}")
