"""Symmetric vs full blocked Gauss-Jordan against the oracle's Cholesky solves on
biharmonic blocks (Delta = 2): which one drifts?"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402
from paper_1504_00907_b200.ddg import DDGError  # noqa: E402

N, b = int(sys.argv[1]), int(sys.argv[2])
pr = P.biharmonic2d(N, b, 1, 5, overlap=2)
r = np.random.default_rng(0).standard_normal(pr.n)
t = time.time()
o = oracle.Oracle.from_problem(pr)
ref = o.forward_sweep(r)
print("oracle", round(time.time() - t, 1), "s; max m", o.m_max, flush=True)
for sym in ("0", "1"):
    os.environ["DDG_GJ_SYM"] = sym
    try:
        s = Solver.from_problem(pr)
        z = s.apply_precond(r)       # whole M r vs the oracle's
        print("sym", sym, "M r rel diff vs oracle", np.linalg.norm(z - o.apply_precond(r)) / np.linalg.norm(z), flush=True)
        s.close()
    except DDGError as e:
        print("sym", sym, str(e)[:100])
