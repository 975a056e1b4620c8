"""Bitwise repeatability of the sparse (dataflow) coarse solve: one context,
coarse_correct and a full solve repeated; prints the number of distinct results."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402

os.environ.setdefault("DDG_ND_LEAF", "64")
for name, pr in (("lognormal32", P.lognormal3d(32, 4, 1, 1003)), ("biharm128", P.biharmonic2d(128, 16, 3, 1005))):
    s = Solver.from_problem(pr, coarse_variant=2)
    r = np.random.default_rng(6).standard_normal(pr.n)
    zs = [s.coarse_correct(r) for _ in range(20)]
    us = [s.solve(pr.f, 1e-8)[0] for _ in range(5)]
    dz = len({z.tobytes() for z in zs})
    du = len({u.tobytes() for u in us})
    print(name, "distinct coarse_correct:", dz, "distinct u:", du,
          "max rel spread:", max(float(np.linalg.norm(z - zs[0]) / np.linalg.norm(zs[0])) for z in zs), flush=True)
    s.close()
