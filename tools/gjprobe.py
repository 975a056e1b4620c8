import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
from ddg_gen import problems as P
from paper_1504_00907_b200 import Solver
from paper_1504_00907_b200.ddg import DDGError
for (N, b, ov) in [(256, 64, 2), (384, 96, 2), (512, 128, 2), (1000, 125, 2)]:
    pr = P.biharmonic2d(N, b, 1, 5, overlap=ov)
    r = np.random.default_rng(0).standard_normal(pr.n)
    out = {}
    for sym in ("0", "1"):
        os.environ["DDG_GJ_SYM"] = sym
        try:
            s = Solver.from_problem(pr)
            out[sym] = s.apply_precond(r)
            s.close()
        except DDGError as e:
            out[sym] = str(e)[:90]
    a, b_ = out["0"], out["1"]
    if isinstance(a, str) or isinstance(b_, str):
        print(N, b, "full:", a if isinstance(a, str) else "ok", "| sym:", b_ if isinstance(b_, str) else "ok", flush=True)
    else:
        print(N, b, "rel diff", np.linalg.norm(a - b_) / np.linalg.norm(a), flush=True)
