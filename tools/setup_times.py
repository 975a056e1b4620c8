"""ddg_setup stage timings (verbose) for the given configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402

for cfg in sys.argv[1:]:
    t0 = time.time()
    pr = P.make(cfg)
    t1 = time.time()
    s = Solver.from_problem(pr, device=0, verbose=True)
    t2 = time.time()
    print(f"{cfg}: generate {t1-t0:.1f} s, ddg_setup {t2-t1:.1f} s", flush=True)
    s.close()
