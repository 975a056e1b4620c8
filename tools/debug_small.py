import sys
import numpy as np
sys.path.insert(0, ".")
from ddg_gen import problems as P
from paper_1504_00907_b200 import Solver, DDGError
pr = P.poisson3d(32, 4, 2, 22)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    try:
        s = Solver(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, pr.part, pr.nparts, overlap=1,
                   block_coords=None, coarse_variant=2)
        print("rep", rep, "ok", flush=True)
        del s
    except DDGError as e:
        print("rep", rep, "ERROR", e, flush=True)
