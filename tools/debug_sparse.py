"""Debug: sparse vs dense coarse correction on mid-size problems (GPU)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from ddg_gen import problems as P
from paper_1504_00907_b200 import Solver, DDGError

cases = [("biharm512", lambda: P.biharmonic2d(512, 16, 3, 5)),
         ("poisson3d_64_b8_p2", lambda: P.poisson3d(64, 8, 2, 6)),
         ("C2", lambda: P.make("C2")),
         ("C5", lambda: P.make("C5"))]
for name, mk in cases:
    pr = mk()
    r = np.random.default_rng(0).standard_normal(pr.n)
    res = {}
    for cv, geom in ((2, True), (2, False), (2, True), (1, True)):
        if cv == 1 and pr.nparts * pr.k > 50000:
            continue
        t = time.time()
        try:
            s = Solver(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, pr.part, pr.nparts, overlap=1,
                       block_coords=pr.block_coords if geom else None, coarse_variant=cv, verbose=False)
            z = s.coarse_correct(r)
            res[(cv, geom)] = z
            print(name, "cv", cv, "geom", geom, "ok", round(time.time() - t, 2), "s; coarse bytes",
                  s.info.coarse_factor_bytes, flush=True)
            del s
        except DDGError as e:
            print(name, "cv", cv, "geom", geom, "ERROR", e, flush=True)
    keys = list(res)
    for a in keys:
        for b in keys:
            if a < b:
                print("   diff", a, b, np.linalg.norm(res[a] - res[b]) / np.linalg.norm(res[b]))
