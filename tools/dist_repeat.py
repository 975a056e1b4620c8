"""Which loopback coarse path is not bitwise repeatable: the distributed
sparse coarse solve or the replicated one (DDG_COARSE_REPLICATED=1), against
the single-context coarse correction, over repeated runs."""
import os
import sys
import threading

os.environ.setdefault("DDG_ND_LEAF", "64")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402
from paper_1504_00907_b200.ddg import LoopGroup  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 4
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pr = P.biharmonic2d(128, 16, 3, 1005)
r = np.random.default_rng(6).standard_normal(pr.n)
s1 = Solver.from_problem(pr, coarse_variant=2)
z1 = s1.coarse_correct(r)
s1.close()
for mode in ("dist", "replicated", "dist"):
    if mode == "replicated":
        os.environ["DDG_COARSE_REPLICATED"] = "1"
    else:
        os.environ.pop("DDG_COARSE_REPLICATED", None)
    seen = {}
    for t in range(trials):
        g = LoopGroup(nr)
        out = [None] * nr

        def body(k):
            s = Solver.from_problem(pr, comm=g.comm(k), coarse_variant=2)
            out[k] = [s.coarse_correct(r) for _ in range(3)]
            s.close()

        th = [threading.Thread(target=body, args=(k,)) for k in range(nr)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        g.close()
        for k in range(nr):
            for j, z in enumerate(out[k]):
                key = z.tobytes()
                seen.setdefault(key, []).append((t, k, j))
    print(mode, "distinct results:", len(seen), "equal to single-context:",
          any(np.array_equal(np.frombuffer(kk), z1) for kk in seen), flush=True)
    for kk, where in seen.items():
        zz = np.frombuffer(kk)
        print("   ", len(where), "times, rel diff to single", float(np.linalg.norm(zz - z1) / np.linalg.norm(z1)),
              "first at", where[0], flush=True)
