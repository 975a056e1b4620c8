"""material-aware generating vectors,
problem (C) "Non-smooth Poisson" of BigResultsTable on the GPU path.

div(D grad u) = f with D = S + 100 J (two materials, J an indicator), on a
structured square grid (ddg_gen.problems.material2d; the paper's annulus mesh
is out of scope), block partitions that do not conform to the material
boundary, Delta = 0, 10^-9 residual reduction after the first preconditioner
application (stop mode 1, reading R1), Gaussian right-hand side.

For every size, H/h and p it runs the plain F (k columns) and the
material-aware F = [F (1 - J), F J] (2k columns; R7 drops the columns that
vanish on a part), and reports iterations and n_c.  The paper: "it makes no
difference with the piecewise constant basis.  However, with the piecewise
cubic basis, this material-aware F reduces the iteration count by nearly one
half"; its BigResultsTable row is quoted
for the two-level columns.

  python tools/material_sweep.py [m ...]   -> JSON lines, then a markdown table
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from ddg_gen import rng  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402
from paper_1504_00907_b200.ddg import STOP_RES1  # noqa: E402

# BigResultsTable, nabla . D nabla rows: two-level H/h=10 P0..P3, H/h=20 P0..P3
PAPER = {200: ([43, 19, 15, 12], [56, 27, 22, 16]), 400: ([46, 20, 15, 13], [64, 28, 22, 19]),
         800: ([48, 21, 16, 13], [67, 31, 23, 18]), 1600: ([52, 21, 17, 14], [69, 33, 23, 20]),
         3200: ([58, 24, 17, 13], [69, 31, 24, 19])}


def run(m, hh, p, aware):
    pr = P.material2d(m, hh, p, 5000 + m, overlap=0, aware=aware)
    pr.f = rng.normal(5000 + m, pr.n)
    t0 = time.time()
    s = Solver.from_problem(pr, device=0, stop_mode=STOP_RES1, max_iter=1000)
    ts = time.time() - t0
    f = torch.from_numpy(pr.f).cuda()
    u = torch.empty_like(f)
    it, hist, rep = s.solve_device(f.data_ptr(), u.data_ptr(), 1e-9)
    torch.cuda.synchronize()
    out = {"m": m, "hh": hh, "p": p, "aware": aware, "n": pr.n, "k": pr.k, "n_c": int(s.info.n_c),
           "dropped": int(s.info.dropped), "iters": it, "converged": bool(rep.converged),
           "frac": round(float(rep.frac_iters), 2), "cond_est": round(float(rep.cond_est), 2),
           "setup_s": round(ts, 2), "solve_ms": round(float(rep.t_solve) * 1e3, 2)}
    s.close()
    del f, u
    torch.cuda.empty_cache()
    return out


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [200, 400, 800, 1600]
    res = {}
    for m in sizes:
        for hh in (10, 20):
            for p in range(4):
                for aware in (False, True):
                    r = run(m, hh, p, aware)
                    res[(m, hh, p, aware)] = r
                    print(json.dumps(r), flush=True)
    print("\nProblem (C), two materials: iterations plain F / material-aware F (paper's row, "
          "material-aware, in brackets)\n")
    print("| m | H/h=10 P0 | P1 | P2 | P3 | H/h=20 P0 | P1 | P2 | P3 |")
    print("|---|" + "---|" * 8)
    for m in sizes:
        cells = []
        for col, hh in enumerate((10, 20)):
            for p in range(4):
                a, b = res[(m, hh, p, False)], res[(m, hh, p, True)]
                pv = PAPER.get(m, (None, None))[col]
                cells.append(f"{a['iters']} / {b['iters']}" + (f" [{pv[p]}]" if pv else ""))
        print(f"| {m} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
