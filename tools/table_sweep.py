"""the paper's iteration-count table (BigResultsTable,
PAPER.md:675-740) for the two problems on regular grids, run on the GPU path.

  (A) Poisson 3D, 7-point FD, one Dirichlet face, Neumann elsewhere
      (ddg_gen.problems.poisson3d_mixed, reading R21),
      Delta = 0, 10^-9 residual reduction after the first preconditioner
      application (stop mode 1, reading R1), Gaussian right-hand side;
  (F) biharmonic, 13-point FD, clamped, Delta = 1,
      10^-6 reduction.

Columns: two-level at H/h = 10 and 20, three-level at H/h = 10 (second-level
parts = the blocks grouped round(blocks / 10) per axis).
CG is stopped at 1000 iterations; then the Lanczos bound is reported, as the
paper does.  Partitions are blocks, not the paper's
recursive inertial bisection (out of scope), and (A) stops at the sizes whose
dense local inverses fit one B200 (m = 160 at H/h = 10, m = 80 at H/h = 20).

  python tools/table_sweep.py A|F [m ...]   -> JSON lines, then a markdown table
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
from paper_1504_00907_b200.ddg import DDGError, STOP_RES1  # noqa: E402

# BigResultsTable as printed in PAPER.md:697-702 (∇·∇ 3D) and 733-736 (∇⁴): per n^{1/d},
# two-level H/h=10 P0..P3, two-level H/h=20 P0..P3, three-level H/h=10 P0..P3 (the
# three-level P0 column is hidden by the "H" column type when rendered, reading R18;
# None = "too small", i.e. the paper's x).  Values above 1000 are Lanczos bounds.
PAPER = {
    "A": {40: ([36, 20, 15, 12], [35, 23, 18, 15], [36, None, None, None]),
          80: ([41, 20, 16, 13], [51, 28, 21, 18], [41, None, None, None]),
          160: ([44, 21, 16, 13], [61, 30, 23, 19], [73, 39, 29, 23]),
          320: ([44, 21, 16, 14], [63, 30, 23, 19], [92, 43, 32, 26]),
          640: ([46, 22, 16, 14], [65, 31, 23, 19], [100, 48, 35, 34])},
    "F": {200: ([698, 62, 20, 12], [600, 154, 44, 24], [722, 119, 40, 22]),
          400: ([2900, 68, 21, 12], [3500, 188, 53, 27], [4300, 376, 112, 37]),
          800: ([5700, 77, 25, 15], [6900, 184, 55, 32], [7900, 961, 156, 51]),
          1600: ([9500, 99, 31, 15], [11000, 246, 70, 30], [14000, 2100, 169, 58])},
}
# sizes whose dense local inverses fit (bytes ~ parts * 4 (H/h)^6 for (A))
FITS = {"A": {10: [40, 80, 160], 20: [40, 80]}, "F": {10: [200, 400, 800, 1600], 20: [200, 400, 800, 1600]}}


def make(prob, m, hh, p):
    if prob == "A":
        return P.poisson3d_mixed(m, hh, p, 3000 + m, overlap=0), 1e-9
    pr = P.biharmonic2d(m, hh, p, 4000 + m, overlap=1)
    pr.f = rng.normal(4000 + m, pr.n)
    return pr, 1e-6


def run(prob, m, hh, p, levels):
    pr, tol = make(prob, m, hh, p)
    kw = {}
    if levels == 3:
        try:
            p2, n2, bc2 = P.coarse_parts(pr, 10, coords=True, nearest=True)
        except ValueError:
            return {"prob": prob, "m": m, "hh": hh, "p": p, "levels": 3, "too_small": True}
        kw = dict(part2=p2, nparts2=n2, block_coords2=bc2)
    t0 = time.time()
    try:
        s = Solver.from_problem(pr, device=0, stop_mode=STOP_RES1, max_iter=1000, **kw)
    except DDGError as e:
        if "too small" in str(e):
            return {"prob": prob, "m": m, "hh": hh, "p": p, "levels": 3, "too_small": True}
        if "out of memory" in str(e):
            torch.cuda.empty_cache()
            return {"prob": prob, "m": m, "hh": hh, "p": p, "levels": levels, "oom": True}
        raise
    ts = time.time() - t0
    f = torch.from_numpy(pr.f).cuda()
    u = torch.empty_like(f)
    torch.cuda.synchronize()
    t0 = time.time()
    it, hist, rep = s.solve_device(f.data_ptr(), u.data_ptr(), tol)
    torch.cuda.synchronize()
    tsol = time.time() - t0
    out = {"prob": prob, "m": m, "hh": hh, "p": p, "levels": levels, "n": pr.n, "n_c": int(s.info.n_c),
           "n_c2": int(s.info.n_c2), "iters": it, "converged": bool(rep.converged),
           "frac": float(rep.frac_iters), "cond_est": float(rep.cond_est), "bound": float(rep.iter_bound),
           "setup_s": round(ts, 2), "solve_s": round(tsol, 3)}
    s.close()
    del f, u
    torch.cuda.empty_cache()
    return out


def cell(r):
    if r is None:
        return "—"
    if r.get("too_small"):
        return "✕"
    if r.get("oom"):
        return "(memory)"
    if not r["converged"]:
        return f"≥1000 ({r['bound']:.0f})"
    return f"{r['iters']}"


def main():
    prob = sys.argv[1] if len(sys.argv) > 1 else "A"
    ps = [int(x) for x in os.environ.get("TABLE_P", "0,1,2,3").split(",")]
    if os.environ.get("TABLE_FITS"):                # e.g. "10:320" to try a size outside FITS
        for item in os.environ["TABLE_FITS"].split(";"):
            hh, ms = item.split(":")
            FITS[prob][int(hh)] = sorted(set(FITS[prob][int(hh)]) | {int(m) for m in ms.split(",")})
    sizes = [int(x) for x in sys.argv[2:]] or sorted(set(FITS[prob][10]) | set(FITS[prob][20]))
    res = {}
    for m in sizes:
        for hh, lv in ((10, 2), (20, 2), (10, 3)):
            if m not in FITS[prob][hh]:
                continue
            for p in ps:
                r = run(prob, m, hh, p, lv)
                res[(m, hh, lv, p)] = r
                print(json.dumps(r), flush=True)
    name = {"A": "∇·∇ 3D (problem A)", "F": "∇⁴ (problem F)"}[prob]
    print(f"\n{name}: ours / paper, iterations to the paper's tolerance (PCG stopped at 1000: Lanczos bound)\n")
    print("| n^(1/d) | 2L H/h=10 P0 | P1 | P2 | P3 | 2L H/h=20 P0 | P1 | P2 | P3 | 3L H/h=10 P0 | P1 | P2 | P3 |")
    print("|---|" + "---|" * 12)
    for m in sizes:
        pap = PAPER[prob].get(m)
        cells = []
        for col, (hh, lv) in enumerate(((10, 2), (20, 2), (10, 3))):
            for p in range(4):
                ours = cell(res.get((m, hh, lv, p)))
                pv = pap[col][p] if pap else None
                cells.append(f"{ours} / {'✕' if pv is None and pap else pv}")
        print(f"| {m} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
