"""SURVEY.md §8(f) f2 evidence on one GPU: the distributed coarse solve's
split of a BASELINE config's nested-dissection tree over P ranks (the plan
libddg makes: top fronts replicated, subtrees below the depth-ceil(log2 P)
cut owned by one rank each), as coarse solve bytes read per rank.

  python tools/coarse_split.py C3 [C5 ...]   -> markdown table on stdout"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver, ddg  # noqa: E402

L = ddg.load()
L.ddg_debug_coarse_split.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
print("| cfg | P | subtrees | top fronts (GB) | per rank, top split: max (GB) | max / replicated | "
      "per rank, top replicated: max (GB) | max / replicated | replicated solve (GB) |")
print("|---|---|---|---|---|---|---|---|---|")
for cfg in sys.argv[1:] or ["C3"]:
    pr = P.make(cfg)
    s = Solver.from_problem(pr, device=0)
    full = s.info.coarse_solve_bytes
    for nr in (1, 2, 4, 8):
        b = (C.c_double * nr)()
        top = C.c_double()
        ns = L.ddg_debug_coarse_split(s._h, nr, b, C.byref(top))
        split = max(b) + top.value / nr
        rep = max(b) + top.value
        print(f"| {cfg} | {nr} | {ns} | {top.value / 1e9:.2f} | {split / 1e9:.2f} | {split / full:.3f} | "
              f"{rep / 1e9:.2f} | {rep / full:.3f} | {full / 1e9:.2f} |", flush=True)
    s.close()
