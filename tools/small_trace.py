"""k_pcg_small phase timeline: %globaltimer at every cluster barrier of CTA 0
(debug entry ddg_debug_small_trace) for one C1 solve; with DDG_SMALL_TRACE=2
also (globaltimer, clock64) pairs inside the colour steps, giving the SM clock."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver, ddg  # noqa: E402

pr = P.poisson2d(64, 8, 1, 1001)
s = Solver.from_problem(pr)
for _ in range(20):
    s.solve(pr.f, 1e-8)
lib = ddg.load()
lib.ddg_debug_small_trace.argtypes = [C.c_int, C.c_void_p, C.c_int]
lib.ddg_debug_small_trace(1, None, 0)
s.launch_count(reset=True)
u, it, hist, rep = s.solve(pr.f, 1e-8)
print("launches", s.launch_count())
buf = np.zeros(4096, np.uint64)
n = lib.ddg_debug_small_trace(0, buf.ctypes.data, 4096)
raw = buf[:n]
clk = raw >> np.uint64(63)
tm = raw[clk == 0].astype(np.float64)
# (globaltimer, clock) pairs: the stamp entries are followed by a flagged clock
pairs = [(float(raw[i]), float(raw[i + 1] & np.uint64((1 << 63) - 1))) for i in range(n - 1)
         if clk[i] == 0 and clk[i + 1] == 1]
if len(pairs) > 2:
    (t0, c0), (t1, c1) = pairs[0], pairs[-1]
    print(f"SM clock {1e3 * (c1 - c0) / (t1 - t0):.0f} MHz over {(t1 - t0) / 1e3:.1f} us")
d = np.diff(tm) / 1e3
print(f"iters {it}, {len(tm)} stamps, span {(tm[-1] - tm[0]) / 1e3:.1f} us, per iteration {(tm[-1] - tm[0]) / 1e3 / it:.1f} us")
print("gaps (us):", " ".join(f"{x:.2f}" for x in d[:48]))
s.close()
