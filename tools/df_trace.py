"""Dataflow coarse-solve timeline (DDG_DF_TRACE=1): per phase/level spans."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["DDG_DF_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver, ddg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
pr = P.make(cfg)
s = Solver.from_problem(pr, device=0, use_graphs=False)
f = torch.from_numpy(pr.f).cuda()
u = torch.empty_like(f)
s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8, max_iter=1)
L = ddg.load()
cap = 1 << 22
tr = np.zeros(cap * 4, np.uint64)
wk = np.zeros(cap, np.int32)
n = L.ddg_debug_df_trace(s._h, C.c_void_p(tr.ctypes.data), C.c_void_p(wk.ctypes.data), cap)
tr = tr[: 4 * n].reshape(n, 4)
wk = wk[:n]
t0 = tr[:, 0].astype(np.int64)
base = t0.min()
nct = 296
t = [t0 - base] + [tr[:, k].astype(np.int64) - base for k in (1, 2, 3)]
kind = np.where(wk & (1 << 29), 0, np.where(wk & (1 << 30), 2, 1)) + np.where(wk & (1 << 28), 2, 0)
end = t[3].max()
print(f"{cfg}: {n} entries, span {end/1e3:.1f} us")
for k, nm in enumerate(["assemble", "fwd item", "bwd item", "fwd red", "bwd red"]):
    m = kind == k
    if not m.any():
        continue
    st, dep, done, fin = t[0][m], t[1][m], t[2][m], t[3][m]
    wait = np.where(dep > 0, dep - st, 0)
    work = np.where(done > 0, done - np.maximum(dep, st), 0)
    tail = fin - np.where(done > 0, done, st)
    print(f"  {nm:9s} n={m.sum():5d} first start {st.min()/1e3:7.1f} last finish {fin.max()/1e3:7.1f} us | "
          f"wait mean {wait.mean()/1e3:6.2f} max {wait.max()/1e3:6.1f} | item mean {work.mean()/1e3:6.2f} "
          f"max {work.max()/1e3:6.1f} | finisher tail mean {tail.mean()/1e3:6.2f} max {tail.max()/1e3:6.1f}")
# busy fraction over time
busy = np.sum(np.where(t[2] > 0, t[2] - np.maximum(t[1], t[0]), 0))
print(f"  item-busy CTA-time {busy/1e3:.0f} us of {nct*end/1e3:.0f} us CTA-time ({busy/(nct*end):.1%})")
# occupancy timeline: CTAs busy on items / reductions per 100 us bucket
B = 100_000
nb = int(end // B) + 1
occ_item = np.zeros(nb)
occ_red = np.zeros(nb)
for k in range(n):
    a, b = max(t[1][k], t[0][k]), t[2][k]
    if b <= 0:
        continue
    tgt = occ_red if kind[k] >= 3 else occ_item
    for q in range(int(a // B), int(b // B) + 1):
        lo, hi = max(a, q * B), min(b, (q + 1) * B)
        if hi > lo:
            tgt[q] += (hi - lo) / B
print("  busy CTAs per 100 us (items + reductions, of %d):" % nct)
print("  " + " ".join("%d" % (occ_item[q] + occ_red[q]) for q in range(nb)))
s.close()
