"""the paper's p-sweep on the biharmonic problem on the GPU
path: 1000^2 grid, H/h = 125 (64
subdomains of ~16.6k unknowns with overlap 2), generating vectors of degree
<= p, stopping rule "10^-9 reduction in residual after the first application
of the preconditioner" (stop mode 1, reading R1).  The figure data is not in
PAPER.md, so this is a trend check: iterations should fall as p grows.

  python tools/p_sweep.py [p ...]   -> markdown table on stdout"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402
from paper_1504_00907_b200.ddg import STOP_RES1  # noqa: E402

ps = [int(x) for x in sys.argv[1:]] or [0, 1, 3, 5, 7]
print("| p | k | n_c | iterations | fractional | κ (Lanczos) | setup s | solve ms |")
print("|---|---|---|---|---|---|---|---|")
for p in ps:
    pr = P.biharmonic2d(1000, 125, p, 2000 + p, overlap=2)
    t0 = time.time()
    s = Solver.from_problem(pr, device=0, stop_mode=STOP_RES1, max_iter=1000)
    ts = time.time() - t0
    f = torch.from_numpy(pr.f).cuda()
    u = torch.empty_like(f)
    s.solve_device(f.data_ptr(), u.data_ptr(), 1e-9)
    torch.cuda.synchronize()
    t0 = time.time()
    it, hist, rep = s.solve_device(f.data_ptr(), u.data_ptr(), 1e-9)
    torch.cuda.synchronize()
    tsol = (time.time() - t0) * 1e3
    print(f"| {p} | {pr.k} | {s.info.n_c} | {it} | {rep.frac_iters:.2f} | {rep.cond_est:.1f} | {ts:.1f} | {tsol:.1f} |",
          flush=True)
    s.close()
    del f, u
    torch.cuda.empty_cache()
