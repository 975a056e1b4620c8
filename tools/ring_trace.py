"""k_symv_ring role/wait breakdown (DDG_RING_TRACE=1) over one device solve's colour sweeps."""
import ctypes as C
import os
import sys

os.environ["DDG_RING_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver, ddg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
pr = P.make(cfg)
s = Solver.from_problem(pr, device=0)
f = torch.from_numpy(pr.f).cuda()
u = torch.empty_like(f)
L = ddg.load()
out = np.zeros(24, np.uint64)
s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8)
L.ddg_debug_ring_trace(C.c_void_p(out.ctypes.data))          # discard warm-up
s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8)
L.ddg_debug_ring_trace(C.c_void_p(out.ctypes.data))
o = out.astype(np.float64)
prod, epi, cons = o[0:8], o[8:16], o[16:24]
print(f"{cfg}: producer wait sempty {prod[0]/prod[3]:.1%} wait empty {prod[1]/prod[3]:.1%} "
      f"desc loads {prod[2]/prod[3]:.1%} chunk issue {prod[6]/prod[3]:.1%} (total {prod[3]/1e9:.2f} Gcyc)")
print(f"   epilogue wait pdone {epi[0]/epi[3]:.1%}")
print(f"   consumers wait sfull {cons[0]/cons[3]:.1%} wait pfree {cons[1]/cons[3]:.1%} wait full {cons[2]/cons[3]:.1%} "
      f"| tiles {cons[4]:.0f} flushes {cons[5]:.0f} ({cons[5]/max(cons[4],1):.2f}/tile) "
      f"| busy cycles per tile per warp {(cons[3]-cons[0]-cons[1]-cons[2])/max(cons[4],1):.0f}")
s.close()
