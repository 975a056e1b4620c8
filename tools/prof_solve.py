"""Profile ONE device-resident PCG solve of a BASELINE config under ncu.

Setup and a warm-up solve run outside the profiled range; the solve is
bracketed by cudaProfilerStart/Stop, so `ncu --profile-from-start off` sees
only the hot path:

  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --csv --log-file out.csv python tools/prof_solve.py C3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 2          # 3: three-level method
factor = int(sys.argv[3]) if len(sys.argv) > 3 else None        # parts grouped per axis
pr = P.make(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
kw = {}
if levels == 3:
    p2, n2, bc2 = P.coarse_parts(pr, factor, coords=True)
    kw = dict(part2=p2, nparts2=n2, block_coords2=bc2)
kw["local_variant"] = int(os.environ.get("LOCAL_VARIANT", "0"))   # 1: Cholesky substitutions
s = Solver.from_problem(pr, device=0, stream=stream.cuda_stream, verbose=int(os.environ.get("VERBOSE", "0")), **kw)
inf = s.info
print(f"levels={inf.levels} n_c={inf.n_c} colours={inf.ncolours} n_c2={inf.n_c2} parts2={inf.nparts2} "
      f"colours2={inf.ncolours2} variant2={inf.coarse_variant2}", flush=True)
f = torch.from_numpy(pr.f).cuda()
u = torch.empty_like(f)
s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8)
torch.cuda.synchronize()
torch.cuda.profiler.start()
it, hist, rep = s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{cfg}: iters={it} coarse_bytes={s.info.coarse_factor_bytes} local_bytes={s.info.local_factor_bytes} "
      f"n_c={s.info.n_c}", flush=True)
s.close()
