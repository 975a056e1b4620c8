"""Time kernel variants of one config: each variant is a fresh setup with
different ddg_opts / env knobs; prints per-class kernel ms of one profiled
solve and the device time of 3 unprofiled solves.
  python tools/variants.py C3 "small=1,fuse=0" "small=0,symv=tma" ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402

cfg = sys.argv[1]
pr = P.make(cfg)
f = torch.from_numpy(pr.f).cuda()
u = torch.empty_like(f)
for spec in sys.argv[2:]:
    kv = dict(x.split("=") for x in spec.split(",") if x)
    kw = {}
    if "small" in kv:
        kw["small_kernel"] = int(kv["small"])
    if "fuse" in kv:
        kw["fuse_gather"] = int(kv["fuse"])
    for k, v in kv.items():
        if k.startswith("DDG_"):
            os.environ[k] = v
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    t0 = time.time()
    s = Solver.from_problem(pr, device=0, stream=stream.cuda_stream, **kw)
    ts = time.time() - t0
    s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        it, hist, rep = s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    s.set_profiling(True)
    s.solve_device(f.data_ptr(), u.data_ptr(), 1e-8)
    st = s.kernel_stats()
    s.set_profiling(False)
    print(f"{cfg} [{spec}] it={it} ms/solve={ms:.2f} DoF*it/s={pr.n*it/ms*1e3:.3e} setup={ts:.1f}s | "
          f"symv {st.symv_ms:.2f} gather {st.gather_ms:.2f} coarse {st.coarse_ms:.2f} vec {st.vec_ms:.2f} "
          f"symv_GBps {st.symv_alg_bytes/max(st.symv_ms,1e-9)/1e6:.0f} res={hist[-1]/hist[0]:.2e}", flush=True)
    s.close()
    for k in kv:
        if k.startswith("DDG_"):
            del os.environ[k]
