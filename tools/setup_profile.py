"""Where ddg_setup's device time goes: CUPTI kernel activity (torch.profiler)
around Solver construction, summed per kernel name.

  python tools/setup_profile.py C3 [local_variant]   -> table on stdout"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402

cfg = sys.argv[1]
lv = int(sys.argv[2]) if len(sys.argv) > 2 else 0
pr = P.make(cfg)
torch.cuda.init()
t0 = time.time()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s = Solver.from_problem(pr, device=0, local_variant=lv)
    torch.cuda.synchronize()
t = time.time() - t0
tot = {}
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    k = ev.name.split("(")[0].split("<")[0]
    a = tot.setdefault(k, [0.0, 0])
    a[0] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    a[1] += 1
print(f"{cfg} local_variant={lv}: setup wall {t:.2f} s (under the profiler)")
print("| kernel | launches | ms |")
print("|---|---|---|")
for k, (us, c) in sorted(tot.items(), key=lambda x: -x[1][0])[:20]:
    print(f"| {k} | {c} | {us / 1e3:.1f} |")
s.close()
