"""Colour-sweep SYMV throughput of one config under the current switches
(DDG_RING_WHOLE, DDG_WHOLE_WARPS, ...): CUDA-event timing of every SYMV launch
of a few preconditioner applications (no PCG, so debug switches that break
the arithmetic can still be timed).

  python tools/symv_probe.py C3 [applications]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import numpy as np  # noqa: E402

from ddg_gen import problems as P  # noqa: E402
from paper_1504_00907_b200 import Solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pr = P.make(cfg)
s = Solver.from_problem(pr)
r = np.random.default_rng(0).standard_normal(pr.n)
s.apply_precond(r)
s.set_profiling(True)
for _ in range(reps):
    s.apply_precond(r)
st = s.kernel_stats()
s.set_profiling(False)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.5) \
    if os.path.exists("MEASURED_PEAKS.json") else 6548.5
gbs = st.symv_alg_bytes / (st.symv_ms * 1e-3) / 1e9
print(json.dumps({"cfg": cfg, "env": {k: v for k, v in os.environ.items() if k.startswith("DDG_")},
                  "symv_ms_per_apply": st.symv_ms / reps, "launches": int(st.symv_launches),
                  "alg_GBps": gbs, "frac": gbs / peak}))
s.close()
