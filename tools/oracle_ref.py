"""Full-size oracle references for the GPU parity tests (calls only oracle/ and ddg_gen/).

For a BASELINE config this runs the CPU oracle (oracle/, PAPER.md:547-564 and
605-608) from the seeded generator and writes

  refcache/<cfg>.u.npy            the oracle's u (fp64, git-ignored, ships with gpurun)
  refcache_perturb/<cfg>.perturb.u.npy   the floor-mode u (--perturb; not shipped)
  tests/golden/oracle_full_<cfg>.json
      iterations, converged, residual history, ||u||, sha256 of u's bytes,
      4096 sampled entries of u at seeded positions (so the GPU test can check
      u element by element even where refcache/ is absent), timings; after
      --floor also the floor |u - u_perturbed| / |u| and the history spread
  tests/golden/oracle_full_<cfg>_perturb.json   the floor-mode run's record

Every stored value is produced here by the oracle; nothing comes from the CUDA
path.  Usage:  python tools/oracle_ref.py C2 [--perturb] [--scratch DIR];  ... C2 --floor
Configs: C1..C5 (BASELINE.json) and C3m (the C3 recipe at 128^3: n_c = 131072,
a 4096-unknown root front).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from ddg_gen import problems as P  # noqa: E402

CACHE = os.path.join(ROOT, "refcache")
GOLD = os.path.join(ROOT, "tests", "golden")
SAMPLE = 4096
SAMPLE_SEED = 20260


def problem(cfg):
    if cfg == "C3m":
        return P.lognormal3d(128, 4, 1, 1003)
    return P.make(cfg)


def coarse_mode(pr):
    # the envelope Cholesky of oracle.c where its envelope fits (C1, C2, C4, C5);
    # the nested-dissection multifrontal solve for the C3 family
    return "nd" if pr.name.startswith("lognormal3d") and pr.n > 1_000_000 else "envelope"


def sample_positions(n):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n, size=min(SAMPLE, n), replace=False))


def run(cfg, perturb, scratch):
    t0 = time.time()
    pr = problem(cfg)
    t1 = time.time()
    o = oracle.Oracle.from_problem(pr, coarse=coarse_mode(pr), perturb=perturb, scratch=scratch)
    t2 = time.time()
    u, it, hist, conv = o.pcg(pr.f, 1e-8, 1000)
    t3 = time.time()
    info = dict(n=o.n, nc=o.nc, nparts=o.nparts, ncolours=o.ncolours, m_min=o.m_min, m_max=o.m_max,
                dropped=o.dropped, min_rank_ratio=o.min_rank_ratio(), coarse=coarse_mode(pr))
    tim = dict(generate_s=t1 - t0, setup_s=t2 - t1, solve_s=t3 - t2, threads_solve=1)
    print(f"{cfg}{' perturb' if perturb else ''}: iters={it} conv={conv} setup {t2 - t1:.0f}s "
          f"solve {t3 - t2:.0f}s", flush=True)
    return pr, u, it, hist, conv, info, tim


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--perturb", action="store_true")
    ap.add_argument("--scratch", default=None)
    ap.add_argument("--floor", action="store_true", help="only combine the two runs' floor")
    a = ap.parse_args()
    os.makedirs(CACHE, exist_ok=True)
    gpath = os.path.join(GOLD, f"oracle_full_{a.cfg}.json")
    if a.floor:
        # floor: |u - u_perturbed| / |u| (SURVEY.md §8(c) "an unavoidable floor")
        g = json.load(open(gpath))
        gp = json.load(open(os.path.join(GOLD, f"oracle_full_{a.cfg}_perturb.json")))
        u0 = np.load(os.path.join(CACHE, f"{a.cfg}.u.npy"))
        up = np.load(os.path.join(CACHE + "_perturb", f"{a.cfg}.perturb.u.npy"))
        h0, hp = np.array(g["hist"]), np.array(gp["hist"])
        m = min(len(h0), len(hp))
        g["floor"] = dict(u_rel=float(np.linalg.norm(u0 - up) / np.linalg.norm(u0)),
                          hist_rel_max=float(np.max(np.abs(h0[:m] - hp[:m]) / h0[:m])),
                          iters=[int(g["iters"]), int(gp["iters"])])
        print(a.cfg, g["floor"])
    else:
        pr, u, it, hist, conv, info, tim = run(a.cfg, a.perturb, a.scratch)
        tag = a.cfg + (".perturb" if a.perturb else "")
        np.save(os.path.join(CACHE + ("_perturb" if a.perturb else ""), f"{tag}.u.npy"), u)
        g = dict(config=a.cfg, perturb=bool(a.perturb), iters=int(it), converged=bool(conv),
                 hist=[float(x) for x in hist], u_norm=float(np.linalg.norm(u)),
                 u_sha256=hashlib.sha256(u.tobytes()).hexdigest(), info=info, timing=tim,
                 provenance=("tools/oracle_ref.py: the CPU oracle (oracle/) on the seeded generator "
                             "(ddg_gen/), rtol 1e-8, stop rule R1(i), u_0 = 0; PAPER.md:547-564, "
                             "605-608" + ("; floor mode (oracle.h or_opts.perturb)" if a.perturb else "")))
        if not a.perturb:
            pos = sample_positions(pr.n)
            g.update(sample_pos=[int(x) for x in pos], sample_u=[float(x) for x in u[pos]])
        else:
            gpath = os.path.join(GOLD, f"oracle_full_{a.cfg}_perturb.json")
    with open(gpath, "w") as fh:
        json.dump(g, fh, indent=1)
    print("wrote", gpath)


if __name__ == "__main__":
    main()
