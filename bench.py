#!/usr/bin/env python
"""bench.py — DDG-preconditioned PCG on B200 (BASELINE.json metric).

One "step" = one full PCG solve A u = f to rtol 1e-8 from u_0 = 0 with the
two-level DDG Schwarz preconditioner (every §8(a) row: SpMV+dot, update,
colour sweeps, coarse restrict/solve/prolong, reverse sweeps, r^T z,
direction), f already resident in HBM.  value = DoF * iterations / s over all
ranks (time-to-rtol = ms_per_step).  e2e = the same metric through
ddg_pcg_solve with pinned HOST f/u (H2D of f and D2H of u inside the timed
region).  Workload at N=1: C3 (3D lognormal 256^3, 4^3 blocks, p=1) -- the
largest BASELINE config that fits one GPU and the one BASELINE quotes at
1/2/4/8 GPUs; --config C1..C5 selects the others.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ddg|reference] [--config Cx]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG DoF*iterations/s (fp64) and time-to-rtol; % HBM roofline"
UNIT = "DoF*it/s"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "100", "-i", str(self.dev)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 8:
                try:
                    rows.append((float(p[1]), float(p[2]), p[4:8]))
                except ValueError:
                    pass
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i in range(4) if r[i].lower().startswith("active")})
        sm = [r[0] for r in rows]
        load_sm = [s for s in sm if s > 0.3 * rows[0][1]] or sm
        return {"sm_mhz": float(np.median(load_sm)), "sm_max_mhz": rows[0][1], "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def model_bytes_per_iter(pr, info, sizes):
    """Algorithmic bytes of one PCG iteration for THIS implementation:
    local operators read once per visit (2 sweeps), the coarse operator bytes one solve reads
    (ddg_info.coarse_solve_bytes),
    per-visit vectors and the O(n) vector work (SURVEY.md §8(d) formula, a = CSR bytes/row)."""
    m = sizes.astype(np.float64)
    a = 12.0 * pr.nnz / pr.n + 4.0
    local = 2 * np.sum(8.0 * m * (m + 1) / 2)
    coarse = float(info.coarse_solve_bytes)     # dense: packed inverse; sparse: 2|G| + |H|
    visits = (64 + 2 * a) * m.sum()
    vec = (144 + 2 * a + 16 * pr.k) * pr.n
    return local + coarse + visits + vec, local


# Bounded CPU samples of each workload for the oracle (the same generator
# recipe -- stencil, coefficient law, block size, p, overlap -- on a smaller
# grid, so that the oracle's setup and solve take seconds, not hours)
CPU_SAMPLES = {
    "C1": (lambda P: P.poisson2d(64, 8, 1, 1001), "C1 itself: 2D Poisson 64^2, 8^2 blocks, p=1"),
    "C2": (lambda P: P.poisson3d(40, 8, 2, 1002), "C2 recipe at 40^3: 7-point Poisson, 8^3 blocks, p=2"),
    "C3": (lambda P: P.lognormal3d(48, 4, 1, 1003), "C3 recipe at 48^3: lognormal 7-point, 4^3 blocks, p=1"),
    "C4": (lambda P: P.elasticity3d(16, 8, 1004), "C4 recipe at 16^3 elements: Q1 elasticity, 8^3-element blocks"),
    "C5": (lambda P: P.biharmonic2d(256, 16, 3, 1005), "C5 recipe at 256^2: 13-point biharmonic, 16^2 blocks, p=3"),
}


def run_cpu_baseline(rtol, config, steps=1):
    """The oracle as it stands (1 thread) on the bounded sample of `config`:
    solve phase timed (setup untimed), DoF*it/s = n * iterations / t_solve."""
    import oracle
    from ddg_gen import problems as P
    mk, desc = CPU_SAMPLES[config]
    pr = mk(P)
    t0 = time.time()
    o = oracle.Oracle.from_problem(pr)
    t_setup = time.time() - t0
    ts, its = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        u, it, hist, conv = o.pcg(pr.f, rtol)
        ts.append(time.perf_counter() - t0)
        its.append(it)
    t = float(np.mean(ts))
    out = {"value": pr.n * its[0] / t, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"{desc}; n={pr.n}, {its[0]} iterations, {t:.2f} s per solve (solve phase), "
                     f"setup {t_setup:.1f} s untimed; 1 thread",
           "ms_per_step": t * 1e3, "iters": its[0], "n": pr.n}
    # context: the full-size oracle run behind the parity goldens (tools/oracle_ref.py),
    # timed on the development container's host, not on this box
    g = os.path.join(ROOT, "tests", "golden", f"oracle_full_{config}.json")
    if os.path.exists(g):
        try:
            gj = json.load(open(g))
            ts_full = gj["timing"]["solve_s"]
            out["full_size_offline"] = {"value": gj["info"]["n"] * gj["iters"] / ts_full, "unit": UNIT,
                                        "solve_s": ts_full, "setup_s": gj["timing"]["setup_s"],
                                        "iters": gj["iters"], "where": "dev container, 1 thread"}
        except Exception:
            pass
    return out


def bench_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    for _ in range(args.warmup if args.warmup < 1 else 1):
        pass
    cb = run_cpu_baseline(args.rtol, args.config, steps=max(1, args.steps))
    out = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config} (bounded CPU sample of its recipe)", "sample": cb["sample"]},
           "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "full_size_offline")
                            if k in cb},
           "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def bench_ddg(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from ddg_gen import problems as P
    from paper_1504_00907_b200 import Solver

    pr = P.make(args.config)
    stream = torch.cuda.Stream()           # the library launches on this stream; events too
    torch.cuda.set_stream(stream)
    comm = None
    if world > 1:
        # libddg owns its NCCL communicator; torch.distributed only bootstraps it
        from paper_1504_00907_b200 import ddg
        obj = [ddg.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = ddg.Comm(rank, world, obj[0], local)
    t0 = time.time()
    kw = {}
    if args.levels == 3:   # three-level method: second level on A_c
        p2, n2, bc2 = P.coarse_parts(pr, args.factor, coords=True)
        kw = dict(part2=p2, nparts2=n2, block_coords2=bc2)
    if args.local_variant == "cholesky":   # forward + back substitution against Cholesky factors
        kw["local_variant"] = 1
    s = Solver.from_problem(pr, device=local, stream=stream.cuda_stream, comm=comm, **kw)
    t_setup = time.time() - t0
    sizes = s.subdomain_sizes()
    f_d = torch.from_numpy(pr.f).cuda()
    u_d = torch.empty_like(f_d)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        it, hist, rep = s.solve_device(f_d.data_ptr(), u_d.data_ptr(), args.rtol)
    torch.cuda.synchronize()
    # ---------------- timed region: K device-resident solves ----------------
    clk = Clocks(local)
    clk.start()
    s.launch_count(reset=True)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters = []
    for _ in range(args.steps):
        it, hist, rep = s.solve_device(f_d.data_ptr(), u_d.data_ptr(), args.rtol)
        iters.append(it)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = s.launch_count(reset=True)
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    t_dev = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms = float(t_dev.item())
    ms_step = ms / args.steps
    it = iters[0]
    value = pr.n * it / (ms_step * 1e-3)          # one global problem shared by all ranks
    # ---------------- e2e: host buffers through ddg_pcg_solve ----------------
    f_h = torch.from_numpy(pr.f.copy()).pin_memory()
    u_h = torch.empty(pr.n, dtype=torch.float64).pin_memory()
    s.solve_host_ptr(f_h.data_ptr(), u_h.data_ptr(), args.rtol)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        it_e, hist_e, _ = s.solve_host_ptr(f_h.data_ptr(), u_h.data_ptr(), args.rtol)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e = e0.elapsed_time(e1)
    t_dev = torch.tensor([ms_e], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms_e = float(t_dev.item()) / args.steps
    e2e_val = pr.n * it_e / (ms_e * 1e-3)
    assert np.array_equal(u_h.numpy(), u_d.cpu().numpy()), "e2e and device paths disagree"
    # ---------------- live kernel timing for the roofline ----------------
    s.set_profiling(True)
    s.solve_device(f_d.data_ptr(), u_d.data_ptr(), args.rtol)
    st = s.kernel_stats()
    s.set_profiling(False)
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    per_launch_bytes = st.symv_alg_bytes / max(1, st.symv_launches)
    per_launch_s = st.symv_ms * 1e-3 / max(1, st.symv_launches)
    achieved = per_launch_bytes / per_launch_s / 1e9
    # ncu dram bytes per launch of this workload's dominant kernel (one --set full
    # capture per config, profiles/symv_traffic_<workload>.json), or null
    traffic = None
    workload = args.config + ("-3level" if args.levels == 3 else "") + (
        "-cholesky" if args.local_variant == "cholesky" else "")
    tpath = os.path.join(ROOT, "profiles", f"symv_traffic_{workload}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    b_iter, b_local = model_bytes_per_iter(pr, s.info, sizes)
    iter_gbs = b_iter * it / (ms_step * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "desc": P.CONFIG_TEXT[args.config], "n": pr.n,
                   "iterations": it, "rtol": args.rtol, "n_c": int(s.info.n_c),
                   "nparts": int(s.info.nparts), "colours": int(s.info.ncolours),
                   "coarse": {1: "dense packed inverse", 2: "sparse nested dissection",
                              3: "three levels: two-level DDG on A_c (second level %s, n_c2=%d, %d parts)" % (
                                  "dense" if s.info.coarse_variant2 == 1 else "sparse", s.info.n_c2,
                                  s.info.nparts2)}[s.info.coarse_variant],
                   "levels": int(s.info.levels), "parallelism": f"subdomain-sharded x{world} (NCCL halos, boundary subdomains first; "
                                  f"split reductions; coarse solve {'distributed over the ranks' if s.info.coarse_variant == 2 else 'replicated (dense)'})" if world > 1 else "1gpu",
                   "l2": "inputs larger than L2 (local inverses %.1f GB)" % (s.info.local_factor_bytes / 1e9),
                   "time_to_rtol_ms": ms_step, "t_setup_s": round(t_setup, 2),
                   "cond_est_lanczos": round(float(rep.cond_est), 3),
                   "cg_iteration_bound": round(float(rep.iter_bound), 2),
                   "true_residual_rel": float(rep.true_res) / float(np.linalg.norm(pr.f)),
                   "local_operator_bytes": int(s.info.local_factor_bytes),
                   "coarse_solve_bytes": int(s.info.coarse_solve_bytes)},
        "roofline": {"bound": "hbm", "kernel": "k_chol_solve (colour sweep, a4/a8; one factor read per visit "
                     "counted)" if args.local_variant == "cholesky" else "k_symv (colour sweep, a4/a8)",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"
                     if not pk.get("_fallback") else "fallback 6650 GB/s",
                     "alg_bytes_per_launch": per_launch_bytes, "launch_ms": per_launch_s * 1e3,
                     "launches_profiled": int(st.symv_launches),
                     "share_of_step": st.symv_ms / max(1e-9, st.symv_ms + st.gather_ms + st.reduce_ms
                                                        + st.coarse_ms + st.vec_ms),
                     "iteration_model_GBps": iter_gbs, "iteration_frac": iter_gbs / hbm,
                     "iteration_model_bytes": b_iter},
        "kernel_ms_per_solve": {"symv": st.symv_ms, "gather": st.gather_ms, "reduce": st.reduce_ms,
                                "coarse": st.coarse_ms, "vector": st.vec_ms},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * pr.n,
                "d2h_bytes_per_step": 8 * pr.n + 8 * (it_e + 1), "ms_per_step": ms_e},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = run_cpu_baseline(args.rtol, args.config)
        out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "full_size_offline")
                               if k in cb}
    if rank == 0:
        print(json.dumps(out), flush=True)
    s.close()
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ddg", choices=["ddg", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--levels", type=int, default=2, choices=[2, 3])
    ap.add_argument("--factor", type=int, default=None,
                    help="three levels: parts grouped per axis into a second-level part (default H/h)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--local-variant", default="inverse", choices=["inverse", "cholesky"],
                    help="exact local solves: explicit inverse (default) or Cholesky substitutions")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one rank per GPU: re-launch under torchrun (rank 0 prints the line)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
               os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ddg(args)


if __name__ == "__main__":
    sys.exit(main())
