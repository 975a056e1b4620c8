"""Multi-GPU decomposition, checked on the CPU with world_size 2 and 3 (gloo).

libddg's host-only plan (ddg_plan_create: part -> rank assignment, owned rows,
and the p / r / z-per-colour halo lists) drives a numpy re-enactment of the
distributed algorithm the GPU path enqueues (setup.cpp: enqueue_step_a,
enqueue_precond, enqueue_step_b).  Every rank keeps full-length views; values
it does not own start as NaN (p, q) or stale (r, z) and are refreshed ONLY
through the plan's exchanges, run with torch.distributed over gloo.  The
result must equal the oracle's single-process PCG: a missing or wrong halo
row makes it diverge or go NaN.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P

CASES = {
    "poisson2d": lambda: P.poisson2d(32, 8, 1, 31),
    "biharm": lambda: P.biharmonic2d(48, 8, 3, 32),
    "poisson3d": lambda: P.poisson3d(16, 4, 1, 33),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, geom, out_dir):
    import torch.distributed as dist
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1504_00907_b200 import ddg

    pr = CASES[case]()
    plan = ddg.Plan(pr, rank=rank, nranks=world, block_coords=pr.block_coords if geom else None)
    o = oracle.Oracle.from_problem(pr)
    A = pr.scipy()
    Pm = o.P_dense()
    Ac = o.Ac_dense()
    cptr = o.coarse_offsets()
    n = pr.n
    owned = plan.query("OWNED_ROWS")
    subs = plan.query("OWNED_SUBS")
    colours = plan.colours
    prolong = plan.query("PROLONG_PARTS")
    sets = {i: plan.query("OVERLAP", peer=int(i)) for i in subs}
    Ad = pr.dense() if n <= 4096 else None
    inv = {i: np.linalg.inv(Ad[np.ix_(sets[i], sets[i])]) for i in subs}
    peers = [q for q in range(world) if q != rank]

    def halo(v, kind, c=0):
        reqs, bufs = [], {}
        for q in peers:
            s_idx = plan.query(kind + "_SEND", colour=c, peer=q)
            r_idx = plan.query(kind + "_RECV", colour=c, peer=q)
            if len(s_idx):
                reqs.append(dist.isend(torch.from_numpy(v[s_idx].copy()), q))
            if len(r_idx):
                bufs[q] = (r_idx, torch.empty(len(r_idx), dtype=torch.float64))
                reqs.append(dist.irecv(bufs[q][1], q))
        for rq in reqs:
            rq.wait()
        for q, (r_idx, b) in bufs.items():
            v[r_idx] = b.numpy()

    def allsum(x):
        t = torch.tensor(np.atleast_1d(x), dtype=torch.float64)
        dist.all_reduce(t)
        return t.numpy() if np.ndim(x) else float(t[0])

    def colour_step(c, r, z):
        for i in subs:
            if colours[i] != c:
                continue
            idx = sets[i]
            s = r[idx] - (A[idx] @ z)
            z[idx] += inv[i] @ s
        halo(z, "Z", c)

    def precond(r):
        z = np.zeros(n)
        for c in range(plan.ncolours):
            colour_step(c, r, z)
        bc = np.zeros(o.nc)
        for I in subs:                       # coarse restriction on owned parts
            rows = np.nonzero(pr.part == I)[0]
            res = r[rows] - A[rows] @ z
            bc[cptr[I]:cptr[I + 1]] = Pm[rows, cptr[I]:cptr[I + 1]].T @ res
        bc = allsum(bc)
        y = np.linalg.solve(Ac, bc)
        for I in prolong:
            rows = np.nonzero(pr.part == I)[0]
            z[rows] += Pm[rows, cptr[I]:cptr[I + 1]] @ y[cptr[I]:cptr[I + 1]]
        for c in range(plan.ncolours - 1, -1, -1):
            colour_step(c, r, z)
        return z

    f = pr.f
    r = f.copy()
    u = np.zeros(n)
    p = np.full(n, np.nan)
    q = np.full(n, np.nan)
    res0 = np.sqrt(allsum(np.sum(f[owned] ** 2)))
    hist = [res0]
    z = precond(r)
    rho = allsum(np.dot(r[owned], z[owned]))
    p[owned] = z[owned]
    halo(p, "P")
    it = 0
    for it in range(1, 200):
        q[owned] = A[owned] @ p
        sigma = allsum(np.dot(p[owned], q[owned]))
        alpha = rho / sigma
        u[owned] += alpha * p[owned]
        r[owned] -= alpha * q[owned]
        res = np.sqrt(allsum(np.sum(r[owned] ** 2)))
        hist.append(res)
        if res <= 1e-8 * res0:
            break
        halo(r, "R")
        z = precond(r)
        rho1 = allsum(np.dot(r[owned], z[owned]))
        beta = rho1 / rho
        rho = rho1
        p[owned] = z[owned] + beta * p[owned]
        halo(p, "P")
    ufull = np.zeros(n)
    ufull[owned] = u[owned]
    ufull = allsum(ufull)
    if rank == 0:
        np.savez(os.path.join(out_dir, "dist.npz"), u=ufull, hist=np.array(hist), it=it,
                 part_rank=plan.query("PART_RANK"))
    dist.destroy_process_group()


@pytest.mark.parametrize("case,geom,world", [("poisson2d", True, 2), ("poisson2d", False, 3),
                                             ("biharm", True, 3), ("biharm", False, 2),
                                             ("poisson3d", True, 2)])
def test_distributed_pcg_equals_oracle(case, geom, world, tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, case, geom, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    d = np.load(os.path.join(tmp_path, "dist.npz"))
    pr = CASES[case]()
    o = oracle.Oracle.from_problem(pr)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)
    assert int(d["it"]) == ito
    m = min(len(histo), len(d["hist"]))
    assert np.max(np.abs(d["hist"][:m] - histo[:m]) / histo[:m]) <= 1e-8
    assert np.linalg.norm(d["u"] - uo) <= 1e-10 * np.linalg.norm(uo)
    pr_rank = d["part_rank"]
    assert set(pr_rank.tolist()) == set(range(world))     # every rank owns parts


def test_plan_partition_properties():
    """Owned rows partition the unknowns; sends equal the peer's receives."""
    from paper_1504_00907_b200 import ddg
    pr = P.poisson3d(16, 4, 2, 3)
    world = 4
    plans = [ddg.Plan(pr, rank=r, nranks=world) for r in range(world)]
    owned = np.concatenate([pl.query("OWNED_ROWS") for pl in plans])
    assert np.array_equal(np.sort(owned), np.arange(pr.n))
    for g in range(world):
        for h in range(world):
            if g == h:
                continue
            for kind in ("P", "R"):
                assert np.array_equal(plans[g].query(kind + "_SEND", peer=h),
                                      plans[h].query(kind + "_RECV", peer=g))
            for c in range(plans[g].ncolours):
                assert np.array_equal(plans[g].query("Z_SEND", colour=c, peer=h),
                                      plans[h].query("Z_RECV", colour=c, peer=g))
    # geometric split: each rank's parts form a box of the block grid
    pr_rank = plans[0].query("PART_RANK")
    for r in range(world):
        bc = pr.block_coords[pr_rank == r]
        ext = bc.max(axis=0) - bc.min(axis=0) + 1
        assert np.prod(ext) == len(bc)
