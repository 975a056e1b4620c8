"""The distributed exact coarse solve,
re-enacted on the CPU with world size 2 and 4 over gloo.

The algorithm libddg runs on the ranks (coarse_sparse.cpp dist_split /
sparse_coarse_enqueue_solve), here on the oracle's nested-dissection Cholesky
of A_0 (oracle/coarse_nd.py: the same PAPER.md:282-287 block structure, a
different elimination kernel):
  * the tree is cut at depth D = ceil(log2 P); subtrees below the cut go to
    ranks greedily by size, the fronts above it (the top separators) are shared;
  * forward: each rank eliminates its own subtrees on its copy of the right-
    hand side; the subtrees' updates of the top unknowns are summed over the
    ranks (one allreduce);
  * the top fronts, their work split over the ranks: for every top front each
    rank applies its share of the off-diagonal block's columns, the partial
    updates are allreduced, every rank does the (small) diagonal solves;
  * backward: each rank substitutes over its own subtrees;
  * y: every unknown is contributed by exactly one rank, one allreduce.
Every rank must end with A_0^{-1} b (the single-process oracle solve) to
rounding, although it only ever touched its own subtrees.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from ddg_gen import problems as P

CASES = {
    "poisson3d": lambda: P.poisson3d(24, 4, 1, 41),      # C3-shaped block graph
    "biharm": lambda: P.biharmonic2d(96, 8, 3, 42),      # C5-shaped, 13-point couplings
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def split(nodes, sizes, P_):
    """dist_split: depth cut, subtree roots, greedy owners (postorder nodes)."""
    nn = len(nodes)
    parent = np.full(nn, -1)
    for t, (_, kids) in enumerate(nodes):
        for ch in kids:
            parent[ch] = t
    depth = np.zeros(nn, int)
    for t in reversed(range(nn)):                      # parents come after children
        depth[t] = 0 if parent[t] < 0 else depth[parent[t]] + 1
    D = 0
    while (1 << D) < P_:
        D += 1
    top = depth < D
    sub = np.array(sizes, float)
    for t in range(nn):
        if parent[t] >= 0:
            sub[parent[t]] += sub[t]
    roots = [t for t in range(nn) if not top[t] and (parent[t] < 0 or top[parent[t]])]
    owner = np.full(nn, -1)
    load = np.zeros(P_)
    for r in sorted(roots, key=lambda t: -sub[t]):
        k = int(np.argmin(load))
        owner[r] = k
        load[k] += sub[r]
    for t in reversed(range(nn)):
        if not top[t] and owner[t] < 0:
            owner[t] = owner[parent[t]]
    return top, owner, roots


def _worker(rank, world, port, case, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pr = CASES[case]()
    o = oracle.Oracle.from_problem(pr)
    from oracle.coarse_nd import NDCholesky
    nd = NDCholesky(o.Ac_sparse(), o.coarse_offsets(), pr.block_coords, leaf=24)
    nn = len(nd.nodes)
    sizes = [len(nd.S[t]) ** 2 + 2 * len(nd.S[t]) * len(nd.B[t]) for t in range(nn)]
    top, owner, roots = split(nd.nodes, sizes, world)
    b = np.random.default_rng(7).standard_normal(nd.nc)

    def allsum(v):
        t = torch.from_numpy(np.ascontiguousarray(v, np.float64))
        dist.all_reduce(t)
        return t.numpy().copy()

    mine = [t for t in range(nn) if not top[t] and owner[t] == rank]
    x = b.copy()
    # forward over own subtrees (postorder: children first)
    for t in mine:
        S, Bt = nd.S[t], nd.B[t]
        y = sla.solve_triangular(nd.LSS[t], x[S], lower=True)
        x[S] = y
        if len(Bt):
            x[Bt] -= nd.LBS[t] @ y
    # the subtrees' updates of the top unknowns, summed over the ranks
    topS = np.concatenate([nd.S[t] for t in range(nn) if top[t]])
    x[topS] = b[topS] + allsum(x[topS] - b[topS])
    tops = [t for t in range(nn) if top[t]]                  # postorder = deepest first
    # forward over the top fronts, off-diagonal block columns split over the ranks
    for t in tops:
        S, Bt = nd.S[t], nd.B[t]
        y = sla.solve_triangular(nd.LSS[t], x[S], lower=True)
        x[S] = y
        if len(Bt):
            c0, c1 = len(S) * rank // world, len(S) * (rank + 1) // world
            part = nd.LBS[t][:, c0:c1] @ y[c0:c1]
            x[Bt] -= allsum(part)
    # backward over the top fronts (root first), block rows split
    for t in reversed(tops):
        S, Bt = nd.S[t], nd.B[t]
        if len(Bt):
            r0, r1 = len(Bt) * rank // world, len(Bt) * (rank + 1) // world
            part = nd.LBS[t][r0:r1, :].T @ x[Bt[r0:r1]]
            rhs = x[S] - allsum(part)
        else:
            rhs = x[S]
        x[S] = sla.solve_triangular(nd.LSS[t], rhs, lower=True, trans="T")
    # backward over own subtrees (root first)
    for t in reversed(mine):
        S, Bt = nd.S[t], nd.B[t]
        rhs = x[S] - (nd.LBS[t].T @ x[Bt] if len(Bt) else 0.0)
        x[S] = sla.solve_triangular(nd.LSS[t], rhs, lower=True, trans="T")
    # y: each unknown from exactly one rank (its subtree's owner, rank 0 the top)
    mask = np.zeros(nd.nc, bool)
    for t in range(nn):
        if (top[t] and rank == 0) or (not top[t] and owner[t] == rank):
            mask[nd.S[t]] = True
    y = allsum(np.where(mask, x, 0.0))
    touched = sum(len(nd.S[t]) for t in mine)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), y=y, b=b, touched=touched, nsub=len(roots),
             ntop=int(top.sum()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", list(CASES))
def test_distributed_coarse_solve_equals_replicated(case, world, tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    pr = CASES[case]()
    o = oracle.Oracle.from_problem(pr)
    A0 = o.Ac_dense()
    res = [np.load(os.path.join(tmp_path, f"r{k}.npz")) for k in range(world)]
    b = res[0]["b"]
    ref = np.linalg.solve(A0, b)                          # A_0^{-1} b, dense
    for d in res:
        assert np.linalg.norm(d["y"] - ref) <= 1e-11 * np.linalg.norm(ref)
        assert np.array_equal(d["y"], res[0]["y"])       # every rank holds the same y_c
    assert int(res[0]["nsub"]) >= world                   # every rank owns a subtree
    assert sum(int(d["touched"]) for d in res) < A0.shape[0]   # the top is shared, not owned


def test_split_plan_properties():
    """dist_split: the cut is at depth ceil(log2 P); subtree owners cover every
    rank; every non-top node's owner is its subtree root's."""
    pr = CASES["poisson3d"]()
    o = oracle.Oracle.from_problem(pr)
    from oracle.coarse_nd import NDCholesky
    nd = NDCholesky(o.Ac_sparse(), o.coarse_offsets(), pr.block_coords, leaf=24)
    nn = len(nd.nodes)
    sizes = [len(nd.S[t]) ** 2 for t in range(nn)]
    for P_ in (2, 3, 4, 8):
        top, owner, roots = split(nd.nodes, sizes, P_)
        assert set(owner[roots].tolist()) == set(range(P_))
        assert np.all((owner >= 0) == ~top)
        for t, (_, kids) in enumerate(nd.nodes):
            for ch in kids:
                if not top[ch] and not top[t]:
                    assert owner[ch] == owner[t]
