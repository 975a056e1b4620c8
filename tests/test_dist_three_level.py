"""The distributed three-level method, re-enacted on the CPU at world size 2 and 3 (gloo).

With three levels and a communicator, libddg distributes the second level (the
two-level method on A_c) over the same ranks with its own
decomposition plan (setup.cpp build_child with opts.comm; coarse_add assembles
y_c with one allreduce).  This test drives a numpy re-enactment of exactly that
schedule from the library's host-only plans -- the fine plan on A and the
second-level plan on A_c's structural pattern (reading R19) with the
second-level block coordinates -- and every value a rank does not own moves
only through the plans' exchanges.  The result must equal the oracle's
single-process three-level PCG.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P
from tests.test_dist_plan import _free_port

CASES = {
    "poisson2d": (lambda: P.poisson2d(32, 4, 1, 41), 2),
    "poisson3d": (lambda: P.poisson3d(16, 4, 1, 43), 2),
}


def _second_level(pr, o3, p2):
    """A_c (dense and CSR with the part-adjacency pattern), the coarse unknowns'
    second-level parts, from the oracle's P (pinned in test_oracle_three_level)."""
    Pm = o3.P_dense()
    A0 = Pm.T @ pr.dense() @ Pm
    cptr = o3.coarse_offsets()
    owner = np.repeat(np.arange(pr.nparts), np.diff(cptr))
    adj = np.zeros((pr.nparts, pr.nparts), bool)
    rows = np.repeat(np.arange(pr.n), np.diff(pr.row_ptr))
    adj[pr.part[rows], pr.part[pr.col]] = True
    S = adj[owner][:, owner]
    rp = np.zeros(len(owner) + 1, np.int64)
    rp[1:] = np.cumsum(S.sum(1))
    col = np.nonzero(S)[1].astype(np.int32)
    return Pm, A0, rp, col, p2[owner].astype(np.int32)


def _worker(rank, world, port, case, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1504_00907_b200 import ddg

    mk, f2 = CASES[case]
    pr = mk()
    p2, n2, bc2 = P.coarse_parts(pr, f2, coords=True)
    o3 = oracle.Oracle.from_problem(pr, part2=p2, nparts2=n2)
    ch = o3.child()
    Pm, A0, rp0, col0, part0 = _second_level(pr, o3, p2)
    nc = A0.shape[0]
    A = pr.dense()
    Asp = pr.scipy().tocsr()
    plan = ddg.Plan(pr, rank=rank, nranks=world)
    plan2 = ddg.Plan(nc, rp0, col0, part0, n2, pr.overlap, block_coords=bc2, rank=rank, nranks=world)
    peers = [q for q in range(world) if q != rank]

    def halo(pl, v, kind, c=0):
        reqs, bufs = [], {}
        for q in peers:
            s_idx = pl.query(kind + "_SEND", colour=c, peer=q)
            r_idx = pl.query(kind + "_RECV", colour=c, peer=q)
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

    class Level:
        """One two-level method on matrix M with a plan; its coarse step is the
        exact solve (second level) or the second level's V-cycle (first)."""

        def __init__(self, M, pl, part, nparts, Pc, coarse):
            self.M, self.pl, self.part, self.Pc, self.coarse = M, pl, part, Pc, coarse
            self.subs = pl.query("OWNED_SUBS")
            self.prolong = pl.query("PROLONG_PARTS")
            self.sets = {i: pl.query("OVERLAP", peer=int(i)) for i in self.subs}
            self.inv = {i: np.linalg.inv(M[np.ix_(s, s)]) for i, s in self.sets.items()}
            cols = np.argmax(np.abs(Pc) > 0, axis=0)        # each coarse column lives in one part
            self.cpart = part[cols]

        def sweep(self, cs, r, z):
            for c in cs:
                for i in self.subs:
                    if self.pl.colours[i] != c:
                        continue
                    idx = self.sets[i]
                    z[idx] += self.inv[i] @ (r[idx] - self.M[idx] @ z)
                halo(self.pl, z, "Z", c)

        def apply(self, r):
            z = np.zeros(len(r))
            nc_ = self.pl.ncolours
            self.sweep(range(nc_), r, z)
            bc = np.zeros(self.Pc.shape[1])
            for I in self.subs:                             # restriction on owned parts
                rows = np.nonzero(self.part == I)[0]
                cc = np.nonzero(self.cpart == I)[0]
                bc[cc] = self.Pc[np.ix_(rows, cc)].T @ (r[rows] - self.M[rows] @ z)
            y = self.coarse(allsum(bc))
            for I in self.prolong:
                rows = np.nonzero(self.part == I)[0]
                cc = np.nonzero(self.cpart == I)[0]
                z[rows] += self.Pc[np.ix_(rows, cc)] @ y[cc]
            self.sweep(range(nc_ - 1, -1, -1), r, z)
            return z

    P2 = ch.P_dense()
    A1 = P2.T @ A0 @ P2
    second = Level(A0, plan2, part0, n2, P2, lambda b: np.linalg.solve(A1, b))
    owned2 = plan2.query("OWNED_ROWS")

    def vcycle(b):                                          # y_c assembled from owned rows
        y = second.apply(b)
        full = np.zeros(nc)
        full[owned2] = y[owned2]
        return allsum(full)

    first = Level(A, plan, pr.part, pr.nparts, Pm, vcycle)
    owned = plan.query("OWNED_ROWS")
    n = pr.n
    f = pr.f
    r = f.copy()
    u = np.zeros(n)
    p = np.full(n, np.nan)
    res0 = np.sqrt(allsum(np.sum(f[owned] ** 2)))
    hist = [res0]
    z = first.apply(r)
    rho = allsum(np.dot(r[owned], z[owned]))
    p[owned] = z[owned]
    halo(plan, p, "P")
    it = 0
    for it in range(1, 200):
        q = np.full(n, np.nan)
        q[owned] = Asp[owned] @ p                           # stored entries only: p is NaN off the halo
        sigma = allsum(np.dot(p[owned], q[owned]))
        alpha = rho / sigma
        u[owned] += alpha * p[owned]
        r[owned] -= alpha * q[owned]
        res = np.sqrt(allsum(np.sum(r[owned] ** 2)))
        hist.append(res)
        if res <= 1e-8 * res0:
            break
        halo(plan, r, "R")
        z = first.apply(r)
        rho1 = allsum(np.dot(r[owned], z[owned]))
        beta = rho1 / rho
        rho = rho1
        p[owned] = z[owned] + beta * p[owned]
        halo(plan, p, "P")
    ufull = np.zeros(n)
    ufull[owned] = u[owned]
    ufull = allsum(ufull)
    if rank == 0:
        np.savez(os.path.join(out_dir, "dist3.npz"), u=ufull, hist=np.array(hist), it=it,
                 ranks2=plan2.query("PART_RANK"))
    dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("poisson2d", 2), ("poisson2d", 3), ("poisson3d", 2)])
def test_distributed_three_level_equals_oracle(case, world, tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    d = np.load(os.path.join(tmp_path, "dist3.npz"))
    mk, f2 = CASES[case]
    pr = mk()
    p2, n2 = P.coarse_parts(pr, f2)
    o3 = oracle.Oracle.from_problem(pr, part2=p2, nparts2=n2)
    uo, ito, histo, conv = o3.pcg(pr.f, 1e-8)
    assert conv and int(d["it"]) == ito
    m = min(len(histo), len(d["hist"]))
    assert np.max(np.abs(d["hist"][:m] - histo[:m]) / histo[:m]) <= 1e-8
    assert np.linalg.norm(d["u"] - uo) <= 1e-10 * np.linalg.norm(uo)
    assert set(d["ranks2"].tolist()) == set(range(world))   # the second level is shared too
