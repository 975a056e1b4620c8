"""The multi-rank CUDA path on one GPU: P virtual ranks through the loopback
communicator (include/ddg.h ddg_loop_group_create), against the oracle.

Every rank is a full libddg context driven by its own host thread: it owns the
rows and subdomains of its box of parts, applies only its own
subdomains, and exchanges z halos after every colour, p/r halos per
iteration, the coarse right-hand side and the CG scalars -- the same code as
over NCCL, with the data movement done by device copies and a fixed-order
sum kernel on the group's stream (no kernel waits on another, so this is safe
on one GPU).  u is assembled on every rank.

Bar (BASELINE.json north_star): u within 1e-10 relative, iterations +-1,
history within 1e-8 relative, against the oracle; M r of the sharded path
equals the single-context M r (the paper's method does not depend on how the
subdomains are spread over processors).
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P

pytestmark = pytest.mark.gpu

U_TOL, H_TOL = 1e-10, 1e-8


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_00907_b200 import build
    build.build()


def run_ranks(P_, fn):
    """fn(rank, comm) on P_ threads; returns the per-rank results (re-raises)."""
    from paper_1504_00907_b200.ddg import LoopGroup
    g = LoopGroup(P_)
    out, err = [None] * P_, []

    def body(r):
        try:
            out[r] = fn(r, g.comm(r))
        except BaseException as e:          # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(P_)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    g.close()
    if err:
        raise err[0]
    return out


CASES = {
    "lognormal_32_b4": lambda: P.lognormal3d(32, 4, 1, 1003),      # C3 recipe, 512 parts
    "biharm_128_b16_p3": lambda: P.biharmonic2d(128, 16, 3, 1005),  # C5 recipe, 64 parts
    "poisson3d_32_b8_p2": lambda: P.poisson3d(32, 8, 2, 1002),     # C2 recipe, multi-item operators
    "elasticity_16_be8": lambda: P.elasticity3d(16, 8, 1004),      # C4 recipe, CSR rows
}


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("name", list(CASES))
def test_loopback_pcg_matches_oracle(name, nranks):
    from paper_1504_00907_b200 import Solver
    pr = CASES[name]()
    if nranks > pr.nparts:
        pytest.skip("fewer parts than ranks")
    o = oracle.Oracle.from_problem(pr)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)
    r = np.random.default_rng(4).standard_normal(pr.n)
    s1 = Solver.from_problem(pr)
    z1 = s1.apply_precond(r)
    s1.close()

    def rank(rk, comm):
        s = Solver.from_problem(pr, comm=comm)
        z = s.apply_precond(r)
        u, it, hist, rep = s.solve(pr.f, 1e-8)
        s.close()
        return z, u, it, hist, bool(rep.converged)

    res = run_ranks(nranks, rank)
    for z, u, it, hist, cv in res:
        assert cv and conv
        assert abs(it - ito) <= 1, (it, ito)
        m = min(len(hist), len(histo))
        assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
        assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
        assert np.linalg.norm(z - z1) <= 1e-13 * np.linalg.norm(z1)
    # every rank holds the same assembled u and the same history
    for z, u, it, hist, _ in res[1:]:
        assert np.array_equal(u, res[0][1]) and np.array_equal(hist, res[0][3])


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("name,factor", [("lognormal_32_b4", 2), ("biharm_128_b16_p3", 2)])
def test_loopback_three_level(name, factor, nranks):
    """The distributed second level (three levels): its parts
    spread over the same virtual ranks, its own halos, y_c assembled by one
    allreduce."""
    from paper_1504_00907_b200 import Solver
    pr = CASES[name]()
    p2, n2, bc2 = P.coarse_parts(pr, factor, coords=True)
    o = oracle.Oracle.from_problem(pr, part2=p2, nparts2=n2)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)

    def rank(rk, comm):
        s = Solver.from_problem(pr, comm=comm, part2=p2, nparts2=n2, block_coords2=bc2)
        u, it, hist, rep = s.solve(pr.f, 1e-8)
        s.close()
        return u, it, hist

    for u, it, hist in run_ranks(nranks, rank):
        assert abs(it - ito) <= 1
        m = min(len(hist), len(histo))
        assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
        assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)


def test_loopback_rejects_mismatched_collectives():
    """A rank that calls a different collective than its peers is an error,
    not a hang (DDG_E_NCCL from the rendezvous)."""
    from paper_1504_00907_b200 import Solver, DDGError
    pr = P.poisson2d(32, 8, 1, 1001)

    def rank(rk, comm):
        s = Solver.from_problem(pr, comm=comm)
        try:
            if rk == 0:
                s.solve(pr.f, 1e-8)          # allreduce first
            else:
                s.apply_precond(pr.f)        # z halo exchange first
            return None
        except DDGError as e:
            return e.code
        finally:
            s.close()

    codes = run_ranks(2, rank)
    assert 9 in codes


@pytest.mark.parametrize("nranks", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("name", ["lognormal_32_b4", "biharm_128_b16_p3", "poisson3d_32_b8_p2"])
def test_loopback_distributed_coarse_solve(name, nranks, monkeypatch):
    """the sparse coarse solve distributed over the ranks --
    the nested-dissection tree cut at depth ceil(log2 P), the top fronts solved
    by every rank, each subtree below by one rank (forward, an allreduce of
    the subtree roots' contributions, the top fronts, backward), y_c assembled
    by one allreduce.  Against the oracle (north-star bar), bitwise equal to
    the replicated solve (DDG_COARSE_REPLICATED=1: every rank the whole tree),
    and each rank reads fewer coarse bytes per solve.  The top fronts' items are
    split over the ranks too (their partial segments allreduced, the reductions
    run by every rank)."""
    from paper_1504_00907_b200 import Solver
    monkeypatch.setenv("DDG_ND_LEAF", "64")       # a deep tree on a test-sized A_c
    pr = CASES[name]()
    o = oracle.Oracle.from_problem(pr)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)
    r = np.random.default_rng(6).standard_normal(pr.n)

    def rank(rk, comm):
        s = Solver.from_problem(pr, comm=comm, coarse_variant=2)
        zc = s.coarse_correct(r)
        u, it, hist, rep = s.solve(pr.f, 1e-8)
        nb = (s.info.coarse_solve_bytes, s.info.coarse_factor_bytes)
        s.close()
        return zc, u, it, hist, nb

    res = run_ranks(nranks, rank)
    monkeypatch.setenv("DDG_COARSE_REPLICATED", "1")
    rep_ = run_ranks(nranks, rank)
    s1 = Solver.from_problem(pr, coarse_variant=2)
    full = (s1.info.coarse_solve_bytes, s1.info.coarse_factor_bytes)
    zc1 = s1.coarse_correct(r)
    s1.close()
    for (zc, u, it, hist, nb), (zr, ur, itr, histr, nbr) in zip(res, rep_):
        assert abs(it - ito) <= 1, (it, ito)
        m = min(len(hist), len(histo))
        assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
        assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
        assert np.array_equal(zc, zr) and np.array_equal(u, ur) and np.array_equal(hist, histr)
        assert np.linalg.norm(zc - zc1) <= 1e-13 * np.linalg.norm(zc1)
        assert nbr == full
        assert nb[0] < full[0] and nb[1] < full[1]      # reads and stores a share of the factor
    assert sum(r[4][1] for r in res) == full[1]          # the shares partition it: each operator on one rank


@pytest.mark.parametrize("nranks", [2, 4])
def test_loopback_three_level_with_distributed_sparse_coarse(nranks, monkeypatch):
    """three levels over the ranks with the second level's own coarse problem
    solved by the distributed sparse solve (coarse_variant 2 on A_1)"""
    from paper_1504_00907_b200 import Solver
    monkeypatch.setenv("DDG_ND_LEAF", "32")
    pr = CASES["lognormal_32_b4"]()
    p2, n2, bc2 = P.coarse_parts(pr, 2, coords=True)
    o = oracle.Oracle.from_problem(pr, part2=p2, nparts2=n2)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)

    def rank(rk, comm):
        s = Solver.from_problem(pr, comm=comm, part2=p2, nparts2=n2, block_coords2=bc2, coarse_variant=2)
        u, it, hist, rep = s.solve(pr.f, 1e-8)
        s.close()
        return u, it, hist

    res = run_ranks(nranks, rank)
    for u, it, hist in res:
        assert abs(it - ito) <= 1
        m = min(len(hist), len(histo))
        assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
        assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
    for u, it, hist in res[1:]:
        assert np.array_equal(u, res[0][0])
