"""Pins of the oracle's three-level method (oracle.c or_setup3).

The three-level preconditioner is the two-level one with A_0^{-1} replaced by
one application M_2 of the two-level method built on A_0, with coarsened
generating vectors F_0 = R_0 F and a second-level partition of the parts.
Each test pins it to something other than itself:

- exact recursion: one second-level part makes M_2 = A_0^{-1} (the forward
  sweep solves exactly), so M_3 = M_2level to rounding;
- "the coarsened coarse problem is equivalent to directly coarsening the
  original problem with larger subdomains": the second
  level's Galerkin correction, lifted by P, equals the two-level coarse
  correction of a separately built method whose parts are the unions;
- Loewner order: with B = P M_2 P^T <= P A_0^{-1} P^T (M_2 A_0 has spectrum
  in (0, 1]), M_3 <= M_2level and both are SPD;
- the spectrum of M_3 A lies in (0, 1] (each factor of I - M A is an
  A-norm contraction);
- the second level's matrix is dense P^T A P and its overlap is the graph
  distance in the structural pattern of A_0 (reading R19).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P
from tests.helpers import graph_distance_sets


def _three(pr, factor=2, overlap=None, allow_single=False):
    p2, n2 = P.coarse_parts(pr, factor, allow_single=allow_single)
    return oracle.Oracle.from_problem(pr, overlap=overlap, part2=p2, nparts2=n2), p2, n2


def _dense_op(apply, n):
    M = np.empty((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        M[:, j] = apply(e)
    return M


def test_levels_reported_and_child_sizes():
    pr = P.poisson2d(32, 4, 1)
    o3, p2, n2 = _three(pr)
    assert o3.levels == 3 and n2 == 16
    ch = o3.child()
    assert ch.levels == 2 and ch.n == o3.nc and ch.nparts == n2
    assert o3.nc2 == ch.nc
    # rank at level 2 <= k * nparts2
    assert ch.nc <= pr.k * n2
    o2 = oracle.Oracle.from_problem(pr)
    assert o2.levels == 2 and o2.child() is None


def test_single_second_level_part_is_exact_recursion():
    pr = P.poisson2d(24, 4, 1)
    o3, _, n2 = _three(pr, factor=64, allow_single=True)
    assert n2 == 1
    o2 = oracle.Oracle.from_problem(pr)
    rng = np.random.default_rng(5)
    for _ in range(3):
        r = rng.standard_normal(pr.n)
        z2, z3 = o2.apply_precond(r), o3.apply_precond(r)
        assert np.linalg.norm(z3 - z2) <= 1e-12 * np.linalg.norm(z2)


@pytest.mark.parametrize("mk,factor", [(lambda: P.poisson2d(32, 4, 1), 2),
                                       (lambda: P.poisson3d(12, 3, 1), 2),
                                       (lambda: P.biharmonic2d(32, 4, 2), 2)])
def test_second_level_equals_direct_coarsening(mk, factor):
    pr = mk()
    o3, p2, n2 = _three(pr, factor)
    assert o3.dropped == 0
    ch = o3.child()
    assert ch.dropped == 0
    Pm = o3.P_dense()                           # n x n_c
    merged = p2[pr.part].astype(np.int32)       # fine node -> union part
    od = oracle.Oracle(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, merged, n2, pr.overlap)
    rng = np.random.default_rng(11)
    for _ in range(3):
        r = rng.standard_normal(pr.n)
        lifted = Pm @ ch.coarse_correct(Pm.T @ r)
        direct = od.coarse_correct(r)
        assert np.linalg.norm(lifted - direct) <= 1e-9 * np.linalg.norm(direct)


def test_second_level_matrix_and_overlap():
    pr = P.poisson2d(32, 4, 1)
    for delta in (0, 1, 2):
        o3, p2, n2 = _three(pr, overlap=delta)
        ch = o3.child()
        A = pr.dense()
        Pm = o3.P_dense()
        A0 = Pm.T @ A @ Pm
        rng = np.random.default_rng(3)
        x = rng.standard_normal(o3.nc)
        assert np.allclose(ch.spmv(x), A0 @ x, rtol=0, atol=1e-12 * np.abs(A0).sum(1).max() * np.abs(x).max())
        # structural pattern of A_0: parts I, J adjacent in the graph of A (R19)
        cptr = o3.coarse_offsets()
        adj = np.zeros((pr.nparts, pr.nparts), bool)
        rows = np.repeat(np.arange(pr.n), np.diff(pr.row_ptr))
        adj[pr.part[rows], pr.part[pr.col]] = True
        owner = np.repeat(np.arange(pr.nparts), np.diff(cptr))
        S = adj[owner][:, owner].astype(float)
        parts2 = [np.nonzero(p2[owner] == J)[0] for J in range(n2)]
        ref = graph_distance_sets(S, parts2, delta)
        for J in range(n2):
            assert ch.overlap_set(J).tolist() == ref[J].tolist()


def test_three_level_spd_below_two_level_and_contracting():
    pr = P.poisson2d(16, 4, 1)
    o3, _, _ = _three(pr)
    o2 = oracle.Oracle.from_problem(pr)
    n = pr.n
    M3 = _dense_op(o3.apply_precond, n)
    M2 = _dense_op(o2.apply_precond, n)
    sc = np.abs(M2).max()
    assert np.abs(M3 - M3.T).max() <= 1e-12 * sc
    w3 = np.linalg.eigvalsh(0.5 * (M3 + M3.T))
    assert w3.min() > 0
    # M_3 <= M_2 (Loewner): B_3 - B_2 = P (M_2 - A_0^{-1}) P^T <= 0
    wd = np.linalg.eigvalsh(0.5 * ((M2 - M3) + (M2 - M3).T))
    assert wd.min() >= -1e-12 * sc
    assert wd.max() > 1e-6 * sc                 # and the inexact level is visible
    A = pr.dense()
    lam = np.sort(np.linalg.eigvals(M3 @ A).real)
    assert lam[0] > 0 and lam[-1] <= 1 + 1e-10
    lam2 = np.sort(np.linalg.eigvals(M2 @ A).real)
    assert lam[0] <= lam2[0] * (1 + 1e-10)


def test_three_level_pcg_converges_with_moderate_inflation():
    """SPEC.md:567 sanity: builds, converges, and at most 3x the two-level
    iterations at the same p (Table 3 three-level columns)."""
    pr = P.poisson2d(64, 8, 1)
    o3, _, n2 = _three(pr, factor=2)
    assert n2 == 16
    o2 = oracle.Oracle.from_problem(pr)
    u3, it3, h3, c3 = o3.pcg(pr.f, 1e-8)
    u2, it2, h2, c2 = o2.pcg(pr.f, 1e-8)
    assert c3 and c2
    assert it2 <= it3 <= 3 * it2
    A = pr.scipy()
    assert np.linalg.norm(A @ u3 - pr.f) <= 1e-7 * np.linalg.norm(pr.f)


def test_too_small_rejected():
    pr = P.poisson2d(16, 8, 1)                  # 2x2 parts grouped 8 per axis: 1 group
    with pytest.raises(ValueError, match="too small"):
        P.coarse_parts(pr, 8)
    with pytest.raises(oracle.OracleError):
        oracle.Oracle.from_problem(pr, part2=np.zeros(pr.nparts, np.int32), nparts2=2)  # empty part
