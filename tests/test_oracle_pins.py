"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here is CPU-only (`-m "not gpu"`).  None compares the oracle with
itself: each pins a step to a closed form, a worked example (tests/golden/,
each with its citation), an invariant, or an independent dense numpy
re-derivation on a tiny grid.  A plausible mistake anywhere in oracle.c (a
dropped term, a wrong sign or index, a transposed operand, the coarse step in
the wrong place, a non-reversed post-smoother) fails at least one of them.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P
from tests.helpers import csr_from_dense, dense_two_level, graph_distance_sets, laplace1d

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def make_oracle_dense(A, F, part, nparts, overlap=1, rank_tol=1e-8):
    rp, c, v = csr_from_dense(A)
    return oracle.Oracle(A.shape[0], rp, c, v, np.asfortranarray(F), np.asarray(part, np.int32),
                         nparts, overlap, rank_tol)


# ---------------------------------------------------------------- overlap

def test_overlap_path_golden():
    g = GOLD["overlap_path"]
    A = laplace1d(9)
    part = np.zeros(9, np.int32)
    part[4:] = 1
    o = make_oracle_dense(A, np.ones((9, 1)), part, 2, overlap=g["delta"])
    for i, exp in enumerate(g["expected"]):
        assert o.overlap_set(i).tolist() == exp


@pytest.mark.parametrize("delta", [0, 1, 2, 3])
def test_overlap_is_graph_distance(delta):
    pr = P.biharmonic2d(16, 8, 1)          # 13-point graph: long-range edges
    A = pr.dense()
    o = oracle.Oracle.from_problem(pr, overlap=delta)
    parts = [np.nonzero(pr.part == I)[0] for I in range(pr.nparts)]
    ref = graph_distance_sets(A, parts, delta)
    for i in range(pr.nparts):
        assert o.overlap_set(i).tolist() == ref[i].tolist()
    if delta == 0:
        for i in range(pr.nparts):
            assert o.overlap_set(i).tolist() == parts[i].tolist()


# ---------------------------------------------------------------- colouring (reading R3)

def _conflict(A, si, sj):
    Nj = np.nonzero(A[sj].any(axis=0))[0]           # Omega~_j and its neighbours
    return len(np.intersect1d(si, Nj)) > 0


@pytest.mark.parametrize("mk,ncol", [(lambda: P.poisson2d(32, 8, 1), 4),
                                     (lambda: P.poisson3d(16, 4, 1), 8),
                                     (lambda: P.biharmonic2d(32, 8, 1), 4),
                                     (lambda: P.elasticity3d(12, 4), 8)])
def test_colouring_valid_and_parity_classes(mk, ncol):
    pr = mk()
    A = pr.dense() != 0
    o = oracle.Oracle.from_problem(pr)
    col = o.colours()
    assert o.ncolours == ncol
    sets = [o.overlap_set(i) for i in range(pr.nparts)]
    for i in range(pr.nparts):
        for j in range(pr.nparts):
            if i != j and col[i] == col[j]:
                assert not _conflict(A, sets[i], sets[j])
    # regular block grid: colour = parity class of the block coordinates
    bc = pr.block_coords
    parity = sum((bc[:, d] % 2) << d for d in range(bc.shape[1]))
    assert np.array_equal(col, parity)


# ---------------------------------------------------------------- coarse basis

def test_p0_restriction_golden():
    g = GOLD["p0_restriction"]
    n = sum(g["sizes"])
    A = laplace1d(n)
    part = np.repeat(np.arange(2), g["sizes"]).astype(np.int32)
    o = make_oracle_dense(A, np.ones((n, 1)), part, 2, overlap=0)
    Pm = o.P_dense()
    assert Pm.shape == (n, 2)
    assert np.allclose(Pm[:4, 0], g["values"][0], rtol=0, atol=1e-15)
    assert np.allclose(Pm[4:, 1], g["values"][1], rtol=0, atol=1e-15)
    assert np.all(Pm[4:, 0] == 0) and np.all(Pm[:4, 1] == 0)


def test_basis_orthonormal_local_and_spans_F():
    pr = P.poisson3d(12, 4, 2)
    o = oracle.Oracle.from_problem(pr)
    Pm = o.P_dense()
    assert np.abs(Pm.T @ Pm - np.eye(o.nc)).max() < 1e-14
    cp = o.coarse_offsets()
    for I in range(pr.nparts):
        cols = Pm[:, cp[I]:cp[I + 1]]
        outside = pr.part != I
        assert np.all(cols[outside] == 0)
        FI = pr.F[pr.part == I]
        QI = cols[pr.part == I]
        assert np.abs(FI - QI @ (QI.T @ FI)).max() < 1e-13


def test_rank_deficiency_dropped():
    """duplicate generating vector => one column discarded per part;
    a 2-node part cannot carry 3 independent linears."""
    pr = P.poisson2d(8, 4, 1)
    F2 = np.asfortranarray(np.concatenate([pr.F, pr.F[:, 1:2]], axis=1))
    o = oracle.Oracle(pr.n, pr.row_ptr, pr.col, pr.val, F2, pr.part, pr.nparts, 1)
    assert o.dropped == pr.nparts and o.nc == 3 * pr.nparts
    A = laplace1d(4)
    F = np.stack([np.ones(4), np.arange(4.0), np.arange(4.0) ** 2], axis=1)
    o = make_oracle_dense(A, F, np.array([0, 0, 1, 1]), 2, overlap=0)
    assert o.nc == 4 and o.dropped == 2


def test_zero_block_and_bad_partition_raise():
    A = laplace1d(6)
    F = np.ones((6, 1))
    F[3:] = 0
    with pytest.raises(oracle.OracleError) as e:
        make_oracle_dense(A, F, np.array([0, 0, 0, 1, 1, 1]), 2)
    assert e.value.code == 4
    with pytest.raises(oracle.OracleError) as e:
        make_oracle_dense(A, np.ones((6, 1)), np.array([0, 0, 0, 2, 2, 2]), 3)
    assert e.value.code == 3
    with pytest.raises(oracle.OracleError) as e:
        make_oracle_dense(A, np.ones((6, 1)), np.array([0, 0, 0, 5, 1, 1]), 2)
    assert e.value.code == 3


def _mp_projector_action(FI, x, dps=50):
    """Exact-input, 50-digit orthonormal basis of span(FI) (mpmath MGS, twice),
    applied as a projector to x.  FI's fp64 entries convert to mpf exactly."""
    import mpmath as mp
    mp.mp.dps = dps
    m, k = FI.shape
    Q = []
    for j in range(k):
        v = [mp.mpf(float(t)) for t in FI[:, j]]
        for _ in range(2):
            for q in Q:
                s = mp.fsum(a * b for a, b in zip(q, v))
                v = [a - s * b for a, b in zip(v, q)]
        nrm = mp.sqrt(mp.fsum(a * a for a in v))
        Q.append([a / nrm for a in v])
    xs = [mp.mpf(float(t)) for t in x]
    out = [mp.mpf(0)] * m
    for q in Q:
        s = mp.fsum(a * b for a, b in zip(q, xs))
        out = [o + s * a for o, a in zip(out, q)]
    return np.array([float(t) for t in out])


def test_dd_orthonormalisation_resolves_ill_conditioned_span():
    """Reading R6c: F restricted to a small part of a big grid is ill-conditioned
    (cubic monomials of global coordinates on a 16x16 part of a 2048^2 grid:
    cond ~ 1e8).  The oracle's per-part basis must span the stored F_I to fp64
    rounding: compare its projector with a 50-digit mpmath one.  Plain fp64 QR
    misses this bound by orders of magnitude (checked below), so the pin
    discriminates."""
    N, b = 32, 16
    pr = P.biharmonic2d(N, b, 3)
    coords = np.stack([np.tile(np.arange(N), N), np.repeat(np.arange(N), N)], axis=1).astype(float)
    # global coordinates as if the grid were 2048 wide, mapped to [-1, 1]
    Fg = P.monomials(np.vstack([coords, [[2047.0, 2047.0]]]), 3)[:-1]
    o = oracle.Oracle(pr.n, pr.row_ptr, pr.col, pr.val, np.asfortranarray(Fg), pr.part,
                      pr.nparts, 1)
    assert o.dropped == 0
    assert o.min_rank_ratio() < 1e-5          # the blocks really are ill-conditioned
    Pm = o.P_dense()
    cp = o.coarse_offsets()
    rs = np.random.default_rng(7)
    worst_dd, worst_fp64 = 0.0, 0.0
    for I in (0, 3):
        rows = np.nonzero(pr.part == I)[0]
        Q = Pm[rows, cp[I]:cp[I + 1]]
        x = rs.standard_normal(len(rows))
        ref = _mp_projector_action(Fg[rows], x)
        worst_dd = max(worst_dd, np.abs(Q @ (Q.T @ x) - ref).max())
        Qn, _ = np.linalg.qr(Fg[rows])
        worst_fp64 = max(worst_fp64, np.abs(Qn @ (Qn.T @ x) - ref).max())
    assert worst_dd < 1e-13, worst_dd
    assert worst_fp64 > 1e-11, worst_fp64


# ---------------------------------------------------------------- Galerkin matrix

@pytest.mark.parametrize("mk", [lambda: P.poisson2d(16, 4, 1), lambda: P.poisson3d(8, 4, 2),
                                lambda: P.biharmonic2d(16, 8, 3), lambda: P.elasticity3d(4, 2),
                                lambda: P.lognormal3d(8, 4, 1)])
def test_coarse_matrix_is_PtAP_and_spd(mk):
    pr = mk()
    A = pr.dense()
    o = oracle.Oracle.from_problem(pr)
    Pm = o.P_dense()
    Ac = o.Ac_dense()
    ref = Pm.T @ A @ Pm
    assert np.abs(Ac - ref).max() <= 1e-13 * np.abs(ref).max()
    assert np.linalg.eigvalsh(Ac).min() > 0
    # block sparsity = part adjacency
    cp = o.coarse_offsets()
    for I in range(pr.nparts):
        for J in range(pr.nparts):
            blk = Ac[cp[I]:cp[I + 1], cp[J]:cp[J + 1]]
            adj = (A[np.ix_(pr.part == I, pr.part == J)] != 0).any()
            if not adj:
                assert np.all(blk == 0)


def test_galerkin_tiny_worked_example():
    """R = one row of 1/sqrt(n) (p=0, one part), A = 1D Dirichlet
    Laplacian n=4 -> A_0 = 1^T A 1 / n = 2/4 = 0.5."""
    o = make_oracle_dense(laplace1d(4), np.ones((4, 1)), np.zeros(4), 1, overlap=0)
    assert abs(o.Ac_dense()[0, 0] - 0.5) < 1e-15


# ---------------------------------------------------------------- coarse correction

@pytest.mark.parametrize("mk", [lambda: P.poisson2d(32, 8, 1), lambda: P.poisson3d(12, 4, 2),
                                lambda: P.biharmonic2d(32, 8, 3), lambda: P.elasticity3d(4, 2)])
def test_polynomial_reproduction(mk):
    """The coarse Galerkin solution reproduces every generating vector exactly:
    F_j lies in the coarse space, so P A_c^{-1} P^T (A F_j) = F_j."""
    pr = mk()
    o = oracle.Oracle.from_problem(pr)
    for j in range(pr.k):
        Fj = pr.F[:, j]
        z = o.coarse_correct(o.spmv(Fj))
        assert np.linalg.norm(z - Fj) <= 1e-9 * np.linalg.norm(Fj)


def test_galerkin_identity_and_orthogonal_residual():
    pr = P.poisson2d(16, 4, 2)
    o = oracle.Oracle.from_problem(pr)
    Pm = o.P_dense()
    rs = np.random.default_rng(0)
    e = rs.standard_normal(o.nc)
    w = Pm @ e
    assert np.linalg.norm(o.coarse_correct(o.spmv(w)) - w) <= 1e-11 * np.linalg.norm(w)
    r = rs.standard_normal(pr.n)
    r -= Pm @ (Pm.T @ r)                      # orthogonal to every R_0 row
    assert np.abs(o.coarse_correct(r)).max() < 1e-13


def test_coarse_error_non_increasing_in_p():
    """nested spaces, Galerkin optimal => A-norm error never increases with p."""
    errs = []
    base = P.poisson2d(32, 8, 0)
    A = base.dense()
    x = np.tile(np.arange(1, 33), 32) / 33.0
    y = np.repeat(np.arange(1, 33), 32) / 33.0
    for u in (np.sin(np.pi * x) * np.sin(2 * np.pi * y),):   # smooth solution, f = A u
        f = A @ u
        for p in range(4):
            pr = P.poisson2d(32, 8, p)
            o = oracle.Oracle.from_problem(pr)
            e = o.coarse_correct(f) - u
            errs.append(np.sqrt(e @ A @ e))
    for a, b in zip(errs, errs[1:]):
        assert b <= a * (1 + 1e-10)
    assert errs[-1] < 0.5 * errs[0]


# ---------------------------------------------------------------- preconditioner

@pytest.mark.parametrize("mk", [lambda: P.poisson2d(16, 4, 1), lambda: P.biharmonic2d(16, 8, 3),
                                lambda: P.elasticity3d(4, 2), lambda: P.lognormal3d(8, 4, 1)])
def test_apply_matches_literal_dense_composition(mk):
    """The oracle's M r equals the literal dense composition of the update
    equation PAPER.md:555 (forward order, coarse solve on the current residual,
    reverse order), built independently with numpy solves."""
    pr = mk()
    A = pr.dense()
    o = oracle.Oracle.from_problem(pr)
    col = o.colours()
    order = sorted(range(pr.nparts), key=lambda i: (col[i], i))
    sets = [o.overlap_set(i) for i in range(pr.nparts)]
    Pm = o.P_dense()
    r = np.random.default_rng(1).standard_normal(pr.n)
    ref = dense_two_level(A, r, sets, order, Pm)
    z = o.apply_precond(r)
    assert np.linalg.norm(z - ref) <= 1e-11 * np.linalg.norm(ref)
    # the multiplicative result is invariant to the order within a colour
    rs = np.random.default_rng(2)
    order2 = sorted(range(pr.nparts), key=lambda i: (col[i], rs.random()))
    ref2 = dense_two_level(A, r, sets, order2, Pm)
    assert np.linalg.norm(ref2 - ref) <= 1e-13 * np.linalg.norm(ref)


def test_forward_sweep_matches_update_equation():
    pr = P.poisson2d(16, 4, 1)
    A = pr.dense()
    o = oracle.Oracle.from_problem(pr)
    col = o.colours()
    order = sorted(range(pr.nparts), key=lambda i: (col[i], i))
    r = np.random.default_rng(3).standard_normal(pr.n)
    z = np.zeros(pr.n)
    for i in order:
        idx = o.overlap_set(i)
        z[idx] += np.linalg.solve(A[np.ix_(idx, idx)], (r - A @ z)[idx])
    assert np.linalg.norm(o.forward_sweep(r) - z) <= 1e-12 * np.linalg.norm(z)


@pytest.mark.parametrize("mk", [lambda: P.poisson2d(16, 4, 1), lambda: P.biharmonic2d(16, 8, 3),
                                lambda: P.poisson3d(8, 4, 2)])
def test_preconditioner_symmetric_pd_linear(mk):
    pr = mk()
    o = oracle.Oracle.from_problem(pr)
    M = np.stack([o.apply_precond(e) for e in np.eye(pr.n)], axis=1)
    assert np.abs(M - M.T).max() <= 1e-12 * np.abs(M).max()
    assert np.linalg.eigvalsh(0.5 * (M + M.T)).min() > 0
    rs = np.random.default_rng(4)
    a, b = rs.standard_normal(pr.n), rs.standard_normal(pr.n)
    assert np.linalg.norm(o.apply_precond(2 * a - 3 * b) - (2 * M @ a - 3 * M @ b)) < 1e-10 * np.linalg.norm(M @ a)
    assert np.all(o.apply_precond(np.zeros(pr.n)) == 0)


def test_single_subdomain_is_exact_inverse():
    """one subdomain covering everything => M = A^{-1}; PCG takes 1 iteration."""
    pr = P.poisson2d(12, 12, 1)
    assert pr.nparts == 1
    A = pr.dense()
    o = oracle.Oracle.from_problem(pr)
    r = np.random.default_rng(5).standard_normal(pr.n)
    assert np.linalg.norm(o.apply_precond(r) - np.linalg.solve(A, r)) < 1e-12 * np.linalg.norm(r)
    u, it, hist, conv = o.pcg(pr.f, 1e-10)
    assert conv and it == 1


def test_block_diagonal_exact_after_one_sweep():
    """two uncoupled subdomains (Delta=0) => one forward sweep is exact."""
    A = np.zeros((8, 8))
    A[:4, :4] = laplace1d(4)
    A[4:, 4:] = 2 * laplace1d(4)
    part = np.array([0] * 4 + [1] * 4)
    o = make_oracle_dense(A, np.ones((8, 1)), part, 2, overlap=0)
    r = np.arange(1.0, 9.0)
    assert np.linalg.norm(o.forward_sweep(r) - np.linalg.solve(A, r)) < 1e-13
    assert np.linalg.norm(o.apply_precond(r) - np.linalg.solve(A, r)) < 1e-13


def test_cholesky_golden_and_not_spd():
    g = GOLD["cholesky_2x2"]
    A = np.array(g["A"], float)
    o = make_oracle_dense(A, np.ones((2, 1)), np.zeros(2), 1, overlap=0)
    u, it, hist, conv = o.pcg(np.array(g["b"], float), 1e-12)
    assert np.allclose(u, g["x"], rtol=0, atol=1e-14) and it == 1
    # all-Neumann 1D Laplacian (zero row sums): singular => not positive definite
    An = laplace1d(6)
    An[0, 0] = An[-1, -1] = 1
    with pytest.raises(oracle.OracleError) as e:
        make_oracle_dense(An, np.ones((6, 1)), np.zeros(6), 1, overlap=0)
    assert e.value.code == 5


# ---------------------------------------------------------------- PCG

@pytest.mark.parametrize("mk", [lambda: P.poisson2d(24, 8, 1), lambda: P.biharmonic2d(24, 8, 3),
                                lambda: P.elasticity3d(4, 2)])
def test_pcg_matches_direct_solve(mk):
    pr = mk()
    A = pr.dense()
    o = oracle.Oracle.from_problem(pr)
    u, it, hist, conv = o.pcg(pr.f, 1e-12)
    ref = np.linalg.solve(A, pr.f)
    assert conv
    assert np.linalg.norm(u - ref) <= 1e-9 * np.linalg.norm(ref)
    # history entry j is the residual of the j-th iterate: check the last one directly
    assert abs(hist[0] - np.linalg.norm(pr.f)) <= 1e-14 * hist[0]
    assert hist[-1] <= 1e-12 * hist[0]


def test_pcg_identity_one_iteration():
    A = np.eye(5)
    o = make_oracle_dense(A, np.ones((5, 1)), np.zeros(5), 1, overlap=0)
    f = np.arange(1.0, 6.0)
    u, it, hist, conv = o.pcg(f, 1e-12)
    assert it == 1 and conv and np.allclose(u, f)


def test_pcg_stop_modes_and_zero_rhs():
    pr = P.poisson2d(32, 8, 1)
    o = oracle.Oracle.from_problem(pr)
    _, it0, h0, _ = o.pcg(pr.f, 1e-8, stop_mode=0)
    _, it1, h1, _ = o.pcg(pr.f, 1e-8, stop_mode=1)
    assert h0[it0] <= 1e-8 * h0[0] < h0[it0 - 1]
    assert h1[it1] <= 1e-8 * h1[1] < h1[it1 - 1]
    u, it, hist, conv = o.pcg(np.zeros(pr.n), 1e-8)
    assert it == 0 and conv and np.all(u == 0)
    _, it, _, conv = o.pcg(pr.f, 1e-14, max_iter=2)
    assert it == 2 and not conv


def test_iterations_h_independent():
    """at fixed H/h the two-level iteration count is ~constant in h."""
    its = []
    for N in (32, 64, 128):
        pr = P.poisson2d(N, 8, 1)
        o = oracle.Oracle.from_problem(pr)
        its.append(o.pcg(pr.f, 1e-8)[1])
    assert max(its) - min(its) <= 2, its


def test_iterations_fall_with_p_biharmonic():
    """Paper trend: higher p => fewer iterations on the biharmonic."""
    its = []
    for p in (1, 3):
        pr = P.biharmonic2d(64, 8, p)
        its.append(oracle.Oracle.from_problem(pr).pcg(pr.f, 1e-8)[1])
    assert its[1] < its[0], its


def test_fractional_iterations_golden():
    for key in ("fractional_a", "fractional_b"):
        g = GOLD[key]
        assert abs(oracle.fractional_iterations(g["hist"], g["tol"]) - g["expected"]) < 1e-12


def test_spmv_golden():
    g = GOLD["spmv_tridiag"]
    o = make_oracle_dense(laplace1d(3), np.ones((3, 1)), np.zeros(3), 1)
    assert o.spmv(np.array(g["x"], float)).tolist() == g["y"]


# ---------------------------------------------------------------- Lanczos condition estimate
def test_lanczos_condition_estimate_matches_dense_spectrum():
    """PAPER.md:617-621 (iteration bounds from "condition number estimates
    derived from the Lanczos coefficients computed during CG"): on a tiny
    problem run to tight tolerance, the Ritz values of the CG-Lanczos
    tridiagonal lie in the spectrum of M A, and kappa = lambda_max/lambda_min
    matches a dense eigensolve of M A (M built column by column)."""
    pr = P.poisson2d(12, 4, 1, 31)
    o = oracle.Oracle.from_problem(pr)
    A = pr.dense()
    M = np.column_stack([o.apply_precond(e) for e in np.eye(pr.n)])
    ev = np.sort(np.linalg.eigvals(M @ A).real)
    u, it, hist, conv, al, be = o.pcg_lanczos(pr.f, 1e-13, 200)
    assert conv and len(al) == it and len(be) == it - 1
    T = oracle.lanczos_tridiagonal(al, be)
    ritz = np.linalg.eigvalsh(T)
    assert ritz[0] >= ev[0] * (1 - 1e-9) and ritz[-1] <= ev[-1] * (1 + 1e-9)
    kappa, bound = oracle.condition_estimate(al, be, 1e-13)
    assert abs(kappa - ev[-1] / ev[0]) <= 0.02 * (ev[-1] / ev[0]), (kappa, ev[-1] / ev[0])
    # the classical bound ln(2/tol)/ln((sqrt k + 1)/(sqrt k - 1)) is an upper bound on the count
    assert bound >= it - 1


def test_lanczos_trivial_cases():
    """One subdomain covering everything: M = A^{-1}, one
    iteration, a single coefficient, kappa = 1; alpha = 1 exactly in theory."""
    pr = P.poisson2d(10, 10, 1, 32)
    o = oracle.Oracle.from_problem(pr)
    u, it, hist, conv, al, be = o.pcg_lanczos(pr.f, 1e-10)
    assert it == 1 and conv and len(al) == 1
    assert abs(al[0] - 1.0) <= 1e-10
    assert oracle.condition_estimate(al, be, 1e-10) == (1.0, 1.0)


# ---------------------------------------------------------------- caller's colouring (reading R3)

@pytest.mark.parametrize("mk", [lambda: P.poisson2d(16, 4, 1), lambda: P.biharmonic2d(16, 4, 2)])
@pytest.mark.parametrize("kind", ["natural", "permuted"])
def test_caller_sweep_order_matches_literal_composition(mk, kind):
    """colour[i] = its sweep position: one subdomain per colour is the paper's
    plain sequential sweep "iterating over all subdomains" in
    that order; the oracle's M r equals the literal dense composition."""
    pr = mk()
    A = pr.dense()
    if kind == "natural":
        colour = np.arange(pr.nparts, dtype=np.int32)
    else:
        colour = np.random.default_rng(3).permutation(pr.nparts).astype(np.int32)
    o = oracle.Oracle.from_problem(pr, colour=colour)
    assert o.ncolours == pr.nparts and np.array_equal(o.colours(), colour)
    order = list(np.argsort(colour))
    sets = [o.overlap_set(i) for i in range(pr.nparts)]
    r = np.random.default_rng(1).standard_normal(pr.n)
    ref = dense_two_level(A, r, sets, order, o.P_dense())
    assert np.linalg.norm(o.apply_precond(r) - ref) <= 1e-11 * np.linalg.norm(ref)


def test_caller_colouring_validated():
    pr = P.poisson2d(16, 4, 1)
    greedy = oracle.Oracle.from_problem(pr)
    col = greedy.colours()
    o = oracle.Oracle.from_problem(pr, colour=col)          # the same colouring passed in
    r = np.random.default_rng(2).standard_normal(pr.n)
    assert np.array_equal(o.apply_precond(r), greedy.apply_precond(r))
    bad = col.copy()
    bad[1] = bad[0]                                          # parts 0 and 1 are neighbours
    with pytest.raises(oracle.OracleError) as e:
        oracle.Oracle.from_problem(pr, colour=bad)
    assert e.value.code == 6
    with pytest.raises(oracle.OracleError):
        oracle.Oracle.from_problem(pr, colour=np.full(pr.nparts, -1, np.int32))
