"""Pins of reading R7 ("detect when phi_i is not full rank,
and discard columns as necessary") and of the preconditioned-norm stop rule.

R7: column j of part I is kept iff ||v_j|| >= rank_tol * ||F_I e_j||, v_j its
part orthogonal to the kept earlier columns.  Relative to the column itself,
the test is invariant under scaling a coordinate axis (monomial column j is
multiplied by a constant, and so is v_j), so the coarse space -- and with it
M, which depends only on span(F_I) -- does not change when
the coordinates that generate F are rescaled or (while every column stays
numerically independent) shifted.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P


def _monomials_affine(coords, p, scale, shift):
    """Graded-lex monomials of the coordinates mapped to [-1,1]^d, then x -> scale*x + shift."""
    lo, hi = coords.min(axis=0), coords.max(axis=0)
    xh = (2.0 * (coords - lo) / (hi - lo) - 1.0) * scale + shift
    cols = []
    for e in P.monomial_exponents(coords.shape[1], p):
        c = np.ones(coords.shape[0])
        for d, ed in enumerate(e):
            c = c * xh[:, d] ** ed
        cols.append(c)
    return np.asfortranarray(np.stack(cols, axis=1))


def _oracle_with_F(pr, F):
    return oracle.Oracle(pr.n, pr.row_ptr, pr.col, pr.val, F, pr.part, pr.nparts, pr.overlap)


def _coords2d(N):
    return P.grid_coords((N, N), 1.0, 1.0 / (N + 1))


@pytest.mark.parametrize("p,maps", [
    (3, [(1e-3, 0.0), (1e3, 0.0), (2.5, 0.7), (0.5, -0.3)]),
    (10, [(1e-3, 0.0), (1e3, 0.0), (0.8, 0.1)]),
])
def test_M_invariant_under_affine_coordinates(p, maps):
    N = 32
    pr = P.biharmonic2d(N, 16, 1)                   # 4 parts of 256 nodes
    coords = _coords2d(N)
    o = _oracle_with_F(pr, _monomials_affine(coords, p, 1.0, 0.0))
    k = len(P.monomial_exponents(2, p))
    assert o.dropped == 0 and o.nc == pr.nparts * k
    R = np.random.default_rng(1).standard_normal((pr.n, 3))
    Z = np.stack([o.apply_precond(R[:, t]) for t in range(3)], axis=1)
    for s, t in maps:
        os_ = _oracle_with_F(pr, _monomials_affine(coords, p, s, t))
        assert os_.dropped == 0, (s, t)             # same coarse space dimension
        for c in range(3):
            z = os_.apply_precond(R[:, c])
            assert np.linalg.norm(z - Z[:, c]) <= 1e-9 * np.linalg.norm(Z[:, c]), (s, t)


def test_rank_ratio_is_scale_free():
    """min ||v_j|| / ||F_I e_j|| is the same number for any axis scaling."""
    pr = P.poisson2d(32, 8, 3)
    coords = _coords2d(32)
    r1 = _oracle_with_F(pr, _monomials_affine(coords, 3, 1.0, 0.0)).min_rank_ratio()
    r2 = _oracle_with_F(pr, _monomials_affine(coords, 3, 1e-4, 0.0)).min_rank_ratio()
    assert abs(r1 - r2) <= 1e-12 * r1


def test_dependent_columns_are_dropped():
    """An exactly dependent column (a copy, a linear combination) is discarded
    whatever the coordinate scale; the span and M stay those of the independent set."""
    pr = P.poisson2d(24, 8, 1)
    F = np.asfortranarray(pr.F)
    Fd = np.asfortranarray(np.column_stack([F, 3.0 * F[:, 1] - 0.5 * F[:, 2], F[:, 0]]))
    o = _oracle_with_F(pr, F)
    od = _oracle_with_F(pr, Fd)
    assert od.dropped == 2 * pr.nparts and od.nc == o.nc
    r = np.random.default_rng(2).standard_normal(pr.n)
    z, zd = o.apply_precond(r), od.apply_precond(r)
    assert np.linalg.norm(z - zd) <= 1e-12 * np.linalg.norm(z)


# ---------------------------------------------------------------- stop_mode 2 (reading R1 iii)

def test_stop_mode_preconditioned_norm():
    """stop_mode 2 stops at the first k with sqrt(r_k^T M r_k) <= rtol sqrt(r_0^T M r_0)
    (reading R1 (iii)), with M built densely column by column."""
    pr = P.poisson2d(12, 4, 1)
    o = oracle.Oracle.from_problem(pr)
    n = pr.n
    M = np.stack([o.apply_precond(e) for e in np.eye(n)], axis=1)
    A = pr.dense()
    f = pr.f
    rtol = 1e-7
    u, it, hist, conv = o.pcg(f, rtol, stop_mode=oracle.STOP_PREC)
    assert conv and it >= 3

    def pnorm(r):
        return np.sqrt(r @ M @ r)

    ref = pnorm(f)
    r_k = f - A @ u
    assert pnorm(r_k) <= rtol * ref * (1 + 1e-6)
    u1, it1, _, conv1 = o.pcg(f, rtol, max_iter=it - 1, stop_mode=oracle.STOP_PREC)
    assert it1 == it - 1 and not conv1
    assert pnorm(f - A @ u1) > rtol * ref
    # and the rule is not the plain residual rule
    _, it0, _, _ = o.pcg(f, rtol, stop_mode=oracle.STOP_RES0)
    assert hist[it] > 0 and it0 >= 1
