"""Pins of the oracle's nested-dissection coarse solve (oracle/coarse_nd.py) and
of its floor mode (oracle.h or_opts.perturb).

The nested-dissection multifrontal Cholesky is what lets the oracle reach
C3's 1,048,576-unknown A_0; it is pinned here, on grids
where both run, against a dense numpy solve of A_0 (an independent route to
the definition y = A_0^{-1} b) and against oracle.c's envelope Cholesky.  The
floor mode must still be the same method: it is pinned
against the literal dense composition, exactly like the plain oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P
from oracle.coarse_nd import NDCholesky
from tests.helpers import dense_two_level

FAMILIES = [
    ("poisson3d_16_b4_p1", lambda: P.poisson3d(16, 4, 1)),      # 64 parts, 7-point
    ("poisson3d_12_b2_p2", lambda: P.poisson3d(12, 2, 2)),      # 216 parts, k = 10
    ("lognormal3d_16_b4", lambda: P.lognormal3d(16, 4, 1)),
    ("biharmonic2d_64_b8_p3", lambda: P.biharmonic2d(64, 8, 3)),  # corner-coupled parts
    ("elasticity3d_8_b2", lambda: P.elasticity3d(8, 2)),       # 27-point node graph
]


@pytest.mark.parametrize("name,mk", FAMILIES, ids=[f[0] for f in FAMILIES])
@pytest.mark.parametrize("leaf", [8, 64])
def test_nd_solve_equals_dense_solve(name, mk, leaf):
    pr = mk()
    o = oracle.Oracle.from_problem(pr)
    A0 = o.Ac_sparse()
    assert np.array_equal(A0.toarray(), o.Ac_dense())
    nd = NDCholesky(A0, o.coarse_offsets(), pr.block_coords, leaf=leaf)
    assert len(nd.nodes) > 1                      # a real dissection, not one dense front
    rng = np.random.default_rng(7)
    for _ in range(2):
        b = rng.standard_normal(o.nc)
        y = nd.solve(b.copy())
        yd = np.linalg.solve(o.Ac_dense(), b)
        assert np.linalg.norm(y - yd) <= 1e-11 * np.linalg.norm(yd)
    # every unknown is eliminated exactly once
    assert np.array_equal(np.sort(nd.order), np.arange(o.nc))


@pytest.mark.parametrize("name,mk", FAMILIES, ids=[f[0] for f in FAMILIES])
def test_nd_coarse_pcg_matches_envelope(name, mk):
    pr = mk()
    o = oracle.Oracle.from_problem(pr)
    on = oracle.Oracle.from_problem(pr, coarse="nd", nd_leaf=16)
    r = np.random.default_rng(3).standard_normal(pr.n)
    zc, zn = o.coarse_correct(r), on.coarse_correct(r)
    assert np.linalg.norm(zc - zn) <= 1e-11 * np.linalg.norm(zc)
    u, it, h, conv = o.pcg(pr.f, 1e-8)
    un, itn, hn, convn = on.pcg(pr.f, 1e-8)
    assert conv and convn and it == itn
    assert np.linalg.norm(u - un) <= 1e-10 * np.linalg.norm(u)
    assert np.max(np.abs(h - hn) / h) <= 1e-8


def test_nd_polynomial_reproduction():
    """P A_0^{-1} P^T (A F_j) = F_j for every generating vector (PAPER.md:266-267,
    369-374) through the nested-dissection solve."""
    pr = P.poisson3d(16, 4, 2)
    on = oracle.Oracle.from_problem(pr, coarse="nd", nd_leaf=20)
    A = pr.scipy()
    for j in range(pr.k):
        Fj = pr.F[:, j]
        z = on.coarse_correct(A @ Fj)
        assert np.linalg.norm(z - Fj) <= 1e-10 * np.linalg.norm(Fj)


def test_nd_refuses_a_non_dissection():
    """Block coordinates that do not follow the coupling give no valid elimination tree."""
    pr = P.poisson3d(16, 4, 1)
    o = oracle.Oracle.from_problem(pr)
    bad = pr.block_coords[np.random.default_rng(0).permutation(pr.nparts)]
    with pytest.raises(ValueError):
        NDCholesky(o.Ac_sparse(), o.coarse_offsets(), bad, leaf=8)


def test_nd_not_spd_is_an_error():
    pr = P.poisson3d(8, 4, 1)
    o = oracle.Oracle.from_problem(pr)
    A0 = o.Ac_sparse().tolil()
    A0[3, 3] = -1.0
    with pytest.raises(np.linalg.LinAlgError):
        NDCholesky(A0.tocsr(), o.coarse_offsets(), pr.block_coords, leaf=4)


# ---------------------------------------------------------------- floor mode

FLOOR = [
    ("poisson2d_32_b8_p1", lambda: P.poisson2d(32, 8, 1)),
    ("biharmonic2d_32_b8_p3", lambda: P.biharmonic2d(32, 8, 3)),
    ("elasticity3d_4_b2", lambda: P.elasticity3d(4, 2)),
]


@pytest.mark.parametrize("name,mk", FLOOR, ids=[f[0] for f in FLOOR])
@pytest.mark.parametrize("coarse", ["envelope", "nd"])
def test_floor_mode_is_the_same_method(name, mk, coarse):
    """The perturbed oracle (reversed dot order, reversed local and coarse
    elimination) still applies PAPER.md:555 + 560-564 exactly."""
    pr = mk()
    op = oracle.Oracle.from_problem(pr, perturb=True, coarse=coarse, nd_leaf=16)
    A = pr.dense()
    sets = [op.overlap_set(i) for i in range(pr.nparts)]
    col = op.colours()
    order = sorted(range(pr.nparts), key=lambda i: (col[i], i))
    Pm = op.P_dense()
    r = np.random.default_rng(11).standard_normal(pr.n)
    z = op.apply_precond(r)
    zd = dense_two_level(A, r, sets, order, Pm)
    assert np.linalg.norm(z - zd) <= 1e-9 * np.linalg.norm(zd)


@pytest.mark.parametrize("name,mk", FLOOR, ids=[f[0] for f in FLOOR])
def test_floor_mode_changes_only_rounding(name, mk):
    pr = mk()
    o = oracle.Oracle.from_problem(pr)
    op = oracle.Oracle.from_problem(pr, perturb=True)
    r = np.random.default_rng(5).standard_normal(pr.n)
    z, zp = o.apply_precond(r), op.apply_precond(r)
    d = np.linalg.norm(z - zp) / np.linalg.norm(z)
    assert 0 < d <= 1e-10                      # a different rounding, the same operator
    u, it, h, _ = o.pcg(pr.f, 1e-8)
    up, itp, hp, _ = op.pcg(pr.f, 1e-8)
    assert it == itp
    assert np.linalg.norm(u - up) <= 1e-9 * np.linalg.norm(u)
