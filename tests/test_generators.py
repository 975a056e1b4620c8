"""Input-recipe checks (ddg_gen): stencils, assembly, RNG, F, partitions."""
from __future__ import annotations

import numpy as np
import pytest

from ddg_gen import problems as P
from ddg_gen import rng


def test_rng_deterministic_range_and_moments():
    a = rng.uniform_pm1(1001, 100000)
    b = rng.uniform_pm1(1001, 100000)
    assert np.array_equal(a, b)
    assert a.min() >= -1 and a.max() < 1
    assert abs(a.mean()) < 0.01 and abs(a.var() - 1 / 3) < 0.01
    assert not np.array_equal(a, rng.uniform_pm1(1002, 100000))
    g = rng.normal(7, 200000)
    assert abs(g.mean()) < 0.01 and abs(g.std() - 1) < 0.01
    # SplitMix64 reference value (Steele et al.; first output for state 0 -> 0xE220A8397B1DCDAF)
    assert int(rng.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_poisson_rows():
    pr = P.poisson2d(8, 4, 1)
    A = pr.dense()
    assert np.all(np.diag(A) == 4)
    i = 3 + 8 * 3                                # interior row: 4 - 4 neighbours = 0 row sum
    assert A[i].sum() == 0 and (A[i] != 0).sum() == 5
    pr = P.poisson3d(6, 3, 1)
    A = pr.dense()
    i = 2 + 6 * (2 + 6 * 2)
    assert A[i, i] == 6 and A[i].sum() == 0 and (A[i] != 0).sum() == 7
    assert (A[0] != 0).sum() == 4                # corner: 3 neighbours eliminated


def test_biharmonic_13pt_rows():
    """interior row sum 0; A x^4 = 24 (h = 1) deep inside; diag 20 (c13)."""
    N = 16
    pr = P.biharmonic2d(N, 8, 1)
    A = pr.dense()
    assert np.all(np.diag(A) == 20)
    xi = np.tile(np.arange(N, dtype=float), N)
    i = 8 + N * 8
    assert A[i].sum() == 0 and (A[i] != 0).sum() == 13
    assert abs((A @ xi ** 4)[i] - 24.0) < 1e-9
    assert abs((A @ (xi ** 2))[i]) < 1e-12      # quadratics annihilated by Delta^2


def test_lognormal_harmonic_faces():
    pr = P.lognormal3d(6, 3, 1)
    A = pr.dense()
    assert np.abs(A - A.T).max() == 0
    # interior row: diagonal equals minus the off-diagonal sum (no boundary face)
    i = 2 + 6 * (2 + 6 * 2)
    assert abs(A[i].sum()) < 1e-12 * A[i, i]
    # boundary row: diagonal exceeds the off-diagonal sum by the boundary T = k_a
    assert A[0].sum() > 0
    assert np.linalg.eigvalsh(A).min() > 0


def test_q1_element_rigid_modes_and_spd_after_clamp():
    Ke, lam, mu = P.q1_element_stiffness(0.5, 1.0, 0.3)
    assert np.abs(Ke - Ke.T).max() < 1e-14
    ev = np.linalg.eigvalsh(Ke)
    assert (np.abs(ev) < 1e-12).sum() == 6       # 6 rigid-body modes per element
    assert abs(lam - 0.5769230769230769) < 1e-15 and abs(mu - 0.38461538461538464) < 1e-15
    pr = P.elasticity3d(4, 2, clamp=False)
    A = pr.dense()
    nn = 5
    idx = np.indices((nn, nn, nn))
    x, y, z = [a.ravel(order="F") * 0.25 for a in idx]
    modes = []
    for c in range(3):
        v = np.zeros(pr.n); v[c::3] = 1; modes.append(v)
    for (a, b, ca, cb) in ((x, y, 1, 0), (y, z, 2, 1), (z, x, 0, 2)):
        v = np.zeros(pr.n); v[ca::3] = a; v[cb::3] = -b; modes.append(v)
    for v in modes:
        assert np.abs(A @ v).max() < 1e-13
    pr = P.elasticity3d(4, 2)
    assert pr.n == 5 * 5 * 4 * 3
    assert np.linalg.eigvalsh(pr.dense()).min() > 0
    # DoFs interleaved node-major; partition per node
    assert np.all(pr.part[0::3] == pr.part[1::3]) and np.all(pr.part[1::3] == pr.part[2::3])


def test_monomials_graded_lex_and_partition():
    assert P.monomial_exponents(2, 3) == [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2),
                                          (3, 0), (2, 1), (1, 2), (0, 3)]
    assert len(P.monomial_exponents(3, 2)) == 10
    pr = P.poisson2d(16, 4, 1)
    assert pr.F.shape == (256, 3) and pr.F.flags.f_contiguous
    assert np.all(pr.F[:, 0] == 1) and pr.F[:, 1].min() == -1 and pr.F[:, 1].max() == 1
    assert pr.nparts == 16 and np.all(np.bincount(pr.part) == 16)
    # block coordinates agree with node coordinates
    for I in range(pr.nparts):
        nodes = np.nonzero(pr.part == I)[0]
        assert np.all(nodes % 16 // 4 == pr.block_coords[I, 0])
        assert np.all(nodes // 16 // 4 == pr.block_coords[I, 1])


@pytest.mark.parametrize("mk", [lambda: P.poisson2d(8, 4, 1), lambda: P.poisson3d(6, 3, 2),
                                lambda: P.biharmonic2d(12, 4, 3), lambda: P.elasticity3d(4, 2),
                                lambda: P.lognormal3d(6, 3, 1)])
def test_csr_canonical(mk):
    pr = mk()
    assert pr.row_ptr[0] == 0 and pr.row_ptr[-1] == len(pr.col) == len(pr.val)
    for i in range(pr.n):
        c = pr.col[pr.row_ptr[i]:pr.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    A = pr.dense()
    assert np.abs(A - A.T).max() <= 1e-15 * np.abs(A).max()


@pytest.mark.parametrize("make", [lambda: P.poisson2d(12, 4, 1, 1), lambda: P.poisson3d(6, 3, 1, 2),
                                  lambda: P.lognormal3d(6, 3, 1, 3), lambda: P.biharmonic2d(12, 4, 2, 4)])
def test_stencil_descriptor_reproduces_csr(make):
    """pr.stencil (include/ddg.h ddg_stencil, handed to the library's matrix-free
    row kernels) describes exactly the assembled CSR matrix: rebuilt entry by
    entry from the descriptor, it equals A bitwise."""
    pr = make()
    st = pr.stencil
    d = list(st["dims"]) + [1] * (3 - len(st["dims"]))
    n = pr.n
    A = pr.scipy().toarray()
    B = np.zeros_like(A)
    for v in range(n):
        ix, iy, iz = v % d[0], (v // d[0]) % d[1], v // (d[0] * d[1])
        if st["kind"] == "const":
            for o, c in zip(st["offsets"], st["coef"]):
                o = list(o) + [0] * (3 - len(o))
                a, b, cc = ix + o[0], iy + o[1], iz + o[2]
                if 0 <= a < d[0] and 0 <= b < d[1] and 0 <= cc < d[2]:
                    B[v, v + o[0] + d[0] * (o[1] + d[1] * o[2])] = c
        else:
            cf = st["coef"]
            D, CX, CY, CZ = cf[:n], cf[n:2 * n], cf[2 * n:3 * n], cf[3 * n:]
            B[v, v] = D[v]
            for ok, cv, off in ((ix + 1 < d[0], CX, 1), (iy + 1 < d[1], CY, d[0]), (iz + 1 < d[2], CZ, d[0] * d[1])):
                if ok:
                    B[v, v + off] = cv[v]
                    B[v + off, v] = cv[v]
    assert np.array_equal(A, B)


def test_poisson3d_mixed_boundary_rows():
    """Problem (A) (reading R21): A 1 is the indicator of the
    Dirichlet layer z = 0 (Neumann rows sum to zero), and A is SPD."""
    pr = P.poisson3d_mixed(5, 5, 1)
    A = pr.dense()
    assert np.array_equal(A, A.T)
    z = (np.arange(pr.n) // 25) == 0
    assert np.array_equal(A @ np.ones(pr.n), z.astype(float))
    assert np.linalg.eigvalsh(A).min() > 0
    # the 2x2x2 case by hand: every node has 3 in-grid neighbours, +1 on z = 0
    B = P.poisson3d_mixed(2, 2, 0).dense()
    assert np.array_equal(np.diag(B), [4, 4, 4, 4, 3, 3, 3, 3])
    assert (B[0] == np.array([4, -1, -1, 0, -1, 0, 0, 0])).all()


@pytest.mark.parametrize("mk,nparts", [(lambda: P.lognormal3d(16, 4, 1, 32), 64),
                                        (lambda: P.biharmonic2d(64, 16, 3, 34), 20),
                                        (lambda: P.elasticity3d(8, 4, 35), 10)])
def test_grown_partition_connected_irregular(mk, nparts):
    """grown_partition: every node in one of nparts non-empty parts, each part
    connected in the graph of A, sizes not all equal, deterministic in the seed,
    and the matrix, F and f untouched"""
    import scipy.sparse.csgraph as cg
    pr = mk()
    g = P.grown_partition(pr, nparts, 9)
    assert g.part.shape == (pr.n,) and g.part.min() == 0 and g.part.max() == nparts - 1
    sz = np.bincount(g.part, minlength=nparts)
    assert sz.min() > 0 and sz.min() < sz.max()
    A = pr.scipy()
    for q in range(nparts):
        idx = np.flatnonzero(g.part == q)
        ncomp, _ = cg.connected_components(A[idx][:, idx], directed=False)
        assert ncomp == 1, q
    assert np.array_equal(P.grown_partition(pr, nparts, 9).part, g.part)
    assert not np.array_equal(P.grown_partition(pr, nparts, 10).part, g.part)
    assert g.val is pr.val and g.F is pr.F and g.f is pr.f and g.block_coords is None


def test_node27_descriptor_classes_reproduce_csr():
    """C4's node27 descriptor (include/ddg.h DDG_STENCIL_NODE27): every row is a
    full 27-point node row in ascending column order, and all nodes of one
    boundary class (first / interior / last per axis) have identical rows, so
    the class table the library reads from the CSR reproduces A exactly."""
    pr = P.elasticity3d(4, 2, 5)
    st = pr.stencil
    assert st["kind"] == "node27" and st["dof"] == 3
    nx, ny, nz = st["dims"]
    dof = st["dof"]
    assert nx * ny * nz * dof == pr.n
    table = {}
    for node in range(nx * ny * nz):
        ix, iy, iz = node % nx, (node // nx) % ny, node // (nx * ny)
        cls = tuple(0 if a == 0 else 2 if a == m - 1 else 1 for a, m in ((ix, nx), (iy, ny), (iz, nz)))
        for d in range(dof):
            v = node * dof + d
            cols, vals = [], []
            for dz in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        a, b, c = ix + dx, iy + dy, iz + dz
                        if 0 <= a < nx and 0 <= b < ny and 0 <= c < nz:
                            nb = a + nx * (b + ny * c)
                            cols += [nb * dof + e for e in range(dof)]
            row = slice(pr.row_ptr[v], pr.row_ptr[v + 1])
            assert np.array_equal(pr.col[row], np.array(cols))
            key = (cls, d)
            if key in table:
                assert np.array_equal(table[key], pr.val[row])
            else:
                table[key] = pr.val[row].copy()
    assert len(table) == 27 * dof
