"""Seeded synthetic problem generators for the five BASELINE.json configs.

Input recipe only — this module defines the PDE systems A u = f that the
method is run on (matrix assembly, generating vectors F, block partition,
right-hand side).  It contains none of the method's arithmetic (no overlap,
no orthogonalisation, no Galerkin product, no Schwarz, no CG), so both the
oracle tests and the CUDA path may use it (task rule ③).

Readings of the paper / BASELINE:
  * C1 2D Poisson 5-point (4,-1), Dirichlet 0 eliminated        (BASELINE configs[0])
  * C2 3D Poisson 7-point (6,-1), Dirichlet 0 on all faces
  * C3 cell-centred 7-point, k = exp(g), harmonic face averages  (c11)
  * C4 Q1 hexahedral elasticity, z=0 face clamped, DoF node-major (c12)
  * C5 13-point biharmonic, every off-grid value zero (diag 20)   (c13)
  * stencils unscaled (no 1/h^2, 1/h^4)                           (c14)
  * f ~ U(-1,1) by SplitMix64, seeds 1000 + config id             (c15)
  * F = graded-lex monomials of coordinates mapped to [-1,1]^d    (c8)
  * partition = regular blocks of H/h nodes per axis, x fastest
"""
from __future__ import annotations

import dataclasses
import itertools

import numpy as np

from . import rng


@dataclasses.dataclass
class Problem:
    name: str
    n: int
    row_ptr: np.ndarray        # int64 [n+1]
    col: np.ndarray            # int32 [nnz], strictly increasing per row
    val: np.ndarray            # float64 [nnz]
    F: np.ndarray              # float64 [n, k], Fortran order (column-major)
    part: np.ndarray           # int32 [n]
    nparts: int
    block_coords: np.ndarray   # int32 [nparts, ndim]
    block_dims: tuple
    f: np.ndarray              # float64 [n]
    overlap: int = 1
    meta: dict = dataclasses.field(default_factory=dict)
    # structured-grid description of A for the library's matrix-free row
    # kernels (include/ddg.h ddg_stencil); the CSR above stays the definition
    stencil: dict = None

    @property
    def k(self) -> int:
        return self.F.shape[1]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def dense(self) -> np.ndarray:
        """Dense copy of A (tests on tiny grids only)."""
        A = np.zeros((self.n, self.n))
        for i in range(self.n):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            A[i, self.col[s:e]] = self.val[s:e]
        return A

    def scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.row_ptr), shape=(self.n, self.n))


# ----------------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------------

def monomial_exponents(ndim: int, p: int):
    """Graded-lex exponents: degree 0..p, within a degree x-power descending."""
    out = []
    for d in range(p + 1):
        if ndim == 1:
            out.append((d,))
        elif ndim == 2:
            for a in range(d, -1, -1):
                out.append((a, d - a))
        else:
            for a in range(d, -1, -1):
                for b in range(d - a, -1, -1):
                    out.append((a, b, d - a - b))
    return out


def monomials(coords: np.ndarray, p: int) -> np.ndarray:
    """F[:, j] = prod_d xhat_d^e_jd with coordinates affinely mapped to [-1,1]^d (c8)."""
    lo = coords.min(axis=0)
    hi = coords.max(axis=0)
    span = np.where(hi > lo, hi - lo, 1.0)
    xh = 2.0 * (coords - lo) / span - 1.0
    ex = monomial_exponents(coords.shape[1], p)
    F = np.empty((coords.shape[0], len(ex)), order="F")
    for j, e in enumerate(ex):
        col = np.ones(coords.shape[0])
        for d, ed in enumerate(e):
            if ed:
                col = col * xh[:, d] ** ed
        F[:, j] = col
    return F


def grid_coords(dims, origin=1.0, h=1.0):
    """Node coordinates (x fastest) for a structured grid, index = x + nx*(y + ny*z)."""
    axes = [origin * h + h * np.arange(d) for d in dims]
    mesh = np.meshgrid(*axes, indexing="ij")
    # linear index x fastest => ravel in Fortran order
    return np.stack([m.ravel(order="F") for m in mesh], axis=1)


def block_partition(dims, bsize):
    """Block id per node of a structured grid; blocks of `bsize` nodes per axis
    (the last block along an axis absorbs a remainder), block ids x fastest."""
    ndim = len(dims)
    nb = [max(1, d // b) for d, b in zip(dims, bsize)]
    idx = np.indices(dims, dtype=np.int64)            # [ndim, *dims] C-order
    bid = np.zeros(dims, dtype=np.int64)
    mult = 1
    for ax in range(ndim):
        bax = np.minimum(idx[ax] // bsize[ax], nb[ax] - 1)
        bid += bax * mult
        mult *= nb[ax]
    part = bid.ravel(order="F").astype(np.int32)      # x fastest
    bc = np.array(list(itertools.product(*[range(b) for b in reversed(nb)])), dtype=np.int32)
    bc = bc[:, ::-1].copy()                           # (bx, by, bz) with bx fastest
    return part, int(np.prod(nb)), bc, tuple(nb)


def coarse_parts(pr, factor=None, allow_single=False, coords=False, nearest=False):
    """Second-level partition for the three-level method:
    the parts' block coordinates grouped `factor` per axis (the last group
    along an axis absorbs a remainder), so that H_1/H_0 = H_0/h when factor is
    the blocks' size H/h (the default: the first axis of meta['bsize']).
    Returns (part2 int32[nparts], nparts2) or, with coords=True, also the
    second-level block coordinates int32[nparts2, ndim].  Fewer than 2 groups means the
    problem is "too small to use the three-level solver" (Table 3's
    x entries) and raises ValueError unless allow_single.  nearest=True
    instead splits each axis's blocks evenly into round(blocks / factor)
    groups (the paper's grids are not multiples of (H/h)^2 blocks)."""
    if factor is None:
        factor = int(pr.meta.get("bsize", (2,))[0])
    nb = list(pr.block_dims)
    if nearest:
        ng = [max(1, int(np.floor(b / factor + 0.5))) for b in nb]
    else:
        ng = [max(1, b // factor) for b in nb]
    bc = np.asarray(pr.block_coords, np.int64)
    g = np.zeros(pr.nparts, np.int64)
    mult = 1
    for ax in range(len(nb)):
        if nearest:
            g += (bc[:, ax] * ng[ax] // nb[ax]) * mult
        else:
            g += np.minimum(bc[:, ax] // factor, ng[ax] - 1) * mult
        mult *= ng[ax]
    n2 = int(np.prod(ng))
    if n2 < 2 and not allow_single:
        raise ValueError(f"too small for three levels: {pr.nparts} parts grouped {factor} per axis "
                         f"give {n2} second-level part")
    if coords:
        bc2 = np.array(list(itertools.product(*[range(b) for b in reversed(ng)])), dtype=np.int32)
        return g.astype(np.int32), n2, bc2[:, ::-1].copy()
    return g.astype(np.int32), n2


def stencil_csr(dims, offsets, coef_fn):
    """CSR of a structured-grid operator.

    offsets: list of integer offset tuples (dx, dy[, dz]).
    coef_fn(k, valid) -> array of coefficients for offset k at every node
    (only entries where `valid` is True are kept).  Off-grid neighbours are
    dropped (zero Dirichlet / zero ghost values).  Columns strictly increase
    within each row because offsets are sorted by their linear offset.
    """
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    strides = [int(np.prod(dims[:a])) for a in range(len(dims))]
    lin = [sum(o[a] * strides[a] for a in range(len(dims))) for o in offsets]
    order = np.argsort(lin, kind="stable")
    idx = np.indices(dims, dtype=np.int64)  # idx[a] shaped dims (C order over axes)
    cols = np.empty((n, len(offsets)), dtype=np.int64)
    vals = np.empty((n, len(offsets)), dtype=np.float64)
    keep = np.empty((n, len(offsets)), dtype=bool)
    node = np.arange(n, dtype=np.int64)
    for slot, k in enumerate(order):
        o = offsets[k]
        valid = np.ones(dims, dtype=bool)
        for a in range(len(dims)):
            q = idx[a] + o[a]
            valid &= (q >= 0) & (q < dims[a])
        valid = valid.ravel(order="F")
        keep[:, slot] = valid
        cols[:, slot] = node + lin[k]
        vals[:, slot] = coef_fn(k, valid)
    counts = keep.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col = cols[keep].astype(np.int32)
    val = vals[keep]
    return row_ptr, col, val


def _finish(name, dims, row_ptr, col, val, coords, p, bsize, seed, overlap, meta):
    n = int(np.prod(dims))
    F = monomials(coords, p)
    part, nparts, bc, nb = block_partition(dims, bsize)
    f = rng.uniform_pm1(seed, n)
    return Problem(name=name, n=n, row_ptr=row_ptr, col=col, val=val, F=F, part=part,
                   nparts=nparts, block_coords=bc, block_dims=nb, f=f, overlap=overlap,
                   meta=dict(meta, dims=tuple(dims), p=p, bsize=tuple(bsize), seed=seed))


# ----------------------------------------------------------------------------
# the five configurations
# ----------------------------------------------------------------------------

def poisson2d(N=64, b=8, p=1, seed=1001, overlap=1):
    """C1: 2D Poisson, 5-point FD (4, -1), N x N interior, Dirichlet 0 (BASELINE configs[0])."""
    offs = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)]
    rp, c, v = stencil_csr((N, N), offs, lambda k, m: np.full(m.shape, 4.0 if k == 0 else -1.0))
    h = 1.0 / (N + 1)
    coords = grid_coords((N, N), 1.0, h)
    pr = _finish("poisson2d", (N, N), rp, c, v, coords, p, (b, b), seed, overlap, dict(stencil="5pt"))
    pr.stencil = dict(kind="const", dims=(N, N, 1), offsets=offs, coef=[4.0, -1, -1, -1, -1])
    return pr


def poisson3d(N=128, b=8, p=2, seed=1002, overlap=1):
    """C2: 3D Poisson, 7-point FD (6, -1), N^3 interior, Dirichlet 0 on all faces (c10)."""
    offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    rp, c, v = stencil_csr((N, N, N), offs, lambda k, m: np.full(m.shape, 6.0 if k == 0 else -1.0))
    h = 1.0 / (N + 1)
    coords = grid_coords((N, N, N), 1.0, h)
    pr = _finish("poisson3d", (N, N, N), rp, c, v, coords, p, (b, b, b), seed, overlap, dict(stencil="7pt"))
    pr.stencil = dict(kind="const", dims=(N, N, N), offsets=offs, coef=[6.0, -1, -1, -1, -1, -1, -1])
    return pr


def poisson3d_mixed(N=40, b=10, p=1, seed=1010, overlap=0):
    """The paper's problem (A), "Poisson 3D": 7-point FD on an
    N^3 grid, one face Dirichlet and the other five Neumann.  Reading R21: the
    graph Laplacian of the grid (off-diagonal -1 to every in-grid neighbour,
    diagonal = number of in-grid neighbours) plus 1 on the diagonal of the
    z = 0 layer (the Dirichlet face's ghost).  f ~ N(0, 1) ("random
    Gaussian-distributed").  Block partition instead of the
    paper's recursive inertial one (out of scope); Delta = 0
    by default as in the paper (only the biharmonic uses Delta = 1)."""
    dims = (N, N, N)
    idx = np.indices(dims, dtype=np.int64)
    cnt = np.zeros(dims, np.float64)
    for a in range(3):
        cnt += (idx[a] > 0).astype(float) + (idx[a] < N - 1).astype(float)
    cnt += (idx[2] == 0).astype(float)
    diag = cnt.ravel(order="F")
    offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    rp, c, v = stencil_csr(dims, offs, lambda k, m: diag.copy() if k == 0 else np.full(m.shape, -1.0))
    h = 1.0 / N
    coords = grid_coords(dims, 0.5, h)
    pr = _finish("poisson3d_mixed", dims, rp, c, v, coords, p, (b, b, b), seed, overlap,
                 dict(stencil="7pt, Dirichlet z=0 face, Neumann elsewhere"))
    pr.f = rng.normal(seed, pr.n)
    return pr


def lognormal3d(N=256, b=4, p=1, seed=1003, overlap=1):
    """C3: cell-centred 7-point, k = exp(g), g ~ N(0,1) per cell; interior face
    T = 2 ka kb / (ka + kb), boundary face T = ka; row = sum_faces T (ua - ub) (c11)."""
    dims = (N, N, N)
    n = N ** 3
    g = rng.normal(seed + 100, n)
    kc = np.exp(g)
    kg = kc.reshape(dims, order="F")                    # kg[x, y, z]
    offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    # face transmissibility towards each of the 6 neighbours (boundary => T = ka)
    T = []
    for o in offs[1:]:
        kn = np.roll(kg, shift=tuple(-x for x in o), axis=(0, 1, 2))
        t = 2.0 * kg * kn / (kg + kn)
        for a in range(3):
            if o[a] == 1:
                sl = [slice(None)] * 3; sl[a] = -1; t[tuple(sl)] = kg[tuple(sl)]
            elif o[a] == -1:
                sl = [slice(None)] * 3; sl[a] = 0; t[tuple(sl)] = kg[tuple(sl)]
        T.append(t.ravel(order="F"))
    diag = np.sum(T, axis=0)

    def coef(k, m):
        return diag if k == 0 else -T[k - 1]

    rp, c, v = stencil_csr(dims, offs, coef)
    h = 1.0 / N
    coords = grid_coords(dims, 0.5, h)                  # cell centres
    pr = _finish("lognormal3d", dims, rp, c, v, coords, p, (b, b, b), seed, overlap,
                 dict(stencil="7pt_harmonic"))
    # couplings towards +x, +y, +z (T[0], T[2], T[4]); the -x/-y/-z entries are
    # the same faces seen from the neighbour (the harmonic mean is symmetric)
    pr.stencil = dict(kind="face7", dims=dims, coef=np.concatenate([diag, -T[0], -T[2], -T[4]]))
    return pr


def material2d(N=256, b=16, p=3, seed=1006, overlap=1, aware=False):
    """Problem (C) of the paper on a structured grid:
    div(D grad u) = f with D = S + 100 J, S = exp(1 + sin(pi (x + y))),
    J = H(0.25 + cos(pi x) cos(2 pi y)) the indicator of a second material.
    The paper's annulus mesh is replaced by the square [-1,1]^2 (N x N cells,
    cell-centred 5-point, harmonic face averages T = 2 Da Db / (Da + Db),
    boundary faces T = Da: Dirichlet at the ghost cell, reading R11's rule in
    2D); the block partition (b x b cells) does not conform to the material
    boundary, as the paper's algebraic partitions did not.

    aware=True gives the material-aware generating vectors: "piecewise
    polynomial with respect to the material domains", [F * (1 - J), F * J]
    (2k columns; a part inside one material keeps only k -- the rank test R7
    drops the columns that vanish on it)."""
    dims = (N, N)
    n = N * N
    h = 2.0 / N
    xc = -1.0 + h * (np.arange(N) + 0.5)
    X, Y = np.meshgrid(xc, xc, indexing="ij")                # X[ix, iy]
    S = np.exp(1.0 + np.sin(np.pi * (X + Y)))
    J = (0.25 + np.cos(np.pi * X) * np.cos(2 * np.pi * Y) > 0).astype(np.float64)
    D = S + 100.0 * J
    offs = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)]
    T = []
    for o in offs[1:]:
        Dn = np.roll(D, shift=tuple(-x for x in o), axis=(0, 1))
        t = 2.0 * D * Dn / (D + Dn)
        for a in range(2):
            if o[a] == 1:
                sl = [slice(None)] * 2; sl[a] = -1; t[tuple(sl)] = D[tuple(sl)]
            elif o[a] == -1:
                sl = [slice(None)] * 2; sl[a] = 0; t[tuple(sl)] = D[tuple(sl)]
        T.append(t.ravel(order="F"))
    diag = np.sum(T, axis=0)

    def coef(k, m):
        return diag if k == 0 else -T[k - 1]

    rp, c, v = stencil_csr(dims, offs, coef)
    coords = np.stack([X.ravel(order="F"), Y.ravel(order="F")], axis=1)
    pr = _finish("material2d", dims, rp, c, v, coords, p, (b, b), seed, overlap,
                 dict(stencil="5pt_harmonic", aware=bool(aware)))
    if aware:
        j = J.ravel(order="F")[:, None]
        pr.F = np.asfortranarray(np.concatenate([pr.F * (1.0 - j), pr.F * j], axis=1))
    pr.meta["material_fraction"] = float(J.mean())
    return pr


def biharmonic2d(N=2048, b=16, p=3, seed=1005, overlap=1):
    """C5: 13-point biharmonic (20; -8 axis; +2 diagonal; +1 at distance 2 on axes),
    restricted to the N x N grid with every off-grid value zero (c13)."""
    offs = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (1, -1), (-1, 1), (-1, -1),
            (2, 0), (-2, 0), (0, 2), (0, -2)]
    cf = [20.0, -8, -8, -8, -8, 2, 2, 2, 2, 1, 1, 1, 1]
    rp, c, v = stencil_csr((N, N), offs, lambda k, m: np.full(m.shape, float(cf[k])))
    h = 1.0 / (N + 1)
    coords = grid_coords((N, N), 1.0, h)
    pr = _finish("biharmonic2d", (N, N), rp, c, v, coords, p, (b, b), seed, overlap, dict(stencil="13pt"))
    pr.stencil = dict(kind="const", dims=(N, N, 1), offsets=offs, coef=cf)
    return pr


# --- C4: Q1 elasticity -------------------------------------------------------

def q1_element_stiffness(h=1.0, E=1.0, nu=0.3):
    """24x24 stiffness of a trilinear hexahedron [0,h]^3, isotropic, 2x2x2 Gauss.
    Local node ordering: d = (dx, dy, dz) in {0,1}^3, index dx + 2 dy + 4 dz;
    DoF = 3 * node + component."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2 * mu
    D[3:, 3:] = np.eye(3) * mu
    gp = np.array([-1.0, 1.0]) / np.sqrt(3.0)
    nodes = np.array([(dx, dy, dz) for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)], float)
    sgn = 2 * nodes - 1                                 # +-1 reference coordinates
    K = np.zeros((24, 24))
    for xi, eta, zeta in itertools.product(gp, gp, gp):
        # dN/dxi_ref, then physical derivative = (2/h) dN/dref
        dN = np.empty((8, 3))
        for a in range(8):
            sx, sy, sz = sgn[a]
            dN[a, 0] = sx * (1 + sy * eta) * (1 + sz * zeta) / 8
            dN[a, 1] = sy * (1 + sx * xi) * (1 + sz * zeta) / 8
            dN[a, 2] = sz * (1 + sx * xi) * (1 + sy * eta) / 8
        dN *= 2.0 / h
        B = np.zeros((6, 24))
        for a in range(8):
            B[0, 3 * a + 0] = dN[a, 0]
            B[1, 3 * a + 1] = dN[a, 1]
            B[2, 3 * a + 2] = dN[a, 2]
            B[3, 3 * a + 0] = dN[a, 1]; B[3, 3 * a + 1] = dN[a, 0]
            B[4, 3 * a + 1] = dN[a, 2]; B[4, 3 * a + 2] = dN[a, 1]
            B[5, 3 * a + 0] = dN[a, 2]; B[5, 3 * a + 2] = dN[a, 0]
        K += B.T @ D @ B * (h / 2) ** 3                # Gauss weights 1, detJ = (h/2)^3
    return K, lam, mu


def elasticity3d(ne=64, be=8, seed=1004, overlap=1, E=1.0, nu=0.3, clamp=True):
    """C4: 3D linear elasticity, Q1 hexahedra on an ne^3 element mesh of the unit
    cube, 3 DoF per node interleaved node-major, face z=0 clamped (its nodes
    eliminated), body force ~ U(-1,1) per DoF used as the load vector (c12).
    F = 12 vector-valued linears (3 components x {1, x, y, z}); partition per
    node block (min(i//be, nb-1), ...), DoFs inherit their node's block."""
    h = 1.0 / ne
    Ke, lam, mu = q1_element_stiffness(h, E, nu)
    nn = ne + 1
    z0 = 1 if clamp else 0
    nz = nn - z0                                        # free node layers
    dims = (nn, nn, nz)
    nnode = nn * nn * nz
    n = 3 * nnode
    idx = np.indices(dims, dtype=np.int64)             # node (i, j, kk); physical k = kk + z0
    ii, jj, kk = [a.ravel(order="F") for a in idx]
    kphys = kk + z0
    locs = [(dx, dy, dz) for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)]
    offs = sorted(itertools.product((-1, 0, 1), repeat=3), key=lambda o: (o[2], o[1], o[0]))
    cols, vals, keep = [], [], []
    node = np.arange(nnode, dtype=np.int64)
    for o in offs:
        blk = np.zeros((nnode, 3, 3))
        for d in locs:
            dd = tuple(d[a] + o[a] for a in range(3))
            if min(dd) < 0 or max(dd) > 1:
                continue
            # element origin e = p - d must be a valid element
            ex, ey, ez = ii - d[0], jj - d[1], kphys - d[2]
            ok = (ex >= 0) & (ex < ne) & (ey >= 0) & (ey < ne) & (ez >= 0) & (ez < ne)
            la = d[0] + 2 * d[1] + 4 * d[2]
            lb = dd[0] + 2 * dd[1] + 4 * dd[2]
            blk[ok] += Ke[3 * la:3 * la + 3, 3 * lb:3 * lb + 3]
        qi, qj, qk = ii + o[0], jj + o[1], kk + o[2]
        valid = (qi >= 0) & (qi < nn) & (qj >= 0) & (qj < nn) & (qk >= 0) & (qk < nz)
        qnode = node + o[0] + nn * (o[1] + nn * o[2])
        for cb in range(3):
            cols.append(3 * qnode + cb)
            vals.append(blk[:, :, cb])                 # [nnode, 3 (row comp)]
            keep.append(valid)
    # assemble rows 3a+ca: entries ordered by (offset, cb) -> increasing column
    C = np.stack(cols, axis=1)                          # [nnode, 81]
    V = np.stack(vals, axis=2)                          # [nnode, 3, 81]
    K = np.stack(keep, axis=1)                          # [nnode, 81]
    # drop exact structural zeros? keep full pattern of valid neighbours
    counts = np.repeat(K.sum(axis=1), 3)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    Cr = np.repeat(C[:, None, :], 3, axis=1).reshape(n, -1)
    Kr = np.repeat(K[:, None, :], 3, axis=1).reshape(n, -1)
    Vr = V.reshape(n, -1)
    col = Cr[Kr].astype(np.int32)
    val = Vr[Kr]
    coords_node = np.stack([ii * h, jj * h, kphys * h], axis=1).astype(float)
    Fs = monomials(coords_node, 1)                      # [nnode, 4]
    F = np.zeros((n, 12), order="F")
    for c in range(3):
        F[c::3, 4 * c:4 * c + 4] = Fs
    # blocks along z are formed from the free layers kphys = 1..ne: kphys//be, capped
    kb = np.minimum(kphys // be, ne // be - 1)
    ib = np.minimum(ii // be, ne // be - 1)
    jb = np.minimum(jj // be, ne // be - 1)
    nbx = ne // be
    npart = (ib + nbx * (jb + nbx * kb)).astype(np.int32)
    nparts = nbx ** 3
    bc = np.array([(x, y, z) for z in range(nbx) for y in range(nbx) for x in range(nbx)],
                  dtype=np.int32)
    part = np.repeat(npart, 3)
    f = rng.uniform_pm1(seed, n)
    pr = Problem(name="elasticity3d", n=n, row_ptr=row_ptr, col=col, val=val, F=F,
                 part=part, nparts=nparts, block_coords=bc, block_dims=(nbx,) * 3, f=f,
                 overlap=overlap,
                 meta=dict(dims=dims, p=1, be=be, ne=ne, lam=lam, mu=mu, seed=seed,
                           stencil="q1_elastic", dof_per_node=3))
    # node-blocked 27-point rows, constant per boundary class (include/ddg.h
    # DDG_STENCIL_NODE27): the library reads the values from the CSR and checks
    # every row against them
    pr.stencil = dict(kind="node27", dims=dims, dof=3)
    return pr


def grown_partition(pr, nparts, seed=77):
    """The same problem with an irregular, non-box partition: `nparts` seeds
    drawn from the SplitMix64 stream `seed`, grown together over the graph of
    A by breadth-first rounds in which every part claims its unclaimed
    neighbours (ties: the lowest part id).  Parts are connected, their
    boundaries follow no grid line, and sizes vary (the paper partitions with
    SCOTCH or inertial bisection).  Components the
    seeds do not reach (none for connected A) join part 0.  No block
    coordinates: the library's nested dissection falls back to its graph
    bisection, the oracle to the envelope coarse factor."""
    n = pr.n
    if not (1 <= nparts <= n):
        raise ValueError("1 <= nparts <= n")
    u = rng.uniform01(seed, n)
    seeds = np.argsort(u, kind="stable")[:nparts]
    part = np.full(n, -1, np.int64)
    part[seeds] = np.arange(nparts)
    rp, col = np.asarray(pr.row_ptr, np.int64), np.asarray(pr.col, np.int64)
    rows = np.repeat(np.arange(n), np.diff(rp))
    while True:
        # every claimed node offers its part to its unclaimed neighbours
        src = part[rows]
        dst = col
        m = (src >= 0) & (part[dst] < 0)
        if not m.any():
            break
        best = np.full(n, np.iinfo(np.int64).max)
        np.minimum.at(best, dst[m], src[m])
        newly = best < np.iinfo(np.int64).max
        part[newly] = best[newly]
    part[part < 0] = 0
    return dataclasses.replace(pr, name=pr.name + f"_grown{nparts}", part=part.astype(np.int32),
                               nparts=int(nparts), block_coords=None, block_dims=None,
                               meta=dict(pr.meta, partition=f"grown({nparts}, seed {seed})"))


CONFIGS = {
    "C1": lambda: poisson2d(64, 8, 1, 1001),
    "C2": lambda: poisson3d(128, 8, 2, 1002),
    "C3": lambda: lognormal3d(256, 4, 1, 1003),
    "C4": lambda: elasticity3d(64, 8, 1004),
    "C5": lambda: biharmonic2d(2048, 16, 3, 1005),
}

CONFIG_TEXT = {
    "C1": "2D Poisson 5-point 64x64, 8x8 blocks, p=1, overlap 1",
    "C2": "3D Poisson 7-point 128^3, 8^3 blocks, p=2, overlap 1",
    "C3": "3D lognormal-coefficient 7-point 256^3, 4^3 blocks, p=1, overlap 1",
    "C4": "3D Q1 elasticity 64^3 elements, 8^3-element blocks, 12 linear modes, overlap 1",
    "C5": "2D biharmonic 13-point 2048^2, 16x16 blocks, p=3, overlap 1",
}


def make(name: str) -> Problem:
    return CONFIGS[name]()
