"""Small dense helpers for tests (independent numpy re-derivations on tiny grids)."""
from __future__ import annotations

import numpy as np


def csr_from_dense(A):
    n = A.shape[0]
    rp = [0]
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(A[i])[0]
        cols.extend(nz.tolist())
        vals.extend(A[i, nz].tolist())
        rp.append(len(cols))
    return (np.array(rp, np.int64), np.array(cols, np.int32), np.array(vals, np.float64))


def laplace1d(n):
    A = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    return A


def graph_distance_sets(A_pattern, parts, delta):
    """Omega~_i by multi-source shortest paths on the unweighted graph of A
    (scipy csgraph; an independent route to PAPER.md:541-542)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import shortest_path
    G = sp.csr_matrix((A_pattern != 0).astype(float))
    G.setdiag(0)
    G.eliminate_zeros()
    D = shortest_path(G, unweighted=True, directed=False)
    out = []
    for p in parts:
        d = D[p].min(axis=0)
        out.append(np.nonzero(d <= delta)[0])
    return out


def dense_two_level(A, r, sets, order, P):
    """Literal dense composition of PAPER.md:555 and :560-564:
    z=0; for i in order: z += R_i^T A_i^{-1} R_i (r - A z); z += P (P^T A P)^{-1} P^T (r - A z);
    for i in reversed(order): same update."""
    z = np.zeros(A.shape[0])
    for i in order:
        idx = sets[i]
        z[idx] += np.linalg.solve(A[np.ix_(idx, idx)], (r - A @ z)[idx])
    Ac = P.T @ A @ P
    z += P @ np.linalg.solve(Ac, P.T @ (r - A @ z))
    for i in reversed(order):
        idx = sets[i]
        z[idx] += np.linalg.solve(A[np.ix_(idx, idx)], (r - A @ z)[idx])
    return z


def block_projectors_local(coords, part, nparts, p):
    """Orthogonal projector onto degree<=p polynomials of LOCAL (block-centred,
    block-scaled) coordinates on every part: the same polynomial space as
    global monomials restricted to the part, computed without ill-conditioning."""
    from ddg_gen.problems import monomial_exponents
    out = []
    for I in range(nparts):
        rows = np.nonzero(part == I)[0]
        X = coords[rows]
        c = X.mean(axis=0)
        s = np.maximum(np.abs(X - c).max(axis=0), 1e-300)
        Xl = (X - c) / s
        cols = []
        for e in monomial_exponents(X.shape[1], p):
            v = np.ones(len(rows))
            for d, ed in enumerate(e):
                v = v * Xl[:, d] ** ed
            cols.append(v)
        Q, _ = np.linalg.qr(np.stack(cols, axis=1))
        out.append((rows, Q @ Q.T))
    return out
