"""Exact coarse solve A_0^{-1} by a nested-dissection multifrontal Cholesky.

CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Used by the
oracle when A_0 is too large for the envelope Cholesky of oracle.c (C3:
n_c = 1,048,576 would need ~1.7e10 envelope entries).  Shares nothing with the
product's coarse factorisation (paper_1504_00907_b200/csrc/coarse_sparse.cpp).

What it computes is plain: the Cholesky factor of A_0 in a nested-dissection
order, and forward then back substitution with it ("A_0 u_0 =
R_0 f"; "the block sparsity pattern of A_0 ... has the same
sparsity pattern as the subdomain adjacency matrix ... efficient numerical
linear algebra using dense storage and operations").  Steps, in order:

  1. ordering (SURVEY.md §8(c) setup step 5): recursive bisection of the box
     of block coordinates along its longest axis, the separator a one-block
     thick layer; boxes of at most `leaf` unknowns are leaves.  The tree is
     checked: every coupling of A_0 must join a node to itself or to one of
     its ancestors (else the ordering is not a dissection and we refuse).
  2. symbolic: for tree node t with unknowns S_t, its boundary B_t = the
     ancestors' unknowns coupled to S_t in A_0 or lying in a child's boundary.
  3. numeric, children before parents (multifrontal):
        F = [A_0[S,S] A_0[S,B]; A_0[B,S] 0] + extend-add of the children's U
        L_SS = chol(F_SS)              (numpy.linalg.cholesky)
        L_BS = F_BS L_SS^{-T}          (scipy.linalg.solve_triangular)
        U    = F_BB - L_BS L_BS^T      (passed to the parent)
  4. solve: forward over the tree (x_S <- L_SS^{-1} x_S; x_B -= L_BS x_S),
     then backward in reverse (x_S <- L_SS^{-T} (x_S - L_BS^T x_B)).

The library routines (LAPACK Cholesky and triangular solve, BLAS products)
are the steps' primitives; nothing is blocked or fused beyond the fronts the
dissection defines.  Pinned in tests/test_oracle_coarse_nd.py against the
envelope Cholesky of oracle.c and a dense numpy solve.
"""
from __future__ import annotations

import os

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


class NDCholesky:
    """A_0 = L L^T in nested-dissection order; solve(x) overwrites x with A_0^{-1} x.

    A0: scipy CSR, full symmetric, coarse order.  cptr: coarse offsets of the
    parts (nparts+1).  block_coords: int [nparts, ndim] block-grid coordinates.
    leaf: maximum unknowns in a leaf box.  perturb: floor mode (separator one
    layer below the middle, the last longest axis first) -- a different but
    equally exact elimination order.  scratch: directory for a file-backed
    factor (the C3 factor is ~30 GB); None keeps it in memory.
    """

    def __init__(self, A0, cptr, block_coords, leaf=256, perturb=False, scratch=None):
        A0 = sp.csr_matrix(A0)
        self.nc = A0.shape[0]
        cptr = np.asarray(cptr, np.int64)
        coords = np.asarray(block_coords, np.int64)
        nparts = len(cptr) - 1
        rank = np.diff(cptr)
        # ---- 1. nested-dissection tree over the parts
        self.nodes = []                     # postorder: (parts, children)
        parent = []

        def dissect(parts):
            box = coords[parts]
            lo, hi = box.min(axis=0), box.max(axis=0)
            ext = hi - lo + 1
            if rank[parts].sum() <= leaf or ext.max() < 3:
                self.nodes.append((np.sort(parts), []))
                parent.append(-1)
                return len(self.nodes) - 1
            ax = int(np.flatnonzero(ext == ext.max())[-1 if perturb else 0])
            mid = lo[ax] + ext[ax] // 2 - (1 if perturb and ext[ax] >= 4 else 0)
            sides = [parts[box[:, ax] < mid], parts[box[:, ax] > mid]]
            kids = [dissect(q) for q in sides if len(q)]
            self.nodes.append((np.sort(parts[box[:, ax] == mid]), kids))
            parent.append(-1)
            t = len(self.nodes) - 1
            for ch in kids:
                parent[ch] = t
            return t

        dissect(np.arange(nparts))
        nn = len(self.nodes)
        node_of_part = np.empty(nparts, np.int64)
        for t, (parts, _) in enumerate(self.nodes):
            node_of_part[parts] = t
        # ancestor test by postorder intervals: u is an ancestor-or-self of t
        # iff first[u] <= t <= u (a subtree is a contiguous postorder range)
        first = np.arange(nn)
        for t, (_, kids) in enumerate(self.nodes):
            for ch in kids:
                first[t] = min(first[t], first[ch])
        coo = A0.tocoo()
        tr, tc = node_of_part[np.searchsorted(cptr, coo.row, "right") - 1], \
            node_of_part[np.searchsorted(cptr, coo.col, "right") - 1]
        hi_, lo_ = np.maximum(tr, tc), np.minimum(tr, tc)
        if not np.all(first[hi_] <= lo_):
            raise ValueError("the block coordinates do not give a nested dissection of A_0")
        del coo, tr, tc, hi_, lo_
        # unknowns of each node, in elimination order (parts ascending)
        self.S = [np.concatenate([np.arange(cptr[I], cptr[I + 1]) for I in parts])
                  if len(parts) else np.zeros(0, np.int64) for parts, _ in self.nodes]
        order = np.concatenate(self.S)
        elim = np.empty(self.nc, np.int64)
        elim[order] = np.arange(self.nc)       # elimination position of each unknown
        self.order = order
        # ---- 2. symbolic: boundary sets B_t (ancestors' unknowns), by elimination position
        self.B = []
        for t, (parts, kids) in enumerate(self.nodes):
            S = self.S[t]
            cols = A0.indices[np.concatenate([np.arange(A0.indptr[v], A0.indptr[v + 1]) for v in S])] \
                if len(S) else np.zeros(0, np.int64)
            cand = [cols[elim[cols] > elim[S].max()]] if len(S) else []
            cand += [self.B[ch] for ch in kids]
            Bt = np.unique(np.concatenate(cand)) if cand else np.zeros(0, np.int64)
            if len(S):
                Bt = Bt[elim[Bt] > elim[S].max()]
            self.B.append(Bt[np.argsort(elim[Bt], kind="stable")])
        # ---- 3. numeric factorisation
        sizes = [(len(self.S[t]), len(self.B[t])) for t in range(nn)]
        total = sum(s * s + b * s for s, b in sizes)
        if scratch:
            os.makedirs(scratch, exist_ok=True)
            fn = os.path.join(scratch, f"nd_factor_{os.getpid()}_{id(self)}.bin")
            self._store = np.memmap(fn, np.float64, "w+", shape=(max(total, 1),))
            os.unlink(fn)                      # freed when the mapping goes
        else:
            self._store = np.empty(max(total, 1))
        self.LSS, self.LBS = [], []
        pos = np.full(self.nc, -1, np.int64)
        upd = {}
        off = 0
        for t, (parts, kids) in enumerate(self.nodes):
            S, Bt = self.S[t], self.B[t]
            s, b = len(S), len(Bt)
            idx = np.concatenate([S, Bt])
            pos[idx] = np.arange(s + b)
            F = np.zeros((s + b, s + b))
            AS = A0[S][:, idx].toarray()        # rows S: every column is in S or B_t
            F[:s, :] = AS
            F[s:, :s] = AS[:, s:].T
            del AS
            for ch in kids:                     # extend-add, children in fixed order
                U = upd.pop(ch)
                p = pos[self.B[ch]]
                F[np.ix_(p, p)] += U
                del U
            pos[idx] = -1
            try:
                Lss = np.linalg.cholesky(F[:s, :s])
            except np.linalg.LinAlgError as e:
                raise np.linalg.LinAlgError(f"coarse factor: A_0 not positive definite in front {t}") from e
            Lbs = sla.solve_triangular(Lss, F[s:, :s].T, lower=True).T if b else np.zeros((0, s))
            if b:
                upd[t] = F[s:, s:] - Lbs @ Lbs.T
            del F
            a = self._store[off: off + s * s].reshape(s, s)
            a[...] = Lss
            off += s * s
            c = self._store[off: off + b * s].reshape(b, s)
            c[...] = Lbs
            off += b * s
            self.LSS.append(a)
            self.LBS.append(c)
        self.factor_bytes = 8 * total

    def solve(self, x):
        """x <- A_0^{-1} x (forward then back substitution over the tree)."""
        for t in range(len(self.nodes)):
            S, Bt = self.S[t], self.B[t]
            if len(S) == 0:
                continue
            y = sla.solve_triangular(self.LSS[t], x[S], lower=True)
            x[S] = y
            if len(Bt):
                x[Bt] -= self.LBS[t] @ y
        for t in reversed(range(len(self.nodes))):
            S, Bt = self.S[t], self.B[t]
            if len(S) == 0:
                continue
            rhs = x[S] - (self.LBS[t].T @ x[Bt] if len(Bt) else 0.0)
            x[S] = sla.solve_triangular(self.LSS[t], rhs, lower=True, trans="T")
        return x
