"""CPU oracle for the DDG-preconditioned CG path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product
(paper_1504_00907_b200/) never imports it and shares no code with it.

The arithmetic lives in oracle.c (plain single-threaded C, fp64, citing
PAPER.md step by step); this module only builds it with gcc and marshals
numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

STOP_RES0, STOP_RES1, STOP_PREC = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (single-threaded, -O2, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                               "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        i64, i32, f64, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        L.or_setup.argtypes = [i64, vp, vp, vp, vp, C.c_int, vp, i32, C.c_int, f64,
                               C.POINTER(vp)]
        L.or_setup.restype = C.c_int
        L.or_setup_coloured.argtypes = [i64, vp, vp, vp, vp, C.c_int, vp, i32, C.c_int, f64, vp,
                                        C.POINTER(vp)]
        L.or_setup_coloured.restype = C.c_int
        L.or_setup_ex.argtypes = [i64, vp, vp, vp, vp, C.c_int, vp, i32, C.c_int, f64, vp,
                                  C.POINTER(vp)]
        L.or_setup_ex.restype = C.c_int
        L.or_set_coarse_solver.argtypes = [vp, vp, vp]
        L.or_set_coarse_solver.restype = None
        L.or_get_Ac_csr.argtypes = [vp, vp, vp, vp]
        L.or_get_Ac_csr.restype = i64
        L.or_setup3.argtypes = [i64, vp, vp, vp, vp, C.c_int, vp, i32, C.c_int, f64, vp, i32,
                                C.POINTER(vp)]
        L.or_setup3.restype = C.c_int
        L.or_child.argtypes = [vp]
        L.or_child.restype = vp
        for name in ("or_apply_precond", "or_forward_sweep", "or_coarse_correct", "or_spmv"):
            getattr(L, name).argtypes = [vp, vp, vp]
            getattr(L, name).restype = C.c_int
        L.or_pcg.argtypes = [vp, vp, f64, C.c_int, C.c_int, vp, C.POINTER(C.c_int), vp,
                             C.POINTER(C.c_int)]
        L.or_pcg.restype = C.c_int
        L.or_pcg_ab.argtypes = [vp, vp, f64, C.c_int, C.c_int, vp, C.POINTER(C.c_int), vp,
                                C.POINTER(C.c_int), vp, vp]
        L.or_pcg_ab.restype = C.c_int
        L.or_info.argtypes = [vp, vp]
        L.or_info.restype = None
        L.or_min_rank_ratio.argtypes = [vp]
        L.or_min_rank_ratio.restype = f64
        L.or_get_colours.argtypes = [vp, vp]
        L.or_get_overlap.argtypes = [vp, i32, vp]
        L.or_get_overlap.restype = i64
        L.or_get_P_dense.argtypes = [vp, vp]
        L.or_get_Ac_dense.argtypes = [vp, vp]
        L.or_get_coarse_offsets.argtypes = [vp, vp]
        L.or_destroy.argtypes = [vp]
        L.or_destroy.restype = None
        L.or_last_error.restype = C.c_char_p
        _lib = L
    return _lib


class _Opts(C.Structure):
    _fields_ = [("colour", C.c_void_p), ("perturb", C.c_int), ("coarse_external", C.c_int)]


_COARSE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.POINTER(C.c_double))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Plain CPU implementation of setup + M r + PCG (see oracle.c)."""

    def __init__(self, n, row_ptr, col, val, F, part, nparts, overlap=1, rank_tol=1e-8,
                 part2=None, nparts2=0, colour=None, coarse="envelope", block_coords=None,
                 perturb=False, nd_leaf=256, scratch=None):
        """part2 (int32[nparts], second-level part of every part) selects the
        three-level method (oracle.c or_setup3).
        coarse="nd" solves A_0 by the nested-dissection multifrontal Cholesky
        of coarse_nd.py (needs block_coords) instead of oracle.c's envelope
        Cholesky.  perturb=True is the floor mode (oracle.h or_opts)."""
        L = lib()
        self._keep = [np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                      np.ascontiguousarray(val, np.float64),
                      np.asfortranarray(F, dtype=np.float64),
                      np.ascontiguousarray(part, np.int32)]
        rp, ci, va, Ff, pa = self._keep
        self.n = int(n)
        self.k = int(Ff.shape[1])
        h = C.c_void_p()
        self._nd = None
        if coarse not in ("envelope", "nd"):
            raise ValueError(coarse)
        if coarse == "nd" or perturb:
            if part2 is not None:
                raise ValueError("coarse='nd' / perturb are two-level options")
            o = _Opts()
            co = None
            if colour is not None:
                co = np.ascontiguousarray(colour, np.int32)
                o.colour = co.ctypes.data
            o.perturb = int(bool(perturb))
            o.coarse_external = int(coarse == "nd")
            st = L.or_setup_ex(self.n, _p(rp), _p(ci), _p(va), _p(Ff), self.k, _p(pa), int(nparts),
                               int(overlap), float(rank_tol), C.byref(o), C.byref(h))
        elif colour is not None:
            co = np.ascontiguousarray(colour, np.int32)
            st = L.or_setup_coloured(self.n, _p(rp), _p(ci), _p(va), _p(Ff), self.k, _p(pa), int(nparts),
                                     int(overlap), float(rank_tol), _p(co), C.byref(h))
        elif part2 is None:
            st = L.or_setup(self.n, _p(rp), _p(ci), _p(va), _p(Ff), self.k, _p(pa), int(nparts),
                            int(overlap), float(rank_tol), C.byref(h))
        else:
            p2 = np.ascontiguousarray(part2, np.int32)
            st = L.or_setup3(self.n, _p(rp), _p(ci), _p(va), _p(Ff), self.k, _p(pa), int(nparts),
                             int(overlap), float(rank_tol), _p(p2), int(nparts2), C.byref(h))
        if st != 0:
            raise OracleError(st, L.or_last_error().decode())
        self._h = h
        self._owner = None
        self._keep = None
        self._read_info()
        if coarse == "nd":
            from .coarse_nd import NDCholesky
            if block_coords is None:
                raise ValueError("coarse='nd' needs block_coords")
            try:
                self._nd = NDCholesky(self.Ac_sparse(), self.coarse_offsets(), block_coords,
                                      leaf=nd_leaf, perturb=perturb, scratch=scratch)
            except np.linalg.LinAlgError as e:
                raise OracleError(5, str(e))
            nd = self._nd

            def _solve(user, nc, x):
                v = np.ctypeslib.as_array(x, shape=(nc,))
                v[:] = nd.solve(v.copy())

            self._cb = _COARSE_FN(_solve)
            L.or_set_coarse_solver(self._h, C.cast(self._cb, C.c_void_p), None)

    def _read_info(self):
        info = np.zeros(10, np.int64)
        lib().or_info(self._h, _p(info))
        (self.n, self.nc, self.nparts, self.ncolours, self.m_min, self.m_max, self.k, self.dropped,
         self.levels, self.nc2) = [int(x) for x in info]

    def child(self):
        """The second-level two-level method on A_0 (three levels only), a
        borrowed view that keeps its parent alive."""
        h = lib().or_child(self._h)
        if not h:
            return None
        o = Oracle.__new__(Oracle)
        o._h = C.c_void_p(h)
        o._owner = self
        o._read_info()
        return o

    @classmethod
    def from_problem(cls, pr, overlap=None, rank_tol=1e-8, part2=None, nparts2=0, colour=None,
                     coarse="envelope", perturb=False, nd_leaf=256, scratch=None):
        return cls(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, pr.part, pr.nparts,
                   pr.overlap if overlap is None else overlap, rank_tol, part2, nparts2, colour,
                   coarse=coarse, block_coords=pr.block_coords, perturb=perturb, nd_leaf=nd_leaf,
                   scratch=scratch)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_owner", None) is None:
            lib().or_destroy(h)
            self._h = None

    def _vec(self, name, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty(self.n)
        st = getattr(lib(), name)(self._h, _p(r), _p(z))
        if st:
            raise OracleError(st, lib().or_last_error().decode())
        return z

    def apply_precond(self, r):
        return self._vec("or_apply_precond", r)

    def forward_sweep(self, r):
        return self._vec("or_forward_sweep", r)

    def coarse_correct(self, r):
        return self._vec("or_coarse_correct", r)

    def spmv(self, x):
        return self._vec("or_spmv", x)

    def pcg(self, f, rtol=1e-8, max_iter=1000, stop_mode=STOP_RES0):
        f = np.ascontiguousarray(f, np.float64)
        u = np.empty(self.n)
        hist = np.zeros(max_iter + 1)
        it = C.c_int(0)
        conv = C.c_int(0)
        st = lib().or_pcg(self._h, _p(f), float(rtol), int(max_iter), int(stop_mode), _p(u),
                          C.byref(it), _p(hist), C.byref(conv))
        if st:
            raise OracleError(st, lib().or_last_error().decode())
        return u, it.value, hist[: it.value + 1].copy(), bool(conv.value)

    def pcg_lanczos(self, f, rtol=1e-8, max_iter=1000, stop_mode=STOP_RES0):
        """pcg plus the CG coefficients: returns (u, iters, hist, converged,
        alphas[iters], betas[iters - 1]) (betas of the directions actually used)."""
        f = np.ascontiguousarray(f, np.float64)
        u = np.empty(self.n)
        hist = np.zeros(max_iter + 1)
        al = np.zeros(max_iter + 1)
        be = np.zeros(max_iter + 1)
        it = C.c_int(0)
        conv = C.c_int(0)
        st = lib().or_pcg_ab(self._h, _p(f), float(rtol), int(max_iter), int(stop_mode), _p(u),
                             C.byref(it), _p(hist), C.byref(conv), _p(al), _p(be))
        if st:
            raise OracleError(st, lib().or_last_error().decode())
        k = it.value
        return u, k, hist[: k + 1].copy(), bool(conv.value), al[:k].copy(), be[: max(k - 1, 0)].copy()

    def colours(self):
        c = np.empty(self.nparts, np.int32)
        lib().or_get_colours(self._h, _p(c))
        return c

    def overlap_set(self, i):
        m = lib().or_get_overlap(self._h, int(i), None)
        idx = np.empty(m, np.int32)
        lib().or_get_overlap(self._h, int(i), _p(idx))
        return idx

    def P_dense(self):
        P = np.zeros((self.nc, self.n))
        lib().or_get_P_dense(self._h, _p(P))
        return P.T.copy()

    def Ac_dense(self):
        A = np.zeros((self.nc, self.nc))
        lib().or_get_Ac_dense(self._h, _p(A))
        return A

    def Ac_sparse(self):
        """A_0 as a full symmetric scipy CSR matrix in coarse order."""
        import scipy.sparse as sp
        nnz = lib().or_get_Ac_csr(self._h, None, None, None)
        rp = np.zeros(self.nc + 1, np.int64)
        ci = np.empty(max(nnz, 1), np.int32)
        va = np.empty(max(nnz, 1))
        lib().or_get_Ac_csr(self._h, _p(rp), _p(ci), _p(va))
        return sp.csr_matrix((va[:nnz], ci[:nnz], rp), shape=(self.nc, self.nc))

    def coarse_offsets(self):
        c = np.empty(self.nparts + 1, np.int32)
        lib().or_get_coarse_offsets(self._h, _p(c))
        return c

    def min_rank_ratio(self):
        return float(lib().or_min_rank_ratio(self._h))


def fractional_iterations(hist, tol_abs):
    """Fractional iteration count: the real k* where the
    linear interpolation of (k, log10 hist[k]) meets log10(tol_abs)."""
    h = np.asarray(hist, float)
    lt = np.log10(tol_abs)
    for k in range(len(h)):
        if h[k] <= tol_abs:
            if k == 0:
                return 0.0
            a, b = np.log10(h[k - 1]), np.log10(h[k])
            return (k - 1) + (a - lt) / (a - b)
    return float("inf")


def lanczos_tridiagonal(alphas, betas):
    """The Lanczos tridiagonal of a (P)CG run from its coefficients (the
    standard CG-Lanczos relation): diagonal 1/a_k + b_{k-1}/a_{k-1}
    (b_{-1}/a_{-1} = 0), off-diagonal sqrt(b_k)/a_k."""
    a = np.asarray(alphas, float)
    b = np.asarray(betas, float)[: max(len(a) - 1, 0)]
    k = len(a)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / a[j] + (b[j - 1] / a[j - 1] if j > 0 else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(b[j]) / a[j]
    return T


def condition_estimate(alphas, betas, tol):
    """kappa = lambda_max / lambda_min of the Lanczos tridiagonal (an estimate
    of cond(M A)) and the classical CG iteration bound
    ln(2/tol) / ln((sqrt(kappa)+1)/(sqrt(kappa)-1)); fewer
    than 2 coefficients: kappa = 1."""
    if len(alphas) < 2:
        return 1.0, 1.0
    ev = np.linalg.eigvalsh(lanczos_tridiagonal(alphas, betas))
    kappa = float(ev[-1] / ev[0])
    sk = np.sqrt(kappa)
    bound = float(np.log(2.0 / tol) / np.log((sk + 1) / (sk - 1))) if kappa > 1 else 1.0
    return kappa, bound
