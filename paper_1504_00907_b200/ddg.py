"""Thin ctypes binding of libddg (include/ddg.h) — argument marshalling only.

Every step of setup and of the PCG hot path runs inside libddg.so (host C++
setup + sm_100a kernels).  There is no CPU fallback: if the library is missing
or no CUDA device is visible, every call raises DDGError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libddg.so")
_lib = None

DDG_OK = 0
STATUS = {0: "DDG_OK", 1: "DDG_E_ARG", 2: "DDG_E_DIM", 3: "DDG_E_PART", 4: "DDG_E_ZERO_BLOCK",
          5: "DDG_E_NOT_SPD", 6: "DDG_E_COLOURING", 7: "DDG_E_BREAKDOWN", 8: "DDG_E_CUDA",
          9: "DDG_E_NCCL", 10: "DDG_E_OOM"}
STOP_RES0, STOP_RES1, STOP_PREC = 0, 1, 2

# symbols declared in include/ddg.h (checked by tests/test_abi.py)
EXPORTS = ["ddg_default_opts", "ddg_setup", "ddg_pcg_solve", "ddg_pcg_solve_device",
           "ddg_apply_precond", "ddg_coarse_correct", "ddg_spmv", "ddg_get_info",
           "ddg_get_colours", "ddg_get_subdomain_sizes", "ddg_launch_count", "ddg_destroy",
           "ddg_status_string", "ddg_last_error", "ddg_set_profiling", "ddg_get_kernel_stats",
           "ddg_get_unique_id", "ddg_comm_init", "ddg_comm_destroy", "ddg_plan_create", "ddg_get_lanczos",
           "ddg_plan_query", "ddg_plan_destroy", "ddg_loop_group_create", "ddg_loop_group_destroy",
           "ddg_comm_init_loopback"]

PLAN = dict(OWNED_ROWS=0, OWNED_SUBS=1, P_SEND=2, P_RECV=3, R_SEND=4, R_RECV=5, Z_SEND=6, Z_RECV=7,
            PROLONG_PARTS=8, COLOURS=9, PART_RANK=10, OVERLAP=11)


class ddg_stencil(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dims", C.c_int32 * 3), ("npts", C.c_int32),
                ("offsets", C.c_void_p), ("coef", C.c_void_p)]


STENCIL_KIND = {"none": 0, "const": 1, "face7": 2, "node27": 3}


class ddg_opts(C.Structure):
    _fields_ = [("overlap", C.c_int), ("rank_tol", C.c_double), ("stop_mode", C.c_int),
                ("max_iter", C.c_int), ("device", C.c_int), ("stream", C.c_void_p),
                ("use_graphs", C.c_int), ("verbose", C.c_int), ("coarse_variant", C.c_int),
                ("block_ndim", C.c_int), ("fuse_gather", C.c_int), ("comm", C.c_void_p),
                ("small_kernel", C.c_int), ("block_coords", C.c_void_p),
                ("stencil", C.POINTER(ddg_stencil)), ("part2", C.c_void_p),
                ("nparts2", C.c_int32), ("block_coords2", C.c_void_p), ("colour", C.c_void_p),
                ("local_variant", C.c_int)]


class ddg_report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iters", C.c_int), ("res0", C.c_double),
                ("res_final", C.c_double), ("t_setup", C.c_double), ("t_solve", C.c_double),
                ("frac_iters", C.c_double), ("cond_est", C.c_double), ("iter_bound", C.c_double),
                ("true_res", C.c_double), ("bytes_per_iter_model", C.c_double)]


class ddg_info(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_c", C.c_int64), ("nparts", C.c_int32),
                ("ncolours", C.c_int32), ("m_min", C.c_int32), ("m_max", C.c_int32),
                ("k", C.c_int32), ("dropped", C.c_int32), ("min_rank_ratio", C.c_double),
                ("local_factor_bytes", C.c_int64), ("coarse_factor_bytes", C.c_int64),
                ("coarse_variant", C.c_int32), ("levels", C.c_int32),
                ("coarse_solve_bytes", C.c_int64), ("n_c2", C.c_int64), ("nparts2", C.c_int32),
                ("ncolours2", C.c_int32), ("coarse_variant2", C.c_int32), ("pad2", C.c_int32)]


class ddg_kstats(C.Structure):
    _fields_ = [("symv_launches", C.c_int64), ("symv_ms", C.c_double),
                ("symv_alg_bytes", C.c_double), ("gather_ms", C.c_double),
                ("reduce_ms", C.c_double), ("coarse_ms", C.c_double), ("vec_ms", C.c_double),
                ("launches", C.c_int64)]


class DDGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def load(path: str = LIB_PATH):
    """Load libddg.so (build it first with paper_1504_00907_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DDGError(8, f"{path} not built (run __graft_entry__.build()); no CPU fallback")
    L = C.CDLL(path)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    L.ddg_default_opts.argtypes = [C.POINTER(ddg_opts)]
    L.ddg_default_opts.restype = None
    L.ddg_setup.argtypes = [i64, vp, vp, vp, vp, C.c_int, vp, i32, C.POINTER(ddg_opts),
                            C.POINTER(vp)]
    L.ddg_setup.restype = C.c_int
    for name in ("ddg_pcg_solve", "ddg_pcg_solve_device"):
        f = getattr(L, name)
        f.argtypes = [vp, vp, dbl, C.c_int, vp, C.POINTER(C.c_int), vp, C.c_int,
                      C.POINTER(ddg_report)]
        f.restype = C.c_int
    for name in ("ddg_apply_precond", "ddg_coarse_correct", "ddg_spmv"):
        getattr(L, name).argtypes = [vp, vp, vp]
        getattr(L, name).restype = C.c_int
    L.ddg_get_info.argtypes = [vp, C.POINTER(ddg_info)]
    L.ddg_get_info.restype = C.c_int
    L.ddg_get_colours.argtypes = [vp, vp]
    L.ddg_get_lanczos.argtypes = [vp, vp, vp, C.c_int]
    L.ddg_get_lanczos.restype = C.c_int
    L.ddg_get_subdomain_sizes.argtypes = [vp, vp]
    L.ddg_launch_count.argtypes = [vp, C.c_int]
    L.ddg_launch_count.restype = i64
    L.ddg_destroy.argtypes = [vp]
    L.ddg_destroy.restype = None
    L.ddg_set_profiling.argtypes = [vp, C.c_int]
    L.ddg_set_profiling.restype = C.c_int
    L.ddg_get_kernel_stats.argtypes = [vp, C.POINTER(ddg_kstats)]
    L.ddg_get_kernel_stats.restype = C.c_int
    L.ddg_get_unique_id.argtypes = [vp]
    L.ddg_get_unique_id.restype = C.c_int
    L.ddg_comm_init.argtypes = [C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]
    L.ddg_comm_init.restype = C.c_int
    L.ddg_loop_group_create.argtypes = [C.c_int, C.c_int, C.POINTER(vp)]
    L.ddg_loop_group_create.restype = C.c_int
    L.ddg_loop_group_destroy.argtypes = [vp]
    L.ddg_loop_group_destroy.restype = None
    L.ddg_comm_init_loopback.argtypes = [vp, C.c_int, C.POINTER(vp)]
    L.ddg_comm_init_loopback.restype = C.c_int
    L.ddg_comm_destroy.argtypes = [vp]
    L.ddg_comm_destroy.restype = None
    L.ddg_plan_create.argtypes = [i64, vp, vp, vp, i32, C.c_int, vp, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(vp)]
    L.ddg_plan_create.restype = C.c_int
    L.ddg_plan_query.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, i64]
    L.ddg_plan_query.restype = i64
    L.ddg_plan_destroy.argtypes = [vp]
    L.ddg_plan_destroy.restype = None
    L.ddg_status_string.argtypes = [C.c_int]
    L.ddg_status_string.restype = C.c_char_p
    L.ddg_last_error.restype = C.c_char_p
    _lib = L
    return L


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _check(st):
    if st != DDG_OK:
        raise DDGError(st, load().ddg_last_error().decode())


def default_opts() -> ddg_opts:
    o = ddg_opts()
    load().ddg_default_opts(C.byref(o))
    return o


class Solver:
    """ddg_setup(A, F, partition, overlap) -> ddg_pcg_solve(f, rtol) (include/ddg.h)."""

    def __init__(self, n, row_ptr, col, val, F, part, nparts, overlap=1, rank_tol=1e-8,
                 stop_mode=STOP_RES0, max_iter=1000, device=0, stream=None, use_graphs=True,
                 verbose=False, coarse_variant=0, block_coords=None, comm=None, fuse_gather=None,
                 small_kernel=None, stencil=None, part2=None, nparts2=0, block_coords2=None, colour=None,
                 local_variant=0):
        """part2 (int32[nparts]: second-level part of every part) selects the
        three-level method (include/ddg.h ddg_opts.part2)."""
        L = load()
        o = default_opts()
        o.overlap, o.rank_tol, o.stop_mode, o.max_iter = overlap, rank_tol, stop_mode, max_iter
        o.device = device
        o.stream = stream
        o.use_graphs = 1 if use_graphs else 0
        o.verbose = 1 if verbose else 0
        o.coarse_variant = int(coarse_variant)
        o.local_variant = int(local_variant)
        if fuse_gather is not None:
            o.fuse_gather = int(fuse_gather)
        if small_kernel is not None:
            o.small_kernel = int(small_kernel)
        o.comm = comm.handle if comm is not None else None
        self._comm = comm
        bc = None
        if block_coords is not None:
            bc = np.ascontiguousarray(block_coords, np.int32)
            o.block_ndim = int(bc.shape[1])
            o.block_coords = bc.ctypes.data
        keep = []
        if colour is not None:
            co = np.ascontiguousarray(colour, np.int32)
            keep.append(co)
            o.colour = co.ctypes.data
        if part2 is not None:
            p2 = np.ascontiguousarray(part2, np.int32)
            keep.append(p2)
            o.part2 = p2.ctypes.data
            o.nparts2 = int(nparts2)
            if block_coords2 is not None:
                bc2 = np.ascontiguousarray(block_coords2, np.int32)
                keep.append(bc2)
                o.block_coords2 = bc2.ctypes.data
        if stencil is not None:
            # {"kind": "const", "dims": (nx, ny, nz), "offsets": [(dx, dy, dz), ...], "coef": [...]}
            # {"kind": "face7", "dims": (nx, ny, nz), "coef": float64[4 n] (diag|cx|cy|cz)}
            # {"kind": "node27", "dims": (nx, ny, nz) nodes, "dof": unknowns per node}
            st = ddg_stencil()
            st.kind = STENCIL_KIND[stencil["kind"]]
            d = list(stencil["dims"]) + [1] * (3 - len(stencil["dims"]))
            st.dims = (C.c_int32 * 3)(*d)
            if stencil["kind"] == "node27":        # values read from the CSR by the library
                st.npts = int(stencil["dof"])
            else:
                cf = np.ascontiguousarray(stencil["coef"], np.float64)
                keep.append(cf)
                st.coef = cf.ctypes.data
            if stencil["kind"] == "const":
                offs = np.zeros((len(stencil["offsets"]), 3), np.int32)
                for i, off in enumerate(stencil["offsets"]):
                    offs[i, :len(off)] = off
                keep.append(offs)
                st.npts = offs.shape[0]
                st.offsets = offs.ctypes.data
            keep.append(st)
            o.stencil = C.pointer(st)
        rp = np.ascontiguousarray(row_ptr, np.int64)
        ci = np.ascontiguousarray(col, np.int32)
        va = np.ascontiguousarray(val, np.float64)
        Ff = np.asfortranarray(F, dtype=np.float64)
        pa = np.ascontiguousarray(part, np.int32)
        self.n = int(n)
        h = C.c_void_p()
        st = L.ddg_setup(self.n, _p(rp), _p(ci), _p(va), _p(Ff), int(Ff.shape[1]), _p(pa),
                         int(nparts), C.byref(o), C.byref(h))
        _check(st)
        self._h = h
        self.max_iter = max_iter
        self.info = ddg_info()
        _check(L.ddg_get_info(self._h, C.byref(self.info)))

    @classmethod
    def from_problem(cls, pr, **kw):
        kw.setdefault("overlap", pr.overlap)
        kw.setdefault("block_coords", pr.block_coords)
        kw.setdefault("stencil", getattr(pr, "stencil", None))
        return cls(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, pr.part, pr.nparts, **kw)

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            load().ddg_destroy(h)
            self._h = None

    __del__ = close

    def solve(self, f, rtol=1e-8, max_iter=None):
        """Host buffers in, host buffers out (end-to-end path)."""
        max_iter = self.max_iter if max_iter is None else max_iter
        f = np.ascontiguousarray(f, np.float64)
        u = np.empty(self.n)
        hist = np.zeros(max_iter + 1)
        it = C.c_int(0)
        rep = ddg_report()
        _check(load().ddg_pcg_solve(self._h, _p(f), float(rtol), int(max_iter), _p(u),
                                    C.byref(it), _p(hist), len(hist), C.byref(rep)))
        return u, it.value, hist[: it.value + 1].copy(), rep

    def solve_device(self, f_ptr, u_ptr, rtol=1e-8, max_iter=None):
        """f and u are device pointers (e.g. torch tensor data_ptr())."""
        max_iter = self.max_iter if max_iter is None else max_iter
        hist = np.zeros(max_iter + 1)
        it = C.c_int(0)
        rep = ddg_report()
        _check(load().ddg_pcg_solve_device(self._h, C.c_void_p(f_ptr), float(rtol), int(max_iter),
                                           C.c_void_p(u_ptr), C.byref(it), _p(hist), len(hist),
                                           C.byref(rep)))
        return it.value, hist[: it.value + 1].copy(), rep

    def solve_host_ptr(self, f_ptr, u_ptr, rtol=1e-8, max_iter=None):
        """f and u are (pinned) HOST pointers; the H2D/D2H copies happen inside."""
        max_iter = self.max_iter if max_iter is None else max_iter
        hist = np.zeros(max_iter + 1)
        it = C.c_int(0)
        rep = ddg_report()
        _check(load().ddg_pcg_solve(self._h, C.c_void_p(f_ptr), float(rtol), int(max_iter),
                                    C.c_void_p(u_ptr), C.byref(it), _p(hist), len(hist),
                                    C.byref(rep)))
        return it.value, hist[: it.value + 1].copy(), rep

    def _vec(self, name, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.n)
        _check(getattr(load(), name)(self._h, _p(x), _p(y)))
        return y

    def apply_precond(self, r):
        return self._vec("ddg_apply_precond", r)

    def coarse_correct(self, r):
        return self._vec("ddg_coarse_correct", r)

    def spmv(self, x):
        return self._vec("ddg_spmv", x)

    def lanczos(self):
        """(alphas[iters], betas[iters - 1]) of the last solve (ddg_get_lanczos)."""
        k = load().ddg_get_lanczos(self._h, None, None, 0)
        if k < 0:
            _check(-k)
        a = np.zeros(max(k, 1))
        b = np.zeros(max(k, 1))
        load().ddg_get_lanczos(self._h, _p(a), _p(b), k)
        return a[:k].copy(), b[: max(k - 1, 0)].copy()

    def colours(self):
        c = np.empty(self.info.nparts, np.int32)
        _check(load().ddg_get_colours(self._h, _p(c)))
        return c

    def subdomain_sizes(self):
        m = np.empty(self.info.nparts, np.int32)
        _check(load().ddg_get_subdomain_sizes(self._h, _p(m)))
        return m

    def launch_count(self, reset=False):
        return int(load().ddg_launch_count(self._h, 1 if reset else 0))

    def set_profiling(self, on=True):
        _check(load().ddg_set_profiling(self._h, 1 if on else 0))

    def kernel_stats(self) -> ddg_kstats:
        st = ddg_kstats()
        _check(load().ddg_get_kernel_stats(self._h, C.byref(st)))
        return st


def unique_id() -> bytes:
    """128-byte NCCL unique id (create on rank 0, broadcast, pass to Comm)."""
    buf = C.create_string_buffer(128)
    _check(load().ddg_get_unique_id(buf))
    return buf.raw


class Comm:
    """ddg_comm_init: one NCCL communicator per rank / GPU (include/ddg.h)."""

    def __init__(self, rank, nranks, uid: bytes, device=0):
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        _check(load().ddg_comm_init(int(rank), int(nranks), buf, int(device), C.byref(h)))
        self.handle = h
        self.rank, self.nranks = rank, nranks

    def close(self):
        if getattr(self, "handle", None):
            load().ddg_comm_destroy(self.handle)
            self.handle = None


class LoopGroup:
    """ddg_loop_group_create: nranks virtual ranks on one device (include/ddg.h).
    comm(r) is rank r's communicator; drive each rank from its own thread."""

    def __init__(self, nranks, device=0):
        h = C.c_void_p()
        _check(load().ddg_loop_group_create(int(nranks), int(device), C.byref(h)))
        self.handle = h
        self.nranks = nranks
        self._comms = []

    def comm(self, rank):
        h = C.c_void_p()
        _check(load().ddg_comm_init_loopback(self.handle, int(rank), C.byref(h)))
        c = Comm.__new__(Comm)
        c.handle, c.rank, c.nranks = h, rank, self.nranks
        self._comms.append(c)
        return c

    def close(self):
        if getattr(self, "handle", None):
            for c in self._comms:
                c.close()
            load().ddg_loop_group_destroy(self.handle)
            self.handle = None


class Plan:
    """Host-only multi-GPU decomposition plan (ddg_plan_create); no device needed."""

    def __init__(self, pr_or_n, row_ptr=None, col=None, part=None, nparts=None, overlap=1,
                 block_coords=None, rank=0, nranks=1):
        if row_ptr is None:
            pr = pr_or_n
            n, row_ptr, col, part, nparts = pr.n, pr.row_ptr, pr.col, pr.part, pr.nparts
            overlap = pr.overlap
            if block_coords is None:
                block_coords = pr.block_coords
        else:
            n = pr_or_n
        self._keep = [np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col, np.int32),
                      np.ascontiguousarray(part, np.int32)]
        bc = None if block_coords is None else np.ascontiguousarray(block_coords, np.int32)
        self._keep.append(bc)
        h = C.c_void_p()
        _check(load().ddg_plan_create(int(n), _p(self._keep[0]), _p(self._keep[1]), _p(self._keep[2]),
                                      int(nparts), int(overlap), None if bc is None else _p(bc),
                                      0 if bc is None else int(bc.shape[1]), int(rank), int(nranks),
                                      C.byref(h)))
        self._h = h
        self.rank, self.nranks, self.nparts = rank, nranks, int(nparts)
        self.colours = self.query("COLOURS")
        self.ncolours = int(self.colours.max()) + 1

    def query(self, what, colour=0, peer=0):
        L = load()
        code = PLAN[what]
        cnt = L.ddg_plan_query(self._h, code, int(colour), int(peer), None, 0)
        if cnt < 0:
            raise DDGError(1, f"bad plan query {what}")
        out = np.empty(cnt, np.int32)
        if cnt:
            L.ddg_plan_query(self._h, code, int(colour), int(peer), _p(out), cnt)
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            load().ddg_plan_destroy(self._h)
            self._h = None
