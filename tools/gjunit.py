"""Blocked Gauss-Jordan (setup) on random SPD matrices: symmetric vs full vs numpy."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1504_00907_b200 import ddg  # noqa: E402

L = ddg.load()
L.ddg_debug_gj.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int]


def to_tiles(A, nT):
    T = np.zeros((nT, nT, 32, 32))
    for I in range(nT):
        for J in range(nT):
            T[J, I] = A[I * 32:(I + 1) * 32, J * 32:(J + 1) * 32].T   # tile (I,J) at J*nT+I, column-major inside
    return np.ascontiguousarray(T.reshape(-1))


def from_tiles(v, nT):
    T = v.reshape(nT, nT, 32, 32)
    A = np.zeros((nT * 32, nT * 32))
    for I in range(nT):
        for J in range(nT):
            A[I * 32:(I + 1) * 32, J * 32:(J + 1) * 32] = T[J, I].T
    return A


rng = np.random.default_rng(0)
sizes = [int(x) for x in sys.argv[1:]] or [97, 161]
mats = []
for nT in sizes:
    n = nT * 32
    X = rng.standard_normal((n, n)) / np.sqrt(n)
    mats.append(X @ X.T + 0.5 * np.eye(n))
for sym in (0, 1):
    v = np.concatenate([to_tiles(A, nT) for A, nT in zip(mats, sizes)])
    nts = np.array(sizes, np.int32)
    st = L.ddg_debug_gj(len(sizes), nts.ctypes.data, v.ctypes.data, sym)
    pos = 0
    errs = []
    for A, nT in zip(mats, sizes):
        ne = nT * nT * 1024
        M = from_tiles(v[pos:pos + ne], nT)
        pos += ne
        S = np.tril(M) + np.tril(M, -1).T
        ref = np.linalg.inv(A)
        errs.append(float(np.abs(np.abs(S) - np.abs(ref)).max() / np.abs(ref).max()))
    print("sym", sym, "status", st, "errors", ["%.1e" % e for e in errs], flush=True)
