"""CPU checks of the C boundary: libddg builds, loads and exports every symbol
include/ddg.h declares; without a GPU it fails loudly (no CPU fallback)."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1504_00907_b200 import build
    build.build()
    from paper_1504_00907_b200 import ddg
    return ddg.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ddg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ddg_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 14
    out = subprocess.check_output(["nm", "-D", "--defined-only",
                                   os.path.join(ROOT, "paper_1504_00907_b200", "libddg.so")]).decode()
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    for s in syms:
        assert s in exported, s
        assert hasattr(lib, s)
    from paper_1504_00907_b200 import ddg
    assert sorted(ddg.EXPORTS) == syms


def test_status_strings_and_defaults(lib):
    from paper_1504_00907_b200 import ddg
    assert lib.ddg_status_string(0) == b"ok"
    assert lib.ddg_status_string(5) == b"matrix not positive definite"
    o = ddg.default_opts()
    assert o.overlap == 1 and o.rank_tol == 1e-8 and o.max_iter == 1000 and o.use_graphs == 1


def test_argument_errors_before_device(lib):
    """Argument validation happens on the host before any device work."""
    from paper_1504_00907_b200 import ddg
    from ddg_gen import problems as P
    pr = P.poisson2d(8, 4, 1)
    with pytest.raises(ddg.DDGError) as e:
        ddg.Solver(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, pr.part, 0)
    assert e.value.code == 1
    bad = pr.part.copy(); bad[3] = 99
    with pytest.raises(ddg.DDGError) as e:
        ddg.Solver(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, bad, pr.nparts)
    assert e.value.code == 3
    with pytest.raises(ddg.DDGError) as e:     # local_variant outside DDG_LOCAL_*
        ddg.Solver(pr.n, pr.row_ptr, pr.col, pr.val, pr.F, pr.part, pr.nparts, local_variant=5)
    assert e.value.code == 1
    col = pr.col.copy(); col[1], col[2] = col[2], col[1]
    with pytest.raises(ddg.DDGError) as e:
        ddg.Solver(pr.n, pr.row_ptr, col, pr.val, pr.F, pr.part, pr.nparts)
    assert e.value.code == 2


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1504_00907_b200 import ddg
    from ddg_gen import problems as P
    pr = P.poisson2d(8, 4, 1)
    with pytest.raises(ddg.DDGError) as e:
        ddg.Solver.from_problem(pr)
    assert e.value.code == 8


def test_product_never_imports_oracle():
    """The product path shares no code with the oracle and never loads it."""
    pkg = os.path.join(ROOT, "paper_1504_00907_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "liboracle" not in txt, f


@pytest.mark.parametrize("n,G,seed", [(0, 148, 0), (5, 148, 1), (148, 148, 2), (4096, 148, 3), (32768, 148, 4),
                                      (1000, 7, 5)])
def test_ring_partition_properties(lib, n, G, seed):
    """Host logic of the persistent SYMV: the byte-balanced contiguous partition
    of a launch's work items over the CTAs (setup.cpp balanced_partition).  It
    covers every item exactly once in order, and no part exceeds its share of
    the total by more than one item's weight."""
    import ctypes as C
    rs = np.random.default_rng(seed)
    w = rs.uniform(0.5, 1.5, n) * rs.choice([1.0, 4.0], n)
    out = np.zeros(G + 1, np.int32)
    f = lib.ddg_debug_partition
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    assert f(w.ctypes.data, n, G, out.ctypes.data) == 0
    assert out[0] == 0 and out[-1] == n and np.all(np.diff(out) >= 0)
    if n:
        loads = np.array([w[out[g]:out[g + 1]].sum() for g in range(G)])
        assert loads.sum() == pytest.approx(w.sum())
        assert loads.max() <= w.sum() / G + 2 * w.max() + 1e-9
