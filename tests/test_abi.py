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
