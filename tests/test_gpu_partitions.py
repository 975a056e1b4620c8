"""GPU parity on irregular (non-box) partitions and on the nested-dissection
code paths the small parity cases do not reach by default.

The paper partitions with SCOTCH or inertial bisection (PAPER.md:246-248,
807-811); `ddg_gen.problems.grown_partition` gives connected parts of varying
size whose boundaries follow no grid line, and no block coordinates, so the
library's coarse nested dissection takes its graph (BFS level-structure)
bisection.  Bar: the north star's (u 1e-10, iterations +-1, history 1e-8).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P

pytestmark = pytest.mark.gpu

U_TOL, H_TOL = 1e-10, 1e-8


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_00907_b200 import build
    build.build()


GROWN = {
    "poisson2d_48_grown40": lambda: P.grown_partition(P.poisson2d(48, 8, 2, 31), 40, 1),
    "lognormal_16_grown64": lambda: P.grown_partition(P.lognormal3d(16, 4, 1, 32), 64, 2),
    "poisson3d_20_grown12_p2": lambda: P.grown_partition(P.poisson3d(20, 8, 2, 33), 12, 3),
    "biharm_64_grown20_p3": lambda: P.grown_partition(P.biharmonic2d(64, 16, 3, 34), 20, 4),
    "elasticity_8_grown10": lambda: P.grown_partition(P.elasticity3d(8, 4, 35), 10, 5),
}


def _check(pr, s, rtol=1e-8, coarse_tol=None):
    o = oracle.Oracle.from_problem(pr)
    assert np.array_equal(s.colours(), o.colours())
    sizes = np.array([len(o.overlap_set(i)) for i in range(pr.nparts)])
    assert np.array_equal(s.subdomain_sizes(), sizes)
    if coarse_tol is not None:
        r = np.random.default_rng(7).standard_normal(pr.n)
        zc, zo = s.coarse_correct(r), o.coarse_correct(r)
        assert np.linalg.norm(zc - zo) <= coarse_tol * np.linalg.norm(zo)
    u, it, hist, rep = s.solve(pr.f, rtol)
    uo, ito, histo, conv = o.pcg(pr.f, rtol)
    assert rep.converged and conv and abs(it - ito) <= 1, (it, ito)
    m = min(len(hist), len(histo))
    assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
    assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
    return it


@pytest.mark.parametrize("name", list(GROWN))
def test_grown_partition_parity(name):
    from paper_1504_00907_b200 import Solver
    pr = GROWN[name]()
    sz = np.bincount(pr.part)
    assert sz.min() < sz.max()                       # genuinely irregular
    _check(pr, Solver.from_problem(pr))


@pytest.mark.parametrize("name", ["lognormal_16_grown64", "biharm_64_grown20_p3", "elasticity_8_grown10"])
def test_grown_partition_sparse_coarse(name):
    """coarse_variant=2 without block coordinates: graph nested dissection"""
    from paper_1504_00907_b200 import Solver
    pr = GROWN[name]()
    s = Solver.from_problem(pr, coarse_variant=2)
    assert s.info.coarse_variant == 2
    _check(pr, s, coarse_tol=1e-9 if "biharm" in name else 1e-12)


PATHS = {
    "ring_everywhere": {"DDG_SMALL_FUSED": "0", "DDG_RING_MIN_MB": "0"},
    "whole_full_tiles": {"DDG_SMALL_FUSED": "0", "DDG_RING_MIN_MB": "0", "DDG_COMPACT": "0"},
    "ring2_everywhere": {"DDG_SMALL_FUSED": "0", "DDG_RING_MIN_MB": "0", "DDG_RING_V2": "1", "DDG_RING_WHOLE": "0"},
    "classic": {"DDG_SMALL_FUSED": "0", "DDG_SYMV": "classic"},
}


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("name", ["lognormal_16_grown64", "biharm_64_grown20_p3", "poisson3d_20_grown12_p2"])
def test_grown_partition_kernel_paths(name, path, monkeypatch):
    from paper_1504_00907_b200 import Solver
    for k, v in PATHS[path].items():
        monkeypatch.setenv(k, v)
    pr = GROWN[name]()
    _check(pr, Solver.from_problem(pr))


# nested-dissection parameters: C3's full size (n_c > 262,144) uses 256-unknown
# leaves; smaller problems 1024.  Force the small leaves (and merged top levels,
# tiny leaves, narrow front items) on problems the oracle checks in seconds.
ND = {
    "leaf256": {"DDG_ND_LEAF": "256"},
    "leaf64": {"DDG_ND_LEAF": "64"},
    "leaf16_merge3": {"DDG_ND_LEAF": "16", "DDG_ND_MERGE": "3"},
    "leaf256_frontbt2": {"DDG_ND_LEAF": "256", "DDG_FRONT_BT": "2"},
    "leaf256_levels": {"DDG_ND_LEAF": "256", "DDG_COARSE_DATAFLOW": "0"},
}


@pytest.mark.parametrize("nd", list(ND))
@pytest.mark.parametrize("name", ["lognormal_32_b4", "biharm_128_b16_p3", "lognormal_16_grown64"])
def test_nested_dissection_paths(name, nd, monkeypatch):
    from paper_1504_00907_b200 import Solver
    for k, v in ND[nd].items():
        monkeypatch.setenv(k, v)
    mk = {"lognormal_32_b4": lambda: P.lognormal3d(32, 4, 1, 23),
          "biharm_128_b16_p3": lambda: P.biharmonic2d(128, 16, 3, 24)}.get(name) or GROWN[name]
    pr = mk()
    s = Solver.from_problem(pr, coarse_variant=2)
    assert s.info.coarse_variant == 2
    _check(pr, s, coarse_tol=1e-9 if "biharm" in name else 1e-12)
