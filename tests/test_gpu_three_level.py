"""GPU parity of the three-level method against the oracle.

libddg builds the second level as its own two-level context on A_c and runs
it as the coarse step (setup.cpp build_child / coarse_add); the oracle nests
or_setup on A_0 (oracle.c or_setup3).  Same bar as the two-level parity:
solution within 1e-10 relative, iterations +-1, residual history within
1e-8 relative; colours and sizes of both levels bit-exact.
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


CASES = {
    "C1_f2": (lambda: P.poisson2d(64, 8, 1, 1001), 2),
    "poisson3d_24_b4_p1": (lambda: P.poisson3d(24, 4, 1, 1002), 2),
    "poisson3d_24_b4_p2_f3": (lambda: P.poisson3d(24, 4, 2, 1012), 3),
    "lognormal_16_b4": (lambda: P.lognormal3d(16, 4, 1, 1003), 2),
    "biharm_64_b8_p2": (lambda: P.biharmonic2d(64, 8, 2, 1005), 2),
    "elasticity_16_be4": (lambda: P.elasticity3d(16, 4, 1004), 2),
    "poisson2d_ragged": (lambda: P.poisson2d(45, 4, 2, 7), 3),
}


def _pair(name, **kw):
    from paper_1504_00907_b200 import Solver
    mk, f = CASES[name]
    pr = mk()
    p2, n2, bc2 = P.coarse_parts(pr, f, coords=True)
    s = Solver.from_problem(pr, part2=p2, nparts2=n2, block_coords2=bc2, **kw)
    o = oracle.Oracle.from_problem(pr, part2=p2, nparts2=n2)
    return pr, s, o


def _check_solve(pr, s, o, rtol=1e-8):
    u, it, hist, rep = s.solve(pr.f, rtol)
    uo, ito, histo, conv = o.pcg(pr.f, rtol)
    assert bool(rep.converged) == conv and conv
    assert abs(it - ito) <= 1, (it, ito)
    m = min(len(hist), len(histo))
    hr = np.abs(hist[:m] - histo[:m]) / histo[:m]
    assert hr.max() <= H_TOL, hr
    ur = np.linalg.norm(u - uo) / np.linalg.norm(uo)
    assert ur <= U_TOL, ur
    return it


@pytest.mark.parametrize("name", list(CASES))
def test_three_level_pcg_parity(name):
    pr, s, o = _pair(name)
    assert s.info.levels == 3 and o.levels == 3
    assert s.info.n_c == o.nc and s.info.n_c2 == o.nc2
    ch = o.child()
    assert s.info.nparts2 == ch.nparts and s.info.ncolours2 == ch.ncolours
    assert np.array_equal(s.colours(), o.colours())
    _check_solve(pr, s, o)


@pytest.mark.parametrize("name", ["C1_f2", "poisson3d_24_b4_p1", "biharm_64_b8_p2", "elasticity_16_be4"])
def test_three_level_apply_parity(name):
    pr, s, o = _pair(name)
    r = np.random.default_rng(0).standard_normal(pr.n)
    tol = 1e-9 if "biharm" in name else 1e-11
    for g, ref in ((s.coarse_correct(r), o.coarse_correct(r)), (s.apply_precond(r), o.apply_precond(r))):
        assert np.linalg.norm(g - ref) <= tol * np.linalg.norm(ref)


@pytest.mark.parametrize("variant", [1, 2])
def test_three_level_second_level_coarse_variants(variant):
    """coarse_variant selects the last level's solve: dense packed inverse or
    the sparse dataflow solve on A_1."""
    pr, s, o = _pair("poisson3d_24_b4_p1", coarse_variant=variant)
    assert s.info.coarse_variant == 3 and s.info.coarse_variant2 == variant
    _check_solve(pr, s, o)


@pytest.mark.parametrize("env", [{"DDG_SYMV": "classic"}, {"DDG_RING_MIN_MB": "0"}])
def test_three_level_kernel_paths(env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    pr, s, o = _pair("lognormal_16_b4")
    _check_solve(pr, s, o)


def test_three_level_symmetric_and_weaker_than_two_level():
    """M_3 is symmetric, SPD, and M_3 <= M_2 (the inexact coarse level only
    removes A-norm reduction; tests/test_oracle_three_level.py derives it)."""
    from paper_1504_00907_b200 import Solver
    pr, s3, _ = _pair("C1_f2")
    s2 = Solver.from_problem(pr)
    rs = np.random.default_rng(4)
    for _ in range(3):
        x, y = rs.standard_normal(pr.n), rs.standard_normal(pr.n)
        Mx, My = s3.apply_precond(x), s3.apply_precond(y)
        assert abs(x @ My - y @ Mx) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(My)
        assert 0 < x @ Mx <= (x @ s2.apply_precond(x)) * (1 + 1e-12)


def test_three_level_bitwise_repeatable_and_launches():
    from paper_1504_00907_b200 import Solver
    pr, s3, _ = _pair("poisson3d_24_b4_p1")
    u1, it1, h1, _ = s3.solve(pr.f)
    u2, it2, h2, _ = s3.solve(pr.f)
    assert it1 == it2 and np.array_equal(u1, u2) and np.array_equal(h1, h2)
    s2 = Solver.from_problem(pr)
    r = np.ones(pr.n)
    s2.launch_count(reset=True)
    s3.launch_count(reset=True)
    s2.apply_precond(r)
    s3.apply_precond(r)
    assert s3.launch_count() > s2.launch_count() > 0


def test_three_level_errors():
    from paper_1504_00907_b200 import Solver
    from paper_1504_00907_b200.ddg import DDGError
    pr = P.poisson2d(32, 8, 1, 3)
    with pytest.raises(DDGError, match="too small"):
        Solver.from_problem(pr, part2=np.zeros(pr.nparts, np.int32), nparts2=1)
    with pytest.raises(DDGError):
        Solver.from_problem(pr, part2=np.full(pr.nparts, 5, np.int32), nparts2=2)
    with pytest.raises(DDGError, match="empty"):
        Solver.from_problem(pr, part2=np.zeros(pr.nparts, np.int32), nparts2=2)


def test_three_level_full_c3():
    """BASELINE C3 at full size with the three-level method as bench.py times
    it (--levels 3 --factor 2): convergence, the true residual, symmetry and
    positivity of M_3 and M_3 <= M_2 on a random vector (derived in
    tests/test_oracle_three_level.py)."""
    import scipy.sparse as sp
    from paper_1504_00907_b200 import Solver
    pr = P.make("C3")
    p2, n2, bc2 = P.coarse_parts(pr, 2, coords=True)
    s3 = Solver.from_problem(pr, part2=p2, nparts2=n2, block_coords2=bc2)
    assert s3.info.levels == 3 and s3.info.nparts2 == n2
    u, it, hist, rep = s3.solve(pr.f, 1e-8)
    assert rep.converged and it <= 12, it
    A = sp.csr_matrix((pr.val, pr.col, pr.row_ptr), shape=(pr.n, pr.n))
    assert np.linalg.norm(pr.f - A @ u) <= 1e-7 * np.linalg.norm(pr.f)
    assert abs(rep.true_res - np.linalg.norm(pr.f - A @ u)) <= 1e-3 * rep.true_res
    rs = np.random.default_rng(8)
    x, y = rs.standard_normal(pr.n), rs.standard_normal(pr.n)
    Mx, My = s3.apply_precond(x), s3.apply_precond(y)
    assert abs(x @ My - y @ Mx) <= 1e-11 * np.linalg.norm(x) * np.linalg.norm(My)
    assert x @ Mx > 0
    s3.close()
    s2 = Solver.from_problem(pr)
    assert x @ Mx <= (x @ s2.apply_precond(x)) * (1 + 1e-10)
    s2.close()


@pytest.mark.parametrize("name", ["C1_f2", "lognormal_16_b4", "poisson3d_24_b4_p1"])
def test_three_level_comm_path_single_rank(name):
    """The distributed three-level path (SURVEY.md §8(f) f2 by the paper's own
    route: the second level is a two-level method distributed over the same
    ranks, only the small A_1 factor replicated) at one NCCL rank: split
    reductions, halo plans and the y_c assembly run, and match the oracle."""
    from paper_1504_00907_b200 import Solver, ddg
    mk, f = CASES[name]
    pr = mk()
    p2, n2, bc2 = P.coarse_parts(pr, f, coords=True)
    comm = ddg.Comm(0, 1, ddg.unique_id(), 0)
    s = Solver.from_problem(pr, comm=comm, part2=p2, nparts2=n2, block_coords2=bc2)
    o = oracle.Oracle.from_problem(pr, part2=p2, nparts2=n2)
    assert s.info.levels == 3
    _check_solve(pr, s, o)
    s.close()
    comm.close()
