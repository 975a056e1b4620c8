"""GPU parity of local_variant = DDG_LOCAL_CHOLESKY (include/ddg.h; chol.cu):
the exact local solves as forward and back substitutions
against per-subdomain Cholesky factors, the kernel the north star names,
instead of the default explicit inverse.

Bar (BASELINE.json north_star), against the CPU oracle (which itself solves
with unblocked Cholesky factors): u within 1e-10 relative, iterations +-1,
history within 1e-8 relative.  A single application of M agrees with the
oracle and with the explicit-inverse variant to ~eps * cond(A_i) (DESIGN.md
§4: 1e-12 for the second-order problems, 1e-9 for the biharmonic blocks).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from ddg_gen import problems as P

pytestmark = pytest.mark.gpu

U_TOL, H_TOL = 1e-10, 1e-8
CHOL, INV = 1, 2


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1504_00907_b200 import build
    build.build()


CASES = {
    "C1": lambda: P.poisson2d(64, 8, 1, 1001),                   # nT = 3
    "poisson3d_24_b8_p2": lambda: P.poisson3d(24, 8, 2, 1002),    # C2 shape: nT up to 28
    "lognormal_16_b4": lambda: P.lognormal3d(16, 4, 1, 1003),    # C3 shape: nT = 4..5
    "elasticity_8_be4": lambda: P.elasticity3d(8, 4, 1004),       # C4 shape: nT up to 47
    "biharm_64_b16_p3": lambda: P.biharmonic2d(64, 16, 3, 1005),  # C5 shape: nT = 11..13, ragged tails
    "poisson2d_ragged": lambda: P.poisson2d(37, 6, 2, 7),        # ragged blocks
}


def _solver(pr, **kw):
    from paper_1504_00907_b200 import Solver
    return Solver.from_problem(pr, **kw)


@pytest.mark.parametrize("path", ["auto", "global"])
@pytest.mark.parametrize("name", list(CASES))
def test_cholesky_pcg_parity(name, path, monkeypatch):
    """auto: factors of <= 6 tile rows (C1, C3 shapes) staged in shared memory by
    bulk copies; global (DDG_CHOL_GLOBAL=1): both passes read global memory"""
    if path == "global":
        monkeypatch.setenv("DDG_CHOL_GLOBAL", "1")
    pr = CASES[name]()
    s = _solver(pr, local_variant=CHOL)
    o = oracle.Oracle.from_problem(pr)
    u, it, hist, rep = s.solve(pr.f, 1e-8)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)
    assert bool(rep.converged) == conv and conv
    assert abs(it - ito) <= 1, (it, ito)
    m = min(len(hist), len(histo))
    assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
    assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
    # factor storage: nT (nT - 1) / 2 full tiles and nT packed diagonal blocks per subdomain
    nT = (s.subdomain_sizes() + 31) // 32
    assert s.info.local_factor_bytes == int(np.sum(nT * (nT - 1) // 2 * 8192 + nT * 528 * 8))


@pytest.mark.parametrize("name", list(CASES))
def test_cholesky_apply_matches_oracle_and_inverse(name):
    pr = CASES[name]()
    sc = _solver(pr, local_variant=CHOL)
    si = _solver(pr, local_variant=INV)
    o = oracle.Oracle.from_problem(pr)
    r = np.random.default_rng(3).standard_normal(pr.n)
    tol = 1e-9 if "biharm" in name else 1e-12
    zc, zi, zo = sc.apply_precond(r), si.apply_precond(r), o.apply_precond(r)
    assert np.linalg.norm(zc - zo) <= tol * np.linalg.norm(zo)
    assert np.linalg.norm(zc - zi) <= tol * np.linalg.norm(zi)
    # symmetric and positive definite (PAPER.md:560-564 is a symmetric method)
    y = np.random.default_rng(4).standard_normal(pr.n)
    zy = sc.apply_precond(y)
    assert abs(r @ zy - y @ zc) <= 1e-12 * np.linalg.norm(r) * np.linalg.norm(zy)
    assert r @ zc > 0


def test_cholesky_bitwise_repeatable_and_default_is_inverse():
    pr = P.lognormal3d(16, 4, 1, 5)
    s = _solver(pr, local_variant=CHOL)
    u1, it1, h1, _ = s.solve(pr.f)
    u2, it2, h2, _ = s.solve(pr.f)
    assert it1 == it2 and np.array_equal(u1, u2) and np.array_equal(h1, h2)
    d = _solver(pr)
    i = _solver(pr, local_variant=INV)
    ud, _, _, _ = d.solve(pr.f)
    ui, _, _, _ = i.solve(pr.f)
    assert np.array_equal(ud, ui)


def test_cholesky_not_spd_and_bad_variant():
    from paper_1504_00907_b200 import DDGError, Solver
    from tests.helpers import csr_from_dense, laplace1d
    An = laplace1d(40)
    An[0, 0] = An[-1, -1] = 1                      # singular (all-Neumann)
    rp, c, v = csr_from_dense(An)
    part = np.repeat(np.arange(4), 10).astype(np.int32)
    with pytest.raises(DDGError) as e:
        Solver(40, rp, c, v, np.ones((40, 1)), part, 4, overlap=1, local_variant=CHOL)
    assert e.value.code == 5
    rp, c, v = csr_from_dense(laplace1d(40))
    with pytest.raises(DDGError) as e:
        Solver(40, rp, c, v, np.ones((40, 1)), part, 4, local_variant=3)
    assert e.value.code == 1


def test_cholesky_three_level_parity():
    """the second level (a two-level context on A_c) inherits local_variant"""
    from paper_1504_00907_b200 import Solver
    pr = P.lognormal3d(16, 4, 1, 1003)
    p2, n2, bc2 = P.coarse_parts(pr, 2, coords=True)
    s = Solver.from_problem(pr, part2=p2, nparts2=n2, block_coords2=bc2, local_variant=CHOL)
    o = oracle.Oracle.from_problem(pr, part2=p2, nparts2=n2)
    u, it, hist, rep = s.solve(pr.f, 1e-8)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)
    assert abs(it - ito) <= 1
    m = min(len(hist), len(histo))
    assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
    assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)


@pytest.mark.parametrize("nranks", [2, 4])
def test_cholesky_loopback_ranks(nranks):
    """the multi-rank path (loopback communicator) with Cholesky local solves"""
    from paper_1504_00907_b200 import Solver
    from tests.test_gpu_loopback import run_ranks
    pr = P.biharmonic2d(128, 16, 3, 1005)
    o = oracle.Oracle.from_problem(pr)
    uo, ito, histo, conv = o.pcg(pr.f, 1e-8)

    def rank(rk, comm):
        s = Solver.from_problem(pr, comm=comm, local_variant=CHOL)
        u, it, hist, rep = s.solve(pr.f, 1e-8)
        s.close()
        return u, it, hist

    for u, it, hist in run_ranks(nranks, rank):
        assert abs(it - ito) <= 1
        m = min(len(hist), len(histo))
        assert np.max(np.abs(hist[:m] - histo[:m]) / histo[:m]) <= H_TOL
        assert np.linalg.norm(u - uo) <= U_TOL * np.linalg.norm(uo)
