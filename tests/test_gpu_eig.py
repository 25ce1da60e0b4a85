"""The hand-written symmetric eigensolvers of the seed SVT (csrc/eig_sym.cu: cooperative Householder
tridiagonalisation, Sturm multisection, inverse iteration, CGS2, back-transformation; csrc/seed_small.cu:
the one-CTA Gram / shared-memory tridiagonal SVT): same singular values, factors and seed solves as the
cuSOLVER syevd path (L1F_OPT_SEED_EIG = 1) and the one-sided Jacobi SVT (L1F_OPT_SEED_SMALL_SVT = 0)
(reference: the SVD inside svt_with_rank, matcore.py:73-105)."""

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import _lib, engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,r", [(600, 500, 20), (400, 700, 35), (1200, 1000, 100)])
def test_gram_svd_matches_syevd(m, n, r):
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn(m, r, dtype=torch.float64, device="cuda", generator=g) @ \
        torch.randn(r, n, dtype=torch.float64, device="cuda", generator=g)
    with _lib.options(seed_eig=0):
        u, s, v = engine.svd_device(a, gram=True)
    with _lib.options(seed_eig=1):
        u1, s1, v1 = engine.svd_device(a, gram=True)
    ref = np.linalg.svd(a.cpu().numpy(), compute_uv=False)
    assert np.abs(s[:r].cpu().numpy() - ref[:r]).max() <= 1e-12 * ref[0]
    rec = (u[:, :r] * s[:r]) @ v[:, :r].T
    assert float((rec - a).norm() / a.norm()) <= 1e-12
    eye = torch.eye(r, dtype=torch.float64, device="cuda")
    assert float((u[:, :r].T @ u[:, :r] - eye).abs().max()) <= 1e-10
    assert float((v[:, :r].T @ v[:, :r] - eye).abs().max()) <= 1e-10


def test_seed_stage_matches_syevd_path():
    m = n = 3000
    r = 60  # 600 x 600 seed: beyond the small-block kernel, the Gram path
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=2)
    cfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    with _lib.options(seed_eig=0):
        k0, s0, a0, _ = engine.seed_stage(mt, cfg)
    with _lib.options(seed_eig=1):
        k1, s1, a1, _ = engine.seed_stage(mt, cfg)
    assert k0 == k1 == "seed" and a0 == a1
    assert s0.r_prime == s1.r_prime == r and s0.pcp_iterations == s1.pcp_iterations
    assert float((s0.seed_l - s1.seed_l).norm() / s1.seed_l.norm()) <= 1e-12


def _pcp_case(m, n, r, seed, rho=0.1):
    rng = np.random.default_rng(seed)
    low = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    sp = np.where(rng.random((m, n)) < rho, rng.uniform(-50, 50, (m, n)), 0.0)
    return torch.from_numpy(low + sp).cuda()


@pytest.mark.parametrize("m,n,r,dsm", [(130, 120, 6, 1), (120, 300, 8, 1), (400, 160, 12, 1), (700, 600, 30, 1),
                                       (130, 120, 6, 0), (120, 300, 8, 0), (400, 160, 12, 0), (700, 600, 30, 0),
                                       (1500, 1300, 40, 1)])
def test_large_block_pcp_matches_syevd(m, n, r, dsm):
    """The ALM loop on blocks beyond the one-CTA kernel with the hand-written eigensolver (shared-
    memory-resident or L2-resident tridiagonalisation; p = min(m, n) from 120, fewer rows than the
    148 blocks, to 1300, where the 512-thread form runs) against the syevd path: same iterations and
    rank, L to 1e-12."""
    from paper_1108_5359_b200 import pcp_adm
    M = _pcp_case(m, n, r, m * 7 + n)
    cfg = pcp_adm.AdmConfig(tol=1e-7)
    with _lib.options(seed_eig=0, seed_eig_dsm=dsm):
        l0, s0, i0 = pcp_adm.solve_pcp_device(M, cfg)
    with _lib.options(seed_eig=1):
        l1, s1, i1 = pcp_adm.solve_pcp_device(M, cfg)
    assert i0["iterations"] == i1["iterations"] and i0["rank"] == i1["rank"]
    assert float((l0 - l1).norm() / l1.norm()) <= 1e-12
    assert float((s0 - s1).abs().max()) <= 1e-9 * float(M.abs().max())


@pytest.mark.parametrize("m,n,r", [(7, 1, 1), (1, 9, 1), (5, 3, 1), (20, 20, 2), (113, 113, 11), (64, 200, 5),
                                   (100, 40, 4)])
def test_small_block_gram_svt_matches_jacobi(m, n, r):
    """The one-CTA ALM kernel's Gram / shared-memory tridiagonal SVT (default) against its one-sided
    Jacobi SVT on edge shapes (a single row or column, rectangular, the 113 x 113 limit): same
    iterations and rank, L to 1e-8 relative."""
    from paper_1108_5359_b200 import pcp_adm
    M = _pcp_case(m, n, r, m * 11 + n)
    cfg = pcp_adm.AdmConfig(tol=1e-7)
    with _lib.options(seed_small_svt=1):
        l0, s0, i0 = pcp_adm.solve_pcp_device(M, cfg)
    with _lib.options(seed_small_svt=0):
        l1, s1, i1 = pcp_adm.solve_pcp_device(M, cfg)
    assert i0["iterations"] == i1["iterations"]
    # a single row / column leaves L at roundoff (~1e-16), its one singular value at the threshold
    roundoff = float(l1.norm()) <= 1e-12 * float(M.norm())
    assert i0["rank"] == i1["rank"] or (roundoff and abs(i0["rank"] - i1["rank"]) <= 1)
    # relative to L, or to M where L is roundoff
    assert float((l0 - l1).norm()) <= 1e-8 * max(float(l1.norm()), 1e-6 * float(M.norm()))


def test_small_block_zero_matrix():
    from paper_1108_5359_b200 import pcp_adm
    M = torch.zeros(50, 60, dtype=torch.float64, device="cuda")
    l, s, info = pcp_adm.solve_pcp_device(M, pcp_adm.AdmConfig(tol=1e-7))
    assert info["iterations"] == 1
    assert float(l.abs().max()) == 0.0 and float(s.abs().max()) == 0.0
