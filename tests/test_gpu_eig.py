"""The hand-written symmetric eigensolver (csrc/eig_sym.cu: cooperative Householder
tridiagonalisation, Sturm multisection, inverse iteration, CGS2, back-transformation) that replaces
cuSOLVER syevd in the large-seed SVT when L1F_OPT_SEED_EIG = 0: same singular values, factors and
seed solves as the syevd path (reference: the SVD inside svt_with_rank, matcore.py:73-105)."""

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
