"""GPU: generator bit-exactness, seed solve, Nystrom/assembly and the full solve against the
reference's golden outputs and the oracle (reference tests: test_pcp_adm.py,
test_l1filter.py, test_matcore.py)."""

import hashlib

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from conftest import load_golden
from oracle import philox_gen, pipeline as opipe, ref_synth
from paper_1108_5359_b200 import _lib, engine

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- generator
@pytest.mark.parametrize("kind,m,n,r,rho,mag", [(0, 150, 260, 7, 0.1, 500.0), (0, 33, 45, 0, 0.05, 100.0),
                                                  (0, 130, 131, 50, 0.05, 500.0), (1, 640, 24, 3, 0.0, 255.0)])
def test_generator_bit_exact_against_oracle(kind, m, n, r, rho, mag):
    mm, l0, x, y = engine.generate_matrix(m, n, r, rho, mag, seed=11, kind=kind, want_l0=True)
    xo, yo = philox_gen.factors(11, kind, m, n, r)
    np.testing.assert_array_equal(x.cpu().numpy(), xo)
    np.testing.assert_array_equal(y.cpu().numpy(), yo)
    mo, l0o = philox_gen.block(11, kind, m, n, r, rho, mag, np.arange(m), np.arange(n), x=xo, y=yo, want_l0=True)
    np.testing.assert_array_equal(l0.cpu().numpy(), l0o)
    np.testing.assert_array_equal(mm.cpu().numpy(), mo)


def test_generator_row_shards_compose():
    m, n, r = 300, 200, 5
    full, _, _, _ = engine.generate_matrix(m, n, r, 0.1, 500.0, seed=3)
    a, _, _, _ = engine.generate_matrix(m, n, r, 0.1, 500.0, seed=3, row0=0, rows=131)
    b, _, _, _ = engine.generate_matrix(m, n, r, 0.1, 500.0, seed=3, row0=131, rows=169)
    assert torch.equal(torch.cat([a, b]), full)


# ---------------------------------------------------------------- dense primitives
def test_matcore_basics():
    assert l1pcp.frobenius_norm([[3, 0], [0, 4]]) == pytest.approx(5.0)
    assert l1pcp.l1_norm([[1, -2], [0, 3]]) == 6.0
    assert l1pcp.l0_count([[1, -2], [0, 3]], 0.0) == 3
    assert l1pcp.linf_norm([[1, -2], [0, 3]]) == 3.0
    assert l1pcp.l0_count(np.array([[100.0, 1e-5], [0.0, 0.0]])) == 1
    assert l1pcp.soft_threshold(np.array([[3.0]]), 1.0)[0, 0] == 2.0
    assert l1pcp.soft_threshold(np.array([[-0.5]]), 1.0)[0, 0] == 0.0
    m = np.random.default_rng(0).standard_normal((6, 5))
    np.testing.assert_array_equal(l1pcp.soft_threshold(m, 0.0), m)


def test_svd_svt_pinv():
    f = l1pcp.svd(np.diag([3.0, 1.0]), rank_tol=0.0)
    np.testing.assert_allclose(f.sigma, [3.0, 1.0])
    a, b = np.array([1.0, 2.0, 2.0]), np.array([0.0, 3.0, 4.0])
    f = l1pcp.svd(np.outer(a, b))
    assert f.rank == 1 and f.sigma[0] == pytest.approx(15.0)
    rng = np.random.default_rng(2)
    for shape in [(20, 10), (50, 50), (200, 120), (120, 200)]:
        m = rng.standard_normal(shape)
        f = l1pcp.svd(m, rank_tol=0.0)
        assert np.linalg.norm(f.reconstruct() - m) <= 1e-8 * np.linalg.norm(m)
        np.testing.assert_allclose(f.u.T @ f.u, np.eye(f.rank), atol=1e-10)
    np.testing.assert_allclose(l1pcp.svt(np.diag([3.0, 1.0]), 2.0), np.diag([1.0, 0.0]), atol=1e-12)
    w = rng.standard_normal((12, 9))
    sig = np.linalg.svd(w, compute_uv=False)
    assert l1pcp.nuclear_norm(l1pcp.svt(w, 0.7)) == pytest.approx(np.maximum(sig - 0.7, 0).sum(), abs=1e-9)
    g1, g2 = rng.standard_normal((20, 3)), rng.standard_normal((15, 3))
    l = g1 @ g2.T
    rhs = l @ rng.standard_normal((15, 4))
    y = l1pcp.pseudo_inverse_apply(l1pcp.svd(l), rhs)
    assert np.linalg.norm(l @ y - rhs) <= 1e-8 * np.linalg.norm(rhs)


# ---------------------------------------------------------------- seed
def test_spectral_norm_and_zero_pcp():
    assert l1pcp.pcp_adm.spectral_norm_estimate(np.diag([5.0, 2.0, 1.0])) == pytest.approx(5.0, rel=1e-6)
    assert l1pcp.pcp_adm.spectral_norm_estimate(np.zeros((3, 3))) == 0.0
    sol = l1pcp.solve_pcp(np.zeros((10, 10)))
    assert sol.converged and sol.iterations == 1 and sol.rank_of_l == 0 and not sol.l.any()


def test_pcp_matches_reference_golden():
    d, meta = load_golden("pcp_rect")
    sol = l1pcp.solve_pcp(d["m"])
    assert sol.converged == meta["converged"]
    assert abs(sol.iterations - meta["iterations"]) <= 1
    assert sol.rank_of_l == meta["rank"]
    assert np.linalg.norm(sol.l - d["l"]) <= 1e-6 * np.linalg.norm(d["l"])
    assert np.linalg.norm(sol.s - d["s"]) <= 1e-6 * np.linalg.norm(d["s"])
    assert l1pcp.pcp_adm.spectral_norm_estimate(d["m"]) == pytest.approx(meta["spectral"], rel=1e-10)


@pytest.mark.parametrize("name", ["seed_clean_rank2", "seed_corrupt_rank5"])
def test_recover_seed_matches_reference_golden(name):
    d, meta = load_golden(name)
    seed = l1pcp.recover_seed(d["block"], l1pcp.AdmConfig(tol=meta["tol"]))
    assert seed.r_prime == meta["r_prime"]
    assert abs(seed.pcp_iterations - meta["pcp_iterations"]) <= 1
    np.testing.assert_allclose(seed.seed_svd.sigma, d["sigma"], rtol=1e-6)
    assert np.linalg.norm(seed.seed_l - d["seed_l"]) <= 1e-6 * np.linalg.norm(d["seed_l"])


def test_recover_seed_zero_block_raises():
    with pytest.raises(l1pcp.SeedRankZeroError):
        l1pcp.recover_seed(np.zeros((20, 20)))


def test_max_iter_exhaustion_is_flagged():
    m, _, _ = ref_synth.generate(100, 100, 0.03, 0.05, rng_seed=0)
    sol = l1pcp.solve_pcp(m, l1pcp.AdmConfig(tol=1e-12, max_iter=3))
    assert not sol.converged and sol.iterations == 3 and sol.final_residual > 1e-12


# ---------------------------------------------------------------- Nystrom / assembly
def test_nystrom_and_assembly_match_reference_golden():
    d, meta = load_golden("nystrom_exact")
    f = l1pcp.SkinnySvd(u=d["u"], sigma=d["sigma"], v=d["v"])
    seed = l1pcp.SeedRecovery(row_idx=d["row_idx"], col_idx=d["col_idx"], seed_svd=f, seed_l=f.reconstruct(),
                              seed_s=None, r_prime=meta["r_prime"])
    fr = l1pcp.FilterResult(q_tilde=d["q"], p_tilde=d["p"], s_col=None, s_row=None)
    comp = l1pcp.nystrom_complete(seed, fr)
    np.testing.assert_allclose(comp, d["completion"], rtol=0, atol=1e-12 * np.abs(comp).max())
    l_hat = l1pcp.assemble(seed, fr, comp, 80, 70)
    np.testing.assert_allclose(l_hat, d["l_hat"], rtol=0, atol=1e-12 * np.abs(l_hat).max())
    # exact re-extraction of the placed blocks (test_l1filter.py:164-177)
    np.testing.assert_array_equal(l_hat[np.ix_(d["row_idx"], d["col_idx"])], seed.seed_l)
    comp_r = np.setdiff1d(np.arange(80), d["row_idx"])
    comp_c = np.setdiff1d(np.arange(70), d["col_idx"])
    np.testing.assert_array_equal(l_hat[np.ix_(comp_r, comp_c)], comp)
    with pytest.raises(RuntimeError):
        l1pcp.assemble(seed, fr, np.zeros((5, 5)), 80, 70)


def test_filter_columns_rows_exact_subspace():
    rng = np.random.default_rng(3)
    u, _ = np.linalg.qr(rng.standard_normal((40, 3)))
    q0 = rng.standard_normal((3, 15))
    q, s_col, _ = l1pcp.filter_columns(u @ q0, u, l1pcp.AdmConfig(tol=1e-10))
    assert np.abs(s_col).max() <= 1e-8 and np.abs(q - q0).max() <= 1e-6
    v, _ = np.linalg.qr(rng.standard_normal((30, 3)))
    p0 = rng.standard_normal((3, 12))
    p, s_row, _ = l1pcp.filter_rows(p0.T @ v.T, v, l1pcp.AdmConfig(tol=1e-10))
    assert s_row.shape == (12, 30) and np.abs(s_row).max() <= 1e-8 and np.abs(p - p0).max() <= 1e-6
    q, s_col, it = l1pcp.filter_columns(np.zeros((40, 0)), u)
    assert q.shape == (3, 0) and s_col.shape == (40, 0) and it == 0


# ---------------------------------------------------------------- full solve
@pytest.mark.parametrize("name", ["pipeline_hint", "pipeline_rect_norank", "pipeline_tol7"])
def test_full_solve_matches_reference_golden(name):
    d, meta = load_golden(name)
    m, l0, _ = ref_synth.generate(**meta["spec"])
    assert hashlib.sha256(m.tobytes()).hexdigest() == meta["m_sha256"]
    cfg = l1pcp.FilterConfig(rank_hint=meta["rank_hint"], rng_seed=meta["rng_seed"],
                             adm=l1pcp.AdmConfig(tol=meta["tol"]))
    sol = l1pcp.estimate_rank_and_solve(m, cfg)
    assert sol.method == meta["method"] == "l1-filter"
    assert sol.rank_of_l == meta["rank"]
    assert sol.stats["seed_rows"] == meta["stats"]["seed_rows"]
    assert sol.stats["attempts"] == meta["stats"]["attempts"]
    assert np.linalg.norm(sol.l - d["l"]) <= 1e-6 * np.linalg.norm(d["l"])
    s_ref = m - d["l"]
    assert np.linalg.norm(sol.s - s_ref) <= 1e-6 * np.linalg.norm(s_ref)
    np.testing.assert_allclose(sol.l + sol.s, m, atol=1e-10)
    assert sol.final_residual == 0.0
    assert l1pcp.rel_err(sol.l, l0) <= max(1e-5, 10 * meta["rel_err"])


def test_full_solve_float32_tensor_path_matches_oracle():
    d, meta = load_golden("pipeline_tol7")
    m, _, _ = ref_synth.generate(**meta["spec"])
    mt = torch.from_numpy(m.astype(np.float32)).cuda()
    cfg = l1pcp.FilterConfig(rank_hint=meta["rank_hint"], rng_seed=meta["rng_seed"],
                             adm=l1pcp.AdmConfig(tol=1e-7))
    sol = l1pcp.estimate_rank_and_solve(mt, cfg)
    assert sol.l.dtype == torch.float32 and sol.l.is_cuda
    ref = opipe.solve(mt.double().cpu().numpy(), meta["rank_hint"], meta["rng_seed"], tol=1e-7)
    l = sol.l.double().cpu().numpy()
    s = sol.s.double().cpu().numpy()
    assert np.linalg.norm(l - ref["l"]) <= 1e-4 * np.linalg.norm(ref["l"])
    assert np.linalg.norm(s - ref["s"]) <= 1e-4 * np.linalg.norm(ref["s"])


def test_degenerate_zero_matrix():
    sol = l1pcp.estimate_rank_and_solve(np.zeros((50, 50)), l1pcp.FilterConfig(rng_seed=0))
    assert sol.method == "degenerate-zero-seed" and sol.rank_of_l == 0 and not sol.l.any()


def test_fallback_to_full_pcp_for_high_rank():
    m, _, _ = ref_synth.generate(100, 100, 0.4, 0.01, rng_seed=0)
    sol = l1pcp.estimate_rank_and_solve(m, l1pcp.FilterConfig(rng_seed=0))
    assert sol.method == "full-pcp-fallback"
    assert np.linalg.norm(m - sol.l - sol.s) / np.linalg.norm(m) <= 1e-7


def test_end_to_end_with_device_generated_instance():
    gt = l1pcp.generate(l1pcp.SynthSpec(m=300, n=300, rho_r=0.01, rho_s=0.01, rng_seed=0))
    sol = l1pcp.estimate_rank_and_solve(gt.m_obs, l1pcp.FilterConfig(rank_hint=3, rng_seed=0))
    assert sol.method == "l1-filter" and sol.rank_of_l == 3
    assert l1pcp.rel_err(sol.l, gt.l0) <= 1e-5
    np.testing.assert_allclose(sol.l + sol.s, gt.m_obs, atol=1e-10)


def test_rank_estimation_and_cross_validation():
    m, l0, _ = ref_synth.generate(400, 400, 0.005, 0.01, rng_seed=1)
    sol = l1pcp.estimate_rank_and_solve(m, l1pcp.FilterConfig(rng_seed=3))
    assert sol.method == "l1-filter" and sol.rank_of_l == 2 and sol.stats["seed_rows"] >= 20
    assert l1pcp.rel_err(sol.l, l0) <= 1e-5
    m, l0, _ = ref_synth.generate(300, 300, 0.01, 0.01, rng_seed=2)
    sol = l1pcp.estimate_rank_and_solve(m, l1pcp.FilterConfig(rng_seed=0, cross_validate=True))
    assert sol.method == "l1-filter" and sol.rank_of_l == 3
    assert l1pcp.rel_err(sol.l, l0) <= 1e-5


def test_sharded_cuda_backend_matches_single_gpu_solve():
    """distributed.solve_sharded with the production CudaBackend (NCCL, world size 1) gives the
    same L/S as the single-GPU engine on the same seed indices."""
    import os
    import socket

    import torch.distributed as dist
    from paper_1108_5359_b200 import distributed as pdist

    mt, _, _, _ = engine.generate_matrix(600, 500, 5, 0.05, 500.0, seed=2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ri, ci = engine.sample_indices(600, 500, 50, 50, np.random.SeedSequence(0).spawn(1)[0])
        plan = pdist.ShardPlan(600, 500, 0, 1, ri, ci)
        adm = l1pcp.AdmConfig(tol=1e-7)
        l, s, info = pdist.solve_sharded(mt, plan, pdist.CudaBackend(), adm)
    finally:
        dist.destroy_process_group()
    sol = l1pcp.estimate_rank_and_solve(mt, l1pcp.FilterConfig(rank_hint=5, rng_seed=0, adm=adm))
    assert info["k"] == sol.rank_of_l == 5
    assert torch.equal(l, sol.l) and torch.equal(s, sol.s)


@pytest.mark.parametrize("m,n,r,stream", [(600, 500, 5, None), (2000, 1800, 30, "0"), (2000, 1800, 30, "1"),
                                          (3000, 2800, 60, "1")])
def test_sharded_timed_step_matches_single_gpu_solve(m, n, r, stream, monkeypatch):
    """The timed multi-GPU step (distributed.CudaShardedStep: column-panel exchange, paired
    filters, Q~ all-gather, factors, reconstruction) at NCCL world size 1 equals the public
    single-GPU solve bitwise, for the FP64 small-k and the fp32 tensor-core filter."""
    import os
    import socket

    import torch.distributed as dist
    from paper_1108_5359_b200 import distributed as pdist

    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=4)
    adm = l1pcp.AdmConfig(tol=1e-7)
    sol = l1pcp.estimate_rank_and_solve(mt, l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=adm))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ri, ci = engine.sample_indices(m, n, 10 * r, 10 * r, np.random.SeedSequence(0).spawn(1)[0])
        plan = pdist.ShardPlan(m, n, 0, 1, ri, ci)
        block = pdist.gather_seed_block(mt, plan, pdist.CudaBackend())
        u, sig, v, _ = pdist.seed_factors(block, plan, pdist.CudaBackend(), adm)
        if stream is not None:  # the paired-filter step, or the streamed one (filter + reconstruction)
            monkeypatch.setitem(_lib.PY_OPTIONS, "sharded_stream", stream == "1")
        stepper = pdist.CudaShardedStep(mt, plan, adm, u, sig, v)
        if stream is not None:
            assert stepper.streamed == (stream == "1")
        for _ in range(2):
            l, s, stats, _ = stepper.step(mt)
            torch.cuda.synchronize()
            assert torch.equal(l, sol.l) and torch.equal(s, sol.s)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,r", [(300, 300, 20), (500, 200, 30), (150, 400, 10)])
def test_svd_gram_matches_gesvd_on_low_rank(m, n, r):
    """l1f_svd_gram_f64 (the seed's final factorisation) vs l1f_svd_f64 on an exactly rank-r
    matrix: singular values, the projectors U U^T / V V^T and orthonormality of the kept triplets."""
    rng = np.random.default_rng(m + n + r)
    x = rng.standard_normal((m, r)) @ np.diag(np.linspace(1.0, 50.0, r)) @ rng.standard_normal((r, n))
    t = torch.from_numpy(x).cuda()
    u1, s1, v1 = engine.svd_device(t)
    u2, s2, v2 = engine.svd_device(t, gram=True)
    s1, s2 = s1.cpu().numpy(), s2.cpu().numpy()
    np.testing.assert_allclose(s2[:r], s1[:r], rtol=1e-11)
    assert (s2[r:] <= 1e-6 * s2[0]).all()
    for a, b in ((u1, u2), (v1, v2)):
        a, b = a[:, :r].cpu().numpy(), b[:, :r].cpu().numpy()
        assert np.abs(a @ a.T - b @ b.T).max() <= 1e-10
        assert np.abs(b.T @ b - np.eye(r)).max() <= 1e-10
    rec = (u2[:, :r] * torch.from_numpy(s2[:r]).cuda()) @ v2[:, :r].T
    assert torch.linalg.norm(rec - t) <= 1e-11 * torch.linalg.norm(t)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_filter_and_full_adm_agree(seed):
    """Acceptance property of the reference (test_acceptance.py:69-81): l1 filtering and the full
    ADM recover the same low-rank part (relative deviation <= 1e-4), both on the device."""
    gt = l1pcp.generate(l1pcp.SynthSpec(m=500, n=500, rho_r=0.01, rho_s=0.01, rng_seed=seed))
    filt = l1pcp.estimate_rank_and_solve(gt.m_obs, l1pcp.FilterConfig(rank_hint=5, rng_seed=seed))
    adm = l1pcp.solve_pcp(gt.m_obs)
    dev = np.linalg.norm(filt.l - adm.l) / np.linalg.norm(adm.l)
    assert dev <= 1e-4, dev


def test_filter_and_full_adm_agree_large_fp32():
    """Same agreement at 2000^2, rank 20, on fp32 device tensors (the full ADM's SVT runs on the
    device through the Gram eigendecomposition)."""
    mt, l0, _, _ = engine.generate_matrix(2000, 2000, 20, 0.05, 500.0, seed=4, want_l0=True)
    filt = l1pcp.estimate_rank_and_solve(mt, l1pcp.FilterConfig(rank_hint=20, rng_seed=0,
                                                                adm=l1pcp.AdmConfig(tol=1e-7)))
    adm = l1pcp.solve_pcp(mt.double(), l1pcp.AdmConfig(tol=1e-7))
    lf, la = filt.l.double(), adm.l.double()
    dev = float(torch.linalg.norm(lf - la) / torch.linalg.norm(la))
    err = float(torch.linalg.norm(lf - l0.double()) / torch.linalg.norm(l0.double()))
    print(f"2000^2 r=20: filter vs ADM {dev:.2e}, filter vs L0 {err:.2e}")
    assert dev <= 1e-4 and err <= 1e-4
