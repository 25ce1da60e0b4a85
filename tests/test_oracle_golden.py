"""CPU: the oracle against the reference's own outputs (tests/golden, made by running the
reference in the build container) and the Philox generator restatement against
numpy.random.Philox and a from-scratch Philox4x64-10."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import adm_filter, philox_gen, pipeline, ref_synth, seed_pcp

L1REG_CASES = ["l1reg_exact_fit", "l1reg_spiked", "l1reg_hand", "l1reg_columnwise", "l1reg_failed",
               "l1reg_cfg1_panel"]


@pytest.mark.parametrize("name", L1REG_CASES)
def test_oracle_filter_matches_reference(name):
    d, meta = load_golden(name)
    c = meta["cfg"]
    z, e, it, res, st = adm_filter.solve_units(d["x"], d["a"], c["tol"], c["rho"], c["beta0"], c["beta_max"],
                                               c["max_iter"])
    iterations, final_residual, failed = adm_filter.summarize(d["x"], it, res, st)
    scale = max(1.0, np.abs(d["x"]).max())
    assert np.abs(z - d["z"]).max() <= 1e-12 * scale
    assert np.abs(e - d["e"]).max() <= 1e-12 * scale
    np.testing.assert_array_equal(it, d["unit_iters"])
    np.testing.assert_allclose(res, d["unit_res"], rtol=1e-9, atol=1e-14 * scale)
    assert iterations == meta["iterations"]
    assert failed == meta["failed"]
    assert final_residual == pytest.approx(meta["final_residual"], rel=1e-6, abs=1e-15)


def test_oracle_known_answer_single_column():
    # the reference's hand-solvable case (test_l1reg.py:37-49): z = 10, E = [0, 3, 0, ...]
    d, _ = load_golden("l1reg_hand")
    z, e, *_ = adm_filter.solve_units(d["x"], d["a"], 1e-10)
    assert z[0, 0] == pytest.approx(10.0, abs=1e-6)
    assert e[1, 0] == pytest.approx(3.0, abs=1e-6)


@pytest.mark.parametrize("name", ["seed_clean_rank2", "seed_corrupt_rank5"])
def test_oracle_seed_matches_reference(name):
    d, meta = load_golden(name)
    u, s, v, seed_l, it = seed_pcp.recover(d["block"], tol=meta["tol"])
    assert s.size == meta["r_prime"]
    assert it == meta["pcp_iterations"]
    np.testing.assert_allclose(s, d["sigma"], rtol=1e-10)
    assert np.abs(seed_l - d["seed_l"]).max() <= 1e-9 * np.abs(d["seed_l"]).max()


def test_oracle_pcp_matches_reference():
    d, meta = load_golden("pcp_rect")
    l, s, it, resid, rank, conv = seed_pcp.pcp(d["m"])
    assert it == meta["iterations"] and rank == meta["rank"] and conv == meta["converged"]
    assert resid == pytest.approx(meta["final_residual"], rel=1e-6)
    assert np.abs(l - d["l"]).max() <= 1e-9 * np.abs(d["l"]).max()
    assert seed_pcp.spectral_norm(d["m"]) == pytest.approx(meta["spectral"], rel=1e-12)


@pytest.mark.parametrize("name", ["pipeline_hint", "pipeline_rect_norank", "pipeline_tol7"])
def test_oracle_pipeline_matches_reference(name):
    d, meta = load_golden(name)
    m, l0, _ = ref_synth.generate(**meta["spec"])
    assert hashlib.sha256(m.tobytes()).hexdigest() == meta["m_sha256"]
    assert hashlib.sha256(l0.tobytes()).hexdigest() == meta["l0_sha256"]
    out = pipeline.solve(m, meta["rank_hint"], meta["rng_seed"], tol=meta["tol"])
    assert out["r_prime"] == meta["rank"]
    assert out["iterations"] == meta["iterations"]
    assert np.linalg.norm(out["l"] - d["l"]) <= 1e-12 * np.linalg.norm(d["l"])


def test_oracle_sampled_blocks_match_full_solve():
    d, meta = load_golden("pipeline_hint")
    m, _, _ = ref_synth.generate(**meta["spec"])
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(m.shape[0], 40, replace=False))
    cols = np.sort(rng.choice(m.shape[1], 50, replace=False))
    out = pipeline.sampled_blocks(m.shape[0], m.shape[1], lambda r, c: m[np.ix_(r, c)], meta["rank_hint"], rows,
                                  cols, meta["rng_seed"], tol=meta["tol"])
    ref = d["l"][np.ix_(rows, cols)]
    assert np.linalg.norm(out["l"] - ref) <= 1e-10 * np.linalg.norm(ref)


def test_oracle_nystrom_matches_reference():
    d, _ = load_golden("nystrom_exact")
    comp = d["p"].T @ (d["q"] / d["sigma"][:, None])
    np.testing.assert_allclose(comp, d["completion"], rtol=0, atol=1e-12 * np.abs(comp).max())
    assert np.linalg.norm(d["l_hat"] - d["l0"]) <= 1e-8 * np.linalg.norm(d["l0"])


# ---------------------------------------------------------------- Philox generator
M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK = (1 << 64) - 1


def _philox_scalar(ctr, key):
    c, k = list(ctr), list(key)
    for r in range(10):
        if r:
            k = [(k[0] + W0) & MASK, (k[1] + W1) & MASK]
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & MASK, (p0 >> 64) ^ c[3] ^ k[1], p0 & MASK]
    return c


@pytest.mark.parametrize("seed,stream,start", [(0, 1, 0), (5, 3, 17), (2**40 + 3, 2, 1001)])
def test_philox_draws_match_independent_implementation(seed, stream, start):
    got = philox_gen.draws(seed, stream, start, 9)
    want = []
    for e in range(start, start + 9):
        want.append(_philox_scalar([e // 4 + 1, 0, 0, 0], [seed, stream])[e % 4])
    assert [int(v) for v in got] == want


def test_normal_transform_statistics():
    v = philox_gen.draws(0, philox_gen.STREAM_X, 0, 200000)
    z = philox_gen.normal_from(v).astype(np.float64)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    assert np.abs(z).max() < 6.5
    # the polynomial log / cos agree with libm to float32 accuracy
    u = np.linspace(1e-6, 1.0, 1001, dtype=np.float32)
    np.testing.assert_allclose(philox_gen.exact_log(u), np.log(u.astype(np.float64)), rtol=2e-6, atol=2e-7)
    t = np.linspace(0, 0.999, 1001, dtype=np.float32)
    np.testing.assert_allclose(philox_gen.exact_cos2pi(t), np.cos(2 * np.pi * t.astype(np.float64)), atol=2e-6)


def test_generator_block_statistics_and_shard_invariance():
    m, n, r = 64, 96, 4
    full, l0 = philox_gen.block(0, philox_gen.GAUSSIAN, m, n, r, 0.1, 500.0, np.arange(m), np.arange(n),
                                want_l0=True)
    s0 = full - l0
    frac = (s0 != 0).mean()
    assert 0.07 < frac < 0.13
    assert np.abs(s0).max() <= 500.0
    part = philox_gen.block(0, philox_gen.GAUSSIAN, m, n, r, 0.1, 500.0, np.arange(10, 30), np.arange(5, 50))
    np.testing.assert_array_equal(part, full[10:30, 5:50])
    x, y = philox_gen.factors(0, philox_gen.GAUSSIAN, m, n, r)
    assert np.linalg.matrix_rank(l0.astype(np.float64), tol=1e-3) == r


def test_video_generator_coverage():
    m, n = 76800, 8
    cover = philox_gen.video_mask(0, np.arange(m), np.arange(n))
    frac = cover.mean()
    assert 0.02 < frac < 0.09
