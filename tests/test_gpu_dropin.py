"""Drop-in contract checks the reference's own tests rely on (reference synth.py:43-64,
l1filter.py:73-87,240-243, l1reg.py:59-137): exact sparse support counts, any dictionary width k,
and bit-exact index gathers against numpy's m[np.ix_(rows, cols)]."""

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from oracle import adm_filter
from paper_1108_5359_b200 import _device as dv
from paper_1108_5359_b200 import _lib, engine
from paper_1108_5359_b200.l1reg import filter_units

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,rho_s,seed", [(200, 200, 0.05, 0), (50, 60, 0.1, 7), (400, 400, 0.1, 0),
                                            (1, 1, 1.0, 3), (37, 1000, 0.999, 1)])
def test_generate_exact_support_count(m, n, rho_s, seed):
    spec = l1pcp.SynthSpec(m=m, n=n, rho_r=0.0, rho_s=rho_s, rng_seed=seed)
    gt = l1pcp.generate(spec)
    assert np.count_nonzero(gt.s0) == spec.n_sparse
    assert np.abs(gt.s0).max() <= spec.magnitude
    gt2 = l1pcp.generate(spec)
    np.testing.assert_array_equal(gt.s0, gt2.s0)
    np.testing.assert_array_equal(gt.m_obs, gt.l0 + gt.s0)


def test_generate_support_is_uniform():
    # positions of 100 draws of 1% support in a 100x100 matrix: every row/column gets ~1%
    spec = l1pcp.SynthSpec(m=100, n=100, rho_r=0.0, rho_s=0.25, rng_seed=11)
    s0 = l1pcp.generate(spec).s0
    frac_rows = (s0 != 0).mean(axis=1)
    assert abs(frac_rows.mean() - 0.25) < 1e-12
    assert frac_rows.std() < 0.08
    vals = s0[s0 != 0]
    assert abs(np.abs(vals).mean() - 250.0) <= 0.05 * 250.0
    assert abs((vals > 0).mean() - 0.5) < 0.05


def test_generate_zero_and_full_and_oversubscribed():
    gt = l1pcp.generate(l1pcp.SynthSpec(m=30, n=30, rho_r=0.1, rho_s=0.0))
    assert not gt.s0.any()
    gt = l1pcp.generate(l1pcp.SynthSpec(m=8, n=9, rho_r=0.0, rho_s=1.0))
    assert np.count_nonzero(gt.s0) == 72
    with pytest.raises(ValueError):
        l1pcp.generate(l1pcp.SynthSpec(m=4, n=4, rho_r=0.25, rho_s=2.0))


def _orth(s, k, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((s, k)))
    return q


@pytest.mark.parametrize("s,k,n", [(600, 300, 12), (520, 257, 5)])
def test_filter_any_k_matches_oracle(s, k, n):
    """k > 256 (the streaming kernel's register limit) runs on the any-k kernel; FP64 per-unit
    results against the oracle restatement of _solve_block (l1reg.py:59-137)."""
    rng = np.random.default_rng(s + k)
    a = _orth(s, k, 1)
    x = a @ rng.standard_normal((k, n))
    mask = rng.random((s, n)) < 0.05
    x[mask] += rng.uniform(-50, 50, mask.sum())
    x[:, 2] = 0.0  # a dead unit
    zo, eo, ito, reso, sto = adm_filter.solve_units(x, a, 1e-9)
    xt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    at = torch.from_numpy(a).cuda()
    z, e, it, res, st = filter_units(xt, at, l1pcp.AdmConfig(tol=1e-9))
    np.testing.assert_array_equal(st.cpu().numpy(), sto)
    assert np.abs(it.cpu().numpy() - ito).max() <= 1
    scale = np.abs(x).max()
    assert np.abs(z.cpu().numpy().T - zo).max() <= 1e-7 * scale
    assert np.abs(e.cpu().numpy().T - eo).max() <= 1e-7 * scale


def test_solve_l1reg_accepts_wide_dictionary():
    a = _orth(700, 280, 2)
    rng = np.random.default_rng(0)
    x = a @ rng.standard_normal((280, 4))
    sol = l1pcp.solve_l1reg(x, a, l1pcp.AdmConfig(tol=1e-9))
    assert sol.converged
    np.testing.assert_allclose(a @ sol.z + sol.e, x, atol=1e-6)


@pytest.mark.parametrize("dt_in,dt_out", [(torch.float32, torch.float32), (torch.float32, torch.float64),
                                          (torch.float64, torch.float64), (torch.float64, torch.float32)])
@pytest.mark.parametrize("transpose", [0, 1])
def test_gather_bit_exact(dt_in, dt_out, transpose):
    """l1f_gather against numpy m[np.ix_(rows, cols)] (l1filter.py:87,242-243), both layouts."""
    rng = np.random.default_rng(5)
    m = rng.standard_normal((333, 517)) * 100
    m_in = m.astype(np.float32) if dt_in == torch.float32 else m
    rows = np.sort(rng.choice(333, 71, replace=False))
    cols = np.sort(rng.choice(517, 130, replace=False))
    mt = torch.from_numpy(m_in).cuda()
    out = torch.empty((130, 71) if transpose else (71, 130), dtype=dt_out, device="cuda")
    rt, ct = torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()  # alive across the call
    _lib.call("l1f_gather", dv.dtype_code(mt), dv.ptr(mt), mt.stride(0), dv.ptr(rt), 71, dv.ptr(ct), 130,
              dv.dtype_code(out), dv.ptr(out), out.stride(0), transpose, dv.stream())
    ref = m_in[np.ix_(rows, cols)].astype(np.float32 if dt_out == torch.float32 else np.float64)
    got = out.cpu().numpy()
    np.testing.assert_array_equal(got.T if transpose else got, ref)


def test_sample_submatrix_and_panels_bit_exact():
    """sample_submatrix (host index draw + device gather) and the pipeline's panel gathers equal
    numpy's fancy indexing bit for bit (l1filter.py:73-87,240-243)."""
    rng = np.random.default_rng(9)
    m = rng.standard_normal((400, 300))
    ri, ci, blk = l1pcp.sample_submatrix(m, 40, 30, 17)
    ref_rng = np.random.default_rng(17)
    r_ref = np.sort(ref_rng.choice(400, 40, replace=False))
    c_ref = np.sort(ref_rng.choice(300, 30, replace=False))
    np.testing.assert_array_equal(ri, r_ref)
    np.testing.assert_array_equal(ci, c_ref)
    np.testing.assert_array_equal(blk, m[np.ix_(r_ref, c_ref)])
    mt = torch.from_numpy(m.astype(np.float32)).cuda()
    comp_c = np.setdiff1d(np.arange(300), ci)
    comp_r = np.setdiff1d(np.arange(400), ri)
    pc = engine.gather(mt, ri, comp_c)
    pr = engine.gather(mt, comp_r, ci)
    m32 = m.astype(np.float32)
    np.testing.assert_array_equal(pc.cpu().numpy(), m32[np.ix_(ri, comp_c)])
    np.testing.assert_array_equal(pr.cpu().numpy(), m32[np.ix_(comp_r, ci)])
