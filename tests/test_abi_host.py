"""CPU: the C-ABI library loads and exports every symbol of include/l1pcp_b200.h; host-side
logic of the drop-in (config validation, index sampling, errors) matches the reference."""

import re

import numpy as np
import pytest

import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import _lib, engine


def _header_functions():
    text = open(_lib.HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(l1f_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = _header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.SIGNATURES) == names


def test_library_version_and_error_string():
    lib = _lib.load()
    assert lib.l1f_version() >= 10000
    assert isinstance(lib.l1f_last_error(), bytes)


def test_workspace_query_needs_no_device():
    n = _lib.load().l1f_filter_workspace_bytes(_lib.F32, 1000, 100, 19000)
    assert n >= 19000 * 4  # at least the per-unit scale array
    assert _lib.load().l1f_filter_workspace_bytes(_lib.F32, 0, 10, 10) == 0


def test_public_api_names_match_reference_exports():
    # pkg/src/l1pcp/__init__.py:5-44
    expected = """SkinnySvd SvdConvergenceError as_dense frobenius_norm l0_count l1_norm linf_norm nuclear_norm
    pseudo_inverse_apply soft_threshold svd svt AdmConfig PcpDivergenceError PcpSolution default_lambda
    solve_pcp L1RegSolution solve_l1reg solve_l1reg_columnwise FilterConfig FilterResult SeedRankZeroError
    SeedRecovery assemble estimate_rank_and_solve filter_columns filter_rows nystrom_complete
    nystrom_complete_via_pinv recover_seed sample_submatrix GroundTruth SynthSpec ave_dif checkerboard
    corrupt_impulsive generate max_dif rel_err""".split()
    for name in expected:
        assert hasattr(l1pcp, name), name
    assert l1pcp.__version__ == "0.1.0"


def test_config_validation_matches_reference():
    with pytest.raises(ValueError):
        l1pcp.AdmConfig(rho=1.0)
    with pytest.raises(ValueError):
        l1pcp.AdmConfig(tol=0.0)
    with pytest.raises(ValueError):
        l1pcp.AdmConfig(beta0=1.0, beta_max=0.5)
    with pytest.raises(ValueError):
        l1pcp.FilterConfig(s_r=1.0)
    with pytest.raises(ValueError):
        l1pcp.FilterConfig(max_seed_fraction=0.0)
    assert l1pcp.FilterConfig().adm.tol == 1e-9
    assert l1pcp.AdmConfig().tol == 1e-7


def test_default_lambda_values():
    assert l1pcp.default_lambda(2000, 2000) == pytest.approx(1 / np.sqrt(2000))
    assert l1pcp.default_lambda(1, 1) == 1.0
    assert l1pcp.default_lambda(100, 400) == pytest.approx(0.05)
    with pytest.raises(ValueError):
        l1pcp.default_lambda(0, 5)


def test_index_sampling_is_the_reference_draw():
    # sample_submatrix (l1filter.py:84-86): sorted choice without replacement
    from oracle import pipeline as op
    for seed in (0, 42, np.random.SeedSequence(3).spawn(1)[0]):
        a = engine.sample_indices(1000, 900, 100, 90, seed)
        b = op.sample_indices(1000, 900, 100, 90, seed)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
        assert np.all(np.diff(a[0]) > 0)
    with pytest.raises(ValueError):
        engine.sample_indices(5, 5, 6, 3, 0)


def test_as_dense_rejects_bad_input():
    with pytest.raises(ValueError):
        l1pcp.as_dense(np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        l1pcp.as_dense(np.array([[np.nan, 0.0]]))
    with pytest.raises(ValueError):
        l1pcp.as_dense(np.array([[np.inf], [1.0]]))
    out = l1pcp.as_dense([[1, 2], [3, 4]])
    assert out.dtype == np.float64 and out.flags.c_contiguous


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.NativeUnavailable):
        l1pcp.soft_threshold(np.ones((2, 2)), 0.5)
    with pytest.raises(_lib.NativeUnavailable):
        l1pcp.estimate_rank_and_solve(np.ones((20, 20)), l1pcp.FilterConfig(rank_hint=1))


def test_overlapped_entry_points_validate_before_device_work():
    """The overlapped filter + reconstruction entry points reject inconsistent shapes with
    L1F_ERR_ARG before touching the device (host-side checks only: runs without a GPU)."""
    lib = _lib.load()
    null = None
    # row units must be the m - s_r non-seed rows
    rc = lib.l1f_rowfilter_reconstruct_f32(null, 100, 100, 10, null, 10, 10, 1e-7, 1.5, 0.0, 0.0, 100, null, 10,
                                           null, null, null, null, null, 5, null, null, null, 5, null, null, 10,
                                           null, 100, 100, 100, null, 100, null, 100, null, null, null)
    assert rc == _lib.L1F_ERR_ARG
    rc = lib.l1f_rowfilter_reconstruct_small(null, 100, 100, 10, null, 10, 10, 1e-7, 1.5, 0.0, 0.0, 100, null, 10,
                                             null, null, null, null, null, 5, null, null, null, 5, null, null, 10,
                                             null, 100, 100, 100, null, 100, null, 100, null, null, null)
    assert rc == _lib.L1F_ERR_ARG
    # leading dimension of the filter panel below the unit length
    rc = lib.l1f_filter_with_gather_f32(null, 10, 100, 5, null, 10, 10, 1e-7, 1.5, 0.0, 0.0, 100, null, 10, null,
                                        null, null, _lib.F32, null, 100, null, 0, null, 0, null, 10, 0, null)
    assert rc == _lib.L1F_ERR_ARG
    assert "need" in _lib.last_error() or "shape" in _lib.last_error()


def test_library_options_are_explicit():
    """Kernel-selection switches are set through l1f_set_option (no environment reads in the
    library): defaults, round trip, restore, and the ValueError mapping for an unknown key."""
    assert _lib.get_option("filter_tc") == 1 and _lib.get_option("recon_stream") == 1
    assert _lib.get_option("wait_timeout_ms") == 10000
    with _lib.options(filter_tc=0, tc_groups=2, wait_timeout_ms=5):
        assert _lib.get_option("filter_tc") == 0 and _lib.get_option("tc_groups") == 2
        assert _lib.get_option("wait_timeout_ms") == 5
    assert _lib.get_option("filter_tc") == 1 and _lib.get_option("tc_groups") == 0
    with pytest.raises(ValueError):
        _lib.call("l1f_set_option", 99, 1)
    with pytest.raises(ValueError):
        _lib.set_option("no_such_option", 1)
    with _lib.options(filter_pair=False):
        assert _lib.get_option("filter_pair") is False
    assert _lib.get_option("filter_pair") is True
