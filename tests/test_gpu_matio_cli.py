"""GPU: DMAT streamed to / from HBM (matio.read_dmat_device / write_dmat_device) and the command
line front end on the device path (cli.py; the reference's tests/test_cli.py cases)."""

import json

import numpy as np
import pytest
import torch

from paper_1108_5359_b200 import matio
from paper_1108_5359_b200.cli import main

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_dmat_device_roundtrip_many_chunks(tmp_path, monkeypatch, dtype):
    monkeypatch.setattr(matio, "_CHUNK_BYTES", 8 * 1000 * 7)  # ~7 rows per chunk
    x = np.random.default_rng(1).standard_normal((101, 1000))
    p = tmp_path / "x.dmat"
    matio.write_dmat(p, x)
    t = matio.read_dmat_device(p, dtype)
    assert t.dtype == dtype and t.is_cuda
    np.testing.assert_array_equal(t.cpu().numpy(), x.astype(np.float32 if dtype == torch.float32 else np.float64))
    q = tmp_path / "y.dmat"
    matio.write_dmat_device(q, t)
    np.testing.assert_array_equal(matio.read_dmat(q), t.double().cpu().numpy())
    bad = tmp_path / "bad.dmat"
    bad.write_bytes(p.read_bytes()[:-16])
    with pytest.raises(ValueError):
        matio.read_dmat_device(bad)


def _synth(tmp_path, m=200, seed=0):
    mp, lp = tmp_path / "m.dmat", tmp_path / "l0.dmat"
    assert main(["synth", "--m", str(m), "--rho-r", "0.01", "--rho-s", "0.01", "--seed", str(seed),
                 "--out-m", str(mp), "--out-l0", str(lp)]) == 0
    return mp, lp


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_decompose_with_truth_stats(tmp_path, capsys, dtype):
    mp, lp = _synth(tmp_path)
    sp, outl, outs = tmp_path / "stats.json", tmp_path / "l.dmat", tmp_path / "s.dmat"
    rc = main(["decompose", str(mp), "--rank-hint", "2", "--truth", str(lp), "--out-l", str(outl), "--out-s",
               str(outs), "--stats-json", str(sp), "--dtype", dtype])
    assert rc == 0
    stats = json.loads(sp.read_text())
    assert stats["method"] == "l1-filter" and stats["rank"] == 2
    assert stats["rel_err"] <= (1e-5 if dtype == "float64" else 1e-4)
    assert stats["t"] >= stats["t1"] + stats["t2"] + stats["t_assemble"] - 1e-3
    assert json.loads(capsys.readouterr().out.strip().splitlines()[-1]) == stats
    l, s, m = matio.read_matrix(outl), matio.read_matrix(outs), matio.read_matrix(mp)
    np.testing.assert_allclose(l + s, m, rtol=0, atol=1e-3 if dtype == "float32" else 1e-10)


def test_decompose_methods_agree(tmp_path, capsys):
    mp, _ = _synth(tmp_path, seed=1)
    lf, la = tmp_path / "lf.dmat", tmp_path / "la.dmat"
    assert main(["decompose", str(mp), "--rank-hint", "2", "--out-l", str(lf)]) == 0
    assert main(["decompose", str(mp), "--method", "adm", "--out-l", str(la)]) == 0
    capsys.readouterr()
    a, b = matio.read_matrix(lf), matio.read_matrix(la)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-4


def test_decompose_exit_codes(tmp_path, capsys):
    z = tmp_path / "zero.csv"
    matio.write_matrix(z, np.zeros((20, 20)))
    assert main(["decompose", str(z), "--rank-hint", "1"]) == 0          # zero matrix: degenerate, ok
    assert main(["decompose", str(tmp_path / "missing.dmat")]) == 1      # unreadable
    mp, _ = _synth(tmp_path)
    other = tmp_path / "other.dmat"
    matio.write_matrix(other, np.zeros((3, 3)))
    assert main(["decompose", str(mp), "--truth", str(other)]) == 3      # dimension mismatch
    capsys.readouterr()


def test_synth_same_seed_identical_and_checkerboard(tmp_path, capsys):
    a, _ = _synth(tmp_path, seed=3)
    b = tmp_path / "again.dmat"
    assert main(["synth", "--m", "200", "--rho-r", "0.01", "--rho-s", "0.01", "--seed", "3", "--out-m", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()
    assert main(["checkerboard", "--m", "64", "--cell", "8", "--fraction", "0.1", "--out", str(tmp_path / "cb")]) == 0
    for suffix in ("_clean.pgm", "_corrupted.pgm", "_clean.dmat", "_corrupted.dmat", "_s0.dmat"):
        assert (tmp_path / f"cb{suffix}").exists()
    capsys.readouterr()


def test_bench_suite_reports(tmp_path, capsys):
    out_csv, out_json = tmp_path / "r.csv", tmp_path / "r.json"
    rc = main(["bench", "--suite", "size-sweep", "--scale", "0.5", "--methods", "l1filter", "adm",
               "--out-csv", str(out_csv), "--out-json", str(out_json)])
    assert rc == 0
    rep = json.loads(out_json.read_text())
    assert rep["suite"] == "size-sweep" and rep["records"]
    assert all(not r["error"] for r in rep["records"])
    assert all(r["rel_err"] <= 1e-3 for r in rep["records"])
    assert set(rep["summary"]["exponents"]) == {"l1filter", "adm"}
    assert out_csv.read_text().splitlines()[0].startswith("method,m,n,r")
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert summary["records"] == len(rep["records"])


def test_parser_rejects_unknown_suite():
    with pytest.raises(SystemExit):
        main(["bench", "--suite", "nope"])
