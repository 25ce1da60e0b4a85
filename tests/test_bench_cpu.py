"""Host logic of the CPU reference arm (bench_cpu.py): the staged reference package times the
pipeline after the seed on a tiny Philox matrix — whole-matrix mode split across steps, the
sampled mode and its extrapolation check.  No GPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench_cpu  # noqa: E402

TINY = dict(name="tiny", m=320, n=300, r=4, rho_s=0.05, magnitude=500.0, kind=0)


@pytest.fixture(scope="module")
def ref():
    mod, kind = bench_cpu.load_reference()
    if kind != "reference":
        pytest.skip("oracle/_ref not staged (build() stages it from /root/reference)")
    return mod


def test_workload_regenerates_the_device_matrix_and_seeds_like_the_reference(ref):
    wl = bench_cpu.Workload(TINY, ref=ref)
    m = bench_cpu.host_matrix(wl, threads=3)
    np.testing.assert_array_equal(m[np.ix_([0, 7, 319], [1, 2, 299])], wl.block(np.array([0, 7, 319]),
                                                                                   np.array([1, 2, 299])))
    # the reference's own pipeline on the same M picks the same seed block and rank
    sol = ref.estimate_rank_and_solve(m, ref.FilterConfig(rank_hint=4, rng_seed=0,
                                                          adm=ref.AdmConfig(tol=bench_cpu.TOL)))
    assert sol.stats["seed_rows"] == wl.seed["row_idx"].size and sol.rank_of_l == wl.seed["sigma"].size


def test_full_measure_covers_every_unit_once(ref):
    wl = bench_cpu.Workload(TINY, ref=ref)
    m = bench_cpu.host_matrix(wl)
    times, detail = bench_cpu.full_measure(ref, wl, m, bench_cpu.Threads(1, 2), steps=3, warmup=1)
    assert len(times) == 3 and all(t > 0 for t in times)
    assert detail["units"] == [wl.comp_c.size, wl.comp_r.size]
    assert detail["t_assemble_s"] > 0 and abs(sum(times) - detail["t_total_s"]) < 1e-9


def test_sampled_mode_and_extrapolation_check(ref):
    wl = bench_cpu.Workload(TINY, ref=ref)
    out = bench_cpu.sample_step(ref, wl, 64, bench_cpu.Threads(1, 1))
    assert out["units"] == [64, 64] and out["t_est"] > out["t_sample"] > 0
    best, settings = bench_cpu.pick_threads(ref, wl, 32)
    assert set(settings) == {"blas=1,parallelism=1", f"blas={os.cpu_count() and len(os.sched_getaffinity(0))},"
                             f"parallelism={len(os.sched_getaffinity(0))}",
                             f"blas=1,parallelism={len(os.sched_getaffinity(0))}"}
    chk = bench_cpu.validate_extrapolation(ref, "reference", TINY, 64, best)
    assert chk["full_s"] > 0 and np.isfinite(chk["rel_err"])


def test_reference_arm_json_contract():
    """`bench.py --impl reference` (the driver's reference arm) on config 1: one JSON line with the
    contract's keys, timed on the staged reference package (kind "reference")."""
    import json
    import subprocess
    if not os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "l1pcp")):
        pytest.skip("oracle/_ref not staged")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
