"""Benchmark of the l1-filtering PCP hot path on B200 (metric of BASELINE.json:
M entries/s = m*n / solve time, plus roofline fractions).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One "step" is one pass of the hot path over the synthetic input of config C (default 3):
panel gathers -> column + row ADM filtering -> rank-k factor build -> reconstruction
L = Af Bf^T, S = M - L (+ residual).  The seed PCP (t1) is solved once before the timed
steps and reported separately (solve time runs from "seed factors resident" to
"L and S written").  M (Philox, fp32) is larger than L2 for configs 2-5, so no flush is
needed between steps.

--impl reference times the reference algorithm's CPU implementation (the numpy oracle,
a restatement of /root/reference/pkg/src/l1pcp) on the host cores, on a bounded sample of
the same workload, extrapolated to the full matrix.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "M entries/s (m*n / solve time)"
UNIT = "M entries/s"
TOL = 1e-7  # BASELINE.json: ALM tolerance 1e-7


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-chunks", type=int, default=8, help="row chunks of the pipelined host-buffer solve")
    p.add_argument("--no-extra", action="store_true", help="skip the cfg5 sub-object and the FP64 API legs")
    return p.parse_args()


def cfg_of(c):
    from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
    return dict(BENCHMARK_CONFIGS[c])


def workload_name(cfg):
    return (f"{cfg['name']}: {cfg['m']}x{cfg['n']} r={cfg['r']} "
            f"{'video boxes' if cfg['kind'] else f'rho_s={cfg['rho_s']}'} seed {10 * cfg['r']}^2 tol {TOL}")


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.pre = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes ~0.1-0.3 s to print its first sample: start timing only once it
            # samples, so a short timed region still gets samples (the prior ones are dropped)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.005)
            self.pre = list(self.lines)  # the sample just before the timed region
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        window = "timed region"
        if not self.lines and getattr(self, "pre", None):  # region shorter than the 10 ms sampling period
            self.lines, window = self.pre, "sample taken just before the timed region (region < sampling period)"
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# ---------------------------------------------------------------- CPU legs (bench_cpu.py)
def cpu_leg(cfgd, seed_np, steps, target_s, ref=None, kind=None, validate=True):
    """Time the reference's own code (oracle/_ref, else the port) on bounded samples of the
    workload: returns (per-step extrapolated seconds, description dict)."""
    import bench_cpu
    if ref is None:
        ref, kind = bench_cpu.load_reference()
    wl = bench_cpu.Workload(cfgd, seed=seed_np, ref=ref)
    probe = 256
    best, settings = bench_cpu.pick_threads(ref, wl, probe)
    t_probe = settings[best.label()]["t_est_s"]
    # size the per-step sample so one step takes about target_s of CPU time
    per_unit = t_probe / (wl.comp_c.size + wl.comp_r.size)  # incl. the assembly share
    units = int(max(64, min(wl.comp_c.size, target_s / max(per_unit, 1e-9) / 2)))
    units = 64 * max(1, units // 64)
    t_est, t_sample = [], []
    for i in range(steps):
        out = bench_cpu.sample_step(ref, wl, units, best, rng_seed=1 + i)
        t_est.append(out["t_est"])
        t_sample.append(out["t_sample"])
    val = None
    if validate:
        from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
        small = dict(BENCHMARK_CONFIGS[2])
        if cfgd["name"] != small["name"]:
            val = bench_cpu.validate_extrapolation(ref, kind, small, min(units, 1024), best)
    desc = {"kind": kind, "cores": max(best.blas, best.parallelism), "threads": best.label(),
            "threading_settings": settings,
            "sample": (f"per step: the reference's filter_columns on {out['units'][0]} and filter_rows on "
                       f"{out['units'][1]} sampled units, nystrom_complete + assemble + m - l on the "
                       f"{out['sub_entries']}-entry sub-matrix (seed + sampled rows x cols); extrapolated per unit "
                       f"to {wl.comp_c.size} + {wl.comp_r.size} units and per entry to {wl.m}x{wl.n}; seed excluded "
                       f"(as in the GPU arm)"),
            "sample_seconds_per_step": float(np.mean(t_sample)), "extrapolation_factor":
                float(np.mean(t_est) / max(np.mean(t_sample), 1e-12)),
            "extrapolation_check": val, "cpu": bench_cpu.cpu_info()}
    return t_est, desc


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref) on this workload.  With
    enough host RAM the K timed steps together run the reference pipeline after the seed over the
    WHOLE matrix once (bench_cpu.full_measure: a measurement, not an extrapolation); otherwise each
    step is a bounded sample extrapolated per unit / per entry."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import bench_cpu
    cfgd = cfg_of(args.config)
    m, n = cfgd["m"], cfgd["n"]
    ref, kind = bench_cpu.load_reference()
    t0 = time.perf_counter()
    wl = bench_cpu.Workload(cfgd, ref=ref)  # the reference's own seed stage, untimed (as in the GPU arm)
    t_seed = time.perf_counter() - t0
    need = 6 * m * n * 8  # M, L, S, completion and the gathers, float64
    if kind == "reference" and need < 0.6 * _host_ram_bytes():
        best, settings = bench_cpu.pick_threads(ref, wl, 256)
        t0 = time.perf_counter()
        m_full = bench_cpu.host_matrix(wl)
        t_regen = time.perf_counter() - t0
        times, detail = bench_cpu.full_measure(ref, wl, m_full, best, args.steps, args.warmup)
        del m_full
        t = float(np.sum(times)) / args.steps
        total = float(np.sum(times))
        desc = {"kind": kind, "cores": max(best.blas, best.parallelism), "threads": best.label(),
                "threading_settings": settings,
                "sample": (f"whole matrix: the {args.steps} timed steps together run the reference's panel gathers, "
                           f"filter_columns / filter_rows on all {detail['units'][0]} + {detail['units'][1]} units "
                           f"(1/{args.steps} per step) and nystrom_complete + assemble + m - l on the full {m}x{n} "
                           f"(last step); seed excluded (as in the GPU arm)"),
                "measured": detail, "seed_s_untimed": t_seed, "regen_s_untimed": t_regen,
                "cpu": bench_cpu.cpu_info()}
        value = m * n / total / 1e6
    else:
        steps = args.warmup + args.steps
        target = float(np.clip(150.0 / max(steps, 1), 1.0, 8.0))
        t_est, desc = cpu_leg(cfgd, wl.seed, steps, target, ref=ref, kind=kind)
        t = float(np.mean(t_est[args.warmup:] or t_est))
        value = m * n / t / 1e6
        desc["seed_s_untimed"] = t_seed
    desc.update(value=value, unit=UNIT)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox, BASELINE.json config, regenerated on host)",
            "config": {"workload": workload_name(cfgd), "parallelism": f"cpu {desc['threads']}"},
            "impl": "reference", "cpu_baseline": desc,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or os.environ.get("L1F_FORCE_SHARDED") == "1":  # the latter: test the N-GPU driver on 1 GPU
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_1108_5359_b200 import distributed as pdist
        return pdist.run_bench(args, rank, world, clock_sampler=ClockSampler)
    from paper_1108_5359_b200 import engine
    fma_tflops = engine.fma_peak_tflops()
    line = measure_config(cfg_of(args.config), args, fma_tflops, e2e=not args.no_e2e,
                          cpu=None if args.no_cpu_baseline else "full", local=local)
    torch.cuda.empty_cache()
    if not args.no_extra:
        # the reference's own contract (numpy float64 in / out, FP64 kernels) through the public call
        line["fp64_api"] = {f"cfg{c}": fp64_api_leg(cfg_of(c)) for c in (2, 3)}
        torch.cuda.empty_cache()
        if args.config != 5:
            # BASELINE's largest single-GPU config, timed in the same run
            sub = measure_config(cfg_of(5), argparse.Namespace(**{**vars(args), "steps": min(args.steps, 5)}),
                                 fma_tflops, e2e=False, cpu=None if args.no_cpu_baseline else "sample",
                                 local=local)
            keep = ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "config", "roofline",
                    "roofline_tensor", "roofline_reconstruct", "generate", "phases_ms", "filter", "value_incl_seed",
                    "recovery_rel_err", "gpu_launches", "clocks", "cpu_baseline")
            line["cfg5"] = {k: sub[k] for k in keep if k in sub}
    print(json.dumps(line))
    return 0


def measure_config(cfgd, args, fma_tflops, e2e=True, cpu="full", local=0):
    """The timed hot path on one GPU for one BASELINE config; returns the JSON line (dict)."""
    import torch

    import paper_1108_5359_b200 as l1pcp
    from paper_1108_5359_b200 import engine

    m, n, r = cfgd["m"], cfgd["n"], cfgd["r"]
    peaks = measured_peaks()

    # input: Philox on the device
    t0 = time.perf_counter()
    mt, _, _, _ = engine.generate_matrix(m, n, r, cfgd["rho_s"], cfgd["magnitude"], seed=0, kind=cfgd["kind"])
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    # generation roofline (K1): a warm, event-timed regeneration of M, 4 B written per entry
    ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ga.record()
    engine.generate_matrix(m, n, r, cfgd["rho_s"], cfgd["magnitude"], seed=0, kind=cfgd["kind"], out=mt)
    gb.record()
    torch.cuda.synchronize()
    gen_ms = ga.elapsed_time(gb)

    fcfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=TOL))
    kind, seed, attempts, t1_first = engine.seed_stage(mt, fcfg)
    if kind != "seed":
        raise RuntimeError(f"seed stage ended in {kind}")
    # t1 = the median of three more seed solves on the same matrix (the first call of the process
    # also pays one-time kernel loading and memory-pool growth, reported as t1_first_call_s)
    t1_runs = [engine.seed_stage(mt, fcfg)[3] for _ in range(3)]
    t1 = float(np.median(t1_runs))
    plan = engine.FilterPlan(m, n, seed, mt.dtype, fcfg.adm, want_e=False)
    l_out = torch.empty_like(mt)
    s_out = torch.empty_like(mt)
    stream = torch.cuda.current_stream()

    def step(evs=None):
        f = engine.solve_step(plan, mt, l_out, s_out, evs)
        return f, f["resid_sq"]

    # warm-up steps, eager, with CUDA events around the phases (kernel times for the rooflines;
    # a graph replay carries no timing events)
    n_ev = max(args.warmup, 5)
    ev_all = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n_ev)]
    for i in range(n_ev):
        # a short device-side spin first, so the whole step is enqueued before it starts: the
        # events then time the GPU work, not host enqueue gaps (small configs are launch-bound)
        torch.cuda._sleep(4_000_000)
        f, rs = step(ev_all[i])
        torch.cuda.synchronize()
    ev_all = ev_all[1:]  # the first eager step carries one-time costs
    # the timed steps replay the step captured into a CUDA graph (engine.CapturedStep): the same
    # kernels on the same buffers without per-step host work
    try:
        graph = engine.CapturedStep(plan, mt, l_out, s_out)
        step_form = "CUDA graph of engine.solve_step (engine.CapturedStep), replayed per timed step"
    except Exception as exc:  # capture unavailable: eager steps (same kernels, host enqueue per step)
        graph, step_form = None, f"eager engine.solve_step ({type(exc).__name__} at graph capture)"
        torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            f = graph.replay() if graph is not None else step()[0]
        end.record(stream)
        torch.cuda.synchronize()
    rs = f["resid_sq"]
    ms = start.elapsed_time(end) / args.steps
    # median over the eager steps: an eager launch occasionally runs ~2x long (seen on either
    # filter, never in the graph-replayed timed steps); the samples are reported beside it
    def _med(xs):
        return float(np.median(xs))
    filter_samples = [round(e[1].elapsed_time(e[2]), 4) for e in ev_all]
    t_filter_only = _med([e[1].elapsed_time(e[2]) for e in ev_all])
    streamed = bool(f.get("streamed"))
    if streamed:
        # the reconstruction runs beside the row filter; time the same kernel family alone for
        # its HBM roofline (outside the timed steps), and report the exposed tail of the step
        t_tail = float(_med([e[2].elapsed_time(e[4]) for e in ev_all]))
        af_s, bf_s = engine.build_factors(plan, f["zc"], f["zr"])
        ra, rb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        engine.reconstruct(mt, af_s, bf_s, l_out, s_out)
        reps = 5
        ra.record(stream)
        for _ in range(reps):
            engine.reconstruct(mt, af_s, bf_s, l_out, s_out)
        rb.record(stream)
        torch.cuda.synchronize()
        t_recon = ra.elapsed_time(rb) / reps
        del af_s, bf_s
        f = graph.replay() if graph is not None else step()[0]  # L, S again (the recovery check reads l_out)
        rs = f["resid_sq"]
        torch.cuda.synchronize()
    else:
        t_recon = _med([e[3].elapsed_time(e[4]) for e in ev_all])
        t_tail = t_recon
    value = m * n / (ms * 1e-3) / 1e6

    # algorithmic work of the dominant kernel: sum_u it_u * s * (4k + 12)
    k = seed.r_prime
    itc = f["iters_c"].double().sum().item()
    itr = f["iters_r"].double().sum().item()
    s_r, s_c = len(seed.row_idx), len(seed.col_idx)
    flops = itc * s_r * (4 * k + 12) + itr * s_c * (4 * k + 12)
    achieved = flops / (t_filter_only * 1e-3) / 1e12
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    recon_bytes = 12.0 * m * n
    recon_gbs = recon_bytes / (t_recon * 1e-3) / 1e9
    failed = int(((f["status_c"] == 1) | (f["status_c"] == 2)).sum().item()
                 + ((f["status_r"] == 1) | (f["status_r"] == 2)).sum().item())
    r2, m2 = rs.cpu().tolist()
    if not np.isfinite(r2):  # a timed-out overlapped wait (L1F_OPT_WAIT_TIMEOUT_MS): L, S not trustworthy
        raise RuntimeError("residual is not finite: an overlapped device wait timed out; no bench line")

    # recovery error vs L0 (reported, not gated): regenerate L0 on the device
    rel = recovery_error(cfgd, l_out)

    del graph  # its private memory pool (the step's temporaries) before the e2e and cfg5 legs
    torch.cuda.empty_cache()
    # e2e: host (pinned) M in, L and S out, through the public estimate_rank_and_solve
    e2e_line = None
    if e2e and 3 * mt.numel() * mt.element_size() > 0.5 * _host_ram_bytes():
        e2e_line = {"value": None, "unit": UNIT, "skipped": "3 pinned host copies of M exceed half the host RAM"}
    elif e2e:
        seed_np = None
        del l_out, s_out
        torch.cuda.empty_cache()
        e2e_line = run_e2e_public(mt, fcfg, args)
        l_out = s_out = None

    cpu_line = None
    if cpu:
        seed_np = {"row_idx": seed.row_idx, "col_idx": seed.col_idx, "u": seed.u.cpu().numpy(),
                   "sigma": seed.sigma.cpu().numpy(), "v": seed.v.cpu().numpy(), "seed_l": seed.seed_l.cpu().numpy()}
        cpu_line = cpu_baseline_leg(cfgd, seed_np, cpu)

    small_k = plan.filter_dtype == torch.float64
    if streamed:
        if small_k:  # 2 gathers; unit scale + filter x 2; gate, Bf, strip index, concurrent + trailing
            launches_per_step = 2 + 4 + 6  # reconstruction, residual sum
        else:  # column gather; unit scale + column filter, gate + row gather beside it; unit scale + row
            # filter, gate, Bf, strip index, Bf split, concurrent + trailing reconstruction, residual sum
            launches_per_step = 1 + 4 + 9  # = 14, profiles/r1_launches_cfg3_v5.csv
        phases = {"gather": float(_med([e[0].elapsed_time(e[1]) for e in ev_all])),
                  "column_filter": float(_med([e[1].elapsed_time(e[3]) for e in ev_all])),
                  "row_filter": float(_med([e[3].elapsed_time(e[2]) for e in ev_all])), "filter_samples_ms": filter_samples,
                  "filters": t_filter_only,
                  "reconstruct_exposed": t_tail,
                  "reconstruct_standalone": t_recon,
                  "note": ("the reconstruction of each 128-row strip runs beside the row filter (on the same SMs "
                           "as its blocks) once the strip's row units are done; the rest after it" if small_k else
                           "the reconstruction of each 128-row strip runs beside the row filter on the SMs its "
                           "clusters leave free once the strip's row units are done; the rest after it"),
                  "t1_seed_s": t1, "t1_runs_s": t1_runs, "t1_first_call_s": t1_first, "generate_s": t_gen}
    else:
        launches_per_step = 2 + 2 * 2 + 1 + 4  # gathers, (unit scale + filter) x 2, factors, split x 2 + recon + sum
        phases = {"gather": float(_med([e[0].elapsed_time(e[1]) for e in ev_all])),
                  "filters": t_filter_only, "filter_samples_ms": filter_samples, "factors": float(_med([e[2].elapsed_time(e[3]) for e in ev_all])),
                  "reconstruct": t_recon, "t1_seed_s": t1, "t1_runs_s": t1_runs, "t1_first_call_s": t1_first,
                  "generate_s": t_gen}
    traffic = ncu_traffic(cfgd)
    fp64_filter = plan.filter_dtype == torch.float64
    fp64_tflops = engine.fma_peak_tflops(fp64=True) if fp64_filter else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Philox4x64-10 on device; BASELINE.json config statistics)",
        "config": {"workload": workload_name(cfgd), "m": m, "n": n, "rank": r, "seed_block": [s_r, s_c],
                   "r_prime": k, "tol": TOL, "parallelism": "1 GPU",
                   "filter_dtype": "f64" if plan.filter_dtype == torch.float64 else "f32",
                   "l2": "inputs larger than L2 (M is %.1f GB)" % (m * n * 4 / 1e9)},
        "roofline": ({"bound": "fp64", "kernel": "adm_small_kernel, FP64 (column + row filters)",
                      "achieved": achieved, "peak": fp64_tflops, "unit": "TFLOP/s", "frac": achieved / fp64_tflops,
                      "peak_source": "measured FP64 FMA probe (l1f_fma_peak_probe_f64, this run)",
                      "peak_nominal": 148 * 64 * 2 * 1.965e9 / 1e12, "fp32_frac": achieved / fma_tflops}
                     if fp64_filter else
                     {"bound": "fp32", "kernel": "adm_tc_kernel, tcgen05 bf16x3 (column + row filters)",
                      "achieved": achieved, "peak": fma_tflops, "unit": "TFLOP/s", "frac": achieved / fma_tflops,
                      "peak_source": "measured FP32 FMA probe (l1f_fma_peak_probe, this run)",
                      "peak_nominal": 148 * 128 * 2 * 1.965e9 / 1e12}) | {
                     "traffic": traffic.get("filter", {}).get("dram_bytes_per_launch"),
                     "traffic_source": traffic.get("filter", {}).get("source"),
                     "algorithmic_flops_per_step": flops, "kernel_ms_per_step": t_filter_only,
                     "kernel_ms_source": "CUDA events around the filter launches of eager steps of the same step "
                                         "(the timed steps are CUDA-graph replays, which carry no timing events)"},
        "roofline_tensor": tensor_roofline(plan, seed, itc, itr, t_filter_only, peaks),
        "generate": {"bound": "fp32" if r > 16 else "hbm", "ms": gen_ms,
                     "gbs": 4.0 * m * n / (gen_ms * 1e-3) / 1e9, "hbm_frac": 4.0 * m * n / (gen_ms * 1e-3) / 1e9 / hbm,
                     "tflops": 2.0 * r * m * n / (gen_ms * 1e-3) / 1e12,
                     "fp32_frac": 2.0 * r * m * n / (gen_ms * 1e-3) / 1e12 / fma_tflops,
                     "note": "Philox M = L0 + S0 written once (4 B/entry); L0 = X Y^T costs 2r flops/entry, done "
                             "as separate mul/add in k order so the numpy oracle regenerates M bit for bit: "
                             "compute-bound for r > 16; outside the timed step"},
        "roofline_reconstruct": {"bound": "hbm", "achieved": recon_gbs, "peak": hbm, "unit": "GB/s",
                                 "frac": recon_gbs / hbm, "bytes_per_step": recon_bytes, "kernel_ms_per_step": t_recon,
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                                 "traffic": traffic.get("reconstruct", {}).get("dram_bytes_per_launch"),
                                 "traffic_source": traffic.get("reconstruct", {}).get("source")},
        "phases_ms": phases,
        "filter": {"units": int(f["iters_c"].numel() + f["iters_r"].numel()),
                   "mean_iters": (itc + itr) / max(1, f["iters_c"].numel() + f["iters_r"].numel()),
                   "max_iters": int(max(f["iters_c"].max().item(), f["iters_r"].max().item())),
                   "failed_units": failed},
        # one-shot solve including the seed PCP (t1), for a single call on a fresh matrix
        "value_incl_seed": m * n / (ms * 1e-3 + t1) / 1e6,
        "recovery_rel_err": rel, "residual": float(np.sqrt(r2 / m2)) if m2 else 0.0,
        "gpu_launches": launches_per_step * args.steps,
        "step_form": step_form,
        "untimed_steps": f"{n_ev} eager steps with phase events (median of the last {n_ev - 1} for the kernel times) + 1 graph capture before the {args.steps} timed steps",
        "clocks": clk.summary(),
        "cpu_baseline": cpu_line,
        "e2e": e2e_line,
    }
    del mt, plan, f
    return line


def cpu_baseline_leg(cfgd, seed_np, mode):
    """cpu_baseline of our line: the reference's own code on the host cores, rank 0 at N=1.
    mode "full": the whole matrix once when host RAM allows (else a sample); "sample": a bounded
    sample extrapolated per unit / per entry, with the extrapolation checked on cfg2."""
    import bench_cpu
    ref, kind = bench_cpu.load_reference()
    m, n = cfgd["m"], cfgd["n"]
    if mode == "full" and kind == "reference" and 6 * m * n * 8 < 0.6 * _host_ram_bytes():
        wl = bench_cpu.Workload(cfgd, seed=seed_np, ref=ref)
        best, settings = bench_cpu.pick_threads(ref, wl, 256)
        m_full = bench_cpu.host_matrix(wl)
        times, detail = bench_cpu.full_measure(ref, wl, m_full, best, 4, 0)
        del m_full
        total = float(np.sum(times))
        return {"value": m * n / total / 1e6, "unit": UNIT, "kind": kind, "cores": max(best.blas, best.parallelism),
                "threads": best.label(), "threading_settings": settings,
                "sample": "whole matrix after the seed (the reference's gathers, filter_columns / filter_rows on all "
                          "units, nystrom_complete + assemble + m - l), measured once; seed factors = this run's",
                "measured": detail, "cpu": bench_cpu.cpu_info()}
    t_est, desc = cpu_leg(cfgd, seed_np, 1, 12.0, ref=ref, kind=kind, validate=True)
    desc.update(value=m * n / t_est[0] / 1e6, unit=UNIT)
    return desc


def fp64_api_leg(cfgd):
    """The reference's own contract through the public call: a numpy float64 M in, float64 numpy
    L, S out (FP64 kernels), FilterConfig(rank_hint=r, tol=1e-7).  Host->device and device->host
    copies are inside; the seed (t1) is included and reported."""
    import torch

    import paper_1108_5359_b200 as l1pcp
    from paper_1108_5359_b200 import engine
    m, n, r = cfgd["m"], cfgd["n"], cfgd["r"]
    mt, _, _, _ = engine.generate_matrix(m, n, r, cfgd["rho_s"], cfgd["magnitude"], seed=0, kind=cfgd["kind"])
    m_np = mt.double().cpu().numpy()
    del mt
    torch.cuda.empty_cache()
    cfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=TOL))
    l1pcp.estimate_rank_and_solve(m_np[:2000, :2000], cfg)  # warm-up (library start-up)
    torch.cuda.synchronize()
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        sol = l1pcp.estimate_rank_and_solve(m_np, cfg)
        el = time.perf_counter() - t0
        if best is None or el < best[0]:
            best = (el, sol.stats)
        del sol
    el, st = best
    return {"value_incl_seed": m * n / el / 1e6, "value_excl_seed": m * n / (el - st["t1"]) / 1e6, "unit": UNIT,
            "elapsed_s": el, "t1_s": st["t1"], "t2_s": st["t2"], "t_assemble_s": st["t_assemble"],
            "dtype": "f64", "h2d_bytes": m * n * 8, "d2h_bytes": 2 * m * n * 8,
            "path": "numpy float64 -> as_dense (host) -> device FP64 seed, filters, reconstruction -> numpy L, S"}


def ncu_traffic(cfgd):
    """Per-launch DRAM bytes of the dominant kernels from the committed ncu capture of this
    workload (profiles/ncu_traffic.json), or {} when none was taken."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(cfgd["name"], {})
    except (OSError, ValueError, KeyError):
        return {}


def tensor_roofline(plan, seed, itc, itr, t_ms, peaks):
    """The filter against the tensor-core peak (report vs both peaks when tensor cores
    are used): executed bf16 MMA flops of the tcgen05 filter (csrc/filter_tc.cu variant selection,
    padding included) over the filter time, vs the sustained bf16 GEMM peak."""
    import math

    import torch
    k = seed.r_prime
    if plan.filter_dtype != torch.float32 or k <= 16 or k > 224:
        return None
    if k <= 112:
        kp = 16 * math.ceil(k / 16)
    elif k <= 160:
        kp = 32 * math.ceil(k / 32)
    else:
        kp = 16 * math.ceil(k / 16)
    pc = 3  # residual-form phase c: a0 v0 + a0 v1 + a1 v0 (phase a: the 6 products of 3 x 3 pieces)
    mtc = math.ceil(kp / 128)
    flops = 0.0
    for it_sum, s_units in ((itc, len(seed.row_idx)), (itr, len(seed.col_idx))):
        rows = 128 * math.ceil(s_units / 128)
        flops += float(it_sum) * 2.0 * rows * (6 * kp + pc * 128 * mtc)
    peak = float(peaks.get("bf16_tflops_sustained", 1397.0))
    ach = flops / (t_ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained", "executed_mma_flops_per_step": flops,
            "note": "bf16 pieces: 6 products in phase a, 3 in the residual-form phase c, 128-row tiles"}


def run_e2e_public(mt, fcfg, args):
    """The same workload end to end through the PUBLIC call a user makes:
    estimate_rank_and_solve(M) with M a float32 tensor in pinned host memory -> L, S pinned host
    tensors (l1filter._solve_host_tensor -> engine.HostPipeline: zero-copy seed block and column
    panel, chunked H2D / compute / D2H overlap).  Copies are inside the timed region.  `value`
    excludes the seed stage (t1, as the device-resident `value` does; timed on the device from the
    call's own events), `value_incl_seed` is the whole call by wall clock."""
    import torch

    import paper_1108_5359_b200 as l1pcp
    m_host = torch.empty(mt.shape, dtype=mt.dtype, pin_memory=True)
    m_host.copy_(mt)
    torch.cuda.synchronize()
    sol = l1pcp.estimate_rank_and_solve(m_host, fcfg)  # warm-up: pipeline buffers, pinned output pool
    assert sol.stats.get("path") == "host-pipeline", sol.stats
    del sol
    steps = max(1, min(args.steps, 3))
    t_solve, t_call = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        sol = l1pcp.estimate_rank_and_solve(m_host, fcfg)
        t_call.append(time.perf_counter() - t0)
        t_solve.append(sol.stats["t2"])  # device events around the pipelined solve (copies included)
        _ = float(sol.final_residual)   # device -> host read of the step's result
        del sol
    ms = float(np.mean(t_solve)) * 1e3
    nbytes = mt.numel() * mt.element_size()
    return {"value": mt.numel() / (ms * 1e-3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": 2 * nbytes, "ms_per_step": ms, "steps": steps,
            "value_incl_seed": mt.numel() / float(np.mean(t_call)) / 1e6, "call_s": float(np.mean(t_call)),
            "api": "paper_1108_5359_b200.estimate_rank_and_solve(pinned float32 host tensor) -> pinned host L, S",
            "path": "zero-copy seed block + column panel -> chunked H2D -> filters/factors/reconstruct per chunk -> "
                    "chunked D2H of L, S (engine.HostPipeline)"}


def _host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        return 0


def recovery_error(cfgd, l_out):
    import torch
    from paper_1108_5359_b200 import engine
    m, n = l_out.shape
    rows = min(m, 4096)
    _, l0, _, _ = engine.generate_matrix(cfgd["m"], cfgd["n"], cfgd["r"], cfgd["rho_s"], cfgd["magnitude"], seed=0,
                                         kind=cfgd["kind"], rows=rows, want_l0=True)
    out = engine.rel_err_device(l_out[:rows].contiguous(), l0)
    del l0
    torch.cuda.empty_cache()
    return {"value": out, "rows_checked": rows}


def _json_stdout():
    """Keep stdout for the one JSON line: library output written straight to file descriptor 1
    (e.g. NCCL's version banner at communicator setup) is sent to stderr instead."""
    try:
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        sys.stdout = os.fdopen(saved, "w", buffering=1)
    except OSError:
        pass


def main():
    args = parse()
    _json_stdout()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
