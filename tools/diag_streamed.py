"""Diagnostics of the streamed row filter + reconstruction on a BASELINE config (1 GPU):
step time with the concurrent reconstruction on / off and the classic path, plus the library's
L1F_RECON_DEBUG per-launch report (items, claim / finish times, split and wait costs)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_5359_b200 as l1pcp  # noqa: E402
from paper_1108_5359_b200 import engine  # noqa: E402
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = BENCHMARK_CONFIGS[cfg]
m, n, r = c["m"], c["n"], c["r"]
mt, _, _, _ = engine.generate_matrix(m, n, r, c["rho_s"], c["magnitude"], seed=0, kind=c["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(m, n, seed, mt.dtype, fcfg.adm, want_e=False)
l_out, s_out = torch.empty_like(mt), torch.empty_like(mt)
print("streamed_ok", engine._streamed_ok(plan, mt), "small", engine._streamed_small_ok(plan, mt))


def run(label, env, force, reps=5):
    old = dict(os.environ)
    os.environ.update(env)
    ok, oks = engine._streamed_ok, engine._streamed_small_ok
    if force is not None:
        engine._streamed_ok = lambda p, t: force and p.filter_dtype == torch.float32
        engine._streamed_small_ok = lambda p, t: force and p.filter_dtype == torch.float64
    try:
        for _ in range(2):
            engine.solve_step(plan, mt, l_out, s_out)
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(reps)]
        for e in evs:
            engine.solve_step(plan, mt, l_out, s_out, e)
        torch.cuda.synchronize()
        step = sum(e[0].elapsed_time(e[4]) for e in evs) / reps
        filt = sum(e[1].elapsed_time(e[2]) for e in evs) / reps
        tail = sum(e[2].elapsed_time(e[4]) for e in evs) / reps
        extra = ""
        if force:
            colf = sum(e[1].elapsed_time(e[3]) for e in evs) / reps
            rowf = sum(e[3].elapsed_time(e[2]) for e in evs) / reps
            extra = f" (column filter + Bf {colf:.3f}, row filter {rowf:.3f})"
        print(f"{label}: step {step:.3f} ms, gathers->filters done {filt:.3f} ms{extra}, tail {tail:.3f} ms", flush=True)
        if env.get("L1F_RECON_DEBUG") != "1" and force:
            os.environ["L1F_RECON_DEBUG"] = "1"
            engine.solve_step(plan, mt, l_out, s_out)
            torch.cuda.synchronize()
    finally:
        engine._streamed_ok, engine._streamed_small_ok = ok, oks
        os.environ.clear()
        os.environ.update(old)


run("classic", {}, False)
run("streamed, concurrent", {}, True)
run("streamed, post only", {"L1F_RECON_CONCURRENT": "0"}, True)
