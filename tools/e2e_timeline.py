"""Timeline of the pipelined host-buffer solve (engine.HostPipeline) at cfg3: per chunk, when its
H2D lands, when its L, S are computed and when its D2H ends (ms from the start), to see where the
device->host stream idles.

    python tools/e2e_timeline.py [config] [chunks]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1108_5359_b200 as l1pcp  # noqa: E402
from paper_1108_5359_b200 import engine  # noqa: E402
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = BENCHMARK_CONFIGS[c]
m, n, r = cfg["m"], cfg["n"], cfg["r"]
mt, _, _, _ = engine.generate_matrix(m, n, r, cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(m, n, seed, mt.dtype, fcfg.adm, want_e=False)
m_host = mt.cpu().pin_memory()
l_host = torch.empty((m, n), dtype=mt.dtype).pin_memory()
s_host = torch.empty((m, n), dtype=mt.dtype).pin_memory()
del mt
torch.cuda.empty_cache()
pipe = engine.HostPipeline(plan, n_chunks=chunks)
for _ in range(2):
    pipe.solve(m_host, l_host, s_host)
torch.cuda.synchronize()
# instrument: events after each chunk's H2D, compute and D2H
ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(chunks)] for k in ("h", "c", "d")}
start = torch.cuda.Event(enable_timing=True)
orig = pipe.chunks
for i, ch in enumerate(orig):
    ch["ev_h"] = ev["h"][i]
    ch["ev_c"] = ev["c"][i]
start.record()
pipe.solve(m_host, l_host, s_host)
end = torch.cuda.Event(enable_timing=True)
end.record()
torch.cuda.synchronize()
print(f"cfg{c} chunks={chunks}: total {start.elapsed_time(end):.2f} ms")
for i in range(chunks):
    print(f"  chunk {i}: H2D landed {start.elapsed_time(ev['h'][i]):7.2f}  computed {start.elapsed_time(ev['c'][i]):7.2f}")
