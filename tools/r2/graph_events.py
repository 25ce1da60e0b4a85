import sys, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
l, s = torch.empty_like(mt), torch.empty_like(mt)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for _ in range(2): engine.solve_step(plan, mt, l, s, ev)
torch.cuda.synchronize()
print("eager", [round(ev[0].elapsed_time(e), 3) for e in ev[1:]])
g = torch.cuda.CUDAGraph()
evg = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g):
    f = engine.solve_step(plan, mt, l, s, evg)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
try:
    print("graph", [round(evg[0].elapsed_time(e), 3) for e in evg[1:]])
except Exception as ex:
    print("graph events failed:", ex)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): g.replay()
b.record(); torch.cuda.synchronize()
a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a2.record()
for _ in range(20): engine.solve_step(plan, mt, l, s)
b2.record(); torch.cuda.synchronize()
print(f"cfg{c}: graph {a.elapsed_time(b)/20:.3f} ms/step, eager {a2.elapsed_time(b2)/20:.3f} ms/step")
