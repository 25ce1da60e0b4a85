"""Strong-scaling probe of the whole timed multi-GPU step on ONE GPU (only one GPU is available
this round): for N = 1, 2, 4, 8 the per-rank work of distributed.CudaShardedStep for ranks 0 and
N-1 — local seed-row gather for the column-panel exchange, row panel, paired column + row
filters on that rank's units, factors, reconstruction of the rank's row block — is timed with
CUDA events, with the two NCCL collectives replaced by device copies of the bytes the rank
would receive (recv buffer of the all-to-all, the all-gathered Q~), filled with the true values
so every filter unit iterates exactly as it would on N GPUs.

Reported per N: per-rank compute time (max of the two ranks), the bytes each rank receives in
the collectives, and the projected step = compute + those bytes at an assumed NVLink rate (an
estimate, not a measurement; nothing here runs ranks concurrently on one GPU).

    python tools/scaling_step_probe.py [config] [nvlink_GBps]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1108_5359_b200 as l1pcp  # noqa: E402
from paper_1108_5359_b200 import distributed as pdist  # noqa: E402
from paper_1108_5359_b200 import engine  # noqa: E402
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
link = float(sys.argv[2]) if len(sys.argv) > 2 else 600.0  # GB/s achieved per GPU (assumption)
cfg = BENCHMARK_CONFIGS[c]
m, n, r = cfg["m"], cfg["n"], cfg["r"]
mt, _, _, _ = engine.generate_matrix(m, n, r, cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
adm = l1pcp.AdmConfig(tol=1e-7)
fcfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=adm)
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan1 = engine.FilterPlan(m, n, seed, mt.dtype, adm, want_e=False)
big = 3 * m * n * 4 > 60e9  # cfg5: keep one L, S pair in HBM at a time
l_buf, s_buf = torch.empty_like(mt), torch.empty_like(mt)
ref = engine.solve_step(plan1, mt, l_buf, s_buf)
zc_true = ref["zc"]                                   # Q~ of every column unit (unit order)
torch.cuda.synchronize()
_a, _b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
_a.record()
for _ in range(10 if not big else 3):
    engine.solve_step(plan1, mt, l_buf, s_buf)
_b.record()
torch.cuda.synchronize()
t_single = _a.elapsed_time(_b) / (10 if not big else 3)
if big:
    del l_buf, s_buf
    ref = {k: ref[k] for k in ("zc",)}
    torch.cuda.empty_cache()
print(f"single-GPU step (engine.solve_step, streamed reconstruction): {t_single:.3f} ms")
row_idx, col_idx = seed.row_idx, seed.col_idx
ri = torch.as_tensor(row_idx, device="cuda")


class FakeDist:
    """all_to_all_single -> copy of the rank's true receive buffer (same bytes)."""

    def __init__(self):
        self.recv_true = None

    def all_to_all_single(self, recv, send, out_splits, in_splits, group=None):
        recv.copy_(self.recv_true)


fake = FakeDist()
real_dist, real_ag = pdist.dist, pdist._all_gather_rows
pdist.dist = fake
zc_all_buf = {}


def fake_all_gather(local, counts, group=None):
    buf = zc_all_buf["t"]
    buf[zc_all_buf["c0"]:zc_all_buf["c1"]].copy_(local)  # this rank's slice; the rest is the truth
    return buf


pdist._all_gather_rows = fake_all_gather
base = None
print(f"cfg{c} {m}x{n} r={r}: per-rank work of the sharded step on one GPU (collectives replaced by copies)")
for world in (1, 2, 4, 8):
    worst, rx = 0.0, 0
    for rank in sorted({0, world - 1}):
        plan = pdist.ShardPlan(m, n, rank, world, row_idx, col_idx)
        m_local = mt[plan.r0:plan.r1]
        stepper = pdist.CudaShardedStep(m_local, plan, adm, seed.u, seed.sigma, seed.v)
        c0, c1 = plan.col_units[rank]
        if world > 1:  # the true receive buffer: blocks [g][j][p_g] of M[row_idx, my_cols]
            xc_true = mt[ri][:, torch.as_tensor(plan.my_cols, device="cuda")].T.contiguous()
            counts = [int((plan.seed_owner == g).sum()) for g in range(world)]
            blocks, p0 = [], 0
            for q in counts:
                blocks.append(xc_true[:, p0:p0 + q].reshape(-1))
                p0 += q
            fake.recv_true = torch.cat(blocks)
        zc_all_buf.update(t=zc_true.clone(), c0=c0, c1=c1)
        for _ in range(3):
            stepper.step(m_local)
        torch.cuda.synchronize()
        # the timed multi-GPU bench replays the step captured in a CUDA graph (run_bench): so here
        try:
            cap = engine.CapturedCall(lambda: stepper.step(m_local))
            run = cap.replay
            form = "graph"
        except Exception as exc:  # capture unsupported: eager steps
            run, form = (lambda: stepper.step(m_local)), f"eager ({type(exc).__name__})"
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 10 if not big else 3
        a.record()
        for _ in range(steps):
            l, s, _, _ = run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        if world > 1:
            rx = max(rx, (len(plan.my_cols) * len(row_idx) + (zc_true.shape[0] - (c1 - c0)) * zc_true.shape[1]) * 4)
        if world == 1 and not big:  # the step's L must be the single-GPU solve's
            assert torch.equal(l, ref["l"]) and torch.equal(s, ref["s"])
        worst = max(worst, ms)
        del stepper, l, s
        if form == "graph":
            del cap
        torch.cuda.empty_cache()
        print(f"  N={world} rank {rank}: rows [{plan.r0}, {plan.r1}), {len(plan.my_cols)} column + "
              f"{len(plan.my_rows)} row units: {ms:.3f} ms ({form})", flush=True)
    comm_ms = rx / (link * 1e9) * 1e3
    base = base or worst
    proj = worst + comm_ms
    print(f"N={world}: per-rank compute {worst:.3f} ms (x{base / worst:.2f} over the sharded N=1 step); receives "
          f"{rx / 1e6:.1f} MB -> +{comm_ms:.3f} ms at {link:.0f} GB/s; projected step {proj:.3f} ms "
          f"(x{t_single / proj:.2f} over the single-GPU step), {m * n / (proj * 1e-3) / 1e6:.0f} M entries/s",
          flush=True)
pdist.dist, pdist._all_gather_rows = real_dist, real_ag
