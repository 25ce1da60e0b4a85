"""Row-sharded multi-GPU l1-filtering solve, one process per GPU.

Rank g owns the row block [r0_g, r1_g) of M.  The exchange steps are the ones the algorithm
has; everything else is local:

  1. all-gather of the seed rows M[row_idx, :]   (each rank contributes the seed rows it owns)
  2. rank 0 solves the seed PCP on M[row_idx, col_idx]; U, sigma, V are broadcast
  3. column units (all non-seed columns) are split evenly across ranks; row units are the
     non-seed rows of each rank's own block                          (local ADM filters)
  4. all-gather of the column coefficients Q~ (unit-major Zc) so every rank can build the
     column factors Bf for all n columns
  5. each rank reconstructs L and S = M - L for its own rows            (local)
  6. all-reduce of the statistics (max iterations, failed units)

Per-unit results do not depend on the partition, so L/S are bitwise identical for any
world size.  Compute goes through a backend object (``CudaBackend`` in production: the C-ABI
kernels over NCCL tensors); tests substitute a CPU backend under gloo to check the plumbing.
"""

import time
from dataclasses import dataclass

import numpy as np

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


def row_ranges(m, world):
    """Contiguous, balanced row blocks [r0, r1) per rank."""
    base, extra = divmod(m, world)
    out, r0 = [], 0
    for g in range(world):
        r1 = r0 + base + (1 if g < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


def unit_ranges(n_units, world):
    return row_ranges(n_units, world)


@dataclass
class ShardPlan:
    m: int
    n: int
    rank: int
    world: int
    row_idx: np.ndarray
    col_idx: np.ndarray

    def __post_init__(self):
        self.rows = row_ranges(self.m, self.world)
        self.r0, self.r1 = self.rows[self.rank]
        self.comp_cols = np.setdiff1d(np.arange(self.n), self.col_idx)
        self.col_units = unit_ranges(self.comp_cols.size, self.world)
        c0, c1 = self.col_units[self.rank]
        self.my_cols = self.comp_cols[c0:c1]
        comp_rows = np.setdiff1d(np.arange(self.m), self.row_idx)
        self.my_rows = comp_rows[(comp_rows >= self.r0) & (comp_rows < self.r1)]
        # seed rows owned by each rank, in global row order
        self.seed_owner = np.searchsorted([r1 for _, r1 in self.rows], self.row_idx, side="right")
        self.my_seed_pos = np.flatnonzero(self.seed_owner == self.rank)


def _all_gather_rows(local, counts, group=None):
    """All-gather of variable-height row blocks (padded to the largest)."""
    world = len(counts)
    width = local.shape[1]
    hmax = max(max(counts), 1)
    pad = local.new_zeros((hmax, width))
    pad[: local.shape[0]] = local
    bufs = [local.new_empty((hmax, width)) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def gather_seed_rows(m_local, plan, group=None):
    """Exchange 1: M[row_idx, :] on every rank (each rank contributes the seed rows it owns)."""
    local = m_local[torch.as_tensor(plan.row_idx[plan.my_seed_pos] - plan.r0, device=m_local.device)]
    counts = [int((plan.seed_owner == g).sum()) for g in range(plan.world)]
    return _all_gather_rows(local, counts, group)


def seed_factors(seed_rows, plan, backend, adm, rank_tol=1e-6, group=None):
    """Exchange 2: rank 0 solves the seed PCP, U / sigma / V are broadcast."""
    dev = seed_rows.device
    k_buf = torch.zeros(1, dtype=torch.int64, device=dev)
    pcp_it = 0
    if plan.rank == 0:
        block = seed_rows[:, torch.as_tensor(plan.col_idx, device=dev)]
        u, sig, v, pcp_it = backend.seed(block, adm, rank_tol)
        k_buf[0] = sig.shape[0]
    dist.broadcast(k_buf, 0, group=group)
    k = int(k_buf.item())
    if plan.rank != 0:
        u = backend.empty((plan.row_idx.size, k), torch.float64)
        sig = backend.empty((k,), torch.float64)
        v = backend.empty((plan.col_idx.size, k), torch.float64)
    for tns in (u, sig, v):
        dist.broadcast(tns, 0, group=group)
    return u, sig, v, pcp_it


def solve_from_seed(m_local, plan, backend, adm, u, sig, v, group=None):
    """The timed multi-GPU step: seed-row exchange, local filters, Q~ all-gather, local
    reconstruction, statistics.  Returns (L_local, S_local, info)."""
    t = {}
    t0 = time.perf_counter()
    seed_rows = gather_seed_rows(m_local, plan, group)
    t["seed_rows"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    xc = backend.column_panel(seed_rows, plan.my_cols)                    # (my cols, s_r) unit-major
    xr = backend.row_panel(m_local, plan.my_rows - plan.r0, plan.col_idx)  # (my rows, s_c)
    zc, itc, stc = backend.filter(xc, u, adm)
    zr, itr, st_r = backend.filter(xr, v, adm)
    t["filter"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    zc_all = _all_gather_rows(zc, [c1 - c0 for c0, c1 in plan.col_units], group)  # Q~ in unit order
    t["gather_q"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    l_local, s_local = backend.reconstruct(m_local, plan, u, sig, v, zc_all, zr)
    t["reconstruct"] = time.perf_counter() - t0
    dev = m_local.device
    it_max = max(int(itc.max()) if itc.numel() else 0, int(itr.max()) if itr.numel() else 0)
    failed = int(((stc == 1) | (stc == 2)).sum()) + int(((st_r == 1) | (st_r == 2)).sum())
    mx = torch.tensor([float(it_max)], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    sm = torch.tensor([float(failed), float(xc.shape[0] + xr.shape[0])], dtype=torch.float64, device=dev)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)
    info = {"k": int(sig.shape[0]), "filter_iterations": int(mx.item()), "failed_units": int(sm[0].item()),
            "units": int(sm[1].item()), "times": t}
    return l_local, s_local, info


def solve_sharded(m_local, plan, backend, adm, rank_tol=1e-6, group=None):
    """Whole distributed solve (seed included).  Returns (L_local, S_local, info)."""
    seed_rows = gather_seed_rows(m_local, plan, group)
    u, sig, v, pcp_it = seed_factors(seed_rows, plan, backend, adm, rank_tol, group)
    l_local, s_local, info = solve_from_seed(m_local, plan, backend, adm, u, sig, v, group)
    info["pcp_iterations"] = pcp_it
    return l_local, s_local, info


class CudaBackend:
    """Production backend: the C-ABI kernels on CUDA tensors."""

    def __init__(self):
        from . import _device as dv
        from . import _lib, engine
        self.dv, self.lib, self.engine = dv, _lib, engine

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device="cuda")

    def seed(self, block, adm, rank_tol):
        u, s, v, _, it = self.engine.recover_seed_device(block.to(torch.float64).contiguous(), adm, rank_tol)
        return u, s, v, it

    def column_panel(self, seed_rows, cols):
        return self.engine.gather(seed_rows, None, cols, transpose=True)

    def row_panel(self, m_local, local_rows, cols):
        return self.engine.gather(m_local, local_rows, cols)

    def filter(self, x_um, a64, adm):
        from .l1reg import filter_units
        fdt = self.engine.filter_dtype_for(a64.shape[1], x_um.dtype)  # same rule as the 1-GPU engine
        z, _, it, _, st = filter_units(x_um.to(fdt).contiguous(), a64.to(fdt).contiguous(), adm, want_e=False)
        return z.to(x_um.dtype), it, st

    def reconstruct(self, m_local, plan, u, sig, v, zc_all, zr):
        seed = self.engine.DeviceSeed(row_idx=plan.row_idx, col_idx=plan.col_idx, u=u, sigma=sig, v=v, seed_l=None,
                                      block=None, r_prime=int(sig.shape[0]), pcp_iterations=0)
        fp = _FactorPlan(plan, seed, m_local.dtype, self.engine)
        af, bf = self.engine.build_factors(fp, zc_all, zr)
        l, s, _ = self.engine.reconstruct(m_local, af, bf)
        return l, s


class _FactorPlan:
    """The subset of engine.FilterPlan that build_factors needs, for a row shard."""

    def __init__(self, plan, seed, dtype, engine):
        self.seed = seed
        self.dtype = dtype
        self.k = seed.r_prime
        self.m_rows, self.m_cols = plan.m, plan.n
        self.row_range = (plan.r0, plan.r1)
        self.d_row_idx = engine.index_tensor(plan.row_idx)
        self.d_col_idx = engine.index_tensor(plan.col_idx)


def run_bench(args, rank, world):
    """bench.py --gpus N: strong scaling of one synthetic matrix over N GPUs (NCCL)."""
    import json

    import paper_1108_5359_b200 as l1pcp
    from . import engine
    from .synth import BENCHMARK_CONFIGS

    cfgd = dict(BENCHMARK_CONFIGS[args.config])
    m, n, r = cfgd["m"], cfgd["n"], cfgd["r"]
    tol = 1e-7
    ranges = row_ranges(m, world)
    r0, r1 = ranges[rank]
    m_local, _, _, _ = engine.generate_matrix(m, n, r, cfgd["rho_s"], cfgd["magnitude"], seed=0, kind=cfgd["kind"],
                                              row0=r0, rows=r1 - r0)
    ss = np.random.SeedSequence(0)
    row_idx, col_idx = engine.sample_indices(m, n, 10 * r, 10 * r, ss.spawn(1)[0])
    plan = ShardPlan(m, n, rank, world, row_idx, col_idx)
    adm = l1pcp.AdmConfig(tol=tol)
    backend = CudaBackend()
    # seed (t1, outside the timed steps as on one GPU): rank 0 solves, factors broadcast
    t0 = time.perf_counter()
    seed_rows = gather_seed_rows(m_local, plan)
    u, sig, v, _ = seed_factors(seed_rows, plan, backend, adm)
    torch.cuda.synchronize()
    t1 = time.perf_counter() - t0
    del seed_rows
    for _ in range(max(1, args.warmup)):
        solve_from_seed(m_local, plan, backend, adm, u, sig, v)
    torch.cuda.synchronize()
    dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(args.steps):
        l_local, s_local, info = solve_from_seed(m_local, plan, backend, adm, u, sig, v)
    end.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([start.elapsed_time(end) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms_v = float(ms.item())
        line = {"metric": "M entries/s (m*n / solve time)", "value": m * n / (ms_v * 1e-3) / 1e6, "unit": "M entries/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_v,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (Philox, row shards generated per rank)",
                "config": {"workload": f"{cfgd['name']}: {m}x{n} r={r}", "parallelism": f"row-sharded x{world}",
                           "collectives": "all-gather seed rows, broadcast seed factors, all-gather Q~, "
                                          "all-reduce stats (NCCL)"},
                "phases_ms": {"t1_seed_s": t1}, "gpu_launches": None,
                "filter": {kk: vv for kk, vv in info.items() if kk != "times"}}
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0
