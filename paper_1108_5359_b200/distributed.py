"""Row-sharded multi-GPU l1-filtering solve, one process per GPU.

Rank g owns the row block [r0_g, r1_g) of M.  The exchange steps are the ones the algorithm
has; everything else is local:

  1. all-to-all of the column panel: rank h needs M[row_idx, C_h] for its column units C_h, and
     each rank owns the seed rows inside its row block, so rank g sends M[its seed rows, C_h]
     to rank h (n_c * s_r floats in total, each rank receiving only its own columns; an
     all-gather of whole seed rows would move world x more).  The seed solve (t1, once) uses
     an all-gather of the s_r x s_c seed block's rows.
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

import os
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
    if world == 1:
        return local
    pad = local.new_zeros((hmax, width))
    pad[: local.shape[0]] = local
    out = local.new_empty((world * hmax, width))
    dist.all_gather_into_tensor(out, pad, group=group)
    if all(c == hmax for c in counts):
        return out
    return torch.cat([out[g * hmax:g * hmax + c] for g, c in enumerate(counts)], dim=0)


def gather_seed_block(m_local, plan, backend, group=None):
    """Exchange 0 (once per solve, before the timed steps): the s_r x s_c seed block
    M[row_idx, col_idx] (sample_submatrix, l1filter.py:73-87) on rank 0 only.  Each rank gathers the
    seed rows it owns at the seed columns (P_g x s_c, an l1f_gather) and rank 0 collects the blocks
    with one gather (padded to the largest P_g): s_r * s_c * 4 bytes in total, <= 16 MB at config 5,
    instead of whole seed rows on every rank.  Returns the block on rank 0, None elsewhere."""
    counts = [int((plan.seed_owner == g).sum()) for g in range(plan.world)]
    local = backend.row_panel(m_local, plan.row_idx[plan.my_seed_pos] - plan.r0, plan.col_idx)  # (P_me, s_c)
    if plan.world == 1:
        return local
    hmax = max(max(counts), 1)
    pad = local.new_zeros((hmax, local.shape[1]))
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(plan.world)] if plan.rank == 0 else None
    dist.gather(pad, gather_list=bufs, dst=0, group=group)
    if plan.rank != 0:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def exchange_column_panel(m_local, plan, backend, group=None, out=None):
    """Exchange 1: this rank's column panel Xc[j][p] = M[row_idx[p], my_cols[j]] (unit-major).

    row_idx is sorted and the row blocks are contiguous in rank order, so rank g owns the seed
    positions [p0_g, p0_g + P_g): it gathers M[its seed rows, all non-seed columns] transposed
    (one row per column unit, T[j][p - p0_g]); rows [c0_h, c1_h) of T go to rank h
    (all_to_all_single), and rank h concatenates the received blocks along p in rank order."""
    world = plan.world
    local_rows = plan.row_idx[plan.my_seed_pos] - plan.r0
    if world == 1:
        return backend.panel_t(m_local, local_rows, plan.comp_cols, out=out)
    seed_counts = [int((plan.seed_owner == g).sum()) for g in range(world)]
    col_counts = [c1 - c0 for c0, c1 in plan.col_units]
    p_me, c_me = seed_counts[plan.rank], col_counts[plan.rank]
    t = backend.panel_t(m_local, local_rows, plan.comp_cols)        # (n_c, P_me)
    recv = t.new_empty((c_me * len(plan.row_idx),))
    dist.all_to_all_single(recv, t.reshape(-1), [c_me * p for p in seed_counts], [c * p_me for c in col_counts],
                           group=group)
    blocks, off = [], 0
    for p in seed_counts:
        blocks.append(recv[off:off + c_me * p].view(c_me, p))
        off += c_me * p
    if out is None:
        return torch.cat(blocks, dim=1)
    return torch.cat(blocks, dim=1, out=out)


def seed_factors(seed_block, plan, backend, adm, rank_tol=1e-6, group=None, device=None):
    """Exchange 2: rank 0 solves the seed PCP on the gathered block, U / sigma / V are broadcast
    (<= 6.4 MB at config 5)."""
    dev = seed_block.device if seed_block is not None else device
    k_buf = torch.zeros(1, dtype=torch.int64, device=dev)
    pcp_it = 0
    if plan.rank == 0:
        u, sig, v, pcp_it = backend.seed(seed_block, adm, rank_tol)
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
    xc = exchange_column_panel(m_local, plan, backend, group)             # (my cols, s_r) unit-major
    t["column_panel"] = time.perf_counter() - t0
    t0 = time.perf_counter()
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
    block = gather_seed_block(m_local, plan, backend, group)
    u, sig, v, pcp_it = seed_factors(block, plan, backend, adm, rank_tol, group, device=m_local.device)
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

    def panel_t(self, m_local, local_rows, cols, out=None):
        """M_local[rows][:, cols] transposed (one row per column), into `out` if given."""
        if out is None:
            return self.engine.gather(m_local, local_rows, cols, transpose=True)
        rt, ct = self.engine.index_tensor(local_rows), self.engine.index_tensor(cols)
        self.lib.call("l1f_gather", self.dv.dtype_code(m_local), self.dv.ptr(m_local), m_local.stride(0),
                      self.dv.ptr(rt), len(local_rows), self.dv.ptr(ct), len(cols), self.dv.dtype_code(out),
                      self.dv.ptr(out), out.stride(0), 1, self.dv.stream())
        return out

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


class CudaShardedStep:
    """The timed multi-GPU step on CUDA, with everything that does not depend on M's values
    prepared once (index tensors, cast seed factors, factor slices, workspaces, outputs) so the
    step enqueues without host synchronisation.  Same exchanges and per-unit arithmetic as
    solve_from_seed with CudaBackend (bitwise identical L, S)."""

    def __init__(self, m_local, plan, adm, u, sig, v, group=None):
        from . import _device as dv
        from . import _lib, engine
        self.dv, self.lib, self.e = dv, _lib, engine
        self.plan, self.adm, self.group = plan, adm, group
        self.k = int(sig.shape[0])
        dt = m_local.dtype
        self.dt, self.fdt = dt, engine.filter_dtype_for(self.k, dt)
        self.u64, self.sig, self.v64 = u, sig, v
        self.u, self.v = u.to(self.fdt).contiguous(), v.to(self.fdt).contiguous()
        idx = engine.index_tensor
        self.d_seed_local = idx(plan.row_idx[plan.my_seed_pos] - plan.r0)
        self.seed_counts = [int((plan.seed_owner == g).sum()) for g in range(plan.world)]
        self.col_counts = [c1 - c0 for c0, c1 in plan.col_units]
        self.d_my_cols = idx(plan.my_cols)
        self.d_my_rows_local = idx(plan.my_rows - plan.r0)
        self.d_col_idx = idx(plan.col_idx)
        loc = (plan.row_idx >= plan.r0) & (plan.row_idx < plan.r1)
        self.d_local_seed_rows = idx(plan.row_idx[loc] - plan.r0)
        self.n_local_seed = int(loc.sum())
        self.u_local = u[idx(np.flatnonzero(loc))].contiguous()
        rows = plan.r1 - plan.r0
        self.af = torch.empty((rows, self.k), dtype=dt, device="cuda")
        self.bf = torch.empty((plan.n, self.k), dtype=dt, device="cuda")
        self.l = torch.empty_like(m_local)
        self.s = torch.empty_like(m_local)
        self.xc = torch.empty((len(plan.my_cols), len(plan.row_idx)), dtype=self.fdt, device="cuda")
        self.d_comp_cols = idx(plan.comp_cols)
        if plan.world > 1:  # exchange 1 buffers (all-to-all of the column panel)
            p_me, c_me = self.seed_counts[plan.rank], self.col_counts[plan.rank]
            self.t_send = torch.empty((len(plan.comp_cols), p_me), dtype=self.fdt, device="cuda")
            self.recv = torch.empty((c_me * len(plan.row_idx),), dtype=self.fdt, device="cuda")
            self.out_splits = [c_me * q for q in self.seed_counts]
            self.in_splits = [c * p_me for c in self.col_counts]
            self.recv_blocks, off = [], 0
            for q in self.seed_counts:
                self.recv_blocks.append(self.recv[off:off + c_me * q].view(c_me, q))
                off += c_me * q
        self.xr = torch.empty((len(plan.my_rows), len(plan.col_idx)), dtype=self.fdt, device="cuda")
        code = _lib.F32 if self.fdt == torch.float32 else _lib.F64
        nbytes = max(_lib.load().l1f_filter_workspace_bytes(code, len(plan.row_idx), self.k, max(1, len(plan.my_cols))),
                     _lib.load().l1f_filter_workspace_bytes(code, len(plan.col_idx), self.k, max(1, len(plan.my_rows))))
        self.ws = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
        self._n_units_t = None
        self.launches_per_step = 11  # 2 gathers, 2 scale prologues + 1-2 filter grids, factors, 2 splits, recon, sum
        # large shards (the library's pass model runs the two unit sets as two launches): the
        # column filter with the row panel gathered beside it, Q~ all-gather, then the row filter
        # with the reconstruction of the rank's rows streamed beside it (as engine.solve_step)
        self.streamed = False
        if (self.fdt == torch.float32 and dt == torch.float32 and 16 < self.k <= 224 and len(plan.my_cols) > 0
                and len(plan.my_rows) > 0 and len(plan.row_idx) == len(plan.col_idx)
                and self.lib.get_option("recon_stream") != 0 and m_local.stride(0) % 4 == 0
                and m_local.data_ptr() % 16 == 0):
            import ctypes
            one = ctypes.c_int32(0)
            _lib.call("l1f_filter_pair_plan_f32", len(plan.row_idx), self.k, len(plan.my_cols), len(plan.my_rows),
                      ctypes.addressof(one))
            self.streamed = not one.value
            force = self.lib.PY_OPTIONS["sharded_stream"]  # tests: True / False overrides the pass model
            if force is not None:
                self.streamed = bool(force)
        if self.streamed:
            nc, nr = len(plan.my_cols), len(plan.my_rows)
            self.zc = torch.empty((nc, self.k), dtype=torch.float32, device="cuda")
            self.itc = torch.empty(nc, dtype=torch.int32, device="cuda")
            self.rc = torch.empty(nc, dtype=torch.float32, device="cuda")
            self.stc = torch.empty(nc, dtype=torch.uint8, device="cuda")
            self.zr = torch.empty((nr, self.k), dtype=torch.float32, device="cuda")
            self.itr = torch.empty(nr, dtype=torch.int32, device="cuda")
            self.rr = torch.empty(nr, dtype=torch.float32, device="cuda")
            self.st_r = torch.empty(nr, dtype=torch.uint8, device="cuda")
            self.rs = torch.zeros(2, dtype=torch.float64, device="cuda")
            self.launches_per_step = 14  # 2 gathers, 2 x (scale + filter), gate, Bf, strip index, Bf split,
            #                              concurrent + trailing reconstruction, residual sum

    def _step_streamed(self, m_local, events=None):
        dv, lib, p, adm = self.dv, self.lib, self.plan, self.adm
        s_r = len(p.row_idx)
        beta0 = float(adm.beta0) if adm.beta0 is not None else 0.0
        beta_max = float(adm.beta_max) if adm.beta_max is not None else 0.0
        ev_done = None
        if events is not None:
            events[0].record()
            events[1].record()  # creates the event; re-recorded by the library after the row filter
            ev_done = events[1].cuda_event
        code = lib.load().l1f_filter_with_gather_f32(
            dv.ptr(self.xc), self.xc.stride(0), s_r, len(p.my_cols), dv.ptr(self.u), self.u.stride(0), self.k,
            float(adm.tol), float(adm.rho), beta0, beta_max, int(adm.max_iter), dv.ptr(self.zc), self.zc.stride(0),
            dv.ptr(self.itc), dv.ptr(self.rc), dv.ptr(self.stc), dv.dtype_code(m_local), dv.ptr(m_local),
            m_local.stride(0), dv.ptr(self.d_my_rows_local), len(p.my_rows), dv.ptr(self.d_col_idx), len(p.col_idx),
            dv.ptr(self.xr), self.xr.stride(0), 0, dv.stream())
        lib.check(code, "l1f_filter_with_gather_f32")
        zc_all = _all_gather_rows(self.zc, self.col_counts, self.group)          # exchange 2: Q~
        code = lib.load().l1f_rowfilter_reconstruct_f32(
            dv.ptr(self.xr), self.xr.stride(0), len(p.col_idx), len(p.my_rows), dv.ptr(self.v), self.v.stride(0),
            self.k, float(adm.tol), float(adm.rho), beta0, beta_max, int(adm.max_iter), dv.ptr(self.zr),
            self.zr.stride(0), dv.ptr(self.itr), dv.ptr(self.rr), dv.ptr(self.st_r), dv.ptr(self.d_my_rows_local),
            dv.ptr(self.d_local_seed_rows), self.n_local_seed, dv.ptr(self.u_local), dv.ptr(self.sig),
            dv.ptr(self.d_col_idx), len(p.col_idx), dv.ptr(self.v64), dv.ptr(zc_all), zc_all.stride(0),
            dv.ptr(m_local), p.r1 - p.r0, p.n, m_local.stride(0), dv.ptr(self.l), self.l.stride(0), dv.ptr(self.s),
            self.s.stride(0), dv.ptr(self.rs), ev_done, dv.stream())
        lib.check(code, "l1f_rowfilter_reconstruct_f32")
        return self.zc, self.itc, self.stc, self.zr, self.itr, self.st_r

    def step(self, m_local, events=None):
        from .l1reg import filter_units
        dv, lib, p = self.dv, self.lib, self.plan
        code_in = dv.dtype_code(m_local)
        code_f = lib.F32 if self.fdt == torch.float32 else lib.F64
        # exchange 1 (all-to-all): T[j][p] = M[my seed rows, all non-seed columns]; rows of T for
        # rank h's column units go to h; received blocks concatenate along p into xc
        tgt = self.xc if p.world == 1 else self.t_send
        lib.call("l1f_gather", code_in, dv.ptr(m_local), m_local.stride(0), dv.ptr(self.d_seed_local),
                 self.n_local_seed, dv.ptr(self.d_comp_cols), len(p.comp_cols), code_f, dv.ptr(tgt), tgt.stride(0),
                 1, dv.stream())
        if p.world > 1:
            dist.all_to_all_single(self.recv, self.t_send.reshape(-1), self.out_splits, self.in_splits,
                                   group=self.group)
            torch.cat(self.recv_blocks, dim=1, out=self.xc)
        if self.streamed:
            zc, itc, stc, zr, itr, st_r = self._step_streamed(m_local, events)
            return self._finish(m_local, itc, stc, itr, st_r)
        lib.call("l1f_gather", code_in, dv.ptr(m_local), m_local.stride(0), dv.ptr(self.d_my_rows_local),
                 len(p.my_rows), dv.ptr(self.d_col_idx), len(p.col_idx), code_f, dv.ptr(self.xr), self.xr.stride(0), 0,
                 dv.stream())
        if events is not None:
            events[0].record()
        if self.fdt == torch.float32 and self.xc.shape[1] == self.xr.shape[1] and self.lib.PY_OPTIONS["filter_pair"]:
            # one call for the shard's column and row units (small shards: overlapped drains)
            from .l1reg import filter_units_pair
            (zc, itc, _, stc), (zr, itr, _, st_r) = filter_units_pair(self.xc, self.u, self.xr, self.v, self.adm)
        else:
            zc, _, itc, _, stc = filter_units(self.xc, self.u, self.adm, want_e=False, workspace=self.ws)
            zr, _, itr, _, st_r = filter_units(self.xr, self.v, self.adm, want_e=False, workspace=self.ws)
        if events is not None:
            events[1].record()
        if self.fdt != self.dt:
            zc, zr = zc.to(self.dt), zr.to(self.dt)
        zc_all = _all_gather_rows(zc, self.col_counts, self.group)           # exchange 2: Q~
        code = lib.F32 if self.dt == torch.float32 else lib.F64
        lib.call("l1f_build_factors", code, p.r1 - p.r0, p.n, self.k, dv.ptr(self.d_local_seed_rows),
                 self.n_local_seed, dv.ptr(self.d_col_idx), len(p.col_idx), dv.ptr(self.u_local), dv.ptr(self.sig),
                 dv.ptr(self.v64), dv.ptr(zc_all), zc_all.stride(0), dv.ptr(zr), max(zr.stride(0), self.k),
                 dv.ptr(self.af), dv.ptr(self.bf), dv.stream())
        self.e.reconstruct(m_local, self.af, self.bf, self.l, self.s)
        return self._finish(m_local, itc, stc, itr, st_r)

    def _finish(self, m_local, itc, stc, itr, st_r):
        dev = m_local.device
        it = torch.stack([itc.max() if itc.numel() else torch.zeros((), dtype=itc.dtype, device=dev),
                          itr.max() if itr.numel() else torch.zeros((), dtype=itr.dtype, device=dev)]).max()
        failed = ((stc == 1) | (stc == 2)).sum() + ((st_r == 1) | (st_r == 2)).sum()
        if self._n_units_t is None:  # a device constant: no host->device copy inside the step
            self._n_units_t = torch.full((), float(itc.numel() + itr.numel()), dtype=torch.float64, device=dev)
        stats = torch.stack([it.double(), failed.double(), self._n_units_t, itc.double().sum() + itr.double().sum()])
        return self.l, self.s, stats, (itc, itr)


def run_bench(args, rank, world, clock_sampler=None):
    """bench.py --gpus N: strong scaling of one synthetic matrix over N GPUs (NCCL).  Same
    contract keys as the 1-GPU line; times are the max over ranks of CUDA-event times."""
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
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    block = gather_seed_block(m_local, plan, backend)
    u, sig, v, _ = seed_factors(block, plan, backend, adm, device=m_local.device)
    torch.cuda.synchronize()
    t1 = time.perf_counter() - t0
    del block
    stepper = CudaShardedStep(m_local, plan, adm, u, sig, v)
    # eager warm-up steps with events around the filters (kernel times; queued behind a device spin
    # so the events time GPU work), then the step with its statistics all-reduce captured in a
    # CUDA graph (kernels and NCCL collectives) for the timed steps; eager if capture fails
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(max(3, args.warmup))]
    for i in range(len(evs)):
        torch.cuda._sleep(4_000_000)
        l_local, s_local, stats, (itc, itr) = stepper.step(m_local, evs[i])
        torch.cuda.synchronize()
    evs = evs[1:]
    dist.barrier()

    def one_step():
        out = stepper.step(m_local)
        dist.all_reduce(out[2], group=None)  # statistics (exchange 3); sum over ranks
        return out

    try:
        graph = engine.CapturedCall(one_step)
        step_form, ok = "CUDA graph (kernels + NCCL collectives), replayed", 1.0
    except Exception as exc:  # capture unsupported: eager steps
        graph, step_form, ok = None, f"eager ({type(exc).__name__} at capture)", 0.0
    # the choice must be the same on every rank (a replayed graph's collectives pair with the
    # other ranks' graph collectives only)
    flag = torch.tensor([ok], dtype=torch.float64, device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if flag.item() < 1.0 and graph is not None:
        graph, step_form = None, "eager (capture failed on another rank)"
    dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = clock_sampler(int(os.environ.get("LOCAL_RANK", "0"))) if clock_sampler else None
    if sampler:
        sampler.__enter__()
    torch.cuda.synchronize()
    start.record()
    for i in range(args.steps):
        l_local, s_local, stats, (itc, itr) = graph.replay() if graph is not None else one_step()
    end.record()
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__(None, None, None)
    dist.barrier()
    filt_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    its = float((itc.double().sum() + itr.double().sum()).item())
    t = torch.tensor([start.elapsed_time(end) / args.steps, filt_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    flops = torch.tensor([its * len(row_idx) * (4 * stepper.k + 12)], dtype=torch.float64, device="cuda")
    dist.all_reduce(flops)  # algorithmic filter work of all ranks (s_r = s_c here)
    # e2e: each rank's row block from pinned host memory, L and S back to pinned host memory
    m_host = torch.empty(m_local.shape, dtype=m_local.dtype, pin_memory=True)
    m_host.copy_(m_local)
    l_host = torch.empty_like(m_host, pin_memory=True)
    s_host = torch.empty_like(m_host, pin_memory=True)
    m_dev = torch.empty_like(m_local)
    e_steps = max(1, min(args.steps, 3))

    def e2e_step():
        m_dev.copy_(m_host, non_blocking=True)
        l_d, s_d, st, _ = stepper.step(m_dev)
        l_host.copy_(l_d, non_blocking=True)
        s_host.copy_(s_d, non_blocking=True)
        dist.all_reduce(st)
        return st

    e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(e_steps):
        st = e2e_step()
        st_host = st.cpu()  # device -> host read of the step's result
    b.record()
    torch.cuda.synchronize()
    te = torch.tensor([a.elapsed_time(b) / e_steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    stats_h = stats.cpu().numpy()
    if rank == 0:
        ms_v, filt_v = float(t[0].item()), float(t[1].item())
        fma = engine.fma_peak_tflops()
        ach = float(flops.item()) / (filt_v * 1e-3) / 1e12
        nbytes = m * n * m_local.element_size()
        line = {"metric": "M entries/s (m*n / solve time)", "value": m * n / (ms_v * 1e-3) / 1e6, "unit": "M entries/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_v,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (Philox, row shards generated per rank)",
                "config": {"workload": f"{cfgd['name']}: {m}x{n} r={r}", "m": m, "n": n, "rank": r,
                           "parallelism": f"row-sharded x{world}",
                           "collectives": "per step: all-to-all of the column panel, all-gather Q~, all-reduce "
                                          "stats (NCCL); once: seed block gathered to rank 0, seed factors broadcast",
                           "l2": "inputs larger than L2 (row block %.2f GB per GPU)" % (nbytes / world / 1e9)},
                "roofline": {"bound": "fp32", "kernel": "adm_tc_kernel (column + row filters, max over ranks)",
                             "achieved": ach, "peak": fma * world, "unit": "TFLOP/s", "frac": ach / (fma * world),
                             "peak_source": "measured FP32 FMA probe x N GPUs", "traffic": None,
                             "kernel_ms_per_step": filt_v},
                "phases_ms": {"t1_seed_s": t1, "filters": filt_v},
                "filter": {"units": int(stats_h[2]), "mean_iters": float(stats_h[3] / max(stats_h[2], 1)),
                           "max_iters_summed_over_ranks": int(stats_h[0]), "failed_units": int(stats_h[1])},
                "gpu_launches": stepper.launches_per_step * args.steps * world,
                "step_form": step_form,
                "gpu_launches_per_rank": stepper.launches_per_step * args.steps,
                "clocks": sampler.summary() if sampler else None,
                "e2e": {"value": m * n / (float(te.item()) * 1e-3) / 1e6, "unit": "M entries/s",
                        "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 2 * nbytes,
                        "ms_per_step": float(te.item()), "steps": e_steps,
                        "path": "per rank: pinned host row block -> H2D -> sharded step -> D2H of L, S rows"}}
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0
