"""CPU baseline legs of bench.py: the reference's own l1-filtering code timed on the host cores.

TEST/BENCH INFRASTRUCTURE ONLY — imported by bench.py, never by the product package.

The timed code is the unmodified reference package staged at oracle/_ref/l1pcp by
__graft_entry__.build() (a copy of /root/reference/pkg/src/l1pcp; `kind: "reference"`).  When that
copy is missing the oracle port stands in (`kind: "port"`).  What is timed per step is the
reference pipeline after the seed (l1filter.py:239-254):

  filter_columns on a sample of column units   (l1filter.py:116-122 -> l1reg.py:163-214)
  filter_rows    on a sample of row units      (l1filter.py:125-134)
  nystrom_complete + assemble + (m - l)        (l1filter.py:137-167, :253) on the sub-matrix
                                               (seed rows + sampled rows) x (seed cols + sampled cols)

and the full-matrix time is extrapolated per unit (filters) and per entry (assembly).  The inputs
are the GPU arm's Philox matrix, regenerated bit for bit on the host by oracle/philox_gen (outside
the timed region), so both arms solve the same M.  `validate_extrapolation` runs the reference's
complete estimate_rank_and_solve on a config small enough to time whole (cfg2) and reports the
extrapolation error of the same sampling scheme there.
"""

import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-7


def load_reference():
    """(module, kind): the staged reference package, or the oracle port."""
    pkg = os.path.join(ROOT, "oracle", "_ref", "l1pcp")
    if os.path.isfile(os.path.join(pkg, "__init__.py")):
        # imported under its own name from its own path: the module name "l1pcp" may be aliased
        # to the drop-in elsewhere in the process (tests/reference_suite)
        if "l1pcp_reference" not in sys.modules:
            import importlib.util
            spec = importlib.util.spec_from_file_location("l1pcp_reference", os.path.join(pkg, "__init__.py"),
                                                          submodule_search_locations=[pkg])
            mod = importlib.util.module_from_spec(spec)
            sys.modules["l1pcp_reference"] = mod
            spec.loader.exec_module(mod)
        return sys.modules["l1pcp_reference"], "reference"
    return _PortShim(), "port"


class _PortShim:
    """The reference functions the CPU leg calls, restated by the oracle port (fallback only)."""

    def __init__(self):
        from dataclasses import dataclass

        from oracle import adm_filter, seed_pcp
        self._adm, self._seed = adm_filter, seed_pcp

        @dataclass
        class AdmConfig:
            tol: float = 1e-7
        self.AdmConfig = AdmConfig

    def filter_columns(self, m_c, u, cfg=None, parallelism=1):
        z, e, it, _, _ = self._adm.solve_units(m_c, u, cfg.tol)
        return z, e, int(it.max(initial=0))

    def filter_rows(self, m_r, v, cfg=None, parallelism=1):
        z, e, it, _, _ = self._adm.solve_units(m_r.T, v, cfg.tol)
        return z, e.T, int(it.max(initial=0))


def cpu_info():
    info = {"affinity_cores": len(os.sched_getaffinity(0)), "machine": platform.machine()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                info["model"] = ln.split(":", 1)[1].strip()
            if ln.startswith("Socket(s):") or ln.startswith("Core(s) per socket:") or ln.startswith("Thread(s) per core:"):
                info[ln.split(":")[0].strip().lower().replace("(s)", "s").replace(" ", "_")] = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
                        for d in threadpool_info() if d.get("user_api") == "blas"]
    except ImportError:
        pass
    info["numpy"] = np.__version__
    return info


class Threads:
    """BLAS threads + the reference's `parallelism` (l1reg.py:179-181) for one setting."""

    def __init__(self, blas, parallelism):
        self.blas, self.parallelism = blas, parallelism

    def __enter__(self):
        try:
            from threadpoolctl import threadpool_limits
            self._ctl = threadpool_limits(limits=self.blas, user_api="blas")
        except ImportError:
            self._ctl = None
        return self

    def __exit__(self, *a):
        if self._ctl is not None:
            self._ctl.unregister() if hasattr(self._ctl, "unregister") else self._ctl.restore_original_limits()

    def label(self):
        return f"blas={self.blas},parallelism={self.parallelism}"


class Workload:
    """A BASELINE config's M regenerated on the host (oracle/philox_gen), with the seed factors."""

    def __init__(self, cfgd, seed=None, ref=None):
        from oracle import philox_gen
        self.cfgd = cfgd
        self.m, self.n, self.r = cfgd["m"], cfgd["n"], cfgd["r"]
        self._pg = philox_gen
        self.x, self.y = philox_gen.factors(0, cfgd["kind"], self.m, self.n, self.r)
        if seed is None:  # the reference's own seed stage (l1filter.py:185-237 with the hint)
            seed = self.reference_seed(ref)
        self.seed = seed  # dict(row_idx, col_idx, u, sigma, v, seed_l)
        self.comp_r = np.setdiff1d(np.arange(self.m), seed["row_idx"])
        self.comp_c = np.setdiff1d(np.arange(self.n), seed["col_idx"])

    def block(self, rows, cols):
        c = self.cfgd
        return self._pg.block(0, c["kind"], self.m, self.n, self.r, c["rho_s"], c["magnitude"], rows, cols,
                              x=self.x, y=self.y).astype(np.float64)

    def reference_seed(self, ref):
        ss = np.random.SeedSequence(0)
        s = 10 * self.r
        rng = np.random.default_rng(ss.spawn(1)[0])
        ri = np.sort(rng.choice(self.m, size=s, replace=False))
        ci = np.sort(rng.choice(self.n, size=s, replace=False))
        rec = ref.recover_seed(self.block(ri, ci), ref.AdmConfig(tol=TOL), 1e-6, ri, ci)
        f = rec.seed_svd
        return {"row_idx": ri, "col_idx": ci, "u": f.u, "sigma": f.sigma, "v": f.v, "seed_l": rec.seed_l,
                "pcp_iterations": rec.pcp_iterations}


def sample_step(ref, wl, n_units, threads, rng_seed=1):
    """One bounded sample of the reference pipeline after the seed; returns timings and the
    full-matrix extrapolation (seconds)."""
    seed = wl.seed
    ri, ci = seed["row_idx"], seed["col_idx"]
    rng = np.random.default_rng(rng_seed)
    sc = np.sort(rng.choice(wl.comp_c, min(n_units, wl.comp_c.size), replace=False))
    sr = np.sort(rng.choice(wl.comp_r, min(n_units, wl.comp_r.size), replace=False))
    m_c = wl.block(ri, sc)
    m_r = wl.block(sr, ci)
    adm = ref.AdmConfig(tol=TOL)
    with threads:
        t0 = time.perf_counter()
        q, s_col, _ = ref.filter_columns(m_c, seed["u"], adm, threads.parallelism)
        t_c = time.perf_counter() - t0
        t0 = time.perf_counter()
        p, s_row, _ = ref.filter_rows(m_r, seed["v"], adm, threads.parallelism)
        t_r = time.perf_counter() - t0
    t_asm, sub_entries = None, 0
    if hasattr(ref, "assemble"):
        # the sub-problem (seed rows + sampled rows) x (seed cols + sampled cols) in the reference's
        # own bookkeeping: seed positions re-indexed into the sub-matrix
        rows = np.union1d(ri, sr)
        cols = np.union1d(ci, sc)
        m_sub = wl.block(rows, cols)
        f = ref.SkinnySvd(u=seed["u"], sigma=seed["sigma"], v=seed["v"])
        sub_seed = ref.SeedRecovery(row_idx=np.searchsorted(rows, ri), col_idx=np.searchsorted(cols, ci),
                                    seed_svd=f, seed_l=seed["seed_l"], seed_s=np.zeros_like(seed["seed_l"]),
                                    r_prime=int(seed["sigma"].size))
        fr = ref.FilterResult(q_tilde=q, p_tilde=p, s_col=s_col, s_row=s_row)
        with threads:
            t0 = time.perf_counter()
            completion = ref.nystrom_complete(sub_seed, fr)
            l_sub = ref.assemble(sub_seed, fr, completion, rows.size, cols.size)
            s_sub = m_sub - l_sub
            t_asm = time.perf_counter() - t0
        del s_sub, l_sub
        sub_entries = rows.size * cols.size
    t_est = t_c * wl.comp_c.size / sc.size + t_r * wl.comp_r.size / sr.size
    if t_asm is not None:
        t_est += t_asm * (wl.m * wl.n) / sub_entries
    return {"t_cols": t_c, "t_rows": t_r, "t_assemble_sub": t_asm, "units": [int(sc.size), int(sr.size)],
            "sub_entries": int(sub_entries), "t_sample": t_c + t_r + (t_asm or 0.0), "t_est": t_est}


def pick_threads(ref, wl, units_probe):
    """Time the threading settings of SURVEY 8(d) — (i) one BLAS thread, parallelism 1; (ii) BLAS
    threads = parallelism = cores — plus (iii) one BLAS thread per worker, parallelism = cores, on
    a small probe; returns (best, per-setting)."""
    cores = len(os.sched_getaffinity(0))
    settings = [Threads(1, 1), Threads(cores, cores), Threads(1, cores)]
    res = {}
    for th in settings:  # best of two probes: oversubscribed settings are noisy run to run
        outs = [sample_step(ref, wl, units_probe, th, rng_seed=99 + rep) for rep in range(2)]
        res[th.label()] = {"t_est_s": min(o["t_est"] for o in outs), "units": outs[0]["units"]}
    best = min(settings, key=lambda th: res[th.label()]["t_est_s"])
    return best, res


def validate_extrapolation(ref, kind, cfgd_small, n_units, threads):
    """Full reference solve (after the seed) on a small config vs the sampled extrapolation.
    Returns dict(full_s, extrapolated_s, rel_err)."""
    if kind != "reference":
        return None
    wl = Workload(cfgd_small, ref=ref)
    m_full = wl.block(np.arange(wl.m), np.arange(wl.n))
    seed = wl.seed
    f = ref.SkinnySvd(u=seed["u"], sigma=seed["sigma"], v=seed["v"])
    rec = ref.SeedRecovery(row_idx=seed["row_idx"], col_idx=seed["col_idx"], seed_svd=f, seed_l=seed["seed_l"],
                           seed_s=np.zeros_like(seed["seed_l"]), r_prime=int(seed["sigma"].size))
    adm = ref.AdmConfig(tol=TOL)
    with threads:
        t0 = time.perf_counter()
        # l1filter.py:239-254, verbatim order of operations
        m_c = m_full[np.ix_(rec.row_idx, wl.comp_c)]
        m_r = m_full[np.ix_(wl.comp_r, rec.col_idx)]
        q, s_col, it_c = ref.filter_columns(m_c, f.u, adm, threads.parallelism)
        p, s_row, it_r = ref.filter_rows(m_r, f.v, adm, threads.parallelism)
        fr = ref.FilterResult(q_tilde=q, p_tilde=p, s_col=s_col, s_row=s_row, iterations=max(it_c, it_r))
        t2 = time.perf_counter() - t0
        t0 = time.perf_counter()
        completion = ref.nystrom_complete(rec, fr)
        l = ref.assemble(rec, fr, completion, wl.m, wl.n)
        s = m_full - l
        t_asm = time.perf_counter() - t0
    del s, l, m_full
    est = sample_step(ref, wl, n_units, threads, rng_seed=5)
    full = t2 + t_asm
    return {"config": cfgd_small["name"], "full_s": full, "full_t2_s": t2, "full_t_assemble_s": t_asm,
            "extrapolated_s": est["t_est"], "rel_err": (est["t_est"] - full) / full,
            "sample_units": est["units"], "threads": threads.label()}


def host_matrix(wl, threads=None):
    """The whole M on the host (float64), regenerated bit for bit in row blocks on a thread pool."""
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or len(os.sched_getaffinity(0))
    out = np.empty((wl.m, wl.n))
    bounds = np.linspace(0, wl.m, 4 * threads + 1).astype(np.int64)
    cols = np.arange(wl.n)

    def fill(i):
        r0, r1 = int(bounds[i]), int(bounds[i + 1])
        if r1 > r0:
            out[r0:r1] = wl.block(np.arange(r0, r1), cols)

    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(fill, range(len(bounds) - 1)))
    return out


def full_measure(ref, wl, m_full, threads, steps, warmup):
    """The reference pipeline after the seed (l1filter.py:239-254) over the WHOLE matrix, split into
    `steps` timed steps: step i gathers and filters the i-th 1/steps of the column and row units
    (filter work is per unit, so the split changes nothing but the 64-unit chunk boundaries); the
    last step also runs nystrom_complete + assemble + m - l on the full matrix.  Warm-up steps
    repeat step 0's filters untimed.  Returns (per-step seconds, details)."""
    seed = wl.seed
    ri, ci = seed["row_idx"], seed["col_idx"]
    f = ref.SkinnySvd(u=seed["u"], sigma=seed["sigma"], v=seed["v"])
    rec = ref.SeedRecovery(row_idx=ri, col_idx=ci, seed_svd=f, seed_l=seed["seed_l"],
                           seed_s=np.zeros_like(seed["seed_l"]), r_prime=int(seed["sigma"].size))
    adm = ref.AdmConfig(tol=TOL)
    parts_c = np.array_split(wl.comp_c, steps)
    parts_r = np.array_split(wl.comp_r, steps)

    def filt(i):
        m_c = m_full[np.ix_(ri, parts_c[i])]
        m_r = m_full[np.ix_(parts_r[i], ci)]
        q, s_col, it_c = ref.filter_columns(m_c, f.u, adm, threads.parallelism)
        p, s_row, it_r = ref.filter_rows(m_r, f.v, adm, threads.parallelism)
        return q, p, s_col, s_row, max(it_c, it_r)

    times, qs, ps, scs, srs, its = [], [], [], [], [], []
    t_asm = 0.0
    with threads:
        for _ in range(warmup):
            filt(0)
        for i in range(steps):
            t0 = time.perf_counter()
            q, p, sc, sr, it = filt(i)
            qs.append(q); ps.append(p); scs.append(sc); srs.append(sr); its.append(it)
            if i == steps - 1:
                ta = time.perf_counter()
                fr = ref.FilterResult(q_tilde=np.concatenate(qs, axis=1), p_tilde=np.concatenate(ps, axis=1),
                                      s_col=np.concatenate(scs, axis=1), s_row=np.concatenate(srs, axis=0),
                                      iterations=max(its))
                completion = ref.nystrom_complete(rec, fr)
                l = ref.assemble(rec, fr, completion, wl.m, wl.n)
                s = m_full - l
                t_asm = time.perf_counter() - ta
            times.append(time.perf_counter() - t0)
    out = {"mode": "full", "t_total_s": float(sum(times)), "t_assemble_s": t_asm,
           "t_filters_s": float(sum(times) - t_asm), "units": [int(wl.comp_c.size), int(wl.comp_r.size)],
           "filter_iterations": int(max(its))}
    del s, l
    return times, out
