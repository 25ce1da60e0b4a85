"""Oracle: the full l1-filtering solve and its sampled form (TEST INFRASTRUCTURE ONLY).

Restates estimate_rank_and_solve (/root/reference/pkg/src/l1pcp/l1filter.py:174-268) with
the seed loop (:196-237), the panel gathers (:240-243), the column/row filters
(:116-134 via l1reg.py:163-214), the Nystrom completion + assembly (:137-167) and
S = M - L (:253).  ``sampled_blocks`` is the sampled oracle of SURVEY section 8(c'):
the seed solve plus the filter on a subset of columns/rows, giving L and S on
(rows x cols) sub-blocks without forming the whole matrix (per-unit separability,
l1reg.py:8-14).
"""

import numpy as np

from . import adm_filter, seed_pcp


def sample_indices(m_rows, m_cols, n_rows, n_cols, rng):
    """sample_submatrix index sets (l1filter.py:73-87)."""
    rng = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
    return (np.sort(rng.choice(m_rows, size=n_rows, replace=False)),
            np.sort(rng.choice(m_cols, size=n_cols, replace=False)))


def seed_loop(m_rows, m_cols, get_block, rank_hint, rng_seed=0, s_r=10.0, s_c=10.0, tol=1e-9,
              rank_tol=1e-6, max_seed_fraction=0.5):
    """The seed attempts of l1filter.py:185-237 (cross_validate off).
    get_block(row_idx, col_idx) -> float64 block.  Returns dict or a 'fallback'/'degenerate' marker."""
    ss = np.random.SeedSequence(rng_seed)
    r = max(1, rank_hint or 1)
    attempts = 0
    while True:
        attempts += 1
        n_rows, n_cols = int(round(s_r * r)), int(round(s_c * r))
        if max(n_rows / m_rows, n_cols / m_cols) > max_seed_fraction:
            return {"kind": "fallback", "attempts": attempts}
        n_rows, n_cols = min(n_rows, m_rows), min(n_cols, m_cols)
        ri, ci = sample_indices(m_rows, m_cols, n_rows, n_cols, ss.spawn(1)[0])
        rec = seed_pcp.recover(get_block(ri, ci), tol=tol, rank_tol=rank_tol)
        if rec is None:
            return {"kind": "degenerate", "attempts": attempts}
        u, sig, v, seed_l, it = rec
        rp = sig.size
        if n_rows / rp >= s_r and n_cols / rp >= s_c:
            return {"kind": "seed", "row_idx": ri, "col_idx": ci, "u": u, "sigma": sig, "v": v, "seed_l": seed_l,
                    "pcp_iterations": it, "r_prime": rp, "attempts": attempts}
        r = max(rp, r + 1)


def solve(m, rank_hint, rng_seed=0, s_r=10.0, s_c=10.0, tol=1e-9, rank_tol=1e-6, filter_dtype=np.float64):
    """Full solve on an in-memory matrix.  Returns dict(l, s, r_prime, iterations, ...)."""
    m = np.asarray(m, dtype=np.float64)
    m_rows, m_cols = m.shape
    sd = seed_loop(m_rows, m_cols, lambda ri, ci: m[np.ix_(ri, ci)], rank_hint, rng_seed, s_r, s_c, tol, rank_tol)
    if sd["kind"] != "seed":
        return sd
    ri, ci = sd["row_idx"], sd["col_idx"]
    comp_r = np.setdiff1d(np.arange(m_rows), ri)
    comp_c = np.setdiff1d(np.arange(m_cols), ci)
    q, _, it_c, _, st_c = adm_filter.solve_units(m[np.ix_(ri, comp_c)], sd["u"], tol, dtype=filter_dtype)
    p, _, it_r, _, st_r = adm_filter.solve_units(m[np.ix_(comp_r, ci)].T, sd["v"], tol, dtype=filter_dtype)
    q = q.astype(np.float64)
    p = p.astype(np.float64)
    u, sig, v = sd["u"], sd["sigma"], sd["v"]
    l = np.empty((m_rows, m_cols))
    l[np.ix_(ri, ci)] = sd["seed_l"]
    l[np.ix_(ri, comp_c)] = u @ q
    l[np.ix_(comp_r, ci)] = p.T @ v.T
    l[np.ix_(comp_r, comp_c)] = p.T @ (q / sig[:, None])
    s = m - l
    return {"kind": "seed", "l": l, "s": s, "r_prime": sd["r_prime"], "row_idx": ri, "col_idx": ci,
            "iterations": sd["pcp_iterations"] + int(max(it_c.max(initial=0), it_r.max(initial=0))),
            "filter_failed": int(((st_c == 1) | (st_c == 2)).sum() + ((st_r == 1) | (st_r == 2)).sum()),
            "u": u, "sigma": sig, "v": v, "q": q, "p": p, "iters_c": it_c, "iters_r": it_r}


def sampled_blocks(m_rows, m_cols, get_block, rank_hint, sample_rows, sample_cols,
                   rng_seed=0, tol=1e-9, rank_tol=1e-6, filter_dtype=np.float64):
    """L and S on the sample_rows x sample_cols sub-block (SURVEY 8(c')).

    get_block(rows, cols) returns float64 M[np.ix_(rows, cols)] for any index sets (e.g.
    regenerated from the Philox oracle), so M itself is never formed.
    """
    sd = seed_loop(m_rows, m_cols, get_block, rank_hint, rng_seed, tol=tol, rank_tol=rank_tol)
    if sd["kind"] != "seed":
        return sd
    ri, ci = sd["row_idx"], sd["col_idx"]
    u, sig, v = sd["u"], sd["sigma"], sd["v"]
    rows = np.asarray(sample_rows)
    cols = np.asarray(sample_cols)
    seed_row_pos = {int(r): p for p, r in enumerate(ri)}
    seed_col_pos = {int(c): p for p, c in enumerate(ci)}
    nr_rows = np.array([r for r in rows if int(r) not in seed_row_pos], dtype=np.int64)
    nr_cols = np.array([c for c in cols if int(c) not in seed_col_pos], dtype=np.int64)
    # filter the sampled non-seed columns (against U) and rows (against V)
    q, _, it_c, _, st_c = adm_filter.solve_units(get_block(ri, nr_cols), u, tol, dtype=filter_dtype)
    p, _, it_r, _, st_r = adm_filter.solve_units(get_block(nr_rows, ci).T, v, tol, dtype=filter_dtype)
    q = q.astype(np.float64)
    p = p.astype(np.float64)
    qpos = {int(c): j for j, c in enumerate(nr_cols)}
    ppos = {int(r): j for j, r in enumerate(nr_rows)}
    a = np.stack([u[seed_row_pos[int(r)]] if int(r) in seed_row_pos else p[:, ppos[int(r)]] / sig for r in rows])
    b = np.stack([sig * v[seed_col_pos[int(c)]] if int(c) in seed_col_pos else q[:, qpos[int(c)]] for c in cols])
    l = a @ b.T
    s = get_block(rows, cols) - l
    return {"kind": "seed", "l": l, "s": s, "r_prime": sd["r_prime"], "row_idx": ri, "col_idx": ci,
            "iters_c": it_c, "iters_r": it_r, "failed": int(((st_c == 1) | (st_c == 2)).sum()
                                                           + ((st_r == 1) | (st_r == 2)).sum())}
