"""CPU study: does the reformulated FP32 ADM (filter_resident.cu) still meet tol = 1e-7 when its
two contractions (A z, A^T v) run as split-TF32 tensor-core products?

Emulation: operands split into TF32 pieces (cvt.rna: 10 explicit mantissa bits), each piece
product summed exactly per K=8 MMA block (float64) and added into an FP32 accumulator.
Modes: fp32 (sgemm), x3 (hi.hi + hi.lo + lo.hi), x5 (A in 2 pieces, vector in 3: 5 terms).
    python tools/tc_numerics.py [units]
"""
import sys
import numpy as np

sys.path.insert(0, ".")
from oracle import adm_filter


def tf32(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32)


def split(x, n):
    out, r = [], np.asarray(x, np.float32)
    for _ in range(n):
        p = tf32(r)
        out.append(p)
        r = (r - p).astype(np.float32)
    return out


def mm(a_pieces, b_pieces, terms):
    """sum over terms (i, j) of a_i @ b_j with K=8 blocks accumulated in FP32."""
    m, k = a_pieces[0].shape
    n = b_pieces[0].shape[1]
    acc = np.zeros((m, n), np.float32)
    for k0 in range(0, k, 8):
        for (i, j) in terms:
            blk = a_pieces[i][:, k0:k0 + 8].astype(np.float64) @ b_pieces[j][k0:k0 + 8].astype(np.float64)
            acc = (acc + blk.astype(np.float32)).astype(np.float32)  # approx: block sum rounded, then added
    return acc


TERMS = {"x3": ((0, 0), (0, 1), (1, 0)), "x5": ((0, 0), (0, 1), (1, 0), (0, 2), (1, 1)),
         "x6": ((0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0))}


def product(mode, a, at, z_or_v, left):
    if mode == "fp32":
        return (a if left else at) @ z_or_v
    apieces = a["p"] if left else at["p"]
    nv = 3 if mode in ("x5", "x6") else 2
    return mm(apieces, split(z_or_v, nv), TERMS[mode])


def adm_fp32(x, a, tol, mode, max_iter=1000, rho=1.5):
    """The resident kernel's reformulated FP32 iteration (filter_resident.cu phase b)."""
    x = x.astype(np.float32)
    s, n = x.shape
    a32 = a.astype(np.float32)
    na = 3 if mode == "x6" else 2
    A = {"p": split(a32, na)} if mode != "fp32" else a32
    AT = {"p": [p.T.copy() for p in A["p"]]} if mode != "fp32" else a32.T.copy()
    scale = np.abs(x).max(axis=0)
    b0 = (1.0 / scale).astype(np.float32)
    bmax = (np.float32(1e7) * b0).astype(np.float32)
    thresh = np.float32(tol) * scale
    y = np.zeros_like(x); l = np.zeros_like(x); az = np.zeros_like(x)
    bcur = b0.copy(); bnext = b0.copy()
    iters = np.zeros(n, int); status = np.zeros(n, int); res_out = np.zeros(n, np.float32)
    live = np.ones(n, bool); prev = np.full(n, np.inf, np.float32); stall = np.zeros(n, int)
    it = 0
    z = np.zeros((a.shape[1], n), np.float32)
    while live.any() and it <= max_iter:
        tn = (np.float32(1) / bnext).astype(np.float32)
        if it > 0:
            r = (l - az).astype(np.float32)
            res = np.abs(r).max(axis=0)
            rel = np.abs(res - prev) / np.maximum(res, np.finfo(np.float32).tiny)
            stall = np.where(rel < 1e-12, stall + 1, 0)
            prev = res
            ok = res <= thresh
            fin = live & (ok | (stall >= 20) | (it >= max_iter))
            iters[fin] = it; res_out[fin] = res[fin]
            status[fin] = np.where(ok[fin], 0, np.where(stall[fin] >= 20, 1, 2))
            live &= ~fin
            y = (y + bcur * r).astype(np.float32)
        yb = (y * tn).astype(np.float32)
        w = ((x - az) + yb).astype(np.float32)
        sup = np.abs(w) > tn
        sg = np.where(w > 0, np.float32(1), np.float32(-1))
        l = np.where(sup, (az - yb) + sg * tn, x).astype(np.float32)
        v = np.where(sup, az + sg * tn, x + yb).astype(np.float32)
        z = product(mode, A, AT, v, left=False)
        az = product(mode, A, AT, z, left=True)
        it += 1
        bcur = bnext
        bnext = np.minimum(np.float32(rho) * bnext, bmax).astype(np.float32)
    return z, iters, status, res_out


def main():
    nunits = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    rng = np.random.default_rng(0)
    s, k, r = 1000, 100, 100
    # cfg3-like column units: x = (L0 column on the seed rows) + 5% impulses in [-500, 500]
    xf = rng.standard_normal((s, r)); yf = rng.standard_normal((nunits, r))
    l0 = xf @ yf.T
    q, _ = np.linalg.qr(xf)
    a = q[:, :k]
    mask = rng.random((s, nunits)) < 0.05
    x = l0 + mask * rng.uniform(-500, 500, (s, nunits))
    tol = 1e-7
    z64, e64, it64, res64, st64 = adm_filter.solve_units(x, a, tol)
    print(f"fp64 oracle: mean iters {it64.mean():.2f} max {it64.max()} failed {(st64 != 0).sum()}")
    for mode in sys.argv[2:] or ["fp32", "x3", "x5"]:
        z, it, st, res = adm_fp32(x, a, tol, mode)
        dz = np.linalg.norm(z - z64) / np.linalg.norm(z64)
        print(f"{mode:5s}: mean iters {it.mean():.2f} max {it.max()} stalled {(st == 1).sum()} maxiter {(st == 2).sum()} "
              f"iters==fp64 {(it == it64).mean():.2f}  rel dz {dz:.2e}")


if __name__ == "__main__":
    main()
