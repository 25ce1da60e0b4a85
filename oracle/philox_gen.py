"""Oracle: the synthetic-input generator, bit for bit (TEST INFRASTRUCTURE ONLY).

Restates csrc/philox.cuh + the generator epilogue of csrc/dense.cu in numpy, on top of
numpy.random.Philox (a third-party Philox4x64-10; block b of stream (seed, id) is what
Philox(key=[seed, id], counter=[b, 0, 0, 0]) emits first).  Every float transform uses the
same sequence of separately rounded float32 operations as the device, so values agree
exactly.  The random model is that of the reference generator synth.generate
(synth.py:43-64): Gaussian factors, support of density rho_s, values U[-mag, mag].
"""

import numpy as np

STREAM_X, STREAM_Y, STREAM_S, STREAM_BOX = 1, 2, 3, 4
GAUSSIAN, VIDEO = 0, 1
VIDEO_W, VIDEO_H, VIDEO_BOXES = 320, 240, 6

f32 = np.float32
_TWO_M24 = f32("5.9604644775390625e-08")
_SQRT2 = f32("1.41421353816986083984375")
_LN2 = f32("0.693147182464599609375")
_HALF_PI = f32("1.57079637050628662109375")
_LOG_C = [f32(c) for c in ("0.0909090936183929443359375", "0.111111111938953399658203125",
                           "0.14285714924335479736328125", "0.20000000298023223876953125",
                           "0.3333333432674407958984375")]
_COS_C = [f32(c) for c in ("2.08767570e-09", "-2.75573188e-07", "2.48015876e-05", "-1.38888892e-03",
                           "4.16666679e-02", "-0.5")]
_SIN_C = [f32(c) for c in ("1.60590444e-10", "-2.50521079e-08", "2.75573188e-06", "-1.98412701e-04",
                           "8.33333377e-03", "-0.166666672")]


def draws(seed, stream, start, count):
    """Raw 64-bit draws number start .. start+count-1 of stream (seed, stream)."""
    if count <= 0:
        return np.zeros(0, dtype=np.uint64)
    b0 = start // 4
    nb = (start + count + 3) // 4 - b0
    g = np.random.Philox(key=np.array([seed, stream], dtype=np.uint64),
                         counter=np.array([b0, 0, 0, 0], dtype=np.uint64))
    raw = g.random_raw(4 * nb)
    off = start - 4 * b0
    return np.asarray(raw[off:off + count], dtype=np.uint64)


def unit_float(b32):
    return (b32 >> np.uint32(8)).astype(f32) * _TWO_M24


def sym_uniform(b32, mag):
    return f32(mag) * ((f32(2.0) * unit_float(b32)) - f32(1.0))


def exact_log(u):
    bits = u.view(np.uint32)
    e = ((bits >> np.uint32(23)) & np.uint32(0xFF)).astype(np.int32) - 127
    f = ((bits & np.uint32(0x7FFFFF)) | np.uint32(0x3F800000)).view(f32)
    big = f > _SQRT2
    f = np.where(big, f * f32(0.5), f)
    e = e + big.astype(np.int32)
    s = (f - f32(1.0)) / (f + f32(1.0))
    s2 = s * s
    p = _LOG_C[0]
    for c in _LOG_C[1:]:
        p = p * s2 + c
    p = p * s2 + f32(1.0)
    lnf = (f32(2.0) * s) * p
    return e.astype(f32) * _LN2 + lnf


def exact_cos2pi(t):
    t4 = t * f32(4.0)
    qf = np.floor(t4)
    q = qf.astype(np.int32)
    th = (t4 - qf) * _HALF_PI
    x = th * th
    c = _COS_C[0]
    for k in _COS_C[1:]:
        c = c * x + k
    c = c * x + f32(1.0)
    sn = _SIN_C[0]
    for k in _SIN_C[1:]:
        sn = sn * x + k
    sn = sn * x + f32(1.0)
    sn = th * sn
    return np.select([q == 0, q == 1, q == 2], [c, -sn, -c], sn).astype(f32)


def normal_from(v):
    hi = (v >> np.uint64(32)).astype(np.uint32)
    lo = (v & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    u1 = ((hi >> np.uint32(8)) + np.uint32(1)).astype(f32) * _TWO_M24
    u2 = unit_float(lo)
    rad = np.sqrt(f32(-2.0) * exact_log(u1))
    return rad * exact_cos2pi(u2)


def factors(seed, kind, m, n, r):
    """X (m x r), Y (n x r) float32 (l1f_generate_factors_f32)."""
    vx = draws(seed, STREAM_X, 0, m * r)
    vy = draws(seed, STREAM_Y, 0, n * r)
    if kind == GAUSSIAN:
        x, y = normal_from(vx), normal_from(vy)
    else:
        yscale = f32(255.0) / f32(r) if r else f32(0.0)
        x = unit_float((vx >> np.uint64(32)).astype(np.uint32))
        y = unit_float((vy >> np.uint64(32)).astype(np.uint32)) * yscale
    return x.reshape(m, r), y.reshape(n, r)


def _boxes(seed):
    out = []
    for b in range(VIDEO_BOXES):
        v = draws(seed, STREAM_BOX, 4 * b, 4)
        hi = [int(w) >> 32 for w in v]
        lo = [int(w) & 0xFFFFFFFF for w in v]
        out.append(dict(w=10 + hi[0] % 31, h=10 + lo[0] % 31, x0=hi[1] % VIDEO_W, y0=lo[1] % VIDEO_H,
                        vx=hi[2] % 7 - 3, vy=lo[2] % 7 - 3))
    return out


def video_mask(seed, rows, cols):
    """Coverage of pixels `rows` in frames `cols` by the moving boxes."""
    rows = np.asarray(rows, dtype=np.int64)[:, None]
    f = np.asarray(cols, dtype=np.int64)[None, :]
    px, py = rows % VIDEO_W, rows // VIDEO_W
    hit = np.zeros((rows.shape[0], f.shape[1]), dtype=bool)
    for B in _boxes(seed):
        bx = (B["x0"] + B["vx"] * f) % VIDEO_W
        by = (B["y0"] + B["vy"] * f) % VIDEO_H
        hit |= ((px - bx) % VIDEO_W < B["w"]) & ((py - by) % VIDEO_H < B["h"])
    return hit


def threshold_u32(rho_s):
    t = np.floor(np.float64(f32(rho_s)) * 4294967296.0)
    return np.uint32(0xFFFFFFFF) if t >= 4294967295.0 else np.uint32(t)


def block(seed, kind, m, n, r, rho_s, magnitude, rows, cols, x=None, y=None, want_l0=False):
    """M[np.ix_(rows, cols)] (float32, bit-exact with l1f_generate_f32) and optionally L0."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if x is None:
        x, y = factors(seed, kind, m, n, r)
    xr, yc = x[rows], y[cols]
    l0 = np.zeros((rows.size, cols.size), dtype=f32)
    for t in range(r):  # separately rounded multiply and add, in t order
        l0 = l0 + xr[:, t:t + 1] * yc[:, t][None, :]
    # per-entry draws: e = i*n + j
    idx = rows[:, None] * n + cols[None, :]
    v = np.empty(idx.shape, dtype=np.uint64)
    for a, i in enumerate(rows):
        lo, hi = int(i * n + cols.min()), int(i * n + cols.max()) + 1 if cols.size else 0
        span = draws(seed, STREAM_S, lo, hi - lo)
        v[a] = span[idx[a] - lo]
    hi32 = (v >> np.uint64(32)).astype(np.uint32)
    lo32 = (v & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    if kind == GAUSSIAN:
        hit = hi32 < threshold_u32(rho_s)
    else:
        hit = video_mask(seed, rows, cols)
    s0 = np.where(hit, sym_uniform(lo32, magnitude), f32(0.0)).astype(f32)
    mm = l0 + s0
    return (mm, l0) if want_l0 else mm
