"""CPU ORACLE of the saliency front-end (§3 and §7.2,
P:516-570, Itti's model as SPEC's `saliency` module fixes its gaps) -- TEST INFRASTRUCTURE
ONLY (same rules as oracle/__init__.py).

Plain numpy float32, every arithmetic step in the order include/gc.h documents for
gc_saliency (products and sums never fused), exact reductions (min / max, and the mean of the
local maxima from an integer fixed-point sum), so the device result must equal this one bit
for bit.  Readings: DESIGN.md c18-c23.

  features ("intensity, color opponents, edge orientation and optical flow"):
      I = (r + g + b) / 3, RG = (r - g) / I, BY = (b - (r + g) / 2) / I (0 where I < 0.1),
      M = |I - I_prev| (frame difference for the motion feature, SPEC saliency decisions)
  Gaussian pyramid: [1 4 6 4 1]/16 separable blur, clamped border, decimation by 2
  orientation: |G_theta * I| with 9 x 9 even Gabor filters ("filter convolution")
  centre-surround: |L_c - up(L_s)|, c in {2,3,4}, s = c + {3,4}, bilinear up-sampling
  N(.) ("global and local [extrema]"): rescale to [0,1], local maxima in a
      radius-7 window, times (1 - mean of the local maxima except the global one)^2
  weighted addition: per class at level 4, then N of each class, their mean, N.

Parity status: pinned (tests/test_saliency_oracle.py: SPEC's worked examples for N(.),
constant / grey images, filter symmetries, closed forms of the pyramid and the up-sampling).
"""
from __future__ import annotations

import math

import numpy as np

F = np.float32
NLEV = 9
LMR = 7
CENTERS = (2, 3, 4)
DELTAS = (3, 4)


def gabor_kernels():
    """[4, 9, 9] float32: even Gabor, sigma 2, wavelength 6, aspect 0.5, mean removed."""
    out = np.zeros((4, 9, 9), np.float32)
    for t in range(4):
        th = t * math.pi / 4.0
        g = np.zeros((9, 9))
        for j in range(9):
            for i in range(9):
                x, y = i - 4, j - 4
                xr = x * math.cos(th) + y * math.sin(th)
                yr = -x * math.sin(th) + y * math.cos(th)
                g[j, i] = math.exp(-(xr * xr + 0.25 * yr * yr) / (2.0 * 2.0 * 2.0)) * math.cos(2.0 * math.pi * xr / 6.0)
        mean = 0.0
        for v in g.reshape(-1):  # the same summation order as the library's host code
            mean += v
        mean /= 81
        out[t] = (g - mean).astype(np.float32)
    return out


def features(img, prev=None):
    c = img.astype(np.float32) / F(255.0)
    r, g, b = c[..., 0], c[..., 1], c[..., 2]
    I = ((r + g) + b) / F(3.0)
    ok = I >= F(0.1)
    safe = np.where(ok, I, F(1.0))
    RG = np.where(ok, (r - g) / safe, F(0.0)).astype(np.float32)
    BY = np.where(ok, (b - (r + g) / F(2.0)) / safe, F(0.0)).astype(np.float32)
    if prev is None:
        M = np.zeros_like(I)
    else:
        p = prev.astype(np.float32) / F(255.0)
        pin = ((p[..., 0] + p[..., 1]) + p[..., 2]) / F(3.0)
        M = np.abs(I - pin)
    return I.astype(np.float32), RG, BY, M.astype(np.float32)


def down(a):
    """Blur [1 4 6 4 1]/16 (clamped) and decimate: out(y,x) = sum_j w_j sum_i w_i a(2y+j-2, 2x+i-2)."""
    h, w = a.shape
    h2, w2 = (h + 1) // 2, (w + 1) // 2
    wt = [F(1.0) / F(16.0), F(4.0) / F(16.0), F(6.0) / F(16.0), F(4.0) / F(16.0), F(1.0) / F(16.0)]
    ys = np.arange(h2)
    xs = np.arange(w2)
    acc = np.zeros((h2, w2), np.float32)
    for j in range(5):
        yy = np.clip(2 * ys + j - 2, 0, h - 1)
        row = np.zeros((h2, w2), np.float32)
        for i in range(5):
            xx = np.clip(2 * xs + i - 2, 0, w - 1)
            row = row + wt[i] * a[yy][:, xx]
        acc = acc + wt[j] * row
    return acc


def pyramid(a):
    levels = [a]
    for _ in range(1, NLEV):
        levels.append(down(levels[-1]))
    return levels


def gabor(a, k):
    h, w = a.shape
    ys, xs = np.arange(h), np.arange(w)
    acc = np.zeros((h, w), np.float32)
    for j in range(9):
        yy = np.clip(ys + j - 4, 0, h - 1)
        rows = a[yy]
        for i in range(9):
            xx = np.clip(xs + i - 4, 0, w - 1)
            acc = acc + k[j, i] * rows[:, xx]
    return np.abs(acc)


def bilinear(s, hc, wc):
    """Sample s (hs x ws) at the centres of an hc x wc grid."""
    hs, ws = s.shape
    y = np.arange(hc, dtype=np.float32)[:, None]
    x = np.arange(wc, dtype=np.float32)[None, :]
    sy = (y + F(0.5)) * (F(hs) / F(hc)) - F(0.5)
    sx = (x + F(0.5)) * (F(ws) / F(wc)) - F(0.5)
    fy0, fx0 = np.floor(sy), np.floor(sx)
    ay, ax = sy - fy0, sx - fx0
    y0 = np.clip(fy0.astype(np.int64), 0, hs - 1)
    y1 = np.clip(fy0.astype(np.int64) + 1, 0, hs - 1)
    x0 = np.clip(fx0.astype(np.int64), 0, ws - 1)
    x1 = np.clip(fx0.astype(np.int64) + 1, 0, ws - 1)
    top = (F(1.0) - ax) * s[y0, x0] + ax * s[y0, x1]
    bot = (F(1.0) - ax) * s[y1, x0] + ax * s[y1, x1]
    return ((F(1.0) - ay) * top + ay * bot).astype(np.float32)


def window_max(v, r=LMR):
    h, w = v.shape
    xs, ys = np.arange(w), np.arange(h)
    rm = v.copy()
    for d in range(1, r + 1):
        rm = np.maximum(rm, np.maximum(v[:, np.clip(xs - d, 0, w - 1)], v[:, np.clip(xs + d, 0, w - 1)]))
    cm = rm.copy()
    for d in range(1, r + 1):
        cm = np.maximum(cm, np.maximum(rm[np.clip(ys - d, 0, h - 1)], rm[np.clip(ys + d, 0, h - 1)]))
    return cm


def normalize(v):
    """N(.): rescale to [0,1]; times (1 - mbar)^2, mbar = mean of the local maxima (>= every
    pixel of their radius-7 window, > 0) other than one instance of the global maximum."""
    lo, hi = v.min(), v.max()
    if not hi > lo:
        return np.zeros_like(v)
    r = ((v - lo) / (hi - lo)).astype(np.float32)
    wm = window_max(r)
    loc = (r > 0) & (r == wm)
    cnt = int(loc.sum())
    fac = F(1.0)
    if cnt > 1:
        s = int(np.floor(r[loc].astype(np.float64) * 16777216.0).astype(np.int64).sum())
        mb = float(s - 16777216) / 16777216.0 / float(cnt - 1)
        m = F(mb)
        fac = (F(1.0) - m) * (F(1.0) - m)
    return (r * fac).astype(np.float32)


def to_level4(v, l):
    for _ in range(l, 4):
        v = down(v)
    return v


def saliency(img, prev=None):
    """One frame: RGB [H,W,3] uint8 (+ previous frame) -> saliency at level 4 (float32)."""
    I, RG, BY, M = features(img, prev)
    P = [pyramid(x) for x in (I, RG, BY, M)]
    ks = gabor_kernels()
    O = [[None, None] + [gabor(P[0][l], ks[t]) for l in range(2, NLEV)] for t in range(4)]
    h4, w4 = P[0][4].shape
    cls = [np.zeros((h4, w4), np.float32) for _ in range(4)]
    chans = [(P[0], 0), (P[1], 1), (P[2], 1), (P[3], 3)] + [(O[t], 2) for t in range(4)]
    for ch, (pyr, k) in enumerate(chans):
        acc = np.zeros((h4, w4), np.float32) if ch >= 4 else cls[k]
        for c in CENTERS:
            for dl in DELTAS:
                s = c + dl
                hc, wc = pyr[c].shape
                fm = np.abs(pyr[c] - bilinear(pyr[s], hc, wc)).astype(np.float32)
                acc = acc + to_level4(normalize(fm), c)
        if ch >= 4:
            cls[2] = cls[2] + normalize(acc)
        else:
            cls[k] = acc
    n = [normalize(c) for c in cls]
    return normalize((((n[0] + n[1]) + n[2]) + n[3]) / F(4.0))


def prior_code(sal, H, W):
    v = bilinear(sal, H, W)
    c = np.floor(F(65535.0) * v + F(0.5))
    return np.clip(c, 0, 65535).astype(np.uint16)
