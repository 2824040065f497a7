"""CPU ORACLE of the prior update (§6) -- TEST
INFRASTRUCTURE ONLY (same rules as oracle/__init__.py).

Written from the paper's §6 and the integer conventions include/gc.h documents for
gc_prior_update:

  f(A_{t-1}, x)     the previous mask smoothed by a Gaussian: separable, integer
                    taps g_i = floor(1024 exp(-i^2 / (2 sigma^2)) + 0.5), |i| <= radius, border
                    replicated; f = S / G^2 with S the 2-D tap-weighted sum, G = sum_i g_i
  p(A_t = 1)        = w_f f + (1 - w_f) q (P:428-436 as printed, reading c10), w_f = s1 /
                    (s1 + s2 + v(t-1)), v(t) = s1 (s2 + v(t-1)) / (s1 + s2 + v(t-1))
  frame edge        p = 0 within `band` px of the border
  output code       round(65535 p) in exact integers:
                    (wf S 65535 + (4096 - wf) q G^2 + 2048 G^2) // (4096 G^2), wf = round(4096 w_f)

Plain numpy int64 (the 2-D sum as an explicit double loop over taps) and Python floats for
the scalar recursion.  Parity status: pinned (tests/test_prior_oracle.py: impulse response =
outer product of the taps, constant masks, the steady state of the recursion in closed form and
the weights SURVEY.md §8(c) c10 prints).
"""
from __future__ import annotations

import math

import numpy as np


def gauss_taps(sigma: float, radius: int):
    return [int(math.floor(1024.0 * math.exp(-(i * i) / (2.0 * sigma * sigma)) + 0.5)) for i in range(radius + 1)]


def kalman_step(s1: float, s2: float, v_prev: float):
    """(w_f, v_next) of one step of §6 as printed."""
    den = s1 + s2 + v_prev
    return s1 / den, s1 * (s2 + v_prev) / den


def wf_q12(w_f: float) -> int:
    return int(math.floor(4096.0 * w_f + 0.5))


def smooth_sum(mask, taps):
    """S(y, x) = sum_{i,j} g_|i| g_|j| m(clamp(y+j), clamp(x+i)) (int64), border replicated."""
    m = (np.asarray(mask) != 0).astype(np.int64)
    H, W = m.shape
    R = len(taps) - 1
    ys = np.arange(H)
    xs = np.arange(W)
    S = np.zeros((H, W), np.int64)
    for j in range(-R, R + 1):
        rows = m[np.clip(ys + j, 0, H - 1)]
        for i in range(-R, R + 1):
            S += taps[abs(j)] * taps[abs(i)] * rows[:, np.clip(xs + i, 0, W - 1)]
    return S


def prior_update(mask_prev, q, wf: int, taps, band: int):
    """One frame: mask_prev [H,W], q [H,W] uint16 codes, wf in 1/4096 -> prior codes [H,W] uint16."""
    S = smooth_sum(mask_prev, taps)
    G = taps[0] + 2 * sum(taps[1:])
    G2 = G * G
    qv = np.asarray(q, np.int64)
    num = wf * S * 65535 + (4096 - wf) * qv * G2 + 2048 * G2
    out = num // (4096 * G2)
    H, W = S.shape
    y = np.arange(H)[:, None]
    x = np.arange(W)[None, :]
    edge = (y < band) | (x < band) | (y >= H - band) | (x >= W - band)
    out = np.where(edge, 0, out)
    return out.astype(np.uint16)
