"""CPU ORACLE of the energy -> capacity construction -- TEST
INFRASTRUCTURE ONLY (same rules as oracle/__init__.py: only tests/, smoke() and bench.py's
baseline legs may use it; the product never imports it).

Plain numpy float64, written from PAPER.md §4 under the readings of DESIGN.md:

  energy (Eq. 1): E(A|D) = sum_x psi1(D|A_x) + xi1(A_x)
                                   + sum_{y in N_x} psi2(D|A_x,A_y) + xi2(A_x,A_y)
  psi1(D|A_x) = -log p(C_x|A_x), p(C|A) a Gaussian mixture over RGB
  xi1(A_x)    = -log p(A_x), p(A_x = 1) the prior, p(A_x = 0) = 1 - p(A_x = 1)
  psi2 + xi2  = lambda exp(-(I_x - I_y)^2 / (2 sigma^2)) / ||x - y|| + kappa if A_x != A_y
                (P:310-321 with the sign / scale reading c5; I scaled to [0, 1] by /255)
  t-links: c(s, v) = psi1(A=0) + xi1(A=0), c(v, t) = psi1(A=1) + xi1(A=1)
  n-links: c(v_x, v_y) = psi2 + xi2

plus the library's documented conventions (include/gc.h gc_energy_params): intensity = the
integer luma (77 R + 150 G + 29 B + 128) >> 8; p = clamp(u / 65535, eps, 1 - eps) for prior
code u; quantisation q(x) = floor(scale x + 0.5) clamped to [0, 2^26 - 1].

The mixture density is evaluated from its definition, sum_m w_m N(C; mu_m, S_m) with
N = exp(-d^T S^-1 d / 2) / sqrt((2 pi)^3 det S) (numpy inv / det), as a log-sum-exp.
Parity status: pinned (tests/test_energy_oracle.py: scipy multivariate_normal, closed forms,
symmetry and monotonicity of the n-links, hand-computed values).
"""
from __future__ import annotations

import numpy as np

CAP_MAX = (1 << 26) - 1
DY = [0, 0, 1, -1, 1, -1, 1, -1]
DX = [1, -1, 0, 0, 1, -1, -1, 1]


def luma(rgb):
    """Integer luma of uint8 RGB [..., 3] (gc.h gc_energy_params)."""
    r = rgb[..., 0].astype(np.int64)
    g = rgb[..., 1].astype(np.int64)
    b = rgb[..., 2].astype(np.int64)
    return (77 * r + 150 * g + 29 * b + 128) >> 8


def gmm_nll(C, weights, means, covs):
    """-log sum_m w_m N(C; mu_m, S_m) for colours C [..., 3] (float64)."""
    C = np.asarray(C, np.float64)
    terms = []
    for w, mu, S in zip(weights, means, covs):
        S = np.asarray(S, np.float64)
        d = C - np.asarray(mu, np.float64)
        P = np.linalg.inv(S)
        quad = np.einsum("...i,ij,...j->...", d, P, d)
        terms.append(np.log(w) - 0.5 * quad - 0.5 * np.log((2.0 * np.pi) ** 3 * np.linalg.det(S)))
    T = np.stack(terms)
    mx = T.max(axis=0)
    return -(mx + np.log(np.exp(T - mx).sum(axis=0)))


def nlink_value(dI, dist, lam, sigma, kappa):
    """psi2 + xi2 of an n-link between intensities differing by dI (0..255) at distance dist."""
    x = np.asarray(dI, np.float64) / 255.0
    return lam * np.exp(-(x * x) / (2.0 * sigma * sigma)) / dist + kappa


def quantize(x, scale):
    v = np.floor(scale * np.asarray(x, np.float64) + 0.5)
    return np.clip(v, 0, CAP_MAX).astype(np.int64)


def caps(rgb, prior, gmm0, gmm1, K, lam=10.0, sigma=0.1, kappa=0.05, eps=1e-6, scale=64.0, raw=False):
    """One frame: rgb [H,W,3] uint8, prior [H,W] uint16, gmm0 / gmm1 = (weights, means, covs)
    of label 0 / 1 -> (cs, ct, nb[K]) int32 (off-grid n-links 0); with raw=True also the
    unrounded values scale * cost (for the rounding-boundary tolerance of DESIGN.md)."""
    H, W, _ = rgb.shape
    p = np.clip(prior.astype(np.float64) / 65535.0, eps, 1.0 - eps)
    C = rgb.astype(np.float64)
    u0 = gmm_nll(C, *gmm0) - np.log(1.0 - p)  # c(s, v) = psi1(A=0) + xi1(A=0)
    u1 = gmm_nll(C, *gmm1) - np.log(p)        # c(v, t) = psi1(A=1) + xi1(A=1)
    I = luma(rgb)
    nb = np.zeros((K, H, W), np.int64)
    nraw = np.zeros((K, H, W), np.float64)
    for k in range(K):
        dy, dx = DY[k], DX[k]
        y0, y1 = max(0, -dy), H - max(0, dy)
        x0, x1 = max(0, -dx), W - max(0, dx)
        dI = np.abs(I[y0:y1, x0:x1] - I[y0 + dy:y1 + dy, x0 + dx:x1 + dx])
        v = nlink_value(dI, np.sqrt(2.0) if k >= 4 else 1.0, lam, sigma, kappa)
        nb[k, y0:y1, x0:x1] = quantize(v, scale)
        nraw[k, y0:y1, x0:x1] = scale * v
    out = (quantize(u0, scale).astype(np.int32), quantize(u1, scale).astype(np.int32), nb.astype(np.int32))
    if raw:
        return out, (scale * u0, scale * u1, nraw)
    return out
