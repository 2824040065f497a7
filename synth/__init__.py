"""Seeded synthetic input generator (test/bench infrastructure, not the method).

Wraps ``libsynth.so`` (synth_host.c + synth_cuda.cu).  The generator draws int32
t-link / n-link capacities shaped like the paper's saliency-driven frames
(DESIGN.md "Input recipe").  It holds none of the min-cut
arithmetic, so both the oracle side and the CUDA side may use it.

Kinds: ``blob`` (realistic saliency-blob video, configs C1-C4), ``serpentine``
(adversarial long-path caps, C5), ``random`` (uniform stress caps).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

KINDS = {"blob": 0, "serpentine": 1, "random": 2}
BASE_SEED = 10080502  # config i uses BASE_SEED + i
CAP_MAX = (1 << 26) - 1


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        L.sy_gen_host.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.sy_gen_host.restype = None
        L.sy_gen_cuda.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.sy_gen_cuda.restype = ctypes.c_int
        L.sy_kalman_weights.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.sy_set_random_params.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.sy_set_serp_params.argtypes = [ctypes.c_int, ctypes.c_int]
        L.sy_gen_energy_host.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.sy_gen_energy_host.restype = None
        L.sy_gen_energy_cuda.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.sy_gen_energy_cuda.restype = ctypes.c_int
        _LIB = L
    return _LIB


def set_random_params(rmax_t=1000, rmax_n=1000, rzero_pct=20):
    lib().sy_set_random_params(int(rmax_t), int(rmax_n), int(rzero_pct))


def set_serpentine_params(lane=64, big=1 << 20):
    lib().sy_set_serp_params(int(lane), int(big))


def kalman_weights(seq_t: int):
    """(w_f, w_q, sigma^2_xi(t-1)) for the seq_t-th frame, Sec. 6 as printed."""
    wf, wq, v = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().sy_kalman_weights(int(seq_t), ctypes.byref(wf), ctypes.byref(wq), ctypes.byref(v))
    return wf.value, wq.value, v.value


def gen_host(kind: str, seed: int, t0: int, n: int, H: int, W: int, K: int = 4, garbage: bool = True,
             seq_len: int = 0):
    """CPU twin: returns (cap_s [n,H,W], cap_t [n,H,W], cap_nb [n,K,H,W]) int32 numpy arrays."""
    cs = np.empty((n, H, W), np.int32)
    ct = np.empty((n, H, W), np.int32)
    nb = np.empty((n, K, H, W), np.int32)
    lib().sy_gen_host(KINDS[kind], seed, t0, n, H, W, K, int(garbage), int(seq_len),
                      cs.ctypes.data, ct.ctypes.data, nb.ctypes.data)
    return cs, ct, nb


def gen_cuda(kind: str, seed: int, t0: int, n: int, H: int, W: int, K: int, cs_ptr: int, ct_ptr: int,
             nb_ptr: int, stream: int = 0, garbage: bool = True, seq_len: int = 0):
    """CUDA twin: fills caller-owned device buffers (raw pointers) with the same caps as gen_host."""
    rc = lib().sy_gen_cuda(KINDS[kind], seed, t0, n, H, W, K, int(garbage), int(seq_len),
                           ctypes.c_void_p(cs_ptr), ctypes.c_void_p(ct_ptr), ctypes.c_void_p(nb_ptr),
                           ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"sy_gen_cuda failed rc={rc}")


def gen_torch(kind: str, seed: int, t0: int, n: int, H: int, W: int, K: int, device="cuda", garbage=True,
              seq_len=0):
    """Allocate torch device tensors and fill them with the CUDA twin."""
    import torch
    cs = torch.empty((n, H, W), dtype=torch.int32, device=device)
    ct = torch.empty((n, H, W), dtype=torch.int32, device=device)
    nb = torch.empty((n, K, H, W), dtype=torch.int32, device=device)
    gen_cuda(kind, seed, t0, n, H, W, K, cs.data_ptr(), ct.data_ptr(), nb.data_ptr(),
             torch.cuda.current_stream().cuda_stream, garbage=garbage, seq_len=seq_len)
    return cs, ct, nb


def random_caps(rng: np.random.Generator, H: int, W: int, K: int, tmax: int = 20, nmax: int = 20,
                zero_frac: float = 0.2, garbage: bool = True, n: int = 1):
    """Plain numpy random caps (small stress instances for tests). Off-grid entries get garbage."""
    cs = rng.integers(0, tmax + 1, size=(n, H, W), dtype=np.int64).astype(np.int32)
    ct = rng.integers(0, tmax + 1, size=(n, H, W), dtype=np.int64).astype(np.int32)
    nb = rng.integers(0, nmax + 1, size=(n, K, H, W), dtype=np.int64).astype(np.int32)
    nb[rng.random(nb.shape) < zero_frac] = 0
    if garbage:
        g = rng.integers(-(1 << 31), (1 << 31) - 1, size=nb.shape, dtype=np.int64).astype(np.int32)
        mask = offgrid_mask(H, W, K)[None]
        nb = np.where(mask, g, nb).astype(np.int32)
    return cs, ct, nb


DY = [0, 0, 1, -1, 1, -1, 1, -1]
DX = [1, -1, 0, 0, 1, -1, -1, 1]


def offgrid_mask(H: int, W: int, K: int):
    """[K,H,W] bool: True where n-link k of pixel (y,x) points outside the grid."""
    y = np.arange(H)[:, None]
    x = np.arange(W)[None, :]
    out = np.zeros((K, H, W), bool)
    for k in range(K):
        y2, x2 = y + DY[k], x + DX[k]
        out[k] = (y2 < 0) | (y2 >= H) | (x2 < 0) | (x2 >= W)
    return out


# ---------------------------------------------------------------- energy inputs (NEXT-1)
def gen_energy_host(seed: int, t0: int, n: int, H: int, W: int, seq_len: int = 0):
    """Blob frames as energy inputs: RGB image [n,H,W,3] uint8 and prior code [n,H,W] uint16."""
    rgb = np.empty((n, H, W, 3), np.uint8)
    prior = np.empty((n, H, W), np.uint16)
    lib().sy_gen_energy_host(seed, t0, n, H, W, int(seq_len), rgb.ctypes.data, prior.ctypes.data)
    return rgb, prior


def gen_energy_torch(seed: int, t0: int, n: int, H: int, W: int, seq_len: int = 0, device="cuda"):
    """CUDA twin of gen_energy_host (bit-identical)."""
    import torch
    rgb = torch.empty((n, H, W, 3), dtype=torch.uint8, device=device)
    prior = torch.empty((n, H, W), dtype=torch.uint16, device=device)
    rc = lib().sy_gen_energy_cuda(seed, t0, n, H, W, int(seq_len), ctypes.c_void_p(rgb.data_ptr()),
                                  ctypes.c_void_p(prior.data_ptr()),
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"sy_gen_energy_cuda failed rc={rc}")
    return rgb, prior


def energy_gmms():
    """The colour model of the synthetic blob frames as two 2-component RGB GMMs (weights [2],
    means [2,3], covariances [2,3,3]) for label 0 (background ~ 80-120 grey) and label 1
    (objects ~ 200 grey); grey colours make the channels strongly correlated.  Input data for
    gc_solve_energy (the paper fits these with EM, P:293-301, P:580-582 -- out of scope)."""
    J = np.ones((3, 3))
    I3 = np.eye(3)
    bg = (np.array([0.6, 0.4]), np.array([[100.0, 100.0, 100.0], [85.0, 88.0, 92.0]]),
          np.stack([30.0 ** 2 * (0.95 * J + 0.05 * I3), 20.0 ** 2 * (0.9 * J + 0.1 * I3)]))
    ob = (np.array([0.7, 0.3]), np.array([[200.0, 200.0, 200.0], [190.0, 205.0, 195.0]]),
          np.stack([25.0 ** 2 * (0.95 * J + 0.05 * I3), 20.0 ** 2 * (0.85 * J + 0.15 * I3)]))
    return bg, ob


ENERGY_PARAMS = dict(lam=10.0, sigma=0.1, kappa=0.05, eps=1e-6, scale=64.0)  # reading c5 / c9 / c11
