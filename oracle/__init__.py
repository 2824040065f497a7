"""CPU ORACLE for the per-frame grid min-cut -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1008_0502_b200``) never imports it and shares no code with it.

It computes what PAPER.md §4 defines: the maximum s-t flow F* of the pixel
graph and the canonical minimum cut, mask = pixels reachable from s in the residual of a
maximum flow (readings c1, c2, c7).  Two independent exact
solvers (Dinic, Boykov-Kolmogorov) in ``oracle.cpp``; a brute-force enumerator of
cut(S) over all 2^N labelings for N <= 24.  Pins: tests/test_oracle.py.

Parity status per function:
  solve(algo="dinic"|"bk")  pinned: python brute force (tiny grids), scipy maximum_flow
                            (F on medium grids), closed forms, SPEC worked examples,
                            duality, Dinic == BK cross-check
  brute                     pinned: independent python enumeration in tests
  cut_value                 pinned: hand-computed examples
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
ALGOS = {"dinic": 0, "bk": 1}


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        L.oracle_solve.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp]
        L.oracle_solve.restype = ctypes.c_int64
        L.oracle_cut_value.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]
        L.oracle_cut_value.restype = ctypes.c_int64
        L.oracle_brute.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]
        L.oracle_brute.restype = ctypes.c_int64
        L.oracle_solve_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         vp, vp, vp, vp, vp, ctypes.c_int]
        L.oracle_solve_batch.restype = None
        _LIB = L
    return _LIB


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def solve(cs, ct, nb, algo: str = "dinic", want_flow: bool = False):
    """One frame: cs, ct [H,W], nb [K,H,W] int32 -> (F, mask[H,W] uint8[, flow_fwd[K/2,H,W]])."""
    cs, ct, nb = _c(cs, np.int32), _c(ct, np.int32), _c(nb, np.int32)
    K, H, W = nb.shape
    mask = np.zeros((H, W), np.uint8)
    fw = np.zeros((K // 2, H, W), np.int32) if want_flow else None
    F = lib().oracle_solve(ALGOS[algo], H, W, K, cs.ctypes.data, ct.ctypes.data, nb.ctypes.data,
                           mask.ctypes.data, fw.ctypes.data if want_flow else None)
    return (int(F), mask, fw) if want_flow else (int(F), mask)


def cut_value(cs, ct, nb, mask) -> int:
    cs, ct, nb = _c(cs, np.int32), _c(ct, np.int32), _c(nb, np.int32)
    m = _c(mask, np.uint8)
    K, H, W = nb.shape
    return int(lib().oracle_cut_value(H, W, K, cs.ctypes.data, ct.ctypes.data, nb.ctypes.data, m.ctypes.data))


def brute(cs, ct, nb):
    """Exhaustive min over all 2^N labelings (N <= 24): (F*, intersection of minimisers)."""
    cs, ct, nb = _c(cs, np.int32), _c(ct, np.int32), _c(nb, np.int32)
    K, H, W = nb.shape
    mask = np.zeros((H, W), np.uint8)
    F = lib().oracle_brute(H, W, K, cs.ctypes.data, ct.ctypes.data, nb.ctypes.data, mask.ctypes.data)
    if F < 0:
        raise ValueError("brute force limited to N <= 24 pixels")
    return int(F), mask


def solve_batch(cs, ct, nb, algo: str = "bk", threads: int | None = None):
    """n frames on a host thread pool: cs, ct [n,H,W], nb [n,K,H,W] -> (F [n] int64, mask [n,H,W])."""
    cs, ct, nb = _c(cs, np.int32), _c(ct, np.int32), _c(nb, np.int32)
    n, K, H, W = nb.shape
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    F = np.zeros(n, np.int64)
    mask = np.zeros((n, H, W), np.uint8)
    lib().oracle_solve_batch(ALGOS[algo], n, H, W, K, cs.ctypes.data, ct.ctypes.data, nb.ctypes.data,
                             mask.ctypes.data, F.ctypes.data, int(threads))
    return F, mask


def _splitmix64(z):
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def mask_digest(mask):
    """(popcount, H) of one [H,W] mask, H = sum over set pixels p = y*W + x of splitmix64(p + 1)
    mod 2^64, returned as a signed int64 -- the digest include/gc.h documents for
    gc_frame_digest, written out here independently (numpy) for comparing oracle masks."""
    idx = np.flatnonzero(np.asarray(mask).reshape(-1)).astype(np.uint64)
    with np.errstate(over="ignore"):
        h = _splitmix64(idx + np.uint64(1)).sum(dtype=np.uint64)
    return int(idx.size), int(np.array(h, dtype=np.uint64).view(np.int64))
