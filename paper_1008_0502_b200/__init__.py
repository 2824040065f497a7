"""B200-native batched grid min-cut (the hot path of arXiv 1008.0502, §4 / §7.3).

Thin ctypes binding over ``libgc.so`` (include/gc.h).  Argument marshalling only:
every step of the solve runs in the library's sm_100a kernels.  There is no CPU or
PyTorch fallback -- importing this package raises if the library is missing.

Functions carry the C names (``gc_create``, ``gc_solve_batch``, ``gc_solve_batch_host``,
``gc_destroy``, ``gc_last_error``, ...); :class:`GridCut` is a convenience wrapper
that allocates outputs as torch tensors (device path) or numpy arrays (host path).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["GridCut", "GcError", "gc_create", "gc_destroy", "gc_solve_batch", "gc_solve_batch_host", "gc_solve_sequences",
           "gc_solve_energy", "gc_gmm_prepare", "gc_gauss_taps", "gc_kalman_step", "gc_prior_update",
           "gc_saliency", "gc_saliency_dims", "gc_gabor_kernels",
           "gc_frame_digest", "gc_last_error", "gc_last_launches", "gc_set_profiling", "gc_get_profile", "gc_get_kernel_ms",
           "gc_set_partitions", "CAP_MAX", "PARTS_MAX",
           "STATUS", "lib_path"]

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libgc.so")
CAP_MAX = (1 << 26) - 1
STATUS = {0: "GC_OK", 1: "GC_ERR_ARG", 2: "GC_ERR_RANGE", 3: "GC_ERR_OOM", 4: "GC_ERR_CUDA", 5: "GC_ERR_NOCONV"}
PROFILE_CLASSES = ("init", "bfs", "push", "sched", "closure", "export")

if not os.path.exists(lib_path):
    raise ImportError(f"{lib_path} is missing: build it with __graft_entry__.build() (make). "
                      "There is no fallback implementation.")
_lib = ctypes.CDLL(lib_path)


class gc_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("neighborhood", ctypes.c_int), ("max_h", ctypes.c_int),
                ("max_w", ctypes.c_int), ("max_batch", ctypes.c_int), ("rounds_per_launch", ctypes.c_int),
                ("relabel_period", ctypes.c_int), ("max_launches", ctypes.c_longlong)]


class gc_batch(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("H", ctypes.c_int), ("W", ctypes.c_int),
                ("cap_s", ctypes.c_void_p), ("cap_t", ctypes.c_void_p), ("cap_nb", ctypes.c_void_p),
                ("warm_flow", ctypes.c_void_p), ("flow_out", ctypes.c_void_p), ("mask_out", ctypes.c_void_p),
                ("flow_state_out", ctypes.c_void_p), ("stats_out", ctypes.c_void_p)]


class gc_seq_batch(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int), ("L", ctypes.c_int), ("H", ctypes.c_int), ("W", ctypes.c_int),
                ("cap_s", ctypes.c_void_p), ("cap_t", ctypes.c_void_p), ("cap_nb", ctypes.c_void_p),
                ("warm_flow", ctypes.c_void_p), ("flow_out", ctypes.c_void_p), ("mask_out", ctypes.c_void_p),
                ("flow_state_out", ctypes.c_void_p), ("stats_out", ctypes.c_void_p), ("warm", ctypes.c_int)]


GMM_MAX = 4


class gc_gmm(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int), ("pad", ctypes.c_int), ("lognorm", ctypes.c_double * GMM_MAX),
                ("mean", (ctypes.c_double * 3) * GMM_MAX), ("prec", (ctypes.c_double * 6) * GMM_MAX)]


class gc_energy_params(ctypes.Structure):
    _fields_ = [("lambda_", ctypes.c_double), ("sigma", ctypes.c_double), ("kappa", ctypes.c_double),
                ("eps", ctypes.c_double), ("scale", ctypes.c_double)]


class gc_energy_batch(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("H", ctypes.c_int), ("W", ctypes.c_int),
                ("image", ctypes.c_void_p), ("prior", ctypes.c_void_p), ("gmm", ctypes.c_void_p),
                ("params", gc_energy_params),
                ("warm_flow", ctypes.c_void_p), ("flow_out", ctypes.c_void_p), ("mask_out", ctypes.c_void_p),
                ("flow_state_out", ctypes.c_void_p), ("stats_out", ctypes.c_void_p), ("caps_out", ctypes.c_void_p)]


PRIOR_RMAX = 16


class gc_prior_params(ctypes.Structure):
    _fields_ = [("radius", ctypes.c_int), ("taps", ctypes.c_int * (PRIOR_RMAX + 1)), ("band", ctypes.c_int)]


class gc_saliency_batch(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("H", ctypes.c_int), ("W", ctypes.c_int), ("image", ctypes.c_void_p),
                ("prev", ctypes.c_void_p), ("sal_out", ctypes.c_void_p), ("q_out", ctypes.c_void_p)]


_lib.gc_create.argtypes = [ctypes.POINTER(gc_config), ctypes.POINTER(ctypes.c_void_p)]
_lib.gc_create.restype = ctypes.c_int
_lib.gc_destroy.argtypes = [ctypes.c_void_p]
_lib.gc_destroy.restype = None
_lib.gc_solve_batch.argtypes = [ctypes.c_void_p, ctypes.POINTER(gc_batch), ctypes.c_void_p]
_lib.gc_solve_batch.restype = ctypes.c_int
_lib.gc_solve_sequences.argtypes = [ctypes.c_void_p, ctypes.POINTER(gc_seq_batch), ctypes.c_void_p]
_lib.gc_solve_sequences.restype = ctypes.c_int
_lib.gc_solve_energy.argtypes = [ctypes.c_void_p, ctypes.POINTER(gc_energy_batch), ctypes.c_void_p]
_lib.gc_solve_energy.restype = ctypes.c_int
_lib.gc_gmm_prepare.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(gc_gmm)]
_lib.gc_gmm_prepare.restype = ctypes.c_int
_lib.gc_gauss_taps.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
_lib.gc_gauss_taps.restype = ctypes.c_int
_lib.gc_kalman_step.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_int),
                                ctypes.POINTER(ctypes.c_double)]
_lib.gc_kalman_step.restype = ctypes.c_int
_lib.gc_prior_update.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(gc_prior_params), ctypes.c_void_p,
                                 ctypes.c_void_p]
_lib.gc_prior_update.restype = ctypes.c_int
_lib.gc_saliency.argtypes = [ctypes.c_void_p, ctypes.POINTER(gc_saliency_batch), ctypes.c_void_p]
_lib.gc_saliency.restype = ctypes.c_int
_lib.gc_saliency_dims.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
_lib.gc_saliency_dims.restype = ctypes.c_int
_lib.gc_gabor_kernels.argtypes = [ctypes.c_void_p]
_lib.gc_gabor_kernels.restype = ctypes.c_int
_lib.gc_solve_batch_host.argtypes = [ctypes.c_void_p, ctypes.POINTER(gc_batch), ctypes.c_void_p]
_lib.gc_solve_batch_host.restype = ctypes.c_int
_lib.gc_last_error.argtypes = [ctypes.c_void_p]
_lib.gc_last_error.restype = ctypes.c_char_p
_lib.gc_last_launches.argtypes = [ctypes.c_void_p]
_lib.gc_last_launches.restype = ctypes.c_longlong
_lib.gc_set_profiling.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.gc_set_profiling.restype = None
_lib.gc_set_partitions.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.gc_set_partitions.restype = ctypes.c_int
_lib.gc_get_profile.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
_lib.gc_get_profile.restype = None
_lib.gc_debug_counters.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
_lib.gc_debug_counters.restype = None
_lib.gc_get_kernel_ms.argtypes = [ctypes.c_void_p, ctypes.c_int]
_lib.gc_get_kernel_ms.restype = ctypes.c_double
_lib.gc_frame_digest.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
_lib.gc_frame_digest.restype = ctypes.c_int

EXPORTED = ("gc_create", "gc_destroy", "gc_solve_batch", "gc_solve_batch_host", "gc_last_error",
            "gc_last_launches", "gc_set_profiling", "gc_get_profile", "gc_get_kernel_ms", "gc_frame_digest",
            "gc_solve_sequences", "gc_solve_energy", "gc_gmm_prepare", "gc_gauss_taps", "gc_kalman_step",
            "gc_prior_update", "gc_saliency", "gc_saliency_dims", "gc_gabor_kernels", "gc_set_partitions")
PARTS_MAX = 8  # GC_PARTS_MAX


class GcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def gc_create(cfg: gc_config) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    st = _lib.gc_create(ctypes.byref(cfg), ctypes.byref(h))
    if st != 0:
        raise GcError(st, "gc_create failed")
    return h


def gc_destroy(ctx) -> None:
    _lib.gc_destroy(ctx)


def gc_solve_batch(ctx, batch: gc_batch, stream: int) -> int:
    return _lib.gc_solve_batch(ctx, ctypes.byref(batch), ctypes.c_void_p(stream))


def gc_solve_sequences(ctx, batch: gc_seq_batch, stream: int) -> int:
    return _lib.gc_solve_sequences(ctx, ctypes.byref(batch), ctypes.c_void_p(stream))


def gc_solve_energy(ctx, batch: gc_energy_batch, stream: int) -> int:
    return _lib.gc_solve_energy(ctx, ctypes.byref(batch), ctypes.c_void_p(stream))


def gc_gmm_prepare(weights, means, covs) -> gc_gmm:
    """gc_gmm of one label from M weights, means [M,3], covariances [M,3,3] (host, double)."""
    w = np.ascontiguousarray(weights, np.float64)
    mu = np.ascontiguousarray(means, np.float64)
    cv = np.ascontiguousarray(covs, np.float64)
    out = gc_gmm()
    st = _lib.gc_gmm_prepare(int(w.shape[0]), w.ctypes.data, mu.ctypes.data, cv.ctypes.data, ctypes.byref(out))
    if st != 0:
        raise GcError(st, "gc_gmm_prepare: bad mixture")
    return out


def gmm_table(pairs):
    """[n][2] gc_gmm array (label 0, label 1 per frame) as raw bytes (uint8 numpy), from a list
    of (bg, obj) tuples of (weights, means, covs)."""
    arr = (gc_gmm * (2 * len(pairs)))()
    for i, (bg, ob) in enumerate(pairs):
        arr[2 * i] = gc_gmm_prepare(*bg)
        arr[2 * i + 1] = gc_gmm_prepare(*ob)
    return np.frombuffer(bytes(arr), np.uint8).copy()


def gc_gauss_taps(sigma: float, radius: int):
    taps = (ctypes.c_int * (PRIOR_RMAX + 1))()
    st = _lib.gc_gauss_taps(float(sigma), int(radius), taps)
    if st != 0:
        raise GcError(st, "gc_gauss_taps: bad arguments")
    return [taps[i] for i in range(radius + 1)]


def gc_kalman_step(s1: float, s2: float, v_prev: float):
    """(wf in 1/4096, v_next) of one step of the Sec. 6 recursion as printed."""
    wf = ctypes.c_int()
    v = ctypes.c_double()
    st = _lib.gc_kalman_step(float(s1), float(s2), float(v_prev), ctypes.byref(wf), ctypes.byref(v))
    if st != 0:
        raise GcError(st, "gc_kalman_step: bad arguments")
    return wf.value, v.value


def prior_params(sigma: float, radius: int, band: int) -> gc_prior_params:
    p = gc_prior_params()
    p.radius = radius
    p.band = band
    for i, v in enumerate(gc_gauss_taps(sigma, radius)):
        p.taps[i] = v
    return p


def gc_prior_update(ctx, n, H, W, mask_prev, q, wf, params, prior_out, stream) -> int:
    return _lib.gc_prior_update(ctx, n, H, W, ctypes.c_void_p(mask_prev), ctypes.c_void_p(q), ctypes.c_void_p(wf),
                                ctypes.byref(params), ctypes.c_void_p(prior_out), ctypes.c_void_p(stream))


def gc_saliency(ctx, batch: gc_saliency_batch, stream: int) -> int:
    return _lib.gc_saliency(ctx, ctypes.byref(batch), ctypes.c_void_p(stream))


def gc_saliency_dims(H: int, W: int):
    h4, w4 = ctypes.c_int(), ctypes.c_int()
    st = _lib.gc_saliency_dims(H, W, ctypes.byref(h4), ctypes.byref(w4))
    if st != 0:
        raise GcError(st, "gc_saliency_dims: bad dims")
    return h4.value, w4.value


def gc_gabor_kernels():
    out = np.zeros((4, 9, 9), np.float32)
    _lib.gc_gabor_kernels(out.ctypes.data)
    return out


def gc_solve_batch_host(ctx, batch: gc_batch, stream: int) -> int:
    return _lib.gc_solve_batch_host(ctx, ctypes.byref(batch), ctypes.c_void_p(stream))


def gc_last_error(ctx) -> str:
    return _lib.gc_last_error(ctx).decode()


def gc_last_launches(ctx) -> int:
    return int(_lib.gc_last_launches(ctx))


def gc_set_partitions(ctx, parts: int) -> None:
    st = _lib.gc_set_partitions(ctx, int(parts))
    if st != 0:
        raise GcError(st, "gc_set_partitions: parts must be in [1, PARTS_MAX]")


def gc_set_profiling(ctx, enable: bool) -> None:
    _lib.gc_set_profiling(ctx, int(bool(enable)))


def gc_get_profile(ctx, reset: bool = False):
    n = (ctypes.c_longlong * 6)()
    ms = (ctypes.c_double * 6)()
    tl = (ctypes.c_longlong * 6)()
    _lib.gc_get_profile(ctx, n, ms, tl, int(bool(reset)))
    return {c: (int(n[i]), float(ms[i]), int(tl[i])) for i, c in enumerate(PROFILE_CLASSES)}


def debug_counters(ctx, reset: bool = False):
    """Development counters of the push phase (profiling only; not part of gc.h)."""
    out = (ctypes.c_ulonglong * 20)()
    _lib.gc_debug_counters(ctx, out, int(bool(reset)))
    return list(out)


_lib.gc_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int]
_lib.gc_debug_trace.restype = ctypes.c_longlong


def debug_trace(ctx, cap: int = 4 << 20, reset: bool = True):
    """Development per-task trace (profiling level 2; not part of gc.h): [m, 4] uint64 records
    (globaltimer start, duration ns, md << 56 | gcnt << 48 | cta << 32 | frame, tile)."""
    out = np.zeros((cap, 4), np.uint64)
    n = int(_lib.gc_debug_trace(ctx, out.ctypes.data, cap, int(bool(reset))))
    return out[:min(n, cap)]


def gc_get_kernel_ms(ctx, reset: bool = False) -> float:
    return float(_lib.gc_get_kernel_ms(ctx, int(bool(reset))))


def gc_frame_digest(ctx, n: int, H: int, W: int, flow: int, mask: int, out: int, stream: int) -> int:
    return _lib.gc_frame_digest(ctx, n, H, W, ctypes.c_void_p(flow), ctypes.c_void_p(mask), ctypes.c_void_p(out),
                                ctypes.c_void_p(stream))


def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


class GridCut:
    """One solver context (one device, one caller at a time).

    ``solve`` takes torch int32 CUDA tensors cap_s [n,H,W], cap_t [n,H,W], cap_nb [n,K,H,W]
    (and optionally warm_flow [n,K/2,H,W]) and returns int64 flow [n] and uint8 mask [n,H,W]
    on the device.  ``solve_host`` does the same with numpy arrays (host buffers).
    """

    def __init__(self, neighborhood: int = 4, max_h: int = 1080, max_w: int = 1920, max_batch: int = 0,
                 rounds_per_launch: int = 0, relabel_period: int = 0, max_launches: int = 0, device: int | None = None):
        self.K = neighborhood
        if device is None:  # the current CUDA device (gc.h: device < 0)
            device = -1
        cfg = gc_config(device, neighborhood, max_h, max_w, max_batch, rounds_per_launch, relabel_period,
                        max_launches)
        self.ctx = gc_create(cfg)

    def close(self):
        if self.ctx:
            gc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, allow=()):
        if st != 0 and st not in allow:
            raise GcError(st, gc_last_error(self.ctx))
        return st

    def solve(self, cap_s, cap_t, cap_nb, warm_flow=None, flow_state=False, stats=False, stream=None,
              allow=(), out=None):
        import torch
        n, H, W = cap_s.shape
        K = self.K
        assert cap_nb.shape == (n, K, H, W), cap_nb.shape
        for t in (cap_s, cap_t, cap_nb) + ((warm_flow,) if warm_flow is not None else ()):
            assert t.dtype == torch.int32 and t.is_cuda and t.is_contiguous()
        dev = cap_s.device
        if out is None:
            flow = torch.empty(n, dtype=torch.int64, device=dev)
            mask = torch.empty((n, H, W), dtype=torch.uint8, device=dev)
        else:
            flow, mask = out
        fs = torch.empty((n, K // 2, H, W), dtype=torch.int32, device=dev) if flow_state else None
        stt = torch.empty((n, 4), dtype=torch.int32, device=dev) if stats else None
        b = gc_batch(n, H, W, _ptr(cap_s), _ptr(cap_t), _ptr(cap_nb), _ptr(warm_flow), _ptr(flow), _ptr(mask),
                     _ptr(fs), _ptr(stt))
        s = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
        self.last_status = self._check(gc_solve_batch(self.ctx, b, s), allow)
        res = [flow, mask]
        if flow_state:
            res.append(fs)
        if stats:
            res.append(stt)
        return tuple(res)

    def solve_sequences(self, cap_s, cap_t, cap_nb, warm=True, warm_flow=None, flow_state=False, stats=False,
                        stream=None, allow=(), out=None):
        """S sequences of L frames in one device pass (gc_solve_sequences): cap_s, cap_t
        [S, L, H, W], cap_nb [S, L, K, H, W] int32 CUDA tensors; frame t >= 1 of a sequence is
        warm-started from frame t-1's flows when `warm`.  Returns flow [S, L] int64 and mask
        [S, L, H, W] uint8 (+ the last frames' flow state [S, K/2, H, W], + stats [S, L, 4])."""
        import torch
        S, L, H, W = cap_s.shape
        K = self.K
        assert cap_nb.shape == (S, L, K, H, W), cap_nb.shape
        for t in (cap_s, cap_t, cap_nb) + ((warm_flow,) if warm_flow is not None else ()):
            assert t.dtype == torch.int32 and t.is_cuda and t.is_contiguous()
        dev = cap_s.device
        if out is None:
            flow = torch.empty((S, L), dtype=torch.int64, device=dev)
            mask = torch.empty((S, L, H, W), dtype=torch.uint8, device=dev)
        else:
            flow, mask = out
        fs = torch.empty((S, K // 2, H, W), dtype=torch.int32, device=dev) if flow_state else None
        stt = torch.empty((S, L, 4), dtype=torch.int32, device=dev) if stats else None
        b = gc_seq_batch(S, L, H, W, _ptr(cap_s), _ptr(cap_t), _ptr(cap_nb), _ptr(warm_flow), _ptr(flow), _ptr(mask),
                         _ptr(fs), _ptr(stt), int(bool(warm)))
        s = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
        self.last_status = self._check(gc_solve_sequences(self.ctx, b, s), allow)
        res = [flow, mask]
        if flow_state:
            res.append(fs)
        if stats:
            res.append(stt)
        return tuple(res)

    def solve_energy(self, image, prior, gmm, lam=10.0, sigma=0.1, kappa=0.05, eps=1e-6, scale=64.0, warm_flow=None,
                     flow_state=False, stats=False, caps=False, stream=None, allow=(), out=None):
        """gc_solve_energy: image [n,H,W,3] uint8, prior [n,H,W] uint16 (torch CUDA tensors), gmm a
        CUDA uint8 tensor holding the [n][2] gc_gmm table (gmm_table).  Returns flow, mask
        (+ flow state, + stats, + the caps [n, 2+K, H, W] the solve built)."""
        import torch
        n, H, W, _ = image.shape
        K = self.K
        assert image.dtype == torch.uint8 and prior.dtype == torch.uint16 and gmm.dtype == torch.uint8
        assert prior.shape == (n, H, W) and gmm.numel() == n * 2 * ctypes.sizeof(gc_gmm)
        for t in (image, prior, gmm):
            assert t.is_cuda and t.is_contiguous()
        dev = image.device
        if out is None:
            flow = torch.empty(n, dtype=torch.int64, device=dev)
            mask = torch.empty((n, H, W), dtype=torch.uint8, device=dev)
        else:
            flow, mask = out
        fs = torch.empty((n, K // 2, H, W), dtype=torch.int32, device=dev) if flow_state else None
        stt = torch.empty((n, 4), dtype=torch.int32, device=dev) if stats else None
        cp = torch.empty((n, 2 + K, H, W), dtype=torch.int32, device=dev) if caps else None
        b = gc_energy_batch(n, H, W, _ptr(image), _ptr(prior), _ptr(gmm),
                            gc_energy_params(lam, sigma, kappa, eps, scale), _ptr(warm_flow), _ptr(flow),
                            _ptr(mask), _ptr(fs), _ptr(stt), _ptr(cp))
        s = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
        self.last_status = self._check(gc_solve_energy(self.ctx, b, s), allow)
        res = [flow, mask]
        if flow_state:
            res.append(fs)
        if stats:
            res.append(stt)
        if caps:
            res.append(cp)
        return tuple(res)

    def prior_update(self, mask_prev, q, wf, params, out=None, stream=None):
        """gc_prior_update: mask_prev [n,H,W] uint8, q [n,H,W] uint16, wf [n] int32 (CUDA tensors),
        params a gc_prior_params (prior_params) -> prior [n,H,W] uint16 on the device."""
        import torch
        n, H, W = mask_prev.shape
        assert mask_prev.dtype == torch.uint8 and q.dtype == torch.uint16 and wf.dtype == torch.int32
        for t in (mask_prev, q, wf):
            assert t.is_cuda and t.is_contiguous()
        pr = torch.empty((n, H, W), dtype=torch.uint16, device=mask_prev.device) if out is None else out
        s = torch.cuda.current_stream(mask_prev.device).cuda_stream if stream is None else stream
        self._check(gc_prior_update(self.ctx, n, H, W, _ptr(mask_prev), _ptr(q), _ptr(wf), params, _ptr(pr), s))
        return pr

    def saliency(self, image, prev=None, q=True, stream=None):
        """gc_saliency: image (and prev) [n,H,W,3] uint8 CUDA tensors -> saliency [n,h4,w4]
        float32 (and the full-resolution prior code [n,H,W] uint16 if q)."""
        import torch
        n, H, W, _ = image.shape
        assert image.dtype == torch.uint8 and image.is_cuda and image.is_contiguous()
        if prev is not None:
            assert prev.shape == image.shape and prev.dtype == torch.uint8 and prev.is_contiguous()
        h4, w4 = gc_saliency_dims(H, W)
        sal = torch.empty((n, h4, w4), dtype=torch.float32, device=image.device)
        qo = torch.empty((n, H, W), dtype=torch.uint16, device=image.device) if q else None
        b = gc_saliency_batch(n, H, W, _ptr(image), _ptr(prev), _ptr(sal), _ptr(qo))
        s = torch.cuda.current_stream(image.device).cuda_stream if stream is None else stream
        st = gc_saliency(self.ctx, b, s)
        if st != 0:
            raise GcError(st, "gc_saliency failed")
        return (sal, qo) if q else sal

    def solve_host(self, cap_s, cap_t, cap_nb, warm_flow=None, flow_state=False, stats=False, stream=0,
                   allow=(), out=None):
        n, H, W = cap_s.shape
        K = self.K
        assert cap_nb.shape == (n, K, H, W)
        for a in (cap_s, cap_t, cap_nb) + ((warm_flow,) if warm_flow is not None else ()):
            assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
        if out is None:
            flow = np.empty(n, np.int64)
            mask = np.empty((n, H, W), np.uint8)
        else:
            flow, mask = out
        fs = np.empty((n, K // 2, H, W), np.int32) if flow_state else None
        stt = np.empty((n, 4), np.int32) if stats else None
        b = gc_batch(n, H, W, _ptr(cap_s), _ptr(cap_t), _ptr(cap_nb), _ptr(warm_flow), _ptr(flow), _ptr(mask),
                     _ptr(fs), _ptr(stt))
        self.last_status = self._check(gc_solve_batch_host(self.ctx, b, stream), allow)
        res = [flow, mask]
        if flow_state:
            res.append(fs)
        if stats:
            res.append(stt)
        return tuple(res)

    def digest(self, flow, mask, stream=None):
        """Per-frame (F, popcount, mask hash, 0) int64 [n, 4] on the device (gc_frame_digest)."""
        import torch
        n, H, W = mask.shape
        assert flow.dtype == torch.int64 and mask.dtype == torch.uint8 and mask.is_contiguous()
        out = torch.empty((n, 4), dtype=torch.int64, device=mask.device)
        s = torch.cuda.current_stream(mask.device).cuda_stream if stream is None else stream
        self._check(gc_frame_digest(self.ctx, n, H, W, _ptr(flow), _ptr(mask), _ptr(out), s))
        return out

    def launches(self) -> int:
        return gc_last_launches(self.ctx)

    def set_partitions(self, parts: int):
        """NEXT-3: band partition of every frame over `parts` CTA groups (gc.h gc_set_partitions)."""
        gc_set_partitions(self.ctx, parts)

    def set_profiling(self, on):
        """False/True, or 2 for the development per-task trace as well."""
        _lib.gc_set_profiling(self.ctx, int(on))

    def profile(self, reset=False):
        return gc_get_profile(self.ctx, reset)

    def kernel_ms(self, reset=False) -> float:
        return gc_get_kernel_ms(self.ctx, reset)
