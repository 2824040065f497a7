#!/usr/bin/env python
"""bench.py -- batched exact grid min-cut (hot path of arXiv 1008.0502 §4/§7.3) on B200.

One "step" = one pass of the whole hot path (init, global relabels, push launches,
closure, flow value) over one batch of synthetic frames resident in HBM, through the
C ABI (gc_solve_batch).  Default workload: C4 of BASELINE.json -- 1920x1080 8-neighbour
saliency-blob frames, 1024 frames per GPU, frames sharded across ranks (weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Rank 0 prints ONE JSON line.  The reference arm (--impl reference) is the CPU oracle
(Boykov-Kolmogorov, oracle/) on the host cores, as the tier framing prescribes.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixel/s and frames/s min-cut solve (VGA, 1080p) at 1/2/4/8 B200; % HBM peak"
L2_BYTES = 126 * 1024 * 1024
CONFIGS = {
    "c1": dict(workload="C1 64x48 blob, 4-nbr", kind="blob", H=48, W=64, K=4, frames=1, seed_off=0),
    "c2": dict(workload="C2 320x240 QVGA blob clip, 4-nbr, 300 frames", kind="blob", H=240, W=320, K=4,
               frames=300, seed_off=1),
    "c3": dict(workload="C3 640x480 VGA blob sequences, 4-nbr", kind="blob", H=480, W=640, K=4, frames=120,
               seed_off=2),
    "c4": dict(workload="C4 1920x1080 blob batch, 8-nbr, 1024 frames per GPU", kind="blob", H=1080, W=1920, K=8,
               frames=1024, seed_off=3),
    "c5": dict(workload="C5 3840x2160 serpentine adversarial, 4-nbr", kind="serpentine", H=2160, W=3840, K=4,
               frames=8, seed_off=4, oracle_hw=(540, 960)),
    # NEXT-3 workload: single 4K frames, solved one per call with --frames 1
    "c4k": dict(workload="3840x2160 blob frames, 8-nbr", kind="blob", H=2160, W=3840, K=8, frames=8, seed_off=14),
}
# algorithmic bytes per processed 32x32 tile and kernel class


def tile_bytes(cls: str, K: int) -> int:
    """Algorithmic bytes one kernel class moves per processed 32x32 tile."""
    px = 1024
    if cls == "push":      # read e, r[K], h; write e, r[K], h, fl
        return (4 * (2 + K) + 4 * (2 + K) + 2) * px
    if cls == "bfs":       # read fl, h; write h (relax sweeps; the seed sweep moves less)
        return (2 + 4 + 4) * px
    if cls == "init":      # read cs, ct, c[K]; write fl
        return (4 * (2 + K) + 2) * px
    if cls == "closure":   # read fl; write m and the caller's mask
        return (2 + 1 + 1) * px
    if cls == "export":    # read r[K/2] (or caps) ; write f[K/2]
        return (4 * (K // 2) * 2) * px
    return 0


def compulsory_bytes_per_px(K: int, warm: bool = False) -> int:
    """read cs, ct, K n-links, write the mask (+ warm flows in/out)."""
    b = 4 * (2 + K) + 1
    if warm:
        b += 2 * 4 * (K // 2)
    return b


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_id: str | None):
        self.proc = None
        self.path = None
        self.dev_id = dev_id

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
            os.close(fd)
            cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200"]
            if self.dev_id:
                cmd += ["-i", self.dev_id]
            self.proc = subprocess.Popen(cmd, stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9 and f[1].isdigit():
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [int(r[1]) for r in rows]
        mx = max(int(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": int(statistics.median(loaded)), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(cfg, n_frames: int, threads: int, seed: int):
    """Bounded sample of the workload solved by the CPU oracle (BK) on `threads` host threads."""
    import oracle  # test infrastructure: only the cpu_baseline / reference legs use it
    import synth
    H, W = cfg.get("oracle_hw", (cfg["H"], cfg["W"]))
    cs, ct, nb = synth.gen_host(cfg["kind"], seed, 0, n_frames, H, W, cfg["K"])
    t0 = time.perf_counter()
    F, m = oracle.solve_batch(cs, ct, nb, "bk", threads=threads)
    dt = time.perf_counter() - t0
    return dt, F


def proxy_note(cfg) -> str:
    if "oracle_hw" not in cfg:
        return ""
    H, W = cfg["oracle_hw"]
    return (f"; PROXY: the oracle needs hours on one {cfg['W']}x{cfg['H']} frame, so the sample is the same "
            f"generator at {W}x{H} (same lane width; the CPU cost grows faster than the pixel count, so this "
            f"overstates the oracle's rate on the real frames)")


def cpu_baseline(cfg, seed: int):
    cores = host_cores()
    n = max(8, min(cores, 24))
    threads = min(cores, n)
    dt, _ = oracle_sample(cfg, n, threads, seed)
    H, W = cfg.get("oracle_hw", (cfg["H"], cfg["W"]))
    px = n * H * W
    return {"value": round(px / dt / 1e6, 3), "unit": "Mpixel/s", "cores": threads, "kind": "oracle",
            "sample": f"{n} frames of {cfg['workload'].split(',')[0]} solved by the CPU oracle "
                      f"(Boykov-Kolmogorov, oracle/oracle.cpp), one frame per thread, {cpu_model()}"
                      + proxy_note(cfg),
            "seconds": round(dt, 3), "fps": round(n / dt, 3)}


def run_reference(args, cfg):
    """--impl reference: the CPU oracle as it stands, on the host cores (tier framing ④)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    cores = host_cores()
    n = max(8, min(cores, 24))
    threads = min(cores, n)
    seed = synth.BASE_SEED + cfg["seed_off"]
    times = []
    for i in range(args.warmup + args.steps):
        dt, _ = oracle_sample(cfg, n, threads, seed)
        if i >= args.warmup:
            times.append(dt)
    H, W = cfg.get("oracle_hw", (cfg["H"], cfg["W"]))
    px = n * H * W
    tot = sum(times)
    val = px * len(times) / tot / 1e6
    out = {"metric": METRIC, "value": round(val, 3), "unit": "Mpixel/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic", "impl": "reference",
           "config": {"workload": cfg["workload"], "H": cfg["H"], "W": cfg["W"], "K": cfg["K"],
                      "frames_per_step": n, "note": "bounded sample per step (CPU oracle)"},
           "fps": round(n * len(times) / tot, 3),
           "cpu_baseline": {"value": round(val, 3), "unit": "Mpixel/s", "cores": threads, "kind": "oracle",
                            "sample": f"{n} frames per step, Boykov-Kolmogorov, one frame per thread, {cpu_model()}"
                                      + proxy_note(cfg)},
           "e2e": {"value": round(val, 3), "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)


def run_warm(args, cfg):
    """Sequence mode for C3 (BASELINE.json configs[2]): S sequences of L frames solved in ONE
    device pass per step through gc_solve_sequences -- a frame slot holds a sequence and frame
    t is warm-started from the flows frame t-1 exported (Kohli-Torr-style reuse).
    The same pass is also timed cold (warm=0, same schedule); results must agree.  One step =
    the S x L frames; value = warm throughput."""
    import torch

    import paper_1008_0502_b200 as gc
    import synth
    from paper_1008_0502_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    H, W, K = cfg["H"], cfg["W"], cfg["K"]
    S, L = args.seqs, args.seq_len
    seed = synth.BASE_SEED + cfg["seed_off"]
    t0, _ = shard.frame_range(rank, world, S * L)  # each rank takes its own S sequences
    cs, ct, nb = synth.gen_torch(cfg["kind"], seed, t0, S * L, H, W, K, device=dev, seq_len=L)
    cs, ct, nb = (a.view((S, L) + tuple(a.shape[1:])) for a in (cs, ct, nb))
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    flow = torch.empty((S, L), dtype=torch.int64, device=dev)
    mask = torch.empty((S, L, H, W), dtype=torch.uint8, device=dev)
    flow_c = torch.empty_like(flow)
    mask_c = torch.empty_like(mask)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        g.solve_sequences(cs, ct, nb, warm=True, out=(flow, mask))
        g.solve_sequences(cs, ct, nb, warm=False, out=(flow_c, mask_c))
    torch.cuda.synchronize()

    def timed(warm, out):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches = 0
        g.kernel_ms(reset=True)
        e0.record(stream)
        for _ in range(args.steps):
            g.solve_sequences(cs, ct, nb, warm=warm, out=out)
            launches += g.launches()
        e1.record(stream)
        torch.cuda.synchronize()
        return shard.max_over_ranks(e0.elapsed_time(e1), dev, world), launches, g.kernel_ms(reset=True)

    clk = ClockSampler(None)
    clk.start()
    time.sleep(0.3)
    ms_w, lw, kw = timed(True, (flow, mask))
    ms_c, _, kc = timed(False, (flow_c, mask_c))
    clocks = clk.stop()
    assert torch.equal(flow, flow_c) and torch.equal(mask, mask_c), "warm-started results differ from cold ones"
    px = world * S * L * H * W * args.steps
    peak, peak_src = load_peak()
    wb = compulsory_bytes_per_px(K, warm=True)  # + the warm flows read and written per frame
    if rank == 0:
        out = {"metric": METRIC, "value": round(px / (ms_w * 1e-3) / 1e6, 1), "unit": "Mpixel/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_w / args.steps, 3),
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
               "data": "synthetic (seeded saliency-blob sequences, synth/; generated on device before timing)",
               "config": {"workload": f"{cfg['workload']}: {S} sequences x {L} frames in one gc_solve_sequences "
                                      f"pass, frame t warm-started from t-1",
                          "H": H, "W": W, "K": K, "sequences_per_rank": S, "seq_len": L,
                          "parallelism": f"sequence-sharded dp{world}",
                          "l2": f"inputs {S * L * H * W * 4 * (2 + K) / 1e9:.1f} GB per rank >> 126 MB L2"},
               "fps": round(world * S * L * args.steps / (ms_w * 1e-3), 1),
               "roofline": {"bound": "hbm", "kernel": f"k_solve<{K}>", "unit": "GB/s", "peak": peak,
                            "achieved": round(wb * S * L * H * W * args.steps / (kw * 1e-3) / 1e9, 1),
                            "frac": round(wb * S * L * H * W * args.steps / (kw * 1e-3) / 1e9 / peak, 4),
                            "bytes_rule": f"{wb} B/px (caps + 2 warm-flow planes read, mask + 2 flow planes written)",
                            "avg_launch_ms": round(kw / args.steps, 4), "traffic": None, "peak_source": peak_src},
               "cold_same_schedule": {"value": round(px / (ms_c * 1e-3) / 1e6, 1), "unit": "Mpixel/s",
                                      "ms_per_step": round(ms_c / args.steps, 3)},
               "warm_speedup": round(ms_c / ms_w, 3), "warm_equals_cold": True,
               "gpu_launches": int(lw), "clocks": clocks}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_energy(args, cfg):
    """NEXT-1: the same frames given as the energy of PAPER.md §4 -- RGB image,
    prior and colour GMMs -- instead of capacities; gc_solve_energy builds the caps inside the
    solve's init pass.  One step = one gc_solve_energy call over this rank's frames.  The e2e leg
    uploads 5 B/px (image + prior) instead of the 4(2+K) B/px of caps."""
    import numpy as np
    import torch

    import paper_1008_0502_b200 as gc
    import synth
    from paper_1008_0502_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    H, W, K, n = cfg["H"], cfg["W"], cfg["K"], cfg["frames"]
    seed = synth.BASE_SEED + cfg["seed_off"]
    t_first, n = shard.frame_range(rank, world, n)
    img, pri = synth.gen_energy_torch(seed, t_first, n, H, W, device=dev)
    bg, ob = synth.energy_gmms()
    gm = torch.from_numpy(gc.gmm_table([(bg, ob)] * n)).to(dev)
    P = synth.ENERGY_PARAMS
    kw = dict(lam=P["lam"], sigma=P["sigma"], kappa=P["kappa"], eps=P["eps"], scale=P["scale"])
    flow = torch.empty(n, dtype=torch.int64, device=dev)
    mask = torch.empty((n, H, W), dtype=torch.uint8, device=dev)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        g.solve_energy(img, pri, gm, out=(flow, mask), **kw)
    torch.cuda.synchronize()
    clk = ClockSampler(None)
    clk.start()
    time.sleep(0.3)
    g.kernel_ms(reset=True)
    g.profile(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    e0.record(stream)
    for _ in range(args.steps):
        g.solve_energy(img, pri, gm, out=(flow, mask), **kw)
        launches += g.launches()
    e1.record(stream)
    torch.cuda.synchronize()
    kms = g.kernel_ms(reset=True)
    nl = max(g.profile(reset=True)["init"][0], 1)
    clocks = clk.stop()
    ms = shard.max_over_ranks(e0.elapsed_time(e1), dev, world)
    px = world * n * H * W * args.steps
    peak, peak_src = load_peak()
    bpx = 3 + 2 + 1  # read RGB + prior code, write the mask
    avg = kms / nl
    achieved = bpx * n * H * W * args.steps / nl / (avg * 1e-3) / 1e9
    # e2e: pinned host image + prior in, mask + flow out, through GridCut.solve_energy
    ne = min(args.e2e_frames, n)
    himg = torch.empty((ne, H, W, 3), dtype=torch.uint8, pin_memory=True)
    hpri = torch.empty((ne, H, W), dtype=torch.uint16, pin_memory=True)
    himg.copy_(img[:ne]); hpri.copy_(pri[:ne])
    hmask = torch.empty((ne, H, W), dtype=torch.uint8, pin_memory=True)
    hflow = torch.empty(ne, dtype=torch.int64, pin_memory=True)
    dimg = torch.empty_like(img[:ne]); dpri = torch.empty_like(pri[:ne])
    dflow = torch.empty(ne, dtype=torch.int64, device=dev)
    dmask = torch.empty((ne, H, W), dtype=torch.uint8, device=dev)
    gme = gm[: ne * 2 * ctypes_sizeof_gmm(gc)]

    def e2e_step():
        dimg.copy_(himg, non_blocking=True)
        dpri.copy_(hpri, non_blocking=True)
        g.solve_energy(dimg, dpri, gme, out=(dflow, dmask), **kw)
        hmask.copy_(dmask, non_blocking=True)
        hflow.copy_(dflow, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e3.record(stream)
    torch.cuda.synchronize()
    ems = shard.max_over_ranks(e2.elapsed_time(e3), dev, world)
    assert np.array_equal(hflow.numpy(), flow[:ne].cpu().numpy())
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        from oracle import energy as oen
        m = 4
        rgb, pr = synth.gen_energy_host(seed, 0, m, H, W)
        t0 = time.perf_counter()
        capsl = [oen.caps(rgb[i], pr[i], bg, ob, K) for i in range(m)]
        cs = np.stack([c[0] for c in capsl]); ct = np.stack([c[1] for c in capsl]); nb = np.stack([c[2] for c in capsl])
        oracle.solve_batch(cs, ct, nb, "bk", threads=min(host_cores(), m))
        dt = time.perf_counter() - t0
        cpu = {"value": round(m * H * W / dt / 1e6, 3), "unit": "Mpixel/s", "cores": min(host_cores(), m),
               "kind": "oracle", "sample": f"{m} frames: oracle/energy.py caps (numpy float64, one core) + BK "
                                            f"on {min(host_cores(), m)} threads, {cpu_model()}", "seconds": round(dt, 2)}
    if rank == 0:
        out = {"metric": METRIC, "value": round(px / (ms * 1e-3) / 1e6, 1), "unit": "Mpixel/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+int32",
               "data": "synthetic (seeded saliency-blob frames as RGB + prior, synth/; generated on device)",
               "config": {"workload": f"{cfg['workload']} from the energy (NEXT-1: RGB image, prior, colour GMMs -> "
                                      f"caps in the init pass)", "H": H, "W": W, "K": K, "frames_per_rank": n,
                          "parallelism": f"frame-sharded dp{world}", "l2": "inputs >> 126 MB L2"},
               "fps": round(world * n * args.steps / (ms * 1e-3), 1),
               "roofline": {"bound": "hbm", "kernel": f"k_solve<{K},energy>", "unit": "GB/s", "peak": peak,
                            "achieved": round(achieved, 1), "frac": round(achieved / peak, 4),
                            "bytes_rule": f"{bpx} B/px compulsory (read RGB + prior code, write the mask)",
                            "avg_launch_ms": round(avg, 4), "traffic": None, "peak_source": peak_src},
               "e2e": {"value": round(world * ne * H * W * args.steps / (ems * 1e-3) / 1e6, 1), "unit": "Mpixel/s",
                       "h2d_bytes_per_step": int(ne * H * W * 5), "d2h_bytes_per_step": int(ne * H * W + ne * 8),
                       "frames_per_step": ne,
                       "note": "GridCut.solve_energy: pinned host image + prior H2D, mask + flow D2H in the timed region"},
               "cpu_baseline": cpu, "gpu_launches": int(launches), "clocks": clocks}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_prior(args, cfg):
    """NEXT-2: gc_prior_update over this rank's frames -- the previous mask
    smoothed (radius-12 Gaussian, sigma 4) and fused with the saliency prior by the §6 weights
    (P:411-438).  Masks: the synthetic frames' prior > 1/2 (blob shapes); q: their prior codes."""
    import torch

    import paper_1008_0502_b200 as gc
    import synth
    from paper_1008_0502_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    H, W, n = cfg["H"], cfg["W"], cfg["frames"]
    seed = synth.BASE_SEED + cfg["seed_off"]
    t_first, n = shard.frame_range(rank, world, n)
    img, q = synth.gen_energy_torch(seed, t_first, n, H, W, device=dev)
    del img
    mask = (q.to(torch.int32) > 32768).to(torch.uint8)
    wfv, _ = gc.gc_kalman_step(0.03 ** 2, 0.035 ** 2, 6.0308884908e-4)
    wf = torch.full((n,), wfv, dtype=torch.int32, device=dev)
    params = gc.prior_params(4.0, 12, 8)
    out = torch.empty_like(q)
    g = gc.GridCut(neighborhood=4, max_h=H, max_w=W)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        g.prior_update(mask, q, wf, params, out=out)
    torch.cuda.synchronize()
    clk = ClockSampler(None)
    clk.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        g.prior_update(mask, q, wf, params, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = shard.max_over_ranks(e0.elapsed_time(e1), dev, world)
    px = world * n * H * W * args.steps
    peak, peak_src = load_peak()
    bpx = 1 + 2 + 2
    ach = bpx * n * H * W * args.steps / (ms * 1e-3) / 1e9 / world * world
    if rank == 0:
        res = {"metric": METRIC, "value": round(px / (ms * 1e-3) / 1e6, 1), "unit": "Mpixel/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
               "data": "synthetic (blob masks and saliency prior codes, synth/; on device)",
               "config": {"workload": f"NEXT-2 prior update (P:411-438) on {cfg['workload'].split(',')[0]} frames, "
                                      f"{n} per rank, Gaussian radius 12 sigma 4, edge band 8",
                          "H": H, "W": W, "frames_per_rank": n, "parallelism": f"frame-sharded dp{world}",
                          "l2": "inputs >> 126 MB L2"},
               "roofline": {"bound": "hbm", "kernel": "k_prior", "unit": "GB/s", "peak": peak,
                            "achieved": round(ach / world, 1), "frac": round(ach / world / peak, 4),
                            "bytes_rule": "5 B/px (read mask + saliency code, write the prior code)",
                            "traffic": None, "peak_source": peak_src},
               "gpu_launches": args.steps, "clocks": clocks}
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_saliency(args, cfg):
    """NEXT-4: gc_saliency (Itti-style map) over C4-geometry frames
    with motion (previous frame), 64 frames per call (the pyramids take ~88 MB per 1080p frame);
    output: the level-4 map and the full-resolution prior code."""
    import torch

    import paper_1008_0502_b200 as gc
    import synth
    from paper_1008_0502_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    H, W = cfg["H"], cfg["W"]
    n = 64
    seed = synth.BASE_SEED + cfg["seed_off"]
    t_first, _ = shard.frame_range(rank, world, n)
    img, _ = synth.gen_energy_torch(seed, t_first, n + 1, H, W, device=dev)
    cur, prev = img[1:].contiguous(), img[:-1].contiguous()
    g = gc.GridCut(neighborhood=4, max_h=H, max_w=W)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        g.saliency(cur, prev)
    torch.cuda.synchronize()
    clk = ClockSampler(None)
    clk.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    launches = 0
    for _ in range(args.steps):
        g.saliency(cur, prev)
        launches += g.launches()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = shard.max_over_ranks(e0.elapsed_time(e1), dev, world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import saliency as osal
        rgb = img[:2].cpu().numpy()
        t0 = time.perf_counter()
        osal.saliency(rgb[1], rgb[0])
        dt = time.perf_counter() - t0
        cpu = {"value": round(H * W / dt / 1e6, 3), "unit": "Mpixel/s", "cores": 1, "kind": "oracle",
               "sample": f"1 frame, oracle/saliency.py (numpy float32, one core), {cpu_model()}", "seconds": round(dt, 2)}
    if rank == 0:
        peak, peak_src = load_peak()
        bpx = 3 + 3 + 2  # read the frame and the previous frame, write the prior code
        ach = bpx * n * H * W * args.steps / (ms * 1e-3) / 1e9
        res = {"metric": METRIC, "value": round(world * n * H * W * args.steps / (ms * 1e-3) / 1e6, 1),
               "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f32", "data": "synthetic (blob frames as RGB, synth/; on device)",
               "config": {"workload": f"NEXT-4 saliency (P:516-570) on {cfg['workload'].split(',')[0]} frames, "
                                      f"{n} per call, with motion", "H": H, "W": W, "frames_per_rank": n,
                          "parallelism": f"frame-sharded dp{world}"},
               "roofline": {"bound": "hbm", "kernel": "gc_saliency (18 kernels per map set)", "unit": "GB/s",
                            "peak": peak, "achieved": round(ach, 1), "frac": round(ach / peak, 4),
                            "bytes_rule": f"{bpx} B/px compulsory (two RGB frames in, the prior code out); "
                                          "the pyramids and feature maps stay in HBM / L2", "traffic": None,
                            "peak_source": peak_src},
               "cpu_baseline": cpu, "gpu_launches": int(launches), "clocks": clocks}
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def ctypes_sizeof_gmm(gc):
    import ctypes
    return ctypes.sizeof(gc.gc_gmm)


def verify_shard(cfg, seed, t_first, cs, ct, nb, flow, mask, nverify, world):
    """--verify: every frame of this rank's shard (or the first `nverify`) against the CPU oracle
    (Boykov-Kolmogorov), bit-exact in F and mask, outside the timed region.  The caps are the
    ones the GPU solved (the CUDA twin of synth/, bit-identical to the host twin), copied to
    the host in chunks; the oracle runs on this rank's share of the host cores."""
    import numpy as np

    import oracle  # test infrastructure: only the verify / cpu_baseline / reference legs use it
    n = cs.shape[0] if nverify <= 0 else min(nverify, cs.shape[0])
    threads = max(1, host_cores() // max(world, 1))
    chunk = max(threads, 8)
    bad, t0 = [], time.perf_counter()
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        Fo, mo = oracle.solve_batch(cs[a:b].cpu().numpy(), ct[a:b].cpu().numpy(), nb[a:b].cpu().numpy(), "bk",
                                    threads=threads)
        Fg, mg = flow[a:b].cpu().numpy(), mask[a:b].cpu().numpy()
        for i in range(b - a):
            if int(Fg[i]) != int(Fo[i]) or not np.array_equal(mg[i], mo[i]):
                bad.append(t_first + a + i)
    return {"frames": n, "first_frame": t_first, "mismatches": len(bad), "bad_frames": bad[:16],
            "oracle": "Boykov-Kolmogorov (oracle/oracle.cpp)", "threads": threads,
            "seconds": round(time.perf_counter() - t0, 1), "compared": "F (int64) and mask bytes, every frame"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--frames", type=int, default=0, help="frames per rank (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-frames", type=int, default=32)
    ap.add_argument("--profile-steps", type=int, default=1)
    ap.add_argument("--verify", type=int, default=-1, metavar="N",
                    help="after timing, compare the first N frames of each rank's shard with the CPU oracle "
                         "(0: all frames; default: off)")
    ap.add_argument("--cross-check", type=int, default=8, metavar="M",
                    help="N > 1: each rank re-solves the first M frames of the next rank's shard")
    ap.add_argument("--energy", action="store_true",
                    help="NEXT-1: frames given as RGB image + prior + colour GMMs; caps built in the solve's init pass")
    ap.add_argument("--prior", action="store_true", help="NEXT-2: the on-device prior update (gc_prior_update)")
    ap.add_argument("--saliency", action="store_true", help="NEXT-4: the saliency front-end (gc_saliency)")
    ap.add_argument("--warm", action="store_true",
                    help="sequence mode (C3): S sequences x L frames, frame t warm-started from t-1")
    ap.add_argument("--parts", type=int, default=1,
                    help="NEXT-3: band-partition every frame over N CTA groups (gc_set_partitions; 1: off)")
    ap.add_argument("--seqs", type=int, default=8)
    ap.add_argument("--seq-len", type=int, default=120)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no launcher: start one rank per GPU ourselves (the same env torchrun would set)
        from paper_1008_0502_b200 import shard
        sys.exit(shard.launch_local_ranks(args.gpus, [os.path.abspath(__file__)] + sys.argv[1:]))
    cfg = dict(CONFIGS[args.config])
    if args.frames:
        cfg["frames"] = args.frames
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.warm:
        return run_warm(args, cfg)
    if args.energy:
        return run_energy(args, cfg)
    if args.prior:
        return run_prior(args, cfg)
    if args.saliency:
        return run_saliency(args, cfg)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1008_0502_b200 as gc
    import synth
    from paper_1008_0502_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    H, W, K, n = cfg["H"], cfg["W"], cfg["K"], cfg["frames"]
    seed = synth.BASE_SEED + cfg["seed_off"]
    if cfg["kind"] == "serpentine":
        synth.set_serpentine_params(lane=64, big=1 << 20)

    # ---- inputs: this rank's frame shard, generated on the device (CUDA twin of synth/)
    t_first, n = shard.frame_range(rank, world, n)
    cs, ct, nb = synth.gen_torch(cfg["kind"], seed, t_first, n, H, W, K, device=dev)
    flow = torch.empty(n, dtype=torch.int64, device=dev)
    mask = torch.empty((n, H, W), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    if args.parts > 1:  # NEXT-3: band partition of each frame over CTA groups (gc_set_partitions)
        g.set_partitions(args.parts)
    stream = torch.cuda.current_stream(dev)

    def step():
        g.solve(cs, ct, nb, out=(flow, mask))
        return g.launches()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region
    uuid = None
    try:
        uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        pass
    clk = ClockSampler(uuid)
    clk.start()
    time.sleep(0.4)
    barrier()
    torch.cuda.synchronize()
    in_bytes = n * H * W * 4 * (2 + K)
    l2_flush = in_bytes < 4 * L2_BYTES  # small inputs: flush L2 between the timed steps
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if l2_flush else None
    launches = 0
    ms_sum = 0.0
    g.kernel_ms(reset=True)
    g.profile(reset=True)
    if not l2_flush:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            launches += step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_sum = e0.elapsed_time(e1)
    else:
        for _ in range(args.steps):  # each step timed alone, L2 flushed (write > L2) before it
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launches += step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_sum += e0.elapsed_time(e1)
    # the persistent kernel's own device time in the timed steps (CUDA events the library
    # records around every k_solve launch on the launching stream; no profiling counters on)
    kms_timed = g.kernel_ms(reset=True)
    nl_timed = max(g.profile(reset=True)["init"][0], 1)
    barrier()
    clocks = clk.stop()
    ms_max = shard.max_over_ranks(ms_sum, dev, world)
    px_total = world * n * H * W * args.steps
    value = px_total / (ms_max * 1e-3) / 1e6
    fps = world * n * args.steps / (ms_max * 1e-3)

    # ---- final statistics over NCCL (the only collectives: SURVEY.md §8(a) a6, §8(e)):
    # per-frame digests (F, popcount, 64-bit mask hash) computed on the device
    digest = g.digest(flow, mask)
    stats, per_frame = shard.reduce_stats(*shard.frame_stats(digest), world)
    bad_frames = int(stats[2].item())
    cross = None
    if world > 1 and args.cross_check > 0:
        m = min(args.cross_check, n)
        nxt, _ = shard.frame_range((rank + 1) % world, world, cfg["frames"])
        pc, pt, pn = synth.gen_torch(cfg["kind"], seed, nxt, m, H, W, K, device=dev)
        pf, pm = g.solve(pc, pt, pn)
        pdg = g.digest(pf, pm)
        cross = {"frames_per_rank": m, "mismatches": shard.cross_rank_mismatches(
            digest[:m][:, [0, 2]], pdg[:, [0, 2]], world, rank),
            "what": "rank r re-solves the first frames of rank r+1's shard; (F, mask hash) must match"}
        del pc, pt, pn

    # ---- profiled replica step: tile tasks and CTA time per class (diagnostic only)
    g.set_profiling(True)
    g.profile(reset=True)
    g.kernel_ms(reset=True)
    gc.debug_counters(g.ctx, reset=True)
    for _ in range(args.profile_steps):
        g.solve(cs, ct, nb, out=(flow, mask))
    torch.cuda.synchronize()
    prof = g.profile(reset=True)
    kms_prof = g.kernel_ms(reset=True)
    cross_band = gc.debug_counters(g.ctx, reset=True)[19] / max(1, n * args.profile_steps)
    g.set_profiling(False)
    peak, peak_src = load_peak()
    nlp = max(prof["init"][0], 1)

    # ---- roofline of the dominant (only) kernel, k_solve:
    # algorithmic bytes = compulsory bytes per pixel (read cs, ct, K n-link planes, write the
    # mask) x pixels per launch, over the launch's unprofiled device time
    avg_ms = kms_timed / nl_timed
    px_launch = n * H * W * args.steps / nl_timed
    bytes_launch = compulsory_bytes_per_px(K) * px_launch
    achieved = bytes_launch / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else 0.0
    # the kernel's own time cannot exceed the step it is part of (same stream, same steps)
    assert kms_timed <= ms_sum * 1.001 + 0.01, (kms_timed, ms_sum)
    # measured DRAM traffic of the benched launch (ncu dram__bytes_read + write, committed
    # capture of this config and launch size); null when none is committed
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            rec = json.load(open(tp)).get(args.config, {}).get("k_solve")
            if rec and int(rec.get("frames_per_launch", -1)) == int(round(px_launch / (H * W))):
                traffic = int(rec["dram_bytes_per_launch"])
                traffic_src = rec.get("source")
        except Exception:
            traffic = None
    task_bytes = sum(tile_bytes(c, K) * prof[c][2] for c in prof) / nlp
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": f"k_solve<{K}>",
                "bytes_per_launch": int(bytes_launch),
                "bytes_rule": f"{compulsory_bytes_per_px(K)} B/px compulsory (read cs, ct, {K} n-link planes as int32, "
                              f"write the uint8 mask) x {int(px_launch)} px per launch",
                "avg_launch_ms": round(avg_ms, 4), "launches_per_step": round(nl_timed / args.steps, 2),
                "share_of_step": round(min(1.0, kms_timed / ms_sum), 4) if ms_sum > 0 else None,
                "peak_source": peak_src, "traffic_source": traffic_src,
                "task_bytes_diag": {"bytes_per_launch": int(task_bytes),
                                    "profiled_launch_ms": round(kms_prof / nlp, 4),
                                    "classes": {c: {"tiles": v[2], "cta_ms": round(v[1], 3),
                                                    "bytes": tile_bytes(c, K) * v[2]} for c, v in prof.items()}}}
    comp = compulsory_bytes_per_px(K) * n * H * W * world * args.steps / (ms_max * 1e-3) / 1e9

    # ---- end to end through the public API with HOST buffers (pinned), copies inside timing
    e2e = None
    if not args.no_e2e:
        ne = min(args.e2e_frames, n, cfg["frames"])
        hcs = torch.empty((ne, H, W), dtype=torch.int32, pin_memory=True)
        hct = torch.empty((ne, H, W), dtype=torch.int32, pin_memory=True)
        hnb = torch.empty((ne, K, H, W), dtype=torch.int32, pin_memory=True)
        hcs.copy_(cs[:ne]); hct.copy_(ct[:ne]); hnb.copy_(nb[:ne])
        hflow = torch.empty(ne, dtype=torch.int64, pin_memory=True)
        hmask = torch.empty((ne, H, W), dtype=torch.uint8, pin_memory=True)
        hargs = (hcs.numpy(), hct.numpy(), hnb.numpy())
        hout = (hflow.numpy(), hmask.numpy())
        g.solve_host(*hargs, out=hout, stream=stream.cuda_stream)
        torch.cuda.synchronize()
        barrier()
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        for _ in range(args.steps):
            g.solve_host(*hargs, out=hout, stream=stream.cuda_stream)
        e3.record(stream)
        torch.cuda.synchronize()
        ems = shard.max_over_ranks(e2.elapsed_time(e3), dev, world)
        e2e = {"value": round(world * ne * H * W * args.steps / (ems * 1e-3) / 1e6, 1), "unit": "Mpixel/s",
               "h2d_bytes_per_step": int(ne * H * W * 4 * (2 + K)),
               "d2h_bytes_per_step": int(ne * H * W + ne * 8), "frames_per_step": ne,
               "fps": round(world * ne * args.steps / (ems * 1e-3), 1),
               "note": "gc_solve_batch_host on pinned host buffers; H2D caps + D2H mask/flow inside the timed region"}
        # results through the host path must equal the device path
        assert np.array_equal(hflow.numpy(), flow[:ne].cpu().numpy())
        assert np.array_equal(hmask.numpy(), mask[:ne].cpu().numpy())

    verify = None
    if args.verify >= 0:
        verify = verify_shard(cfg, seed, t_first, cs, ct, nb, flow, mask, args.verify, world)
        if world > 1:
            vt = torch.tensor([verify["frames"], verify["mismatches"]], dtype=torch.int64, device=dev)
            dist.all_reduce(vt)
            verify["frames_all_ranks"], verify["mismatches_all_ranks"] = int(vt[0]), int(vt[1])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, seed)

    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 1), "unit": "Mpixel/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
               "data": "synthetic (seeded saliency-blob frames, synth/; generated on device before timing)",
               "config": {"workload": cfg["workload"], "H": H, "W": W, "K": K, "frames_per_rank": n,
                          "frames_total": n * world, "parallelism": f"frame-sharded dp{world}" +
                          (f", each frame band-partitioned over {args.parts} CTA groups (NEXT-3 emulation)"
                           if args.parts > 1 else ""),
                          "partitions": args.parts,
                          "l2": (f"inputs {in_bytes / 1e9:.2f} GB per rank: L2 (126 MB) flushed by a 252 MB write before "
                                 f"each separately timed step" if l2_flush else
                                 f"inputs {in_bytes / 1e9:.1f} GB per rank >> 126 MB L2 (no flush needed)")},
               "fps": round(fps, 1),
               "roofline": roofline,
               "hbm_frac_compulsory": round(comp / peak, 5),
               "cpu_baseline": cpu,
               "e2e": e2e,
               "gpu_launches": int(launches),
               "clocks": clocks,
               "frames_failed": bad_frames,
               "checksum": {"sum_F": int(stats[0].item()), "sum_mask": int(stats[1].item()),
                            "hash_xor": int(np.bitwise_xor.reduce(per_frame[:, 2].cpu().numpy()))},
               "cross_rank": cross,
               "cross_band_handoffs_per_frame": round(cross_band, 1) if args.parts > 1 else None,
               "verify": verify,
               "paper_context": "graph-cut stage 1.47 / 6.65 / 1.41 Mpx/s on a GeForce 9800GT (P:757-762)"}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
