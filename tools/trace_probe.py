"""Development: per-task trace of one solve (profiling level 2) and a utilisation summary.

  python tools/trace_probe.py [config] [frames] [tag]
Writes gpurun_out/trace_<tag>.npy and prints: busy CTAs per time bin and class, per-frame
latency (first task -> last task), and the frames that end the call.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

CLS = {0: "init", 1: "seed", 2: "bfs", 3: "push", 4: "cseed", 5: "clos", 15: "trans"}


def summarize(tr, nctas, bin_us=500.0):
    t0 = tr[:, 0].min()
    st = (tr[:, 0] - t0).astype(np.float64) / 1e3  # us
    du = tr[:, 1].astype(np.float64) / 1e3
    md = (tr[:, 2] >> np.uint64(56)).astype(np.int64)
    fr = (tr[:, 2] & np.uint64(0xffffffff)).astype(np.int64)
    span = (st + du).max()
    out = {"tasks": int(len(tr)), "span_us": round(span, 1)}
    nb = int(np.ceil(span / bin_us))
    busy = {}
    for m, name in CLS.items():
        sel = md == m
        if not sel.any():
            continue
        b = np.zeros(nb + 1)
        for s0, d0 in zip(st[sel], du[sel]):
            i0, i1 = s0 / bin_us, (s0 + d0) / bin_us
            a = int(i0)
            while a < i1:
                lo, hi = max(i0, a), min(i1, a + 1)
                b[a] += hi - lo
                a += 1
        busy[name] = b[:nb] / nctas
        out[f"n_{name}"] = int(sel.sum())
        out[f"mean_us_{name}"] = round(float(du[sel].mean()), 2)
        out[f"cta_ms_{name}"] = round(float(du[sel].sum()) / 1e3 / nctas, 3)
    rows = []
    for i in range(nb):
        rows.append(f"{i * bin_us / 1e3:6.2f}ms " + " ".join(f"{k}={busy[k][i]:.2f}" for k in busy) +
                    f" tot={sum(busy[k][i] for k in busy):.2f}")
    out["timeline"] = rows
    # per frame latency
    fs = {}
    for f in np.unique(fr):
        sel = fr == f
        a, b = st[sel].min(), (st[sel] + du[sel]).max()
        fs[int(f)] = (a, b, int(sel.sum()), int((md[sel] == 15).sum()))
    lat = np.array([v[1] - v[0] for v in fs.values()])
    out["frame_latency_us"] = {"mean": round(float(lat.mean()), 1), "p50": round(float(np.median(lat)), 1),
                               "p90": round(float(np.percentile(lat, 90)), 1), "max": round(float(lat.max()), 1)}
    last = sorted(fs.items(), key=lambda kv: -kv[1][1])[:8]
    out["last_frames"] = [(f, round(v[0], 1), round(v[1], 1), v[2], v[3]) for f, v in last]
    slow = sorted(fs.items(), key=lambda kv: -(kv[1][1] - kv[1][0]))[:8]
    out["slowest_frames"] = [(f, round(v[0], 1), round(v[1] - v[0], 1), v[2], v[3]) for f, v in slow]
    return out


def main():
    import torch

    import paper_1008_0502_b200 as gc
    import synth
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
    seqmode = None
    if cfgname in ("c3warm", "c3cold"):  # gc_solve_sequences, 8 x 120 VGA frames
        seqmode = cfgname == "c3warm"
        cfgname = "c3"
    cfg = dict(bench.CONFIGS[cfgname])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["frames"]
    tag = sys.argv[3] if len(sys.argv) > 3 else cfgname
    H, W, K = cfg["H"], cfg["W"], cfg["K"]
    if cfg["kind"] == "serpentine":
        synth.set_serpentine_params(lane=64, big=1 << 20)
    if seqmode is not None:
        n = 960
    cs, ct, nb = synth.gen_torch(cfg["kind"], synth.BASE_SEED + cfg["seed_off"], 0, n, H, W, K,
                                 seq_len=120 if seqmode is not None else 0)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    if seqmode is not None:
        cs, ct, nb = (a.view((8, 120) + tuple(a.shape[1:])) for a in (cs, ct, nb))
        run = lambda: g.solve_sequences(cs, ct, nb, warm=seqmode)  # noqa: E731
    else:
        run = lambda: g.solve(cs, ct, nb)  # noqa: E731
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    g.kernel_ms(reset=True)
    run()
    plain = g.kernel_ms(reset=True)
    g.set_profiling(2)
    gc.debug_trace(g.ctx, 1, reset=True)
    run()
    torch.cuda.synchronize()
    prof_ms = g.kernel_ms(reset=True)
    tr = gc.debug_trace(g.ctx)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", f"trace_{tag}.npy"), tr)
    nctas = int(((tr[:, 2] >> np.uint64(32)) & np.uint64(0xffff)).max()) + 1
    s = summarize(tr, nctas)
    s.update({"config": cfgname + ("" if seqmode is None else (" seq warm" if seqmode else " seq cold")), "frames": n, "plain_kernel_ms": round(plain, 3), "traced_kernel_ms": round(prof_ms, 3),
              "ctas": nctas})
    tl = s.pop("timeline")
    print(json.dumps(s))
    print("\n".join(tl))


if __name__ == "__main__":
    main()
