"""Development aid: single-frame solve latency (device time) for chosen frames of a config.
usage: latency.py cfg t0,t1,... [seed_off]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1008_0502_b200 as gc
import synth

ALL = {"qvga": ("blob", 240, 320, 4), "vga": ("blob", 480, 640, 4), "1080p": ("blob", 1080, 1920, 8),
       "serp": ("serpentine", 1080, 1920, 4), "4k": ("serpentine", 2160, 3840, 4)}
name = sys.argv[1]
ts = [int(x) for x in sys.argv[2].split(",")]
seed_off = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kind, H, W, K = ALL[name]
if kind == "serpentine":
    synth.set_serpentine_params(lane=64, big=1 << 20)
g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
for t0 in ts:
    cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + seed_off, t0, 1, H, W, K)
    F, m, st = g.solve(cs, ct, nb, stats=True)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.solve(cs, ct, nb); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    g.set_profiling(True); g.profile(reset=True); g.kernel_ms(reset=True)
    g.solve(cs, ct, nb); torch.cuda.synchronize()
    prof = g.profile(reset=True)
    g.set_profiling(False)
    print(json.dumps({"cfg": name, "t": t0, "ms": round(best, 3), "stats": st[0].tolist()[:3],
                      "tasks": {k: v[2] for k, v in prof.items()}, "cta_ms": {k: round(v[1], 3) for k, v in prof.items()}}),
          flush=True)
