"""Development aid: solve time vs frame slots in flight (scratch budget) and per-frame stats.
usage: slots_probe.py cfg frames mb[,mb...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json

import torch

import paper_1008_0502_b200 as gc
import synth

ALL = {"qvga": ("blob", 240, 320, 4), "vga": ("blob", 480, 640, 4), "1080p": ("blob", 1080, 1920, 8),
       "serp": ("serpentine", 1080, 1920, 4), "4k": ("serpentine", 2160, 3840, 4)}
name, n = sys.argv[1], int(sys.argv[2])
mbs = [int(x) for x in sys.argv[3].split(",")]
kind, H, W, K = ALL[name]
if kind == "serpentine":
    synth.set_serpentine_params(lane=64, big=1 << 20)
cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + 3, 0, n, H, W, K)
ref = None
for mb in mbs:
    os.environ["GC_SCRATCH_MB"] = str(mb)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    F, m, st = g.solve(cs, ct, nb, stats=True)
    torch.cuda.synchronize()
    if ref is None:
        ref = (F.clone(), m.clone())
    assert torch.equal(F, ref[0]) and torch.equal(m, ref[1])
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.solve(cs, ct, nb); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    launches = g.launches()
    g.set_profiling(True); g.profile(reset=True)
    g.solve(cs, ct, nb); torch.cuda.synchronize()
    prof = g.profile(reset=True)
    stf = st.float()
    print(json.dumps({"cfg": name, "mb": mb, "ms": round(best, 3), "Mpx_s": round(n * H * W / best / 1e3, 1),
                      "launches": launches,
                      "st_mean": [round(x, 2) for x in stf.mean(0).tolist()], "st_max": st.max(0).values.tolist(),
                      "prof": {k: (v[0], round(v[1], 2), v[2]) for k, v in prof.items()}}), flush=True)
    g.close()
    del g
