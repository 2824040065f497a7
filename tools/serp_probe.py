"""Development aid: solve time and per-frame counters of serpentine (C5-shaped) frames.
usage: serp_probe.py "HxW[:lane]" ... (one frame each; GC_TIMEOUT_S bounds each solve)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1008_0502_b200 as gc
import synth

for spec in sys.argv[1:]:
    hw, _, lane = spec.partition(":")
    H, W = map(int, hw.split("x"))
    n = int(os.environ.get("NF", "1"))
    synth.set_serpentine_params(lane=int(lane or 64), big=1 << 20)
    cs, ct, nb = synth.gen_torch("serpentine", synth.BASE_SEED + 4, 0, n, H, W, 4)
    synth.set_serpentine_params()
    g = gc.GridCut(neighborhood=4, max_h=H, max_w=W, rounds_per_launch=int(os.environ.get("ROUNDS", "0")))
    g.set_profiling(True)
    torch.cuda.synchronize()
    t0 = time.time()
    F, m, st = g.solve(cs, ct, nb, stats=True, allow=(5,))
    torch.cuda.synchronize()
    dt = time.time() - t0
    prof = g.profile(reset=True)
    dbg = gc.debug_counters(g.ctx, reset=True)
    print(json.dumps({"spec": spec, "n": n, "s": round(dt, 3), "status": g.last_status, "F": F.tolist(),
                      "mask": m.flatten(1).sum(1).tolist(), "stats": st.tolist(),
                      "cta_ms": {k: round(v[1], 2) for k, v in prof.items()}, "tasks": {k: v[2] for k, v in prof.items()},
                      "dbg": dbg[:13]}), flush=True)
    g.close()
