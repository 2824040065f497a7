"""Development: push-phase counters of the C4 cold-start frame (frame 0) solved alone."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1008_0502_b200 as gc  # noqa: E402
import synth  # noqa: E402

H, W, K = 1080, 1920, 8
f0 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, f0, 1, H, W, K)
g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
g.solve(cs, ct, nb)
g.set_profiling(True)
gc.debug_counters(g.ctx, reset=True)
g.profile(reset=True)
g.kernel_ms(reset=True)
F, m, st = g.solve(cs, ct, nb, stats=True)
torch.cuda.synchronize()
ms = g.kernel_ms(reset=True)
dbg = gc.debug_counters(g.ctx, reset=True)
names = ["push_tasks", "lower", "absorbed", "sides", "skipped_drain", "rounds", "active_after", "had_inflow", "noprog"]
out = {"frame": f0, "kernel_ms": round(ms, 3), "stats": [int(x) for x in st[0].tolist()],
       **{n: int(dbg[i]) for i, n in enumerate(names)}, "transitions": int(dbg[9])}
out["prof"] = {k: (v[0], round(v[1], 3), v[2]) for k, v in g.profile(reset=True).items()}
# tiles: how many are not uniform
print(json.dumps(out))
