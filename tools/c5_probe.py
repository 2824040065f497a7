"""Development: C5 (4K serpentine) per-class task counts / CTA time and per-frame counters."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1008_0502_b200 as gc  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
H, W = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (2160, 3840)
synth.set_serpentine_params(lane=64, big=1 << 20)
cs, ct, nb = synth.gen_torch("serpentine", synth.BASE_SEED + 4, 0, n, H, W, 4)
g = gc.GridCut(neighborhood=4, max_h=H, max_w=W, rounds_per_launch=int(os.environ.get("C5_ROUNDS", "0")))
g.set_profiling(True)
g.profile(reset=True)
g.kernel_ms(reset=True)
F, m, st = g.solve(cs, ct, nb, stats=True)
torch.cuda.synchronize()
prof = g.profile(reset=True)
print(json.dumps({"n": n, "H": H, "W": W, "kernel_ms": round(g.kernel_ms(reset=True), 1),
                  "classes": {k: {"tasks": v[2], "cta_ms": round(v[1], 2)} for k, v in prof.items()},
                  "stats": st.cpu().tolist(), "F": F.cpu().tolist(),
                  "dbg": gc.debug_counters(g.ctx, reset=True)}))
