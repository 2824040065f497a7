"""Development: latency of the C4 cold-start frame (frame 0) alone and the batch without it."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1008_0502_b200 as gc  # noqa: E402
import synth  # noqa: E402

H, W, K = 1080, 1920, 8
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, 0, n, H, W, K)
g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
out = {}
cases = [("frame0", slice(0, 1)), ("frames0-23", slice(0, min(24, n))), ("frame1", slice(1, 2))]
if n > 24:
    cases += [("without0", slice(1, n)), ("all", slice(0, n))]
for name, sl in cases:
    a, b, c = cs[sl].contiguous(), ct[sl].contiguous(), nb[sl].contiguous()
    g.solve(a, b, c)
    ms = []
    for _ in range(3):
        g.kernel_ms(reset=True)
        F, m, st = g.solve(a, b, c, stats=True)
        ms.append(round(g.kernel_ms(reset=True), 3))
    out[name] = {"ms": ms, "relabels0": int(st[0, 1]), "push0": int(st[0, 0])}
    del a, b, c
print(json.dumps(out))
