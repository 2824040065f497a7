"""Development: C4 frame 0 alone / 24 frames / 1024 frames vs rounds_per_launch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1008_0502_b200 as gc  # noqa: E402
import synth  # noqa: E402

H, W, K = 1080, 1920, 8
cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, 0, 1024, H, W, K)
for r in [int(x) for x in sys.argv[1:]]:
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W, rounds_per_launch=r)
    out = {"rounds": r}
    for name, n in [("f0", 1), ("b24", 24), ("all", 1024)]:
        a, b, c = cs[:n], ct[:n], nb[:n]
        g.solve(a, b, c)
        ms = []
        for _ in range(3):
            g.kernel_ms(reset=True)
            F, m, st = g.solve(a, b, c, stats=True)
            ms.append(round(g.kernel_ms(reset=True), 2))
        out[name] = ms
        out[name + "_push0"] = int(st[0, 0])
    g.close()
    print(json.dumps(out), flush=True)
