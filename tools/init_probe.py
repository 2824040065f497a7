"""Development aid: init-pass throughput.  Frames whose every pixel is a sink (cs = 0,
ct = 1) are solved by the init pass alone (every tile is a uniform sink tile), so the solve
time is the streaming cost of reading the caps.
usage: init_probe.py [frames] [H] [W] [K]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1008_0502_b200 as gc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
H = int(sys.argv[2]) if len(sys.argv) > 2 else 1080
W = int(sys.argv[3]) if len(sys.argv) > 3 else 1920
K = int(sys.argv[4]) if len(sys.argv) > 4 else 8
cs = torch.zeros((n, H, W), dtype=torch.int32, device="cuda")
ct = torch.ones((n, H, W), dtype=torch.int32, device="cuda")
nb = torch.randint(0, 100, (n, K, H, W), dtype=torch.int32, device="cuda")
g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
F, m = g.solve(cs, ct, nb)
torch.cuda.synchronize()
assert int(F[0]) == 0 and int(m.sum()) == 0
best = 1e30
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.solve(cs, ct, nb); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
byts = n * H * W * (4 * (2 + K) + 2 + 1)
print(json.dumps({"frames": n, "H": H, "W": W, "K": K, "ms": round(best, 3), "GB_s": round(byts / best / 1e6, 1),
                  "Mpx_s": round(n * H * W / best / 1e3, 1)}))
