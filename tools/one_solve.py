"""Development aid for ncu captures: generate a batch on the device and solve it twice
(warm-up + the launch to capture: `ncu -k regex:k_solve -s 1 -c 1`).
usage: one_solve.py cfg frames [t0] [seed_off]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1008_0502_b200 as gc
import synth

ALL = {"qvga": ("blob", 240, 320, 4), "vga": ("blob", 480, 640, 4), "1080p": ("blob", 1080, 1920, 8),
       "serp": ("serpentine", 1080, 1920, 4)}
name, n = sys.argv[1], int(sys.argv[2])
t0 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
seed_off = int(sys.argv[4]) if len(sys.argv) > 4 else 3
kind, H, W, K = ALL[name]
cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + seed_off, t0, n, H, W, K)
g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
for _ in range(2):
    F, m = g.solve(cs, ct, nb)
torch.cuda.synchronize()
print("ok", int(F.sum()), int(m.sum()))
