"""Development aid: solve a config and save per-frame F and mask hashes (regression check
between library builds).  usage: dump_results.py cfg frames out.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1008_0502_b200 as gc
import synth

ALL = {"qvga": ("blob", 240, 320, 4, 1), "vga": ("blob", 480, 640, 4, 2), "1080p": ("blob", 1080, 1920, 8, 3)}
name, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
kind, H, W, K, so = ALL[name]
cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + so, 0, n, H, W, K)
g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
F, m = g.solve(cs, ct, nb)
torch.cuda.synchronize()
w = torch.arange(H * W, device="cuda", dtype=torch.int64) % 1000003 + 1
mh = (m.view(n, -1).to(torch.int64) * w).sum(dim=1)
np.savez(out, F=F.cpu().numpy(), mh=mh.cpu().numpy(), pop=m.view(n, -1).sum(dim=1).cpu().numpy())
print("saved", out, int(F.sum()))
