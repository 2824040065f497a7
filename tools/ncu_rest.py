"""Development: one C4 launch for an ncu capture: frames t0..t0+n-1 (default 1..128: the
throughput part, without the cold-start frame 0; `n 0` = the bench's own 1024-frame batch).
  ncu -k regex:k_solve --launch-skip 1 -c 1 python tools/ncu_rest.py [n] [t0]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1008_0502_b200 as gc  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
t0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, t0, n, 1080, 1920, 8)
g = gc.GridCut(neighborhood=8, max_h=1080, max_w=1920)
for _ in range(2):
    g.solve(cs, ct, nb)
torch.cuda.synchronize()
print("ok")
