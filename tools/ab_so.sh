#!/bin/bash
# Same-box A/B of two prebuilt libraries (paper_1008_0502_b200/libgc_A.so, libgc_B.so) on the
# C4 batch without frame 0 (stable: the throughput part) and with it.  usage: tools/ab_so.sh [reps]
set -u
REPS=${1:-3}
P=paper_1008_0502_b200
cat > /tmp/abso.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, synth, paper_1008_0502_b200 as gc
t0 = int(sys.argv[1])
cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, t0, 1024, 1080, 1920, 8)
g = gc.GridCut(neighborhood=8, max_h=1080, max_w=1920)
for _ in range(2): g.solve(cs, ct, nb)
torch.cuda.synchronize()
ms = []
for _ in range(4):
    g.kernel_ms(reset=True); g.solve(cs, ct, nb); ms.append(round(g.kernel_ms(reset=True), 2))
print(json.dumps(ms))
PY
for r in $(seq $REPS); do
  for v in A B; do
    cp $P/libgc_$v.so $P/libgc.so
    echo "$v rest $(timeout 300 python /tmp/abso.py 1 2>&1 | tail -1)  all $(timeout 300 python /tmp/abso.py 0 2>&1 | tail -1)"
  done
done
