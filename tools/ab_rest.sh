#!/bin/bash
# DEV-build A/B of a knob on the C4 batch WITHOUT the cold-start frame 0 (frames 1..1024: the
# throughput part of the step, not frame 0's latency).  usage: tools/ab_rest.sh KNOB "v1 v2" [reps]
set -u
KNOB=$1; VALS=$2; REPS=${3:-3}
mkdir -p gpurun_out
rm -f paper_1008_0502_b200/libgc.so; make -s DEV=1 all > /dev/null 2>&1
cat > /tmp/rest.py <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, synth, paper_1008_0502_b200 as gc
cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, 1, 1024, 1080, 1920, 8)
g = gc.GridCut(neighborhood=8, max_h=1080, max_w=1920)
for _ in range(2): g.solve(cs, ct, nb)
torch.cuda.synchronize()
ms = []
for _ in range(4):
    g.kernel_ms(reset=True); g.solve(cs, ct, nb); ms.append(round(g.kernel_ms(reset=True), 2))
print(json.dumps(ms))
PY
for r in $(seq $REPS); do
  for v in $VALS; do
    echo "$KNOB=$v $(env $KNOB=$v timeout 300 python /tmp/rest.py 2>&1 | tail -1)"
  done
done
rm -f paper_1008_0502_b200/libgc.so; make -s all
