#!/bin/bash
# Same-box A/B of a DEV-build tuning knob on the C4 bench: tools/ab_knob.sh KNOB "v1 v2" [reps] [extra bench args]
set -u
KNOB=$1; VALS=$2; REPS=${3:-2}; EXTRA=${4:-}
mkdir -p gpurun_out
rm -f paper_1008_0502_b200/libgc.so; make -s DEV=1 all > /dev/null 2>&1
for r in $(seq $REPS); do
  for v in $VALS; do
    env $KNOB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 $EXTRA > gpurun_out/ab_${KNOB}_${v}_$r.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_${KNOB}_${v}_$r.log').read().strip().splitlines()[-1]); print('$KNOB=$v', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'])"
  done
done
rm -f paper_1008_0502_b200/libgc.so; make -s all
