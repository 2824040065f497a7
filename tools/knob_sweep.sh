#!/bin/bash
# DEV-build knob sweep: frame-0-alone latency and the full C4 bench per setting.
# usage: tools/knob_sweep.sh "ENV1=a ENV2=b" "ENV1=c" ...
set -u
mkdir -p gpurun_out
rm -f paper_1008_0502_b200/libgc.so; make -s DEV=1 all > /dev/null 2>&1
i=0
for setting in "$@"; do
  i=$((i+1))
  env $setting timeout 300 python tools/frame0_probe.py 24 > gpurun_out/sweep_f0_$i.txt 2>&1
  env $setting timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/sweep_b_$i.log 2>&1
  python - "$setting" $i <<'PY'
import json, sys
s, i = sys.argv[1], sys.argv[2]
try:
    f = json.loads(open(f"gpurun_out/sweep_f0_{i}.txt").read().strip().splitlines()[-1])
    d = json.loads(open(f"gpurun_out/sweep_b_{i}.log").read().strip().splitlines()[-1])
    print(s, "| f0 alone", f["frame0"]["ms"], "rel", f["frame0"]["relabels0"], "| 0-23", f["frames0-23"]["ms"], "| C4", d["ms_per_step"])
except Exception as e:
    print(s, "failed", e)
PY
done
rm -f paper_1008_0502_b200/libgc.so; make -s all
