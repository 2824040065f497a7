#!/bin/bash
# stall-bound sweep on typical and serpentine frames (development; logs in gpurun_out/)
set -u
mkdir -p gpurun_out
for cf in "1080p 1024" "qvga 300" "vga 120"; do
  timeout 600 python tools/sweep.py $cf "GC_STALL=64,1024,100000;GC_STALLX=0,1" >> gpurun_out/sweep3.log 2>&1
done
echo "sweep done"
for kv in "GC_STALL=64 GC_STALLX=1" "GC_STALL=100000" "GC_STALL=1000000 GC_VIS=1000000"; do
  echo "== $kv" >> gpurun_out/serp3.log
  env $kv GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 540x960 1080x1920 2160x3840 >> gpurun_out/serp3.log 2>&1
done
echo "serp done"
