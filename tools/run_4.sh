#!/bin/bash
# stall-doubling threshold sweep on typical and serpentine frames (development)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for cf in "1080p 1024" "qvga 300" "vga 120"; do
  timeout 600 python tools/sweep.py $cf "GC_STALLX=1000000,2,4,6,8" >> gpurun_out/sweep4.log 2>&1
done
done
echo "sweep done"
for x in 2 4 6 8; do
  echo "== $x" >> gpurun_out/serp4.log
  GC_STALLX=$x GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 540x960 1080x1920 2160x3840 >> gpurun_out/serp4.log 2>&1
done
echo "serp done"
