#!/bin/bash
# relabel-bound / push-cap growth per failed attempt (development)
set -u
mkdir -p gpurun_out
T0=0 timeout 300 python tools/sweep.py 1080p 1 "GC_BNDSH=1,2,3;GC_WAVESH=1,2" > gpurun_out/grow8.log 2>&1
T0=0 timeout 300 python tools/sweep.py 1080p 16 "GC_BNDSH=1,2,3;GC_WAVESH=1,2" >> gpurun_out/grow8.log 2>&1
for rep in 1 2; do
timeout 600 python tools/sweep.py 1080p 1024 "GC_BNDSH=1,2;GC_WAVESH=1,2" >> gpurun_out/grow8.log 2>&1
timeout 300 python tools/sweep.py vga 120 "GC_BNDSH=1,2;GC_WAVESH=1,2" >> gpurun_out/grow8.log 2>&1
timeout 300 python tools/sweep.py qvga 300 "GC_BNDSH=1,2;GC_WAVESH=1,2" >> gpurun_out/grow8.log 2>&1
done
echo "sweep rc=$?"
for kv in "GC_BNDSH=1" "GC_BNDSH=2" "GC_BNDSH=2 GC_WAVESH=2"; do
  echo "== $kv" >> gpurun_out/serp8.log
  env $kv GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 >> gpurun_out/serp8.log 2>&1
done
echo "serp done"
