#!/bin/bash
# push self-rerun rule and rounds per task on serpentine and typical frames (development)
set -u
mkdir -p gpurun_out
for kv in "GC_SELFRUN=0" "GC_SELFRUN=1" "ROUNDS=16" "ROUNDS=32" "GC_SELFRUN=1 ROUNDS=16"; do
  echo "== $kv" >> gpurun_out/serp10.log
  env $kv GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 1080x1920 2160x3840 >> gpurun_out/serp10.log 2>&1
done
echo "serp done"
for cf in "1080p 1024" "vga 120" "qvga 300"; do
  timeout 600 python tools/sweep.py $cf "GC_SELFRUN=0,1;ROUNDS=8,16" >> gpurun_out/sweep10.log 2>&1
done
echo "sweep done"
