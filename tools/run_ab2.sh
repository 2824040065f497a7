#!/bin/bash
# A/B of the scheduler variant + serpentine knob sweep (development; logs in gpurun_out/)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_new2.log 2>&1; echo "pytest rc=$?"
AB_REPS=3 timeout 900 bash tools/ab.sh abl/old.so abl/new.so "1080p 1024" "qvga 300" "vga 120" > gpurun_out/ab2.log 2>&1; echo "ab rc=$?"
for kv in "GC_X=0" "GC_STALL=100000" "GC_STALL=100000 GC_VIS=100000" "GC_ALPHA=2" "GC_SELFRUN=0" "GC_WAVE=1000000" "GC_STALL=100000 GC_VIS=100000 GC_ALPHA=5 GC_SELFRUN=0"; do
  echo "== $kv" >> gpurun_out/serp2.log
  env $kv GC_TIMEOUT_S=30 timeout 120 python tools/serp_probe.py 540x960 >> gpurun_out/serp2.log 2>&1
done
echo "serp done"
