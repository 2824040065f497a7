#!/bin/bash
# A/B: urgent ring for hard frames (development; logs in gpurun_out/)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_urg.log 2>&1; echo "pytest rc=$?"
AB_REPS=4 timeout 1200 bash tools/ab.sh abl/base.so abl/urg.so "1080p 1024" "qvga 300" "vga 120" > gpurun_out/ab5.log 2>&1; echo "ab rc=$?"
for lib in base urg; do
  echo "== $lib" >> gpurun_out/serp5.log
  NF=8 GC_LIB_PATH=abl/$lib.so GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 >> gpurun_out/serp5.log 2>&1
done
echo "serp done"
