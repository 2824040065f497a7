#!/bin/bash
# per-warp seed / closure-seed groups: parity + A/B against the block versions (development)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_warp.log 2>&1; echo "pytest rc=$?"
AB_REPS=3 timeout 1200 bash tools/ab.sh abl/urg.so abl/warp.so "1080p 1024" "qvga 300" "vga 120" > gpurun_out/ab6.log 2>&1; echo "ab rc=$?"
for lib in urg warp; do
  echo "== $lib" >> gpurun_out/serp6.log
  GC_LIB_PATH=abl/$lib.so GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 >> gpurun_out/serp6.log 2>&1
done
echo "serp done"
