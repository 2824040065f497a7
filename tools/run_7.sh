#!/bin/bash
# per-warp seed / closure-seed groups + init L2 prefetch: parity + A/B (development)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_l2pf.log 2>&1; echo "pytest rc=$?"
AB_REPS=2 timeout 900 bash tools/ab.sh abl/base.so abl/warp2.so "1080p 1024" "qvga 300" "vga 120" > gpurun_out/ab7.log 2>&1; echo "ab rc=$?"
GC_LIB_PATH=abl/l2pf.so timeout 600 python tools/sweep.py 1080p 1024 "GC_L2PF=0,1,2,4" > gpurun_out/l2pf7.log 2>&1
GC_LIB_PATH=abl/l2pf.so timeout 600 python tools/sweep.py 1080p 1024 "GC_L2PF=0,1,2,4" >> gpurun_out/l2pf7.log 2>&1; echo "l2pf rc=$?"
for lib in base warp2; do
  echo "== $lib" >> gpurun_out/serp7.log
  NF=8 GC_LIB_PATH=abl/$lib.so GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 >> gpurun_out/serp7.log 2>&1
done
echo "serp done"
