#!/bin/bash
set -u
mkdir -p gpurun_out
AB_REPS=3 timeout 900 bash tools/ab.sh abl/gridc2.so abl/minb3.so "1080p 1024" "vga 120" "qvga 300" > gpurun_out/ab23.log 2>&1; echo "ab rc=$?"
for lib in gridc2 minb3; do
  echo "== $lib" >> gpurun_out/serp23.log
  NF=8 GC_LIB_PATH=abl/$lib.so GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 >> gpurun_out/serp23.log 2>&1
done
