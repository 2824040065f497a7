#!/bin/bash
# __grid_constant__ kernel params (no local copy of Dev/IO/Ctl): parity + A/B (development)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_19.log 2>&1; echo "pytest rc=$?"
AB_REPS=3 timeout 900 bash tools/ab.sh abl/base3.so abl/gridc.so "1080p 1024" "vga 120" "qvga 300" > gpurun_out/ab19.log 2>&1; echo "ab rc=$?"
for lib in base3 gridc; do
  echo "== $lib" >> gpurun_out/serp19.log
  NF=8 GC_LIB_PATH=abl/$lib.so GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 >> gpurun_out/serp19.log 2>&1
  GC_LIB_PATH=abl/$lib.so timeout 300 python bench.py --config c3 --warm --steps 2 --warmup 1 > gpurun_out/w19_$lib.log 2>&1
done
echo done
