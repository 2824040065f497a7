#!/bin/bash
# export of untouched tiles at init (templated): parity + A/B against lat (development)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_16.log 2>&1; echo "pytest rc=$?"
AB_REPS=3 timeout 900 bash tools/ab.sh abl/lat.so abl/exp.so "1080p 1024" "vga 120" > gpurun_out/ab16.log 2>&1; echo "ab rc=$?"
for lib in lat exp; do
  GC_LIB_PATH=abl/$lib.so timeout 300 python bench.py --config c3 --warm --steps 2 --warmup 1 > gpurun_out/w16_$lib.log 2>&1; echo "$lib rc=$?"
done
