#!/bin/bash
# init tasks of up to 64 tiles + export of untouched tiles at init: parity + A/B (development)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_15.log 2>&1; echo "pytest rc=$?"
AB_REPS=2 timeout 900 bash tools/ab.sh abl/lat.so abl/init64.so "1080p 1024" "vga 120" "qvga 300" > gpurun_out/ab15.log 2>&1; echo "ab rc=$?"
for lib in lat init64; do
  GC_LIB_PATH=abl/$lib.so timeout 300 python bench.py --config c3 --warm --steps 2 --warmup 1 > gpurun_out/w15_$lib.log 2>&1; echo "$lib rc=$?"
done
GC_LIB_PATH=abl/init64.so timeout 600 python tools/sweep.py 1080p 1024 "GC_INITG=32,63,128" > gpurun_out/sw15.log 2>&1; echo "sweep rc=$?"
