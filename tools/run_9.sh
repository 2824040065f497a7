#!/bin/bash
# initial init groups on the chain ring: C3 sequence steps, C2, C4 (development)
set -u
mkdir -p gpurun_out
for lib in old cur setupq; do
  GC_LIB_PATH=abl/$lib.so timeout 300 python bench.py --config c3 --warm --steps 2 --warmup 1 > gpurun_out/w9_$lib.log 2>&1; echo "$lib rc=$?"
done
AB_REPS=2 timeout 900 bash tools/ab.sh abl/cur.so abl/setupq.so "1080p 1024" "qvga 300" "vga 120" "vga 8" > gpurun_out/ab9.log 2>&1; echo "ab rc=$?"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_setupq.log 2>&1; echo "pytest rc=$?"
