#!/bin/bash
# export fused into the closure seed (no export phase): parity + warm A/B (development)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_17.log 2>&1; echo "pytest rc=$?"
for lib in exp noexp exp noexp; do
  GC_LIB_PATH=abl/$lib.so timeout 300 python bench.py --config c3 --warm --steps 2 --warmup 1 >> gpurun_out/w17_$lib.log 2>&1; echo "$lib rc=$?"
done
AB_REPS=2 timeout 900 bash tools/ab.sh abl/exp.so abl/noexp.so "1080p 1024" "vga 120" > gpurun_out/ab17.log 2>&1; echo "ab rc=$?"
