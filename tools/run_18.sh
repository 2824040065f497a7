#!/bin/bash
# urgent ring (held tickets): parity + A/B against base3 on typical, small and serpentine calls
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_18.log 2>&1; echo "pytest rc=$?"
AB_REPS=3 timeout 900 bash tools/ab.sh abl/base3.so abl/urg2.so "1080p 1024" "vga 120" "qvga 300" "vga 8" > gpurun_out/ab18.log 2>&1; echo "ab rc=$?"
for lib in base3 urg2; do
  echo "== $lib" >> gpurun_out/serp18.log
  NF=8 GC_LIB_PATH=abl/$lib.so GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 >> gpurun_out/serp18.log 2>&1
  GC_LIB_PATH=abl/$lib.so timeout 300 python bench.py --config c3 --warm --steps 2 --warmup 1 > gpurun_out/w18_$lib.log 2>&1
done
echo done
