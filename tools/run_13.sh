#!/bin/bash
# shorter load chains in seed / closure-seed / push prologues: parity + A/B (development)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_13.log 2>&1; echo "pytest rc=$?"
AB_REPS=3 timeout 1200 bash tools/ab.sh abl/head.so abl/lat.so "1080p 1024" "vga 120" "qvga 300" > gpurun_out/ab13.log 2>&1; echo "ab rc=$?"
