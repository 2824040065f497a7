#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_12.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b12_c4.log 2>&1; echo "c4 rc=$?"
timeout 600 python bench.py --config c3 --warm > gpurun_out/b12_c3warm.log 2>&1; echo "c3w rc=$?"
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b12_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/b12_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b12_c5.log 2>&1; echo "c5 rc=$?"
