#!/bin/bash
# Round check under gpurun: gpu tests, smoke, default bench, C5 bench (logs in gpurun_out/).
set -u
mkdir -p gpurun_out
make -s all >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?"
