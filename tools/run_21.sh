#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_21.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_21.log 2>&1; echo "smoke rc=$?"
NF=8 GC_TIMEOUT_S=60 timeout 200 python tools/serp_probe.py 2160x3840 > gpurun_out/serp21.log 2>&1; echo "serp rc=$?"
timeout 300 python bench.py --config c3 --warm --steps 2 --warmup 1 > gpurun_out/w21.log 2>&1; echo "warm rc=$?"
