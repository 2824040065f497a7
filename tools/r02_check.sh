#!/bin/bash
# Round-2 GPU check under gpurun: build, gpu tests (with durations), bench (+ verify leg).
set -u
TAG=${1:-a}
OUT=gpurun_out
mkdir -p $OUT
make -s all > $OUT/make_$TAG.log 2>&1; echo "make rc=$?"
nproc > $OUT/nproc_$TAG.txt; free -g >> $OUT/nproc_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -x -q -s --durations=15 > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --verify 0 > $OUT/bench_c4_$TAG.log 2>&1; echo "bench rc=$?"
