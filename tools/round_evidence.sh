#!/bin/bash
# Round-end evidence under gpurun: gpu tests, smoke, bench lines of every config, the reference
# arm, the k_solve launch list and one full ncu capture (logs and reports in gpurun_out/).
set -u
TAG=${1:-v13}
OUT=gpurun_out
mkdir -p $OUT
make -s all > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $OUT/bench_c4_$TAG.log 2>&1; echo "bench c4 rc=$?"
timeout 600 python bench.py --config c2 > $OUT/bench_c2_$TAG.log 2>&1; echo "bench c2 rc=$?"
timeout 600 python bench.py --config c3 > $OUT/bench_c3_$TAG.log 2>&1; echo "bench c3 rc=$?"
timeout 600 python bench.py --config c3 --warm > $OUT/bench_c3warm_$TAG.log 2>&1; echo "bench c3 warm rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > $OUT/bench_c5_$TAG.log 2>&1; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --frames 128 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 200 --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_solve" -s 2 -c 1 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
