#!/bin/bash
# Round profiling recipe (run under gpurun): plain bench, launch list, full capture of k_solve.
set -u
OUT=gpurun_out
TAG=${1:-cur}
FR=${2:-128}
CMD="python bench.py --frames $FR --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 200 --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_solve" -s 2 -c 1 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
