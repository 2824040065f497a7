#!/bin/bash
# Round profiling recipe (run under gpurun): plain bench, launch list, full capture of the top kernels.
set -u
OUT=gpurun_out
CMD="python bench.py --frames 16 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_push|k_relax|k_seed|k_stream" -s 8 -c 16 -o $OUT/prof_full $CMD > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
