make -s all
CMD="python bench.py --frames 128 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu2_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_solve -s 2 -c 1 -o gpurun_out/prof_r02 $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu rc=$?"
