make -s all
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu1_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c4_1024_r02.csv $CMD > gpurun_out/ncu1.log 2>&1
echo "ncu rc=$?"
