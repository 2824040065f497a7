bash tools/knob_sweep.sh "GC_URGENT=0" "GC_URGENT=1" "GC_URGENT=0" "GC_URGENT=1"
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_u.log 2>&1; tail -c 300 gpurun_out/bench_c5_u.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
timeout 300 python tools/trace_probe.py c4 1024 c4_u > gpurun_out/trace_c4_u.txt 2>&1
