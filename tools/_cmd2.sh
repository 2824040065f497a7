make -s all > gpurun_out/make.log 2>&1 || { cat gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_fast_l.log 2>&1; echo "fast rc=$?"; tail -2 gpurun_out/pytest_fast_l.log
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_l$i.log 2>&1; python tools/tsum.py l$i 2>&1 | head -1; done
timeout 300 python tools/trace_probe.py c4 1024 c4_l > gpurun_out/trace_c4_l.txt 2>&1
