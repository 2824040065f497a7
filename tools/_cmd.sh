make -s all > gpurun_out/make.log 2>&1 || { cat gpurun_out/make.log; exit 1; }
T=${TAG:-x}
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_fast_$T.log 2>&1; echo "pytest fast rc=$?"; tail -3 gpurun_out/pytest_fast_$T.log
timeout 900 python -m pytest tests -m "gpu and slow" -x -q -s > gpurun_out/pytest_slow_$T.log 2>&1; echo "pytest slow rc=$?"; tail -3 gpurun_out/pytest_slow_$T.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?"
timeout 300 python tools/trace_probe.py c4 1024 c4_$T > gpurun_out/trace_c4_$T.txt 2>&1; echo "trace rc=$?"
if [ -n "${MORE:-}" ]; then
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_$T.log 2>&1; echo "c2 rc=$?"
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_$T.log 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --config c3 --warm --steps 2 --warmup 1 > gpurun_out/bench_c3w_$T.log 2>&1; echo "c3w rc=$?"
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$T.log 2>&1; echo "c5 rc=$?"
fi
