python bench.py --config c3 --warm --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_c3w_t5.log 2>&1; tail -1 gpurun_out/bench_c3w_t5.log | cut -c1-200; grep -o '"cold_same_schedule[^}]*}' gpurun_out/bench_c3w_t5.log
python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_c3_t5.log 2>&1; python tools/tsum.py c3_t5 2>/dev/null | head -1
python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_c2_t5.log 2>&1; python tools/tsum.py c2_t5 2>/dev/null | head -1
python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_c4_t5.log 2>&1; python tools/tsum.py c4_t5 2>/dev/null | head -1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_t5.log 2>&1; tail -3 gpurun_out/pytest_t5.log
