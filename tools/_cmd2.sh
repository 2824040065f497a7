make -s all > gpurun_out/make.log 2>&1 || { cat gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_fast_o.log 2>&1; echo "fast rc=$?"; tail -2 gpurun_out/pytest_fast_o.log
timeout 900 python -m pytest tests/test_gpu_scale.py -k "c3" -x -q > gpurun_out/pytest_c3_o.log 2>&1; echo "c3 rc=$?"; tail -2 gpurun_out/pytest_c3_o.log
for i in 1 2; do timeout 600 python bench.py --config c3 --warm --steps 3 --warmup 2 > gpurun_out/bench_c3w_o$i.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_c3w_o$i.log').read().strip().splitlines()[-1]); print('c3w', d['value'], d['ms_per_step'], d['cold_same_schedule'])"; done
timeout 300 python tools/trace_probe.py c3warm 0 c3warm_o > gpurun_out/trace_c3warm_o.txt 2>&1; head -1 gpurun_out/trace_c3warm_o.txt | cut -c1-400
