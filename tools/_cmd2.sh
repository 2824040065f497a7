make -s all > gpurun_out/make.log 2>&1 || { cat gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_prior.py tests/test_gpu_energy.py -x -q > gpurun_out/pytest_prior.log 2>&1; echo "prior rc=$?"; tail -15 gpurun_out/pytest_prior.log
timeout 600 python bench.py --prior > gpurun_out/bench_prior.log 2>&1; echo "bench rc=$?"; tail -c 900 gpurun_out/bench_prior.log
