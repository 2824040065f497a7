make -s all > gpurun_out/make.log 2>&1 || { cat gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_energy.py -x -q > gpurun_out/pytest_energy.log 2>&1; echo "energy rc=$?"; tail -15 gpurun_out/pytest_energy.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_fast_j.log 2>&1; echo "fast rc=$?"; tail -2 gpurun_out/pytest_fast_j.log
