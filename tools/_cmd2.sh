make -s all > gpurun_out/make.log 2>&1 || { cat gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_saliency.py -x -q > gpurun_out/pytest_sal.log 2>&1; echo "sal rc=$?"; tail -25 gpurun_out/pytest_sal.log
