make -s all; python tools/frame0_probe.py > gpurun_out/frame0.txt 2>&1; cat gpurun_out/frame0.txt
