make -s all
python tools/trace_probe.py c4 1 f0alone > gpurun_out/trace_f0alone.txt 2>&1
