#!/bin/bash
# Full ncu capture of busy k_push / k_relax / k_seed launches on 16 1080p 8-nbr frames.
CMD="python tools/frames_probe.py blob 1080 1920 8 16 10080505 0"
timeout 300 $CMD > gpurun_out/fp_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_push|k_relax|k_seed|k_stream" -s 40 -c 16 -o gpurun_out/prof_push $CMD > gpurun_out/ncu_push.log 2>&1
echo "rc=$?"
