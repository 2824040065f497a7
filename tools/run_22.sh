#!/bin/bash
set -u
mkdir -p gpurun_out
AB_REPS=3 timeout 900 bash tools/ab.sh abl/gridc2.so abl/gridc3.so "1080p 1024" "vga 120" "qvga 300" > gpurun_out/ab22.log 2>&1; echo "ab rc=$?"
