#!/bin/bash
set -u
mkdir -p gpurun_out
AB_REPS=2 timeout 900 bash tools/ab.sh abl/base3.so abl/gridc2.so "1080p 1024" "vga 120" > gpurun_out/ab20.log 2>&1; echo "ab rc=$?"
