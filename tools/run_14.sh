#!/bin/bash
# init group size and frames in flight on C4 (development)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python tools/sweep.py 1080p 1024 "GC_INITG=8,16,32" >> gpurun_out/sweep14.log 2>&1
  timeout 600 python tools/sweep.py 1080p 1024 "GC_SLOTS=24,48,96" >> gpurun_out/sweep14.log 2>&1
done
echo done
