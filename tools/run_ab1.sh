#!/bin/bash
# A/B of the two-ring scheduler + serpentine probes (development; logs in gpurun_out/)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"
AB_REPS=2 timeout 900 bash tools/ab.sh abl/old.so abl/new.so "1080p 1024" "qvga 300" "vga 120" > gpurun_out/ab1.log 2>&1; echo "ab rc=$?"
T0=1 AB_REPS=1 timeout 300 bash tools/ab.sh abl/old.so abl/new.so "1080p 1024" >> gpurun_out/ab1.log 2>&1
GC_TIMEOUT_S=60 timeout 600 python tools/serp_probe.py 256x384 540x960 1080x1920 > gpurun_out/serp1.log 2>&1; echo "serp rc=$?"
