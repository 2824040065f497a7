#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (run under gpurun);
# logs in gpurun_out/sanitize_<tool>_<part>.log
set -u
mkdir -p gpurun_out
make -s all > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for part in c1 c2 c4; do
    timeout 1500 $CS --tool $tool --kernel-name regex:"k_solve|k_setup|k_abort|k_digest" \
      python tools/sanitize_run.py $part > gpurun_out/sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_${part}.log | tail -1)"
  done
done
