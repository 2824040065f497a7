#!/bin/bash
# The GPU test suite against a CHECKS=1 build of libgc.so (device invariant checks; the pool
# has no compute-sanitizer), then the default build again.  Logs in gpurun_out/.
set -u
mkdir -p gpurun_out
rm -f paper_1008_0502_b200/libgc.so
make -s CHECKS=1 paper_1008_0502_b200/libgc.so synth/libsynth.so oracle/liboracle.so > gpurun_out/checked_make.log 2>&1 || { cat gpurun_out/checked_make.log; exit 1; }
strings paper_1008_0502_b200/libgc.so | grep -c "device check failed" > gpurun_out/checked_build_marker.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/checked_pytest.log 2>&1; echo "checked pytest rc=$?"; tail -3 gpurun_out/checked_pytest.log
timeout 600 python tools/sanitize_run.py all > gpurun_out/checked_small.log 2>&1; echo "checked small rc=$?"
rm -f paper_1008_0502_b200/libgc.so; make -s all
