#!/bin/bash
# small-call latency (8 VGA frames) across scheduler versions (development)
set -u
mkdir -p gpurun_out
for t0 in 5 0; do
  for lib in old new base2 setupq qnop; do
    T0=$t0 GC_LIB_PATH=abl/$lib.so timeout 120 python tools/sweep.py vga 8 "" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', 'T0=$t0', d['n'], d['ms'], d['st_max'][:2], d['cta_ms'])" >> gpurun_out/lat11.log 2>&1
  done
done
T0=5 GC_STALLX=1000000 GC_LIB_PATH=abl/setupq.so timeout 120 python tools/sweep.py vga 8 "" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('setupq nostallx T0=5', d['ms'], d['cta_ms'])" >> gpurun_out/lat11.log 2>&1
echo done
