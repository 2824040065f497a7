#!/bin/bash
# DEV-build sweep of push-phase knobs on the C4 cold-start frame 0 alone (tools/f0_counters.py).
rm -f paper_1008_0502_b200/libgc.so; make -s DEV=1 all > /dev/null 2>&1
run() { echo "$* $(env "$@" timeout 120 python tools/f0_counters.py 0 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernel_ms"], d["stats"][:3])')"; }
run X=0
run GC_WAVE=4
run GC_WAVE=16
run GC_WAVE=64
run GC_WAVESH=1
run GC_WAVESH=3
run GC_BNDSH=1
run GC_BNDSH=3
run GC_BNDSH=4
run GC_ALPHA=0.05
run GC_ALPHA=1.0
run GC_STALL=16
run GC_STALL=256
run GC_STALLX=2
run GC_SELFRUN=1
run GC_VIS=16
run GC_VIS=256
run GC_WAVE=16 GC_BNDSH=3
run X=0
rm -f paper_1008_0502_b200/libgc.so; make -s all > /dev/null 2>&1
