rm -f paper_1008_0502_b200/libgc.so; make -s DEV=1 all > /dev/null 2>&1
for v in 0 1; do echo "LREL=$v c5 $(GC_LRELABEL=$v timeout 600 python tools/c5_probe.py 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernel_ms"], d["stats"][0][:3])')"; done
for v in 0 1; do echo "LREL=$v f0 $(GC_LRELABEL=$v timeout 600 python tools/f0_counters.py 0 | cut -c1-120)"; done
GC_LRELABEL=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
bash tools/ab_knob.sh GC_LRELABEL "0 1" 2
bash tools/ab_rest.sh GC_LRELABEL "0 1" 1
