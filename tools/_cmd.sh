bash tools/ab_knob.sh GC_BULKG "2 4 8" 2 "--config c2" 2>&1 | grep GC_BULKG
bash tools/ab_rest.sh GC_BULKG "4 8 16" 2 2>&1 | grep GC_BULKG
