#!/bin/bash
# Development aid: A/B timing of two builds of libgc.so on the same box, interleaved.
# Builds under test should be DEV=1 builds (tuning knobs). The last one tested stays installed.
# usage: tools/ab.sh old.so new.so "cfg frames" ["cfg frames" ...]   (reps: AB_REPS, default 3)
old=$1; new=$2; shift 2
for cf in "$@"; do
  for r in $(seq ${AB_REPS:-3}); do
    for lib in "$old" "$new"; do
      cp "$lib" paper_1008_0502_b200/libgc.so && python tools/sweep.py $cf "" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], d['cfg'], d['n'], d['ms'], d['cta_ms'])"
    done
  done
done
