#!/bin/bash
# Development aid: A/B timing of two builds of libgc.so on the same box, interleaved.
# usage: tools/ab.sh old.so new.so "cfg frames" ["cfg frames" ...]   (reps: AB_REPS, default 3)
old=$1; new=$2; shift 2
for cf in "$@"; do
  for r in $(seq ${AB_REPS:-3}); do
    for lib in "$old" "$new"; do
      GC_LIB_PATH=$lib python tools/sweep.py $cf "" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], d['cfg'], d['n'], d['ms'], d['cta_ms'])"
    done
  done
done
