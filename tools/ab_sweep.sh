#!/bin/bash
# A/B all variants/*.so on a sweep subset: tools/ab_sweep.sh CONFIGS
for so in variants/*.so; do
  LWB200_LIB=$so timeout 600 python tools/bench_sweep.py --configs ${1:-C2b,C2u} --no-cpu --reps 10 --dtypes float32 2>/dev/null | \
    python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$(basename $so)'.ljust(18), d['config'], d['matrix'][:30].ljust(30), d['schedule'].ljust(14), d['ms'])
"
done
