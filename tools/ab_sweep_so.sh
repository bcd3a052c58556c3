#!/bin/bash
# A/B library variants on the schedule sweep: SOS="variants/a.so ..." SCHED=group_warp CONFIGS=C2b,C2u
for rep in 1 2; do
for so in $SOS; do
  LWB200_LIB=$so timeout 600 python tools/bench_sweep.py --configs ${CONFIGS:-C2b,C2u,C3,C4} --no-cpu --dtypes ${DTYPES:-float32,float64} --schedules ${SCHED:-group_warp} --reps 20 2>/dev/null | python3 -c "
import sys,json
out=[]
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    out.append(f\"{d['config']}/{d['dtype'][5:]}/{d['schedule'][:8]}:{d['ms']}\")
print('$so', ' '.join(out))"
done; done
