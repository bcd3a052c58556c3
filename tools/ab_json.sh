#!/bin/bash
# A/B library variants (SOS="variants/a.so ...") on the bench line: fp32 hot-x kernel/step,
# unpacked kernel, fp64 step, C5 power step. BENCH_ARGS adds flags.
for rep in 1 2; do
for so in ${SOS:-variants/*.so}; do
  LWB200_LIB=$so timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | tail -1 | \
  python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d.get('power',{}); f=d.get('fp64',{}); u=d.get('unpacked',{})
print('$so', 'hot_kernel', d['roofline']['kernel_ms'], 'step', d['ms_per_step'], 'unpacked_kernel', u.get('kernel_ms'), 'fp64_step', f.get('ms_per_step'), 'power_step', p.get('ms_per_step'), 'spmv_c5', p.get('breakdown_ms',{}).get('spmv_max_rank'))"
done; done
