#!/bin/bash
# A/B library variants built by tools/build_variant.py (SOS="variants/a.so variants/b.so")
for so in ${SOS:-variants/*.so}; do
  r=$(LWB200_LIB=$so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>&1 | tail -1)
  echo "$so $(echo $r | grep -o '"kernel_ms": [0-9.]*') $(echo $r | grep -o '"ms_per_step": [0-9.]*')"
done
