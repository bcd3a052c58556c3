#!/bin/bash
# A/B the headline bench across variants/*.so (3 runs each, ms per SpMV)
for so in variants/*.so; do
  r=""
  for i in 1 2 3; do
    r="$r $(LWB200_LIB=$so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>&1 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2)"
  done
  echo "$(basename $so) $r"
done
