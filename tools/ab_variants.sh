#!/bin/bash
# A/B the work_oriented kernel geometry variants built into variants/*.so
for so in variants/*.so; do
  for kind in c v; do
    r=$(LWB200_LIB=$so LW_WO_KERNEL=$kind timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"ms_per_step": [0-9.]*')
    echo "$(basename $so) kind=$kind $r"
  done
done
