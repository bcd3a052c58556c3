#!/bin/bash
# A/B of work_oriented library builds / shared-memory carveouts:
#   SPECS="carveout:lib ..."  (empty carveout = driver default; lib = variants/*.so)
for spec in ${SPECS:-":" "16:" "0:"}; do
  IFS=: read cv lib <<< "$spec"
  env ${cv:+LW_WO_CARVEOUT=$cv} ${lib:+LWB200_LIB=$lib} timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS > /tmp/ab.log 2>&1
  r=$(tail -1 /tmp/ab.log)
  echo "carve=$cv lib=$lib $(echo $r | grep -o '"kernel_ms": [0-9.]*') $(echo $r | grep -o '"ms_per_step": [0-9.]*')"
done
