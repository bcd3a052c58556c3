#!/bin/bash
# A/B of work_oriented builds / carveouts: KSPECS="kind:carveout:lib ..." (kind is
# informational now that k_wo_chunk is the only SpMV kernel; lib = variants/*.so)
for spec in ${KSPECS:-"c::" "f::" "f:16:" "f:0:"}; do
  IFS=: read k cv lib <<< "$spec"
  env ${cv:+LW_WO_CARVEOUT=$cv} ${lib:+LWB200_LIB=$lib} LW_WO_KERNEL=$k timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS > /tmp/ab.log 2>&1
  r=$(tail -1 /tmp/ab.log)
  echo "kernel=$k carve=$cv lib=$lib $(echo $r | grep -o '"kernel_ms": [0-9.]*') $(echo $r | grep -o '"ms_per_step": [0-9.]*')"
done
