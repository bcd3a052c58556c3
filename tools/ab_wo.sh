#!/bin/bash
# A/B the work_oriented SpMV kernel variants (LW_WO_KERNEL) and carveouts on C3.
mkdir -p gpurun_out
TAG=${TAG:-ab}
if [ -z "$NO_TEST" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_${TAG}.log
fi
for spec in ${SPECS:-"c:" "l:" "l:25" "l:50" "l:0"}; do
  k=${spec%%:*}; cv=${spec#*:}
  if [ -n "$cv" ]; then export LW_WO_CARVEOUT=$cv; else unset LW_WO_CARVEOUT; fi
  r=$(LW_WO_KERNEL=$k timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>&1 | tail -1)
  echo "kernel=$k carve=$cv $(echo $r | grep -o '"ms_per_step": [0-9.]*') $(echo $r | grep -o '"kernel_ms": [0-9.]*') $(echo $r | grep -o '"frac": [0-9.]*')"
done
