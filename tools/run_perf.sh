#!/bin/bash
# Usage: tools/run_perf.sh TAG [items...] — bench variants (+ ncu capture when NCU=1)
TAG=${1:-dev}; shift
ITEMS=${@:-0}
mkdir -p gpurun_out
for it in $ITEMS; do
  timeout 300 python bench.py --steps 30 --warmup 5 --items $it --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/bench_${TAG}_i$it.log 2>&1
  echo "items=$it: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_i$it.log) $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/bench_${TAG}_i$it.log) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_${TAG}_i$it.log)"
  tail -2 gpurun_out/bench_${TAG}_i$it.log | grep -i error
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-k_wo_chunk} -s 3 -c 1 -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/ncu_${TAG}.log 2>&1
echo ncu=$?
fi
