#!/bin/bash
# Round profile session: ncu full capture of the dominant kernel, launch list of the
# bench command, the schedule sweep, and the reference arm. Outputs in gpurun_out/.
set -x
TAG=${1:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wo_chunk -s 3 -c 1 \
  -o gpurun_out/prof_${TAG}_wo_chunk python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1200 python tools/bench_sweep.py --out gpurun_out/sweep_${TAG}.jsonl > gpurun_out/sweep_${TAG}.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_${TAG}.log 2>&1
tail -2 gpurun_out/ref_${TAG}.log
python tools/micro/run_gather_bw.py > gpurun_out/gather_ceiling_${TAG}.log 2>&1
echo done
