#!/bin/bash
# Round profile of the §8(f) kernels + refreshed SpMV schedule sweep. Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python tools/bench_sweep.py --out gpurun_out/sweep_r1c.jsonl > gpurun_out/sweep_r1c.log 2>&1; echo "sweep=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_work -s 2 -c 1 \
  -o gpurun_out/prof_r1_spmm python tools/spmm_one.py C3 16 work_oriented > gpurun_out/ncu_spmm.log 2>&1; echo "ncu_spmm=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_relax_merge -s 8 -c 1 \
  -o gpurun_out/prof_r1_sssp python tools/bench_traversal.py --scale 22 --reps 1 --no-cpu > gpurun_out/ncu_sssp.log 2>&1; echo "ncu_sssp=$?"
