#!/bin/bash
# Round-2 final validation: full GPU suite, smoke, sanitizer over the changed kernels,
# launch list + ncu captures of the fp32 / fp64 headline kernels. Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2g.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/pytest_r2g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2g.log 2>&1; echo "smoke=$?"
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spmm.py -x -q -k "golden or group or vector_scale or integer or edge" > gpurun_out/memcheck_r2g.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv_fp64 or integer_bit_exact or group_general" > gpurun_out/racecheck_r2g.log 2>&1
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv_fp64 or integer_bit_exact" > gpurun_out/synccheck_r2g.log 2>&1
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/memcheck_r2g.log gpurun_out/racecheck_r2g.log gpurun_out/synccheck_r2g.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2g.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-power > /dev/null 2>&1; echo "launches=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wo_chunk -s 3 -c 1 \
  -o gpurun_out/prof_r2g_wo_chunk python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-fp64 --no-power > gpurun_out/ncu_r2g.log 2>&1; echo "ncu32=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wo_chunk64 -s 3 -c 1 \
  -o gpurun_out/prof_r2g_wo_chunk64 python bench.py --dtype fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-fp64 --no-power > gpurun_out/ncu64_r2g.log 2>&1; echo "ncu64=$?"
for f in gpurun_out/prof_r2g_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
