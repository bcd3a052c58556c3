#!/bin/bash
# One GPU session: parity tests, smoke, headline bench, ncu launch list + full capture.
TAG=${1:-val}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke=$?"
timeout 600 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench_${TAG}.log
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_launch=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-k_wo_chunk} -s 3 -c 1 \
  -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu_full=$?"
fi
# optional: SANITIZE=1 runs memcheck / racecheck / synccheck over the GPU tests
if [ -n "$SANITIZE" ]; then
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spmm.py tests/test_gpu_traversal.py tests/test_gpu_edges.py -x -q > gpurun_out/memcheck_${TAG}.log 2>&1
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "integer_bit_exact or edge_cases or spmv_fp64 or one_giant" > gpurun_out/racecheck_${TAG}.log 2>&1
timeout 1800 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "integer_bit_exact or edge_cases or one_giant" > gpurun_out/synccheck_${TAG}.log 2>&1
grep -h "SUMMARY" gpurun_out/*check_${TAG}.log
fi
