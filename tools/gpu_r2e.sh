#!/bin/bash
# full GPU suite + memcheck/racecheck over the work_oriented fp64 kernel and the scale kernel
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2e.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/pytest_r2e.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv_fp64 or integer_bit_exact or vector_scale or normalisation or edge" > gpurun_out/memcheck_r2e.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv_fp64 or integer_bit_exact" > gpurun_out/racecheck_r2e.log 2>&1
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/memcheck_r2e.log gpurun_out/racecheck_r2e.log
