# compute-sanitizer over the round-2 long-row changes: block-tile single-tile runs,
# warp-tile gathers, thread_mapped pipelined loop (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
T="tests/test_gpu_parity.py::test_group_tiles_long_row_runs tests/test_gpu_parity.py::test_power_law_sweep_within_tolerance"
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $T -x -q > gpurun_out/memcheck_r2b.log 2>&1; echo memcheck=$?
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest "tests/test_gpu_parity.py::test_group_tiles_long_row_runs" -x -q > gpurun_out/racecheck_r2b.log 2>&1; echo racecheck=$?
timeout 1800 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest "tests/test_gpu_parity.py::test_group_tiles_long_row_runs" -x -q > gpurun_out/synccheck_r2b.log 2>&1; echo synccheck=$?
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/*check_r2b.log
