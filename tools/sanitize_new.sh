# compute-sanitizer over the kernels added late in round 1: hot-x packing (inspector + packed
# SpMV), the staged group-mapped warp kernel; memcheck, racecheck and synccheck
mkdir -p gpurun_out
T="tests/test_gpu_hotx.py tests/test_gpu_parity.py::test_group_warp_staged_and_cooperative_blocks_bit_exact tests/test_gpu_parity.py::test_power_law_sweep_within_tolerance tests/test_gpu_parity.py::test_integer_bit_exact_all_schedules"
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $T -x -q > gpurun_out/memcheck_new.log 2>&1; echo memcheck=$?
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_hotx.py::test_inspector_matches_rule tests/test_gpu_parity.py::test_group_warp_staged_and_cooperative_blocks_bit_exact -x -q > gpurun_out/racecheck_new.log 2>&1; echo racecheck=$?
timeout 1800 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_hotx.py::test_inspector_matches_rule tests/test_gpu_parity.py::test_group_warp_staged_and_cooperative_blocks_bit_exact -x -q > gpurun_out/synccheck_new.log 2>&1; echo synccheck=$?
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/*check_new.log
