mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_integration_binding.py tests/test_reference_contract.py tests/test_bench_launch.py -m gpu -x -q --durations=15 > gpurun_out/pytest_r2b.log 2>&1; echo "pytest=$?"
tail -25 gpurun_out/pytest_r2b.log
timeout 900 python bench.py > gpurun_out/bench_r2b.log 2>gpurun_out/bench_r2b.err; echo "bench=$?"
tail -1 gpurun_out/bench_r2b.log
timeout 600 python bench.py --impl reference > gpurun_out/ref_r2b.log 2>&1; echo "ref=$?"
tail -1 gpurun_out/ref_r2b.log
