mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_r2c.log 2>&1; echo "pytest=$?"
tail -12 gpurun_out/pytest_r2c.log
timeout 900 python bench.py > gpurun_out/bench_r2c.log 2>gpurun_out/bench_r2c.err; echo "bench=$?"
tail -1 gpurun_out/bench_r2c.log; tail -3 gpurun_out/bench_r2c.err
