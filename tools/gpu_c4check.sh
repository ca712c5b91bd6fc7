mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_c4c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c4c.log
tail -2 gpurun_out/pytest_c4c.log
timeout 900 python bench.py > gpurun_out/bench_c4c.log 2>&1
tail -1 gpurun_out/bench_c4c.log | cut -c1-300
grep -o '"near_ms_per_launch": [0-9.]*\|"fp64_pipe_frac": [0-9.]*\|"ms_per_step": [0-9.]*' gpurun_out/bench_c4c.log
