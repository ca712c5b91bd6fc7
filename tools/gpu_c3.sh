mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "symmetric or sharded or golden or tiers or near_and_far or stokes" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c3.log
tail -2 gpurun_out/pytest_c3.log
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 3 > gpurun_out/bench_c3.log 2>&1
grep -o '"near_ms_per_launch": [0-9.]*\|"fp64_pipe_frac": [0-9.]*' gpurun_out/bench_c3.log
