# Session check after the table-log / table-exp / image-mask changes: GPU tests, the
# N=1e6 bench lines, c2, a c5 slice, then one full-size c5 total_field (logs in gpurun_out/).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
grep -o '"near_ms_per_launch": [0-9.]*\|"ms_per_step": [0-9.]*\|"fp64_pipe_frac": [0-9.]*' gpurun_out/bench_c*.log
echo "c5 slice: $(timeout 600 python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)"
timeout 1800 python tools/run_c5_full.py > gpurun_out/c5_full.json 2> gpurun_out/c5_full.err
cat gpurun_out/c5_full.json
