mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_c1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c1.log
tail -2 gpurun_out/pytest_c1.log
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
grep -o '"ms_per_step": [0-9.]*\|"near_ms_per_launch": [0-9.]*\|"far_ms": [0-9.]*' gpurun_out/bench_c1.log
bash tools/gpu_c1_launches.sh | tail -18
