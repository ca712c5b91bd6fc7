# Parity + the N=1e6 bench lines after a tile change (logs under gpurun_out/).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
for f in gpurun_out/pytest_gpu.log gpurun_out/bench_c4.log gpurun_out/bench_c3.log; do echo "== $f"; tail -n 3 "$f" | cut -c1-300; done
grep -o '"near_ms_per_launch": [0-9.]*\|"fp64_pipe_frac": [0-9.]*\|"ms_per_step": [0-9.]*' gpurun_out/bench_c*.log
