# Screened (modified Helmholtz) tiles after a change: parity, c2 bench line, c5 slice
# with and without the per-tile image mask (logs under gpurun_out/).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 3 > gpurun_out/bench_c2.log 2>&1
echo "c2 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/bench_c2.log)"
echo "c5 slice cull: $(timeout 600 python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)"
echo "c5 slice no cull: $(PWB_NO_CULL=1 timeout 600 python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)"
