# Quick check of a screened-tile change: the screened GPU tests, the c5 slice, c2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "screened or symmetric or golden or sharded or bessel or binned or config_small" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log
echo "c5 slice: $(timeout 600 python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)"
timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 3 > gpurun_out/bench_c2.log 2>&1
echo "c2 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/bench_c2.log)"
