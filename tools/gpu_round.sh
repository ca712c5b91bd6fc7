# One GPU round: GPU tests, then 1-GPU benches (logs under gpurun_out/).
set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
for c in c2 c3; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
PWB_FULL_PRECISION=1 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2_full.log 2>&1
python tools/sort_experiment.py c5 --n 200000 > gpurun_out/sort_c5.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 "$f" | cut -c1-400; done
