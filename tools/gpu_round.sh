# One GPU round: GPU tests, then 1-GPU benches (logs under gpurun_out/).
set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 "$f"; done
