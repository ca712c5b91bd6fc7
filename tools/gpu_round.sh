set -x
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c4.log 2>&1
python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1
python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
(cd paper_2111_01083_b200 && touch csrc/cuda/near_sym.cu && make EXTRA_NVFLAGS=-DPWB_SYM_LAPLACE_MINB=5 > /dev/null 2>&1)
python bench.py --no-cpu-baseline > gpurun_out/bench_c4_minb5.log 2>&1
tail -3 gpurun_out/*.log
