# Last end-of-session set (logs gpurun_out/fin3_*): tests, smoke, bench lines, reference arm,
# c5 slice + full, ncu captures of the c2 / c3-slice / c5-slice near kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin3_gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/fin3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin3_smoke.log
timeout 900 python bench.py > gpurun_out/fin3_bench_c4.log 2>&1
for c in c1 c2 c3; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/fin3_bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin3_bench_ref.log 2>&1
echo "c5 slice: $(timeout 600 python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)" > gpurun_out/fin3_c5_slice.log
timeout 1800 python tools/run_c5_full.py > gpurun_out/fin3_c5_full.json 2> gpurun_out/fin3_c5_full.err
NCU="ncu --set full --clock-control none --import-source on"
python tools/profile_step.py c2 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_tile -c 1 -f -o gpurun_out/fin3_c2_near_tile python tools/profile_step.py c2 --reps 1 > gpurun_out/fin3_ncu_c2.log 2>&1
python tools/profile_step.py c3 --n 300000 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/fin3_c3_near_sym python tools/profile_step.py c3 --n 300000 --reps 1 > gpurun_out/fin3_ncu_c3.log 2>&1
python tools/profile_step.py c5 --n 100000 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/fin3_c5_near_sym python tools/profile_step.py c5 --n 100000 --reps 1 > gpurun_out/fin3_ncu_c5.log 2>&1
for f in gpurun_out/fin3_*.log gpurun_out/fin3_c5_full.json; do echo "== $f"; tail -n 2 "$f" | cut -c1-300; done
