# End-of-session measurement set on one B200 (logs under gpurun_out/final_*):
# GPU tests, smoke, every config's bench line, the reference arm, a c5 slice, one full c5
# total_field, then the c4 ncu capture and the bench launch list (each after its plain run).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final_gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench_c4.log 2>&1
for c in c1 c2 c3; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/final_bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1
echo "c5 slice: $(timeout 600 python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)" > gpurun_out/final_c5_slice.log
timeout 1800 python tools/run_c5_full.py > gpurun_out/final_c5_full.json 2> gpurun_out/final_c5_full.err
NCU="ncu --set full --clock-control none --import-source on"
python tools/profile_step.py c4 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/final_c4_near_sym python tools/profile_step.py c4 --reps 1 > gpurun_out/final_ncu_c4.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_pre_launches.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_ncu_launches.log 2>&1
for f in gpurun_out/final_*.log gpurun_out/final_c5_full.json; do echo "== $f"; tail -n 2 "$f" | cut -c1-300; done
