# Final bench lines + c4 ncu capture / launch list of the last build (logs gpurun_out/last_*).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/last_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/last_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/last_smoke.log
timeout 900 python bench.py > gpurun_out/last_bench_c4.log 2>&1
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/last_bench_c3.log 2>&1
timeout 1800 python tools/run_c5_full.py > gpurun_out/last_c5_full.json 2> gpurun_out/last_c5_full.err
NCU="ncu --set full --clock-control none --import-source on"
python tools/profile_step.py c4 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/last_c4_near_sym python tools/profile_step.py c4 --reps 1 > gpurun_out/last_ncu_c4.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/last_pre.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/last_c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/last_ncu_launches.log 2>&1
for f in gpurun_out/last_*.log gpurun_out/last_c5_full.json; do echo "== $f"; tail -n 2 "$f" | cut -c1-300; done
