# c4 ncu capture of the current near tile + the bench launch list (after plain runs).
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python tools/profile_step.py c4 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/r1e_c4_near_sym python tools/profile_step.py c4 --reps 1 > gpurun_out/r1e_ncu_c4.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1e_pre.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1e_c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1e_ncu_launches.log 2>&1
ls -la gpurun_out | grep r1e
