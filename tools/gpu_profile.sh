# ncu captures of the dominant near kernels + the bench launch list (run through gpurun;
# reports land in gpurun_out/). Each profiled command first runs once without ncu and
# must exit 0. TAG names the capture set (default r1b).
set -x
TAG=${TAG:-r1b}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python tools/profile_step.py c4 --reps 1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/${TAG}_c4_near_sym python tools/profile_step.py c4 --reps 1 > gpurun_out/ncu_c4.log 2>&1
python tools/profile_step.py c3 --n 300000 --reps 1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/${TAG}_c3_near_sym python tools/profile_step.py c3 --n 300000 --reps 1 > gpurun_out/ncu_c3.log 2>&1
python tools/profile_step.py c5 --n 100000 --reps 1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/${TAG}_c5_near_sym python tools/profile_step.py c5 --n 100000 --reps 1 > gpurun_out/ncu_c5.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_pre_launches.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out
