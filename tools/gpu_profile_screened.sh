# ncu captures of the screened tiles (c5 slice symmetric, c2 one-sided at full size) with
# source-level counters (TAG names the set), plus the sharded c5-slice smoke at world size 1.
set -x
TAG=${TAG:-r1c}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python tools/profile_step.py c5 --n 100000 --reps 1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/${TAG}_c5_near_sym python tools/profile_step.py c5 --n 100000 --reps 1 > gpurun_out/ncu_c5.log 2>&1
python tools/profile_step.py c2 --reps 1 && \
  $NCU -k regex:near_tile -c 1 -f -o gpurun_out/${TAG}_c2_near_tile python tools/profile_step.py c2 --reps 1 > gpurun_out/ncu_c2.log 2>&1
ls -la gpurun_out | grep $TAG
