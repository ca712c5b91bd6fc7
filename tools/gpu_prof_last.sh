mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
python tools/profile_step.py c2 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_tile -c 1 -f -o gpurun_out/r1h_c2_near_tile python tools/profile_step.py c2 --reps 1 > gpurun_out/r1h_ncu_c2.log 2>&1
python tools/profile_step.py c3 --n 300000 --reps 1 > /dev/null 2>&1 && \
  $NCU -k regex:near_sym -c 1 -f -o gpurun_out/r1h_c3_near_sym python tools/profile_step.py c3 --n 300000 --reps 1 > gpurun_out/r1h_ncu_c3.log 2>&1
ls gpurun_out | grep r1h
