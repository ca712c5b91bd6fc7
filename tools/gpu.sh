#!/usr/bin/env bash
# One parameterised GPU driver (run on a B200 box through gpurun, from the repo root):
#
#   gpurun --timeout 2400 -- 'TAG=r2a bash tools/gpu.sh tests smoke bench:c4 ncu:c4'
#
# Every task writes gpurun_out/$TAG_<task>.log (scratch; copy what is worth keeping into
# profiles/). Tasks, in the order given:
#   tests[:EXPR]        pytest -m gpu (optionally -k EXPR)
#   smoke               __graft_entry__.smoke()
#   bench:CFG[:ARGS]    python bench.py --config CFG ARGS (ARGS: comma-separated flags)
#   ref:CFG             python bench.py --impl reference --config CFG
#   gpus:N[:CFG]        python bench.py --gpus N --dist-backend gloo --config CFG (N ranks on this box)
#   ncu:CFG[:N[:W]]     ncu --set full capture of the dominant near launch of CFG (N points; W: c5 strip width)
#   launches:CFG        ncu launch list (gpu__time_duration) of a short bench.py run
#   c5full              tools/run_c5_full.py (1e7 points, vs the golden)
#   py:SCRIPT[:ARGS]    python tools/SCRIPT ARGS
#   export:VAR=VAL      set an environment variable for the tasks after it (unset:VAR clears it)
#   ab:TU:FLAGS:CFG     rebuild translation unit csrc/cuda/TU.cu with EXTRA_NVFLAGS=FLAGS (comma-separated
#                       -D... flags; "default" = none), relink, time one warm CFG step (profile_step);
#                       the library stays in that state until the next ab task
# Each profiled command runs once without ncu first and must exit 0.
TAG=${TAG:-r2}
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "gpurun_out/${TAG}_gpu.txt" 2>&1
for task in "$@"; do
  IFS=: read -r kind a b w <<< "$task"
  log="gpurun_out/${TAG}_${kind}${a:+_$a}.log"
  case "$kind" in
    tests)
      if [ -n "$a" ]; then timeout 2400 python -m pytest tests -q -m gpu -k "$a" > "$log" 2>&1
      else timeout 2400 python -m pytest tests -q -m gpu > "$log" 2>&1; fi
      echo "pytest rc=$?" >> "$log" ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$log" 2>&1; echo "smoke rc=$?" >> "$log" ;;
    bench)
      timeout 1200 python bench.py --config "${a:-c4}" ${b//,/ } > "$log" 2>&1 ;;
    ref)
      timeout 1200 python bench.py --impl reference --config "${a:-c4}" --steps 3 --warmup 3 > "$log" 2>&1 ;;
    gpus)
      timeout 1200 python bench.py --gpus "${a:-2}" --dist-backend gloo --config "${b:-c4}" --no-cpu-baseline > "$log" 2>&1 ;;
    ncu)
      n="${b:+--n $b} ${w:+--strip $w}"
      k=near_sym; { [ "$a" = c2 ] || [ "$a" = c1 ]; } && k=near_tile
      timeout 600 python tools/profile_step.py "$a" $n --reps 1 > "$log" 2>&1 && \
        timeout 1800 $NCU -k regex:$k -c 1 -f -o "gpurun_out/${TAG}_${a}_${k}" \
          python tools/profile_step.py "$a" $n --reps 1 >> "$log" 2>&1
      echo "ncu rc=$?" >> "$log" ;;
    launches)
      timeout 900 python bench.py --config "${a:-c4}" --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > "$log" 2>&1 && \
        timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
          --log-file "gpurun_out/${TAG}_${a:-c4}_launches.csv" \
          python bench.py --config "${a:-c4}" --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 >> "$log" 2>&1
      echo "launches rc=$?" >> "$log" ;;
    c5full)
      timeout 1800 python tools/run_c5_full.py > "$log" 2>&1 ;;
    py)
      log="gpurun_out/${TAG}_py_${a%.py}${b:+_${b//[,\/ ]/_}}.log"
      timeout 1800 python "tools/$a" ${b//,/ } > "$log" 2>&1 ;;
    ab)
      flags=""; [ "$b" != default ] && flags="${b//,/ }"
      log="gpurun_out/${TAG}_ab_${a}_${b//[,=\/ ]/_}.log"
      touch "paper_2111_01083_b200/csrc/cuda/$a.cu"
      make -C paper_2111_01083_b200 -j8 EXTRA_NVFLAGS="$flags" > "$log" 2>&1 && \
        timeout 900 python tools/profile_step.py "${w:-c4}" --reps 3 >> "$log" 2>&1
      echo "ab rc=$?" >> "$log" ;;
    export)
      export "$a"; continue ;;
    unset)
      unset "$a"; continue ;;
    *) echo "unknown task $task" > "$log" ;;
  esac
done
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -n 4 "$f" | cut -c1-700; done
