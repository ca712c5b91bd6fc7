# A/B of the reduced-tier log table shape on c4 (near-phase ms from bench.py).
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/ab_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/ab_$1.log)"
}
run base ""
run b7r4 "-DPWB_LOG_TAB_BITS=7 -DPWB_LOG_TAB_REPL=4"
run b7r8m5 "-DPWB_LOG_TAB_BITS=7 -DPWB_SYM_LAPLACE_MINB=5"
run b7r2 "-DPWB_LOG_TAB_BITS=7 -DPWB_LOG_TAB_REPL=2"
