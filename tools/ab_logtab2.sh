mkdir -p gpurun_out
run() {
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/abl_$1.log 2>&1
  echo "$1 c4 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abl_$1.log)"
}
run base ""
run b8r4 "-DPWB_LOG_TAB_BITS=8 -DPWB_SYM_LAPLACE_REPL=4"
run b8r8 "-DPWB_LOG_TAB_BITS=8"
