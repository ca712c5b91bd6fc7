mkdir -p gpurun_out
run() {
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" 2>&1 | grep -A1 "spill" | grep -o "SymLaplaceILb1ELb1EEELi3ELi1ELb0[^']*', [0-9]* bytes spill stores" | head -1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/abtpt_$1.log 2>&1
  echo "$1 c4 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abtpt_$1.log) $(tail -c 300 gpurun_out/abtpt_$1.log | grep -o 'Error.*' | head -1)"
}
run base ""
run t3 "-DPWB_SYM_LAPLACE_TPT=3"
run t3m6 "-DPWB_SYM_LAPLACE_TPT=3 -DPWB_SYM_LAPLACE_MINB=6"
run t5m5 "-DPWB_SYM_LAPLACE_TPT=5 -DPWB_SYM_LAPLACE_MINB=5"
