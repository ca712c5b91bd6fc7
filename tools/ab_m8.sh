mkdir -p gpurun_out
run() {
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" 2>&1 | grep -A1 "spill" | grep -o "SymLaplaceILb1ELb1EEELi3ELi1ELb0[^']*', [0-9]* bytes spill stores" | head -1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/abm8_$1.log 2>&1
  echo "$1 c4 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abm8_$1.log)"
}
run base ""
run m8 "-DPWB_SYM_LAPLACE_MINB=8"
run m6 "-DPWB_SYM_LAPLACE_MINB=6"
