mkdir -p gpurun_out
run() {
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu csrc/cuda/near_sym_stokes.cu && make EXTRA_NVFLAGS="$2" 2>&1 | grep -A1 "spill" | grep -o "SymLaplaceILb1ELb1EEELi3ELi1ELb0[^']*', [0-9]* bytes spill stores" | head -1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/abk_$1.log 2>&1
  python bench.py --config c3 --no-cpu-baseline --steps 2 > gpurun_out/abk3_$1.log 2>&1
  echo "$1 c4 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abk_$1.log) c3 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abk3_$1.log)"
}
run base ""
run keep "-DPWB_SYM_KEEP_SMEM=1"
