# A/B: 7-8 resident blocks for the Laplace tile with 128-point column tiles.
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" 2>&1 | grep -o "spill[^']*" | head -2)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/ab_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/ab_$1.log)"
}
run m7c1 "-DPWB_SYM_LAPLACE_MINB=7 -DPWB_SYM_LAPLACE_CPT=1"
run m8c1 "-DPWB_SYM_LAPLACE_MINB=8 -DPWB_SYM_LAPLACE_CPT=1"
run m8c1r4 "-DPWB_SYM_LAPLACE_MINB=8 -DPWB_SYM_LAPLACE_CPT=1 -DPWB_SYM_LAPLACE_REPL=4"
run m7c1u2 "-DPWB_SYM_LAPLACE_MINB=7 -DPWB_SYM_LAPLACE_CPT=1 -DPWB_SYM_LAPLACE_UNROLL=2"
run m7c1u8 "-DPWB_SYM_LAPLACE_MINB=7 -DPWB_SYM_LAPLACE_CPT=1 -DPWB_SYM_LAPLACE_UNROLL=8"
