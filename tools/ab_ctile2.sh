# A/B: more resident blocks for the Laplace tile now that shared memory allows 7.
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/ab_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/ab_$1.log)"
}
run base ""
run m7 "-DPWB_SYM_LAPLACE_MINB=7"
run m7c1 "-DPWB_SYM_LAPLACE_MINB=7 -DPWB_SYM_LAPLACE_CPT=1"
run base2 ""
