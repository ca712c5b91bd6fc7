# A/B of the Laplace symmetric tile shape on c4 (near-phase ms from bench.py).
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/ab_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/ab_$1.log)"
}
run base ""
run m5 "-DPWB_SYM_LAPLACE_MINB=5"
run u2 "-DPWB_SYM_LAPLACE_UNROLL=2"
run u8 "-DPWB_SYM_LAPLACE_UNROLL=8"
run t2m8 "-DPWB_SYM_LAPLACE_TPT=2 -DPWB_SYM_LAPLACE_MINB=8"
run t2m7 "-DPWB_SYM_LAPLACE_TPT=2 -DPWB_SYM_LAPLACE_MINB=7"
run t2m8u8 "-DPWB_SYM_LAPLACE_TPT=2 -DPWB_SYM_LAPLACE_MINB=8 -DPWB_SYM_LAPLACE_UNROLL=8"
