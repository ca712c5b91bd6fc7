# A/B of the Laplace symmetric tile shape on c4 (near-phase ms from bench.py).
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/ab_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/ab_$1.log)"
}
run base ""
run tpt2_m6 "-DPWB_SYM_LAPLACE_TPT=2"
run tpt8_m3 "-DPWB_SYM_LAPLACE_TPT=8 -DPWB_SYM_LAPLACE_MINB=3"
run tpt8_m4 "-DPWB_SYM_LAPLACE_TPT=8 -DPWB_SYM_LAPLACE_MINB=4"
run u1 "-DPWB_SYM_FAST_UNROLL=1"
run u4 "-DPWB_SYM_FAST_UNROLL=4"
run tpt4_m5 "-DPWB_SYM_LAPLACE_MINB=5"
