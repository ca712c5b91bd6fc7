# Last shape A/B: Laplace tile unroll / TPT at 128-point column tiles; one-sided screened TPT / unroll.
mkdir -p gpurun_out
runl() {
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/abf_$1.log 2>&1
  echo "$1 c4 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abf_$1.log)"
}
runm() {
  (cd paper_2111_01083_b200 && touch csrc/cuda/near.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --config c2 --no-cpu-baseline --steps 3 > gpurun_out/abf_$1.log 2>&1
  echo "$1 c2 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abf_$1.log)"
}
runl base ""
runl u2 "-DPWB_SYM_LAPLACE_UNROLL=2"
runl u8 "-DPWB_SYM_LAPLACE_UNROLL=8"
runl t2m8 "-DPWB_SYM_LAPLACE_TPT=2 -DPWB_SYM_LAPLACE_MINB=8"
(cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make > /dev/null 2>&1)
runm base ""
runm t2 "-DPWB_MH_TPT=2"
runm u2 "-DPWB_MH_SRC_UNROLL=2"
runm u8 "-DPWB_MH_SRC_UNROLL=8"
