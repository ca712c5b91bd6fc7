# A/B of the screened tiles' sweep shape: c2 (one-sided) and a c5 slice (symmetric).
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near.cu csrc/cuda/near_sym_modhelm.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --config c2 --no-cpu-baseline --steps 3 > gpurun_out/abmh_$1.log 2>&1
  echo "$1 c2 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abmh_$1.log)"
  echo "$1 c5 $(python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)"
}
run base ""
run u1 "-DPWB_MH_SRC_UNROLL=1 -DPWB_SYM_MH_SRC_UNROLL=1"
run u4 "-DPWB_MH_SRC_UNROLL=4 -DPWB_SYM_MH_SRC_UNROLL=4"
run t2 "-DPWB_MH_TPT=2 -DPWB_SYM_MH_TPT=4"
run t2u1 "-DPWB_MH_TPT=2 -DPWB_SYM_MH_TPT=4 -DPWB_MH_SRC_UNROLL=1 -DPWB_SYM_MH_SRC_UNROLL=1"
