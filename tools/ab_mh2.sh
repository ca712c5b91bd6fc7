# A/B: code size of the screened sweeps (per-pair-dispatch unroll, near-regime sweep).
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near.cu csrc/cuda/near_sym_modhelm.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --config c2 --no-cpu-baseline --steps 3 > gpurun_out/abmh2_$1.log 2>&1
  echo "$1 c2 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abmh2_$1.log)  c5 $(python tools/sort_experiment.py c5 --n 200000 --reps 2 | tail -1)"
}
run base ""
run g1 "-DPWB_MH_GEN_UNROLL=1 -DPWB_SYM_MH_GEN_UNROLL=1"
run g2 "-DPWB_MH_GEN_UNROLL=2 -DPWB_SYM_MH_GEN_UNROLL=2"
run g1n0 "-DPWB_MH_GEN_UNROLL=1 -DPWB_SYM_MH_GEN_UNROLL=1 -DPWB_MH_NEAR_SWEEP=0"
