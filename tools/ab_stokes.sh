# A/B of the Stokeslet tile shape on c3 (near-phase ms).
mkdir -p gpurun_out
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_stokes.cu && make EXTRA_NVFLAGS="$2" 2>&1 | grep -A1 "spill" | grep -o "SymStokesILb0ELb1EEELi3ELi3ELb1[^']*', [0-9]* bytes spill stores" | head -1)
  python bench.py --config c3 --no-cpu-baseline --steps 2 > gpurun_out/abs_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abs_$1.log)"
}
run base ""
run t1 "-DPWB_SYM_STOKES_TPT=1 -DPWB_SYM_STOKES_CPT=1"
run t1m5 "-DPWB_SYM_STOKES_TPT=1 -DPWB_SYM_STOKES_CPT=1 -DPWB_SYM_STOKES_MINB=5"
