mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "symmetric or sharded or golden or tiers or near_and_far or stokes or split" > gpurun_out/pytest_st.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_st.log
tail -2 gpurun_out/pytest_st.log
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_stokes.cu && make EXTRA_NVFLAGS="$2" 2>&1 | grep -A1 "spill" | grep -o "SymStokesILb0ELb1EEELi3ELi3ELb1[^']*', [0-9]* bytes spill stores" | head -1)
  python bench.py --config c3 --no-cpu-baseline --steps 2 > gpurun_out/abs_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abs_$1.log)"
}
run base ""
run m4 "-DPWB_SYM_STOKES_MINB=4"
