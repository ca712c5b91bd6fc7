# A/B of the Laplace tile's column tile / log-table replicas on c4 (near-phase ms).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "symmetric or sharded or golden or tiers or split" > gpurun_out/pytest_ct.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ct.log
tail -2 gpurun_out/pytest_ct.log
run() {  # $1 label, $2 flags
  (cd paper_2111_01083_b200 && touch csrc/cuda/near_sym_laplace.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --no-cpu-baseline --steps 3 > gpurun_out/ab_$1.log 2>&1
  echo "$1 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/ab_$1.log)"
}
run c2r8 ""
run c4r4 "-DPWB_SYM_LAPLACE_CPT=4 -DPWB_SYM_LAPLACE_REPL=4"
run c2r4 "-DPWB_SYM_LAPLACE_REPL=4"
run c2r8u2 "-DPWB_SYM_LAPLACE_UNROLL=2"
run c1r8 "-DPWB_SYM_LAPLACE_CPT=1"
