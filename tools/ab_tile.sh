mkdir -p gpurun_out
runm() {
  (cd paper_2111_01083_b200 && touch csrc/cuda/near.cu && make EXTRA_NVFLAGS="$2" > /dev/null 2>&1)
  python bench.py --config c2 --no-cpu-baseline --steps 3 > gpurun_out/abt_$1.log 2>&1
  echo "$1 c2 $(grep -o '"near_ms_per_launch": [0-9.]*' gpurun_out/abt_$1.log)"
}
runm base ""
runm t128 "-DPWB_NEAR_TILE=128"
runm t64 "-DPWB_NEAR_TILE=64"
runm t512 "-DPWB_NEAR_TILE=512"
