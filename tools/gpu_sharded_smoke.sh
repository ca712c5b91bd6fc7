# The multi-GPU code path of bench.py (NCCL group, sharded passes, collectives) at world size 1.
mkdir -p gpurun_out
for c in c4 c2 c3; do
  PWB_BENCH_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/sharded_$c.log 2>&1
  echo "$c rc=$?"
done
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ref_arm.log 2>&1; echo "ref rc=$?"
for f in gpurun_out/sharded_*.log gpurun_out/ref_arm.log; do echo "== $f"; tail -n 2 $f | cut -c1-700; done
