# Balanced multi-GPU split: tests, then the per-rank times of count vs cost split (one GPU).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sharded.py -q > gpurun_out/split_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/split_pytest.log
tail -3 gpurun_out/split_pytest.log
true
timeout 900 python tools/shard_balance.py c5 --n 1000000 > gpurun_out/balance_c5_cost.log 2>&1
true
cat gpurun_out/balance_*.log | cut -c1-400
