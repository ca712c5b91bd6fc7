"""bench.py's contract pieces that run without a GPU: the multi-GPU launcher refuses what
it cannot honour, both arms carry the same config, the roofline is an executed-work
fraction (<= 1) reproducible from the committed ncu capture."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=300)


def test_gpus_without_enough_devices_fails_loudly():
    r = _bench("--gpus", "2", env={"CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2 and "needs 2 visible GPUs" in r.stderr


def test_launcher_world_size_must_match_gpus():
    r = _bench("--gpus", "1", env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode == 2 and "launcher started 2 ranks" in r.stderr


def test_both_arms_share_the_config(pw):
    import bench
    import workloads
    from oracle import pyoracle
    from paper_2111_01083_b200 import configs

    for name in ("c1", "c4"):
        ours = configs.generate(name, n_src=2000)
        theirs = workloads.generate(name, n_src=2000, rng=pyoracle.rng_uniform)
        assert bench.bench_config(name, ours) == bench.bench_config(name, theirs)


def test_roofline_is_an_executed_work_fraction():
    import bench

    with open(bench.WORK_MODEL) as f:
        m = json.load(f)["c4"]
    # the capture's own launch: achieved = executed fp64 flops / its duration
    r = bench.roofline("c4", m["n_src"], m["n_tgt"], True, 1, m["launch_ms"], 36.46, 3)
    assert r["achieved"] == pytest.approx(m["fp64_flops_per_launch"] / (m["launch_ms"] * 1e-3) / 1e12)
    assert 0.0 < r["frac"] <= 1.0 and 0.0 < r["fp64_pipe_frac"] <= 1.0
    assert r["model_speedup"] > 1.0  # the survey's model charge, reported apart
    assert r["traffic"] == m["dram_bytes_per_launch"]
    # sharded: each of W ranks evaluates 1/W of the pair-groups in (about) 1/W of the time
    r4 = bench.roofline("c4", m["n_src"], m["n_tgt"], True, 4, m["launch_ms"] / 4, 36.46, 3)
    assert r4["frac"] == pytest.approx(r["frac"]) and r4["traffic"] is None
    # a kernel without a capture reports no roofline instead of a model number
    assert bench.roofline("c4", 1000, 1000, False, 1, 1.0, 36.46, 3)["frac"] is None
