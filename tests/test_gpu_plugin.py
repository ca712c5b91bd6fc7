"""The reference's own total_field with the B200 near field plugged in through its
documented override point, FreeSpaceEvaluator::accumulate (proj/include/periwave/
apply.hpp:36-45; include/periwave_b200_plugin.hpp). The compiled program
(oracle/plugin/test_plugin.cpp, built against the reference's headers and library) checks
c1- and c2-shaped systems and Stokes with pressure against the stock evaluator (<= 1e-13
relative in the full precision tier, one accumulate call per near image, the reference's Counting pattern in
proj/tests/test_apply.cpp:337-357), the empty system, coincidence and length errors."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "test_plugin")


@pytest.mark.parametrize("tier", ["full", "default"])
def test_reference_total_field_with_the_b200_near_plugin(gpu, tier):
    """full: PWB_FULL_PRECISION=1, agreement <= 1e-13; default: the product's own precision
    tier for the periodizer's eps, agreement <= 1e-2 eps."""
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_plugin not built (needs /root/reference at build time)")
    env = dict(os.environ)
    if tier == "full":
        env["PWB_FULL_PRECISION"] = "1"
    r = subprocess.run([BIN] + (["full"] if tier == "full" else []), capture_output=True, text=True, timeout=600,
                       env=env)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    cases = {c["case"]: c for c in lines if "case" in c}
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert set(cases) >= {"c1_poisson_self", "c2_modhelm_skewed", "stokes_pressure_singly", "empty_targets",
                          "coincident_plugin", "coincident_stock", "length_mismatch"}
    assert all(c["ok"] for c in cases.values())
    assert cases["c2_modhelm_skewed"]["calls"] == 15 and cases["c1_poisson_self"]["calls"] == 9
