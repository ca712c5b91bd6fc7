"""The C-ABI boundary: the library loads on a CPU-only box, exports every symbol
include/periwave_b200.h declares, and its host-only entry points behave like the
reference's (no GPU compute here)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "periwave_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pwb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(pw):
    L = pw.lib()
    names = declared_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), n
    assert sorted(pw.EXPORTED) == names


def test_cpp_dropin_api_exported():
    """The drop-in C++ API (include/periwave/periwave.hpp) lives in the same .so."""
    import subprocess

    lib = os.path.join(ROOT, "paper_2111_01083_b200", "libperiwave_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", lib], capture_output=True, text=True).stdout
    for sym in ("periwave::total_field(", "periwave::apply_far(", "periwave::make_periodizer(",
                "periwave::FreeSpaceEvaluator::accumulate(", "periwave::choose_path(", "periwave::nufft_type1(",
                "periwave::brute_force_far(", "periwave::periodicity_residual(", "periwave::bessel_k0("):
        assert sym in out, sym


def test_version_and_device_count(pw):
    assert b"sm_100a" in pw.lib().pwb_version()
    assert pw.device_count() >= 0


def test_error_codes_cross_the_boundary(pw):
    with pytest.raises(pw.PeriwaveError) as e:
        pw.make_unit_cell(0.0, 0.0, 1.0)
    assert e.value.code == pw.ErrorCode.NonPositiveDimension
    with pytest.raises(pw.PeriwaveError) as e:
        pw.make_unit_cell(1.0, 0.3, 1.0)  # d < |e2| for a doubly periodic cell
    assert e.value.code == pw.ErrorCode.OrientationViolation
    with pytest.raises(pw.PeriwaveError) as e:
        pw.make_unit_cell(1.0, 0.6, 1.0, pw.Periodicity.Singly)
    assert e.value.code == pw.ErrorCode.OrientationViolation
    cell = pw.make_unit_cell(1.0, 0.0, 1.0)
    with pytest.raises(pw.PeriwaveError) as e:
        pw.make_periodizer(pw.Pde.ModHelmholtz, 0.0, cell, 1e-10)
    assert e.value.code == pw.ErrorCode.MissingBeta
    with pytest.raises(pw.PeriwaveError) as e:
        pw.make_periodizer(pw.Pde.Poisson, 0.0, cell, 0.5)
    assert e.value.code == pw.ErrorCode.PrecisionOutOfRange
    with pytest.raises(pw.PeriwaveError) as e:
        pw.make_multipole_periodizer(pw.Pde.Poisson, 0.0, 5, cell, 1e-10)
    assert e.value.code == pw.ErrorCode.OrderOutOfRange


def test_unit_cell_and_near_translations(pw):
    c = pw.make_unit_cell(1.0, 0.3, 0.8)
    assert c.m0 == 2
    tr = pw.near_translations(c)
    assert len(tr) == 15 and tr[0][:2] == (-2, -1) and tr[7][:2] == (0, 0)
    assert tr[0][2] == (-2 * 1.0 + -1 * 0.3, -0.8)
    s = pw.make_unit_cell(1.0, 0.0, 1.0, pw.Periodicity.Singly)
    assert [t[:2] for t in pw.near_translations(s)] == [(-1, 0), (0, 0), (1, 0)]
    assert pw.make_unit_cell(100.0, 0.0, 1.0).m0 == 1
    assert pw.make_unit_cell(1.0, -0.9, 0.3).m0 == 3


def test_rng_matches_reference_stream(pw):
    """xorshift64* (util.hpp:83-98) restated in numpy."""
    out = pw.rng_uniform(12345, 1000)
    s = np.uint64(12345)
    want = []
    with np.errstate(over="ignore"):
        for _ in range(1000):
            s ^= s >> np.uint64(12)
            s ^= s << np.uint64(25)
            s ^= s >> np.uint64(27)
            r = s * np.uint64(0x2545F4914F6CDD1D)
            want.append(float(r >> np.uint64(11)) * 2.0 ** -53)
    assert np.array_equal(out, np.array(want))


def test_compute_without_gpu_fails_loudly(pw):
    if pw.device_count() > 0:
        pytest.skip("a GPU is present")
    cell = pw.make_unit_cell(1.0, 0.0, 1.0)
    pz = pw.make_periodizer(pw.Pde.ModHelmholtz, 1.0, cell, 1e-8)
    s = pw.ParticleSystem(sources=np.array([[0.1, 0.2]]), charges=np.array([1.0]), targets=np.array([[0.0, 0.0]]))
    with pytest.raises(pw.PeriwaveError) as e:
        pw.total_field(pz, s)
    assert e.value.status == 64  # PWB_ERR_CUDA: no silent CPU fallback
