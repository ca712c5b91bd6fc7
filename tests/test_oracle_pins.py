"""Pin the CPU checkers before trusting them (CPU only).

* the compiled reference (oracle/_ref) with the own GSL/FFTW shims reproduces the
  reference test-suite's known answers (proj/tests/test_kernels.cpp, test_nufft.cpp);
* the fast Bessel shim agrees with std::cyl_bessel_k (the accuracy shim);
* the C restatement (oracle/port) agrees with the compiled reference on the near
  images, the far contractions and the exact NUFFT sums;
* the committed golden fixtures are reproducible.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, rel_l2


def test_reference_bessel_known_answers(ref, port):
    # proj/tests/test_kernels.cpp:28-48
    for impl in (ref, port):
        assert abs(impl.bessel_kn(0, 1.0) - 0.42102443824070833) <= 1e-14 * 0.421
        assert abs(impl.bessel_kn(1, 1.0) - 0.60190723019723457) <= 1e-14 * 0.602
        assert abs(impl.bessel_kn(2, 1.3) - 0.85139763957996879) <= 1e-14 * 0.851
        assert abs(impl.bessel_kn(3, 0.55) - 46.328915013455511) <= 1e-14 * 46.33
        for l in range(1, 6):
            lhs = impl.bessel_kn(l + 1, 0.8)
            rhs = impl.bessel_kn(l - 1, 0.8) + (2.0 * l / 0.8) * impl.bessel_kn(l, 0.8)
            assert abs(lhs - rhs) <= 1e-13 * abs(rhs)
        assert impl.bessel_kn(0, 800.0) == 0.0 and impl.bessel_kn(1, 800.0) == 0.0


def test_fast_shim_matches_accuracy_shim():
    code = ("import sys, numpy as np; sys.path.insert(0, %r); from oracle.pyoracle import Ref; r = Ref(); "
            "xs = np.concatenate([np.geomspace(1e-4, 2, 60), np.geomspace(2.01, 600, 200)]); "
            "print(' '.join(repr(float(r.bessel_kn(l, x))) for l in (0, 1, 2) for x in xs))") % ROOT
    vals = {}
    for mode in ("fast", "accurate"):
        env = dict(os.environ, ORACLE_BESSEL=mode)
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, check=True)
        vals[mode] = np.array([float(v) for v in out.stdout.split()])
    rel = np.abs(vals["fast"] - vals["accurate"]) / vals["accurate"]
    assert rel.max() <= 2e-15, rel.max()


def test_reference_kernel_known_answers(ref):
    # proj/tests/test_kernels.cpp:50-171
    assert abs(ref.greens_scalar(0, 0.0, (0.3, 0.4)) - 0.1103178000763258) <= 1e-14
    assert abs(ref.greens_scalar(1, 2.5, (0.3, 0.4)) - 0.047365002707153135) <= 1e-14
    g = ref.greens_block(2, 0.0, (0.3, -0.4))
    assert np.allclose(g, [0.083806789794704059, -0.038197186342054881, -0.038197186342054881,
                           0.10608848182756941], rtol=1e-14, atol=0)
    g = ref.greens_block(3, 1.3, (0.7, 0.4))
    assert np.allclose(g[[0, 1, 3]], [0.046161086481584479, 0.025233352638660489, 0.016421778014591761],
                       rtol=1e-13, atol=0)
    g = ref.greens_block(3, 1.3, (0.05, -0.03))
    assert np.allclose(g[[0, 1, 3]], [0.23355962920866488, -0.034933841604551148, 0.19629686483047698],
                       rtol=1e-13, atol=0)
    mh = ref.multipole_kernel(1, 1.1, 3, (0.3, 0.4))
    assert abs(mh - (-43.363864452594358 + 16.30777808473634j)) <= 1e-13 * abs(mh)


def test_host_api_kernels_match_reference(pw, ref):
    """The product's host-side periwave::bessel_k* (same series/polynomials as the
    device tiles, exact host seeds) through pwb-free C++ symbols is exercised via
    the periodizer builders; here its Bessel values are checked via ctypes."""
    import ctypes

    L = ctypes.CDLL(pw.LIB_PATH)
    fn = getattr(L, "_ZN8periwave9bessel_k0Ed")
    fn.restype = ctypes.c_double
    fn.argtypes = [ctypes.c_double]
    for x in (1e-6, 0.3, 1.0, 1.99, 2.0, 2.01, 7.5, 40.0, 300.0):
        want = ref.bessel_kn(0, x)
        assert abs(fn(x) - want) <= (4e-15 + 3e-16 * x) * want


NEAR_CASES = [  # (port kind, pde, beta, order, cell, strength)
    ("LAPLACE", 0, 0.0, 0, (1.0, 0.3, 0.8, 2), "charge"),
    ("LAPLACE", 0, 0.0, 0, (1.0, 0.0, 1.5, 1), "charge"),
    ("MODHELM", 1, 3.0, 0, (1.0, 0.6, 0.7, 2), "charge"),
    ("STOKES", 2, 0.0, 0, (1.0, 0.0, 1.0, 2), "force"),
    ("MODSTOKES", 3, 1.4, 0, (1.0, 0.2, 0.9, 2), "force"),
]


def _pts(rng, cell, n):
    d, xi, eta = cell[:3]
    a, b = rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n)
    return np.ascontiguousarray(np.stack([a * d + b * xi, b * eta], 1))


@pytest.mark.parametrize("case", NEAR_CASES, ids=lambda c: f"{c[0]}-{c[4][3]}")
def test_port_near_matches_reference(ref, port, case):
    from oracle.pyoracle import near_shifts

    kind, pde, beta, order, cell, strength = case
    rng = np.random.default_rng(42)
    src, tgt = _pts(rng, cell, 300), _pts(rng, cell, 120)
    tgt[:10] = src[:10]  # self pairs exercise the identity-image skip
    q = rng.uniform(-1, 1, 300)
    f = rng.uniform(-1, 1, (300, 2))
    if pde in (0, 2):
        q -= q.mean()
        f -= f.mean(axis=0)
    R = ref.make_periodizer(pde, beta, cell, 1e-10)
    kw = dict(charges=q) if strength == "charge" else dict(forces=np.ascontiguousarray(f))
    want = R.apply(2, src, tgt, path=1, with_pressure=strength == "force", **kw)
    shifts, ident = near_shifts(cell)
    got, coinc = port.near(getattr(port, kind), src, tgt, shifts, ident, q=q, vec=f, beta=beta, order=order,
                           with_pressure=strength == "force", threads=3)
    assert not coinc
    if strength == "charge":
        assert rel_l2(got[:, 0], want["scalar"]) <= 1e-13
    else:
        assert rel_l2(got[:, :2], want["velocity"]) <= 1e-13
        assert rel_l2(got[:, 2], want["pressure"]) <= 1e-13


def test_port_far_matches_reference(pw, ref, port):
    rng = np.random.default_rng(7)
    for pde, beta, cell, eps, strength in ((1, 2.0, (1.0, 0.3, 0.8, 2), 1e-10, "charge"),
                                          (0, 0.0, (1.0, 0.0, 1.0, 1), 1e-10, "charge"),
                                          (2, 0.0, (1.0, 0.2, 0.9, 2), 1e-8, "force")):
        src, tgt = _pts(rng, cell, 250), _pts(rng, cell, 90)
        q = rng.uniform(-1, 1, 250)
        f = rng.uniform(-1, 1, (250, 2))
        q -= q.mean()
        f -= f.mean(axis=0)
        f = np.ascontiguousarray(f)
        R = ref.make_periodizer(pde, beta, cell, eps)
        if strength == "charge":
            want = R.apply(1, src, tgt, charges=q, path=1)["scalar"]
            got = port.far(R.parts(0), src, tgt, charges=q, threads=2).scalar[:, 0]
        else:
            want = R.apply(1, src, tgt, forces=f, path=1)["velocity"]
            v = port.far(R.parts(1), src, tgt, forces=f, threads=2).velocity
            got = v[:, [0, 2]]
        assert rel_l2(got, want, gauge=pde in (0, 2)) <= 1e-12


def test_nufft_checkers(ref, port):
    rng = np.random.default_rng(11)
    x = rng.uniform(-np.pi, np.pi, 300)
    c = rng.uniform(-1, 1, 300) + 1j * rng.uniform(-1, 1, 300)
    for n in (1, 7, 64, 513):
        exact = port.nufft_type1(x, c, n)
        assert np.max(np.abs(ref.nufft_type1(0, 1e-12, x, c, n) - exact)) <= 1e-12 * np.abs(c).sum()
        assert np.max(np.abs(ref.nufft_type1(1, 1e-12, x, c, n) - exact)) <= 1e-12 * np.abs(c).sum()
        fm = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        exact2 = port.nufft_type2(x, fm)
        assert np.max(np.abs(ref.nufft_type2(1, 1e-12, x, fm) - exact2)) <= 1e-12 * np.abs(fm).sum()
    s = np.array([-17.25, -3.0, 0.0, 0.5, 9.75, 120.0])
    e3 = port.nufft_type3(x, c, s)
    assert np.max(np.abs(ref.nufft_type3(1, 1e-10, x, c, s) - e3)) <= 1e-10 * np.abs(c).sum()


def test_golden_c1_reproducible(ref):
    from paper_2111_01083_b200 import configs

    path = os.path.join(ROOT, "tests", "golden", "c1.npz")
    g = np.load(path)
    inp = configs.generate("c1")
    c = inp.config
    R = ref.make_periodizer(int(c.pde), c.beta, tuple(float(v) for v in c.cell[:3]) + (int(c.cell[3]),), c.eps)
    want = R.apply(0, inp.sources, np.ascontiguousarray(inp.targets[inp.sample]), charges=inp.charges, path=1,
                   threads=4)["scalar"]
    assert np.array_equal(g["direct"], want)


def test_golden_metadata():
    for name in ("c1", "c2", "c3", "c4", "c5"):
        p = os.path.join(ROOT, "tests", "golden", f"{name}.json")
        if not os.path.exists(p):
            continue
        meta = json.load(open(p))
        g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
        assert len(g["sample"]) == len(g["direct"])
        assert np.all(np.isfinite(g["direct"]))
        assert meta["config"] == name
