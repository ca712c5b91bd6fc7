"""Accelerated (NUFFT) far field on the GPU: the transforms themselves and both
accelerated sweeps of apply_far, against the reference's contracts
(proj/tests/test_nufft.cpp:99-169, proj/tests/test_apply.cpp:250-335,
proj/tests/acceptance.cpp:237-306: Direct vs Accelerated within 10 eps)."""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _cell(pw, c):
    return pw.make_unit_cell(c[0], c[1], c[2], pw.Periodicity(int(c[3])))


def test_transforms_meet_requested_accuracy(pw, gpu, port):
    rng = np.random.default_rng(11)
    for npts, nmodes in ((200, 128), (900, 512), (3000, 4096), (512, 513), (1, 7)):
        x = rng.uniform(-np.pi, np.pi, npts)
        c = rng.uniform(-1, 1, npts) + 1j * rng.uniform(-1, 1, npts)
        for eps in (1e-6, 1e-12):
            exact = port.nufft_type1(x, c, nmodes)
            fast = pw.nufft_type1(pw.NufftBackend.Accelerated, eps, x, c, nmodes)
            assert np.max(np.abs(fast - exact)) <= eps * np.abs(c).sum()
            ref = pw.nufft_type1(pw.NufftBackend.Reference, eps, x, c, nmodes)
            assert np.max(np.abs(ref - exact)) <= 1e-12 * np.abs(c).sum()
            f = rng.uniform(-1, 1, nmodes) + 1j * rng.uniform(-1, 1, nmodes)
            exact2 = port.nufft_type2(x, f)
            fast2 = pw.nufft_type2(pw.NufftBackend.Accelerated, eps, x, f)
            assert np.max(np.abs(fast2 - exact2)) <= eps * np.abs(f).sum()
    x = rng.uniform(-0.7, 0.7, 400)
    c = rng.uniform(-1, 1, 400) + 1j * rng.uniform(-1, 1, 400)
    s = np.concatenate([[-17.25, -3.0, 0.0, 0.5, 9.75, 120.0], rng.uniform(-40, 40, 200)])
    exact3 = port.nufft_type3(x, c, s)
    for eps in (1e-6, 1e-10):
        fast3 = pw.nufft_type3(pw.NufftBackend.Accelerated, eps, x, c, s)
        assert np.max(np.abs(fast3 - exact3)) <= eps * np.abs(c).sum()
    # degenerate extents: every output is sum c (nufft_fast.cpp:498-503)
    z = pw.nufft_type3(pw.NufftBackend.Accelerated, 1e-8, np.zeros(5), np.ones(5), np.array([1.0, 2.0]))
    assert np.allclose(z, 5.0)


VERT_CASES = [  # test_apply.cpp:265-275
    ((1.0, 0.0, 1.0, 2), 1, 1.0, 1e-12, 1e-11, False),
    ((1.0, 0.0, 1.0, 2), 1, 1.0, 1e-6, 1e-5, False),
    ((1.0, 0.0, 1.0 / 12.0, 2), 1, 1.0, 1e-12, 1e-11, False),
    ((1.0, 0.35, 0.8, 2), 1, 2.0, 1e-10, 1e-9, False),
    ((1.0, 0.0, 1.0, 2), 0, 0.0, 1e-12, 1e-11, True),
    ((100.0, 0.0, 1.0, 2), 1, 1.0, 1e-8, 1e-7, False),  # c5 cell
]


def _scalar_system(rng, cell, ns, nt, neutral):
    d, xi, eta = cell[:3]

    def pts(n):
        a, b = rng.uniform(-0.45, 0.45, n), rng.uniform(-0.45, 0.45, n)
        return np.ascontiguousarray(np.stack([a * d + b * xi, b * eta], 1))

    q = rng.uniform(-1, 1, ns)
    if neutral:
        q -= q.mean()
    return pts(ns), pts(nt), np.ascontiguousarray(q)


@pytest.mark.parametrize("case", VERT_CASES, ids=lambda c: f"{c[0]}-{c[1]}-{c[3]}")
def test_vertical_accelerated_matches_direct_and_reference(pw, gpu, ref, case):
    cell, pde, beta, eps, tol, neutral = case
    rng = np.random.default_rng(206)
    src, tgt, q = _scalar_system(rng, cell, 600, 400, neutral)
    pz = pw.make_periodizer(pw.Pde(pde), beta, _cell(pw, cell), eps)
    sysd = pw.ParticleSystem(sources=src, charges=q, targets=tgt)
    fd = pw.apply_far(pz, sysd, pw.ApplyOptions(path=pw.ApplyPath.Direct))
    fa = pw.apply_far(pz, sysd, pw.ApplyOptions(path=pw.ApplyPath.Accelerated))
    assert not fd.accelerated and fa.accelerated
    gauge = pde == 0
    assert rel_l2(fa.scalar, fd.scalar, gauge) <= tol
    R = ref.make_periodizer(pde, beta, cell, eps)
    ra = R.apply(1, src, tgt, charges=q, path=2, threads=8)
    assert ra["accelerated"]
    assert rel_l2(fa.scalar, ra["scalar"], gauge) <= tol


def test_horizontal_type3_matches_direct_and_reference(pw, gpu, ref):
    """test_apply.cpp:310-335: singly periodic strips accelerate through the type-3 transform."""
    rng = np.random.default_rng(207)
    strip = (1.0, 0.0, 2.5, 1)
    src, tgt, q = _scalar_system(rng, strip, 500, 300, False)
    pz = pw.make_periodizer(pw.Pde.ModHelmholtz, 1.0, _cell(pw, strip), 1e-10)
    sysd = pw.ParticleSystem(sources=src, charges=q, targets=tgt)
    fd = pw.apply_far(pz, sysd, pw.ApplyOptions(path=pw.ApplyPath.Direct))
    fa = pw.apply_far(pz, sysd, pw.ApplyOptions(path=pw.ApplyPath.Accelerated))
    assert fa.accelerated and not fd.accelerated
    assert rel_l2(fa.scalar, fd.scalar) <= 1e-9
    R = ref.make_periodizer(1, 1.0, strip, 1e-10)
    assert rel_l2(fa.scalar, R.apply(1, src, tgt, charges=q, path=2, threads=8)["scalar"]) <= 1e-9
    # log kernel: agreement modulo the additive constant (test_apply.cpp:325-334)
    src, tgt, q = _scalar_system(rng, strip, 500, 300, True)
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, _cell(pw, strip), 1e-9)
    sysd = pw.ParticleSystem(sources=src, charges=q, targets=tgt)
    pd = pw.apply_far(pz, sysd, pw.ApplyOptions(path=pw.ApplyPath.Direct)).scalar
    pa = pw.apply_far(pz, sysd, pw.ApplyOptions(path=pw.ApplyPath.Accelerated)).scalar
    d = (pd - pd.mean()) - (pa - pa.mean())
    assert np.max(np.abs(d)) <= 1e-8 * max(np.abs(pd).max(), np.abs(pa).max())


def test_choose_path_matches_reference(pw, gpu, ref):
    assert pw.fast_nufft_available()
    for cell, pde, beta, eps, sizes in (((1.0, 0.0, 1.0, 2), 1, 1.0, 1e-6, [(100000, 100000)]),
                                        ((1.0, 0.0, 1.0 / 30.0, 2), 1, 1.0, 1e-12,
                                         [(3000, 2000), (2000, 2000), (3000, 1097)]),
                                        ((1.0, 0.0, 1.0 / 30.0, 2), 2, 0.0, 1e-6, [(100000, 100000)]),
                                        ((1.0, 0.0, 1.0, 1), 0, 0.0, 1e-10, [(1000000, 1000000), (2048, 2048)]),
                                        ((100.0, 0.0, 1.0, 2), 1, 1.0, 1e-8, [(10000000, 10000000)])):
        pz = pw.make_periodizer(pw.Pde(pde), beta, _cell(pw, cell), eps)
        R = ref.make_periodizer(pde, beta, cell, eps)
        for ns, nt in sizes:
            assert int(pw.choose_path(pz, ns, nt)) == R.choose_path(ns, nt), (cell, pde, ns, nt)


@pytest.mark.parametrize("name,n", [("c4", 20000), ("c5", 20000)])
def test_auto_path_of_the_accelerated_configs(pw, gpu, ref, name, n):
    """c4 (type 3) and c5 (type 1/2) resolve Auto to Accelerated, as upstream."""
    from paper_2111_01083_b200 import configs

    inp = configs.generate(name, n_src=n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, _cell(pw, c.cell), c.eps)
    tgt = np.ascontiguousarray(inp.targets[inp.sample[:300]])
    got = pw.total_field(pz, pw.ParticleSystem(sources=inp.sources, charges=inp.charges, targets=tgt))
    assert got.accelerated
    R = ref.make_periodizer(int(c.pde), c.beta, tuple(float(v) for v in c.cell[:3]) + (int(c.cell[3]),), c.eps)
    want = R.apply(0, inp.sources, tgt, charges=inp.charges, path=1, threads=8)["scalar"]
    assert rel_l2(got.scalar, want, c.pde == pw.Pde.Poisson) <= 10 * c.eps
