"""Product forms of the symmetric tiles (near_sym_impl.cuh SymLaplace / SymStokes PROD): binned
points scaled to period 2; Laplace on singly periodic cells takes the three images' product
in closed form, the Stokeslet on unskewed 3 x 3 image blocks takes each image row's sums
from one reciprocal -- on tile pairs that keep clear of the +-d image columns, the image
loop elsewhere. Checked against the same tiles without it (PWB_NO_PROD=1), the one-sided
full-precision tile and the compiled reference (apply.cpp:481-546)."""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _points(rng, d, n):
    """Uniform background plus clusters hugging both x faces (tile pairs close to a +-d
    image) and one in the middle."""
    k = n // 5
    parts = [np.column_stack([rng.uniform(-0.5 * d, 0.5 * d, n - 4 * k), rng.uniform(-0.5, 0.5, n - 4 * k)])]
    for cx, cy in [(-0.49 * d, 0.1), (0.49 * d, 0.1), (0.45 * d, -0.3), (0.0, 0.2)]:
        p = np.column_stack([rng.normal(cx, 0.02 * d, k), rng.normal(cy, 0.02, k)])
        p[:, 0] = np.clip(p[:, 0], -0.5 * d, 0.5 * d)
        p[:, 1] = np.clip(p[:, 1], -0.5, 0.5)
        parts.append(p)
    return np.ascontiguousarray(rng.permutation(np.vstack(parts)))


@pytest.mark.parametrize("eps", [1e-10, 1e-11])
@pytest.mark.parametrize("d", [1.0, 0.5, 4.0, 1.5, 0.3])  # powers of two: scaled points; the others: unscaled form
def test_product_form_matches_image_loop(pw, gpu, ref, monkeypatch, d, eps):
    rng = np.random.default_rng(int(d * 8) + 3)
    n = 40000
    src = _points(rng, d, n)
    q = rng.standard_normal(n)
    q -= q.mean()
    cell = pw.make_unit_cell(d, 0.0, 1.0, pw.Periodicity.Singly)
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, cell, eps)
    sys_ = pw.ParticleSystem(sources=src, targets=src, charges=q)
    prod = pw.near_field(pz, sys_).scalar
    again = pw.near_field(pz, sys_).scalar
    assert np.array_equal(prod, again)  # fixed-point sums: bitwise deterministic
    monkeypatch.setenv("PWB_NO_PROD", "1")
    loop = pw.near_field(pz, sys_).scalar
    monkeypatch.delenv("PWB_NO_PROD")
    assert not np.array_equal(prod, loop)  # the product form did run
    monkeypatch.setenv("PWB_FULL_PRECISION", "1")
    full = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src.copy(), charges=q)).scalar
    monkeypatch.delenv("PWB_FULL_PRECISION")
    e_prod, e_loop = rel_l2(prod, full), rel_l2(loop, full)
    print("d", d, "eps", eps, "prod vs full", e_prod, "image loop vs full", e_loop)
    # the tier's log budget (coarse table 9.1e-13, reduced 3e-13 absolute per pair-log)
    assert e_prod <= (2e-12 if eps >= 1e-10 else 5e-13)
    assert e_prod <= 2.0 * e_loop + 1e-13  # no worse than the image loop of the same tier
    # and the reference's near images at a target subsample
    idx = rng.choice(n, 200, replace=False)
    tg = np.ascontiguousarray(src[idx])
    R = ref.make_periodizer(int(pw.Pde.Poisson), 0.0, (d, 0.0, 1.0, int(pw.Periodicity.Singly)), eps)
    want = R.apply(2, src, tg, charges=q, threads=8)["scalar"]  # mode 2: the near images
    assert rel_l2(prod[idx], want) <= 1e-11


def test_product_form_unscaled_at_a_power_of_two(pw, gpu, monkeypatch):
    """PWB_PROD_UNSCALED=1 runs the any-period form at d = 1: the same field as the scaled
    form to the tier's accuracy."""
    rng = np.random.default_rng(5)
    n = 36000
    src = _points(rng, 1.0, n)
    q = rng.standard_normal(n)
    q -= q.mean()
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(1.0, 0.0, 1.0, pw.Periodicity.Singly), 1e-10)
    sys_ = pw.ParticleSystem(sources=src, targets=src, charges=q)
    a = pw.near_field(pz, sys_).scalar
    monkeypatch.setenv("PWB_PROD_UNSCALED", "1")
    b = pw.near_field(pz, sys_).scalar
    assert not np.array_equal(a, b)
    assert rel_l2(a, b) <= 2e-12


def test_product_form_duplicates_and_image_coincidence(pw, gpu):
    """Exact zeros keep the reference's meaning on the scaled points (apply.cpp:538-545):
    duplicates are skipped in the identity image; a point on the x face coinciding with
    another point's +-d image raises CoincidentSourceTarget."""
    rng = np.random.default_rng(17)
    n = 40000
    src = _points(rng, 1.0, n)
    src[1000:1010] = src[30000:30010]
    src[5] = src[6]
    q = rng.standard_normal(n)
    q -= q.mean()
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(1.0, 0.0, 1.0, pw.Periodicity.Singly), 1e-10)
    sym = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, charges=q)).scalar
    one = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src.copy(), charges=q)).scalar
    assert np.all(np.isfinite(sym))
    assert rel_l2(sym, one) <= 2e-12
    bad = src.copy()
    bad[7] = [-0.5, 0.25]
    bad[33333] = [0.5, 0.25]  # the +d image of point 7
    with pytest.raises(pw.PeriwaveError) as e:
        pw.near_field(pz, pw.ParticleSystem(sources=bad, targets=bad, charges=q))
    assert e.value.code == pw.ErrorCode.CoincidentSourceTarget


def test_product_form_strength_scales(pw, gpu):
    """Tiny and huge strengths: the fixed-point scale follows them, also on the
    binned, scaled path."""
    rng = np.random.default_rng(23)
    n = 36000
    src = _points(rng, 1.0, n)
    q = rng.standard_normal(n)
    q -= q.mean()
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(1.0, 0.0, 1.0, pw.Periodicity.Singly), 1e-10)
    base = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, charges=q)).scalar
    for s in (2.0 ** -50, 2.0 ** 50):
        got = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, charges=q * s)).scalar
        assert np.array_equal(got, base * s)


# ------------------------------------------------------------------ Stokeslet rows in closed form
def _points2(rng, d, eta, n):
    """Uniform background plus clusters hugging the x faces, the y faces and a corner (tile
    pairs close to images of the +-d columns in every image row)."""
    k = n // 8
    parts = [np.column_stack([rng.uniform(-0.5 * d, 0.5 * d, n - 6 * k), rng.uniform(-0.5 * eta, 0.5 * eta, n - 6 * k)])]
    for cx, cy in [(-0.49, 0.1), (0.49, 0.1), (0.47, -0.48), (-0.48, 0.47), (0.1, 0.49), (0.0, 0.0)]:
        p = np.column_stack([rng.normal(cx * d, 0.02 * d, k), rng.normal(cy * eta, 0.02 * eta, k)])
        out = (np.abs(p[:, 0]) > 0.5 * d) | (np.abs(p[:, 1]) > 0.5 * eta)  # resampled, not clipped onto a face:
        p[out] = np.column_stack([rng.uniform(-0.5 * d, 0.5 * d, out.sum()),  # two clipped corners would coincide
                                  rng.uniform(-0.5 * eta, 0.5 * eta, out.sum())])
        parts.append(p)
    return np.ascontiguousarray(rng.permutation(np.vstack(parts)))


@pytest.mark.parametrize("eps", [1e-8, 1e-11])
@pytest.mark.parametrize("d,eta", [(1.0, 1.0), (2.0, 0.7), (0.5, 0.4), (1.5, 1.0), (3.0, 2.9)])
def test_stokeslet_product_form_matches_image_loop(pw, gpu, ref, monkeypatch, d, eta, eps):
    rng = np.random.default_rng(int(d * 8) + 11)
    n = 36000
    src = _points2(rng, d, eta, n)
    f = rng.standard_normal((n, 2))
    f = np.ascontiguousarray(f - f.mean(axis=0))
    cell = pw.make_unit_cell(d, 0.0, eta)
    if cell.m0 != 1:
        pytest.skip("more than 3 x 3 images")
    pz = pw.make_periodizer(pw.Pde.Stokes, 0.0, cell, eps)
    sys_ = pw.ParticleSystem(sources=src, targets=src, forces=f)
    prod = pw.near_field(pz, sys_).velocity
    assert np.array_equal(prod, pw.near_field(pz, sys_).velocity)  # bitwise deterministic
    monkeypatch.setenv("PWB_NO_PROD", "1")
    loop = pw.near_field(pz, sys_).velocity
    monkeypatch.delenv("PWB_NO_PROD")
    assert not np.array_equal(prod, loop)  # the product form did run
    monkeypatch.setenv("PWB_FULL_PRECISION", "1")
    full = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src.copy(), forces=f)).velocity
    monkeypatch.delenv("PWB_FULL_PRECISION")
    e_prod, e_loop = rel_l2(prod, full), rel_l2(loop, full)
    print("d", d, "eta", eta, "eps", eps, "prod vs full", e_prod, "image loop vs full", e_loop)
    assert e_prod <= 2e-12
    assert e_prod <= 2.0 * e_loop + 2e-13
    idx = rng.choice(n, 200, replace=False)
    tg = np.ascontiguousarray(src[idx])
    R = ref.make_periodizer(int(pw.Pde.Stokes), 0.0, (d, 0.0, eta, int(pw.Periodicity.Doubly)), eps)
    want = R.apply(2, src, tg, forces=f, threads=8)["velocity"]
    assert rel_l2(prod[idx], want) <= 1e-11


def test_stokeslet_product_form_excluded_cases(pw, gpu, monkeypatch):
    """A skewed cell and the pressure output keep the image loop (bitwise the PWB_NO_PROD
    result)."""
    rng = np.random.default_rng(31)
    n = 34000
    for d, xi, eta, pressure in [(1.0, 0.25, 0.9, False), (1.0, 0.0, 1.0, True)]:
        cell = pw.make_unit_cell(d, xi, eta)
        src = np.column_stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n)]) @ np.array([[d, 0.0], [xi, eta]])
        src = np.ascontiguousarray(src)
        f = rng.standard_normal((n, 2))
        f = np.ascontiguousarray(f - f.mean(axis=0))
        pz = pw.make_periodizer(pw.Pde.Stokes, 0.0, cell, 1e-8)
        opt = pw.ApplyOptions(with_pressure=pressure)
        sys_ = pw.ParticleSystem(sources=src, targets=src, forces=f)
        a = pw.near_field(pz, sys_, opt).velocity
        monkeypatch.setenv("PWB_NO_PROD", "1")
        b = pw.near_field(pz, sys_, opt).velocity
        monkeypatch.delenv("PWB_NO_PROD")
        assert np.array_equal(a, b), (d, xi, eta, pressure)


def test_stokeslet_product_form_duplicates_and_image_coincidence(pw, gpu):
    rng = np.random.default_rng(37)
    n = 36000
    src = _points2(rng, 1.0, 1.0, n)
    src[1000:1010] = src[30000:30010]
    src[5] = src[6]
    f = rng.standard_normal((n, 2))
    f = np.ascontiguousarray(f - f.mean(axis=0))
    pz = pw.make_periodizer(pw.Pde.Stokes, 0.0, pw.make_unit_cell(1.0, 0.0, 1.0), 1e-8)
    sym = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, forces=f)).velocity
    one = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src.copy(), forces=f)).velocity
    assert np.all(np.isfinite(sym))
    assert rel_l2(sym, one) <= 3e-12
    for p7, p3 in [([-0.5, 0.25], [0.5, 0.25]), ([0.3, -0.5], [0.3, 0.5]), ([-0.5, -0.5], [0.5, 0.5])]:
        bad = src.copy()
        bad[7] = p7
        bad[33333] = p3  # a near image of point 7
        with pytest.raises(pw.PeriwaveError) as e:
            pw.near_field(pz, pw.ParticleSystem(sources=bad, targets=bad, forces=f))
        assert e.value.code == pw.ErrorCode.CoincidentSourceTarget


# ------------------------------------------------------------------ Laplace, 3 x 3 images
@pytest.mark.parametrize("eps", [1e-10, 1e-11])
@pytest.mark.parametrize("d,eta", [(1.0, 1.0), (2.0, 0.7), (0.5, 0.4), (1.5, 1.0)])
def test_laplace_3x3_product_form_matches_image_loop(pw, gpu, ref, monkeypatch, d, eta, eps):
    """Unskewed doubly periodic Poisson above the symmetric threshold: every image row in
    closed form."""
    rng = np.random.default_rng(int(d * 8) + 41)
    n = 36000
    src = _points2(rng, d, eta, n)
    q = rng.standard_normal(n)
    q -= q.mean()
    cell = pw.make_unit_cell(d, 0.0, eta)
    if cell.m0 != 1:
        pytest.skip("more than 3 x 3 images")
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, cell, eps)
    sys_ = pw.ParticleSystem(sources=src, targets=src, charges=q)
    prod = pw.near_field(pz, sys_).scalar
    assert np.array_equal(prod, pw.near_field(pz, sys_).scalar)
    monkeypatch.setenv("PWB_NO_PROD", "1")
    loop = pw.near_field(pz, sys_).scalar
    monkeypatch.delenv("PWB_NO_PROD")
    assert not np.array_equal(prod, loop)
    monkeypatch.setenv("PWB_FULL_PRECISION", "1")
    full = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src.copy(), charges=q)).scalar
    monkeypatch.delenv("PWB_FULL_PRECISION")
    e_prod, e_loop = rel_l2(prod, full), rel_l2(loop, full)
    print("d", d, "eta", eta, "eps", eps, "prod vs full", e_prod, "image loop vs full", e_loop)
    assert e_prod <= (2e-12 if eps >= 1e-10 else 5e-13)
    assert e_prod <= 2.0 * e_loop + 1e-13
    idx = rng.choice(n, 200, replace=False)
    tg = np.ascontiguousarray(src[idx])
    R = ref.make_periodizer(int(pw.Pde.Poisson), 0.0, (d, 0.0, eta, int(pw.Periodicity.Doubly)), eps)
    want = R.apply(2, src, tg, charges=q, threads=8)["scalar"]
    assert rel_l2(prod[idx], want) <= 1e-11


def test_laplace_3x3_product_form_duplicates_and_image_coincidence(pw, gpu, monkeypatch):
    rng = np.random.default_rng(43)
    n = 36000
    src = _points2(rng, 1.0, 1.0, n)
    src[1000:1010] = src[30000:30010]
    src[5] = src[6]
    q = rng.standard_normal(n)
    q -= q.mean()
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(1.0, 0.0, 1.0), 1e-10)
    sym = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, charges=q)).scalar
    one = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src.copy(), charges=q)).scalar
    assert np.all(np.isfinite(sym))
    assert rel_l2(sym, one) <= 2e-12
    for p7, p3 in [([-0.5, 0.25], [0.5, 0.25]), ([0.3, -0.5], [0.3, 0.5]), ([-0.5, 0.5], [0.5, -0.5])]:
        bad = src.copy()
        bad[7] = p7
        bad[33333] = p3
        with pytest.raises(pw.PeriwaveError) as e:
            pw.near_field(pz, pw.ParticleSystem(sources=bad, targets=bad, charges=q))
        assert e.value.code == pw.ErrorCode.CoincidentSourceTarget
    # a skewed cell keeps the image loop
    sk = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(1.0, 0.25, 0.9), 1e-10)
    pts = np.ascontiguousarray(np.column_stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n)])
                               @ np.array([[1.0, 0.0], [0.25, 0.9]]))
    a = pw.near_field(sk, pw.ParticleSystem(sources=pts, targets=pts, charges=q)).scalar
    monkeypatch.setenv("PWB_NO_PROD", "1")
    b = pw.near_field(sk, pw.ParticleSystem(sources=pts, targets=pts, charges=q)).scalar
    assert np.array_equal(a, b)


@pytest.mark.parametrize("d", [2.0 ** -60, 3.0 * 2.0 ** -28, 2.0 ** 40, 5.0 * 2.0 ** 25])
def test_product_form_extreme_cell_sizes(pw, gpu, monkeypatch, d):
    """Tiny and huge cells (scaled form for powers of two, unscaled form within 2^+-30): the
    products stay normal numbers and the field agrees with the image loop."""
    rng = np.random.default_rng(53)
    n = 34000
    src = np.ascontiguousarray(_points(rng, 1.0, n) * d)
    q = rng.standard_normal(n)
    q -= q.mean()
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(d, 0.0, d, pw.Periodicity.Singly), 1e-10)
    sys_ = pw.ParticleSystem(sources=src, targets=src, charges=q)
    prod = pw.near_field(pz, sys_).scalar
    monkeypatch.setenv("PWB_NO_PROD", "1")
    loop = pw.near_field(pz, sys_).scalar
    assert np.all(np.isfinite(prod))
    assert not np.array_equal(prod, loop)
    assert rel_l2(prod, loop, gauge=True) <= 3e-12
