"""Product form of the symmetric Laplace tile (singly periodic cells, near_sym_impl.cuh
SymLaplace PROD): binned points scaled to period 2, the three images' product in closed
form on tile pairs that keep clear of the +-d images, the image loop elsewhere. Checked
against the same tile without it (PWB_NO_PROD=1), the one-sided full-precision tile and the
compiled reference (apply.cpp:481-546)."""
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
@pytest.mark.parametrize("d", [1.0, 0.5, 4.0])
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


def test_product_form_needs_power_of_two_period(pw, gpu, monkeypatch):
    """d = 1.5: scaling by 2 / d would round the points, so the image loop runs (bitwise the
    PWB_NO_PROD result)."""
    rng = np.random.default_rng(5)
    n = 36000
    src = _points(rng, 1.5, n)
    q = rng.standard_normal(n)
    q -= q.mean()
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(1.5, 0.0, 1.0, pw.Periodicity.Singly), 1e-10)
    sys_ = pw.ParticleSystem(sources=src, targets=src, charges=q)
    a = pw.near_field(pz, sys_).scalar
    monkeypatch.setenv("PWB_NO_PROD", "1")
    b = pw.near_field(pz, sys_).scalar
    assert np.array_equal(a, b)


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
