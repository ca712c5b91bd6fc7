"""The per-tile-pair Chebyshev K0 fit of the screened symmetric tile (pw_math.cuh
cheb_fit_k0, regime 3), emulated on the host with the generated constant matrices
(csrc/cuda/pw_cheb.h): for intervals of the shapes the tiles produce, every fit the rule
accepts meets its relative error bound against an independent K0 (scipy's, ~1e-15 relative;
the bound is 1e-11), and the degree it picks is the smallest of {6, 9, 12} whose bound holds."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_2111_01083_b200", "csrc", "cuda", "pw_cheb.h")


def _tables():
    src = open(HDR).read()
    D = int(re.search(r"kChebMax = (\d+)", src).group(1))

    def arr(name):
        m = re.search(name + r"\[\d+\](?:\[\d+\])? = \{(.*?)\};", src, re.S)
        return np.array([float(x) for x in re.findall(r"[-+0-9.eE]+", m.group(1))])

    return D, arr("pw_cheb_u_dev"), arr("pw_cheb_a_dev").reshape(D + 1, D + 1), arr("pw_cheb_c_dev").reshape(D + 1,
                                                                                                             D + 1)


def _k0(x):
    from scipy.special import k0

    return float(k0(x))


def fit(slo, shi, beta, tol):
    """Host restatement of cheb_fit_k0: (degree or 0, monomial coefficients, s_c)."""
    D, u, A, C = _tables()
    sc, hs = 0.5 * (slo + shi), 0.5 * (shi - slo)
    f = np.array([_k0(beta * np.sqrt(sc + hs * v)) for v in u])
    a = A @ f
    fmn = f.min()
    budget = tol * fmn
    own = 4 * a[D] ** 2
    if not own <= budget * abs(a[D - 1]):
        return 0, None, sc
    own_err = own / abs(a[D - 1])
    tail = np.abs(a[10:]).sum()
    d = D
    if own_err + tail <= budget:
        d = 9
        if own_err + tail + np.abs(a[7:10]).sum() <= budget:
            d = 6
    m = np.array([sum(C[i, k] * a[k] for k in range(i, d + 1)) for i in range(d + 1)])
    return d, m / hs ** np.arange(d + 1), sc


def test_tables_interpolate_exactly():
    D, u, A, C = _tables()
    # the degree-D interpolant of a degree-D polynomial is the polynomial itself
    coef = np.random.default_rng(0).standard_normal(D + 1)
    f = np.polynomial.polynomial.polyval(u, coef)
    m = C @ (A @ f)
    assert np.allclose(m, coef, rtol=0, atol=1e-12)


@pytest.mark.parametrize("beta", [1.0, 10.0])
def test_accepted_fits_meet_the_bound(beta):
    rng = np.random.default_rng(7)
    tol = 1e-11  # 1e-3 eps at c5's eps = 1e-8
    accepted = 0
    for _ in range(120):
        xc = rng.uniform(0.8, 40.0)
        dx = rng.uniform(0.02, 0.5)
        xlo, xhi = max(xc - dx, 0.5), xc + dx
        slo, shi = (xlo / beta) ** 2, (xhi / beta) ** 2
        d, c, sc = fit(slo, shi, beta, tol)
        if not d:
            continue
        accepted += 1
        ss = np.linspace(slo, shi, 41)
        got = np.polynomial.polynomial.polyval(ss - sc, c)
        want = np.array([_k0(beta * np.sqrt(v)) for v in ss])
        err = np.max(np.abs(got - want) / want.min())
        assert err <= tol, (xc, dx, d, err)
    assert accepted > 40


def test_degree_is_the_smallest_that_holds():
    beta, tol = 1.0, 1e-11
    # far and narrow: degree 6; nearer or wider: more
    assert fit(19.9 ** 2, 20.1 ** 2, beta, tol)[0] == 6
    d_mid = fit(4.8 ** 2, 5.2 ** 2, beta, tol)[0]
    assert d_mid in (9, 12)
    assert fit(0.6 ** 2, 1.4 ** 2, beta, tol)[0] == 0  # too wide near the log singularity
