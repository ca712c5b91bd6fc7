"""Validation tools on the GPU: brute_force_far and
periodicity_residual against the reference's (proj/src/oracle.cpp:83-173) and the
oracle-free periodicity bound of the reference CLI (residual <= 5 eps,
proj/tools/periwave_cli.cpp:288)."""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _pts(rng, cell, n, margin=0.02):
    d, xi, eta = cell[:3]
    a = (rng.uniform(size=n) - 0.5) * (1 - 2 * margin)
    b = (rng.uniform(size=n) - 0.5) * (1 - 2 * margin)
    return np.ascontiguousarray(np.stack([a * d + b * xi, b * eta], 1))


def test_brute_force_far_matches_reference_and_plane_waves(pw, gpu, ref):
    rng = np.random.default_rng(31)
    cell = (1.0, 0.3, 0.8, 2)
    src, tgt = _pts(rng, cell, 40), _pts(rng, cell, 15)
    q = np.ascontiguousarray(rng.uniform(-1, 1, 40))
    c = pw.make_unit_cell(*cell[:3], pw.Periodicity(cell[3]))
    pz = pw.make_periodizer(pw.Pde.ModHelmholtz, 3.0, c, 1e-12)
    sysd = pw.ParticleSystem(sources=src, charges=q, targets=tgt)
    bf = pw.brute_force_far(pz, sysd, 12).scalar
    R = ref.make_periodizer(1, 3.0, cell, 1e-12)
    want = R.brute_force_far(12, src, tgt, charges=q)["scalar"]
    assert rel_l2(bf, want) <= 1e-13
    far = pw.apply_far(pz, sysd, pw.ApplyOptions(path=pw.ApplyPath.Direct)).scalar
    assert rel_l2(far, bf) <= 1e-11  # proj/tests/test_periodize.cpp:182-381 (<= 1e-11 ModHelm)


@pytest.mark.parametrize("pde,beta,cell,eps", [
    (0, 0.0, (1.0, 0.0, 1.0, 2), 1e-10),
    (1, 1.0, (1.0, 0.5, 0.8, 2), 1e-12),
    (1, 1.0, (100.0, 0.0, 1.0, 2), 1e-8),
    (0, 0.0, (1.0, 0.0, 1.0, 1), 1e-10),
    (2, 0.0, (1.0, 0.0, 1.0, 2), 1e-8),
])
def test_periodicity_residual_within_5_eps(pw, gpu, ref, pde, beta, cell, eps):
    rng = np.random.default_rng(17)
    n = 400
    src = _pts(rng, cell, n, margin=0.0)
    c = pw.make_unit_cell(*cell[:3], pw.Periodicity(cell[3]))
    pz = pw.make_periodizer(pw.Pde(pde), beta, c, eps)
    if pde == 2:
        f = rng.uniform(-1, 1, (n, 2))
        f -= f.mean(axis=0)
        kw = dict(forces=np.ascontiguousarray(f))
    else:
        q = rng.uniform(-1, 1, n)
        if pde == 0:
            q -= q.mean()
        kw = dict(charges=np.ascontiguousarray(q))
    rep = pw.periodicity_residual(pz, pw.ParticleSystem(sources=src, targets=np.zeros((0, 2)), **kw), 50)
    assert rep["rel"] <= 5 * eps, rep
    R = ref.make_periodizer(pde, beta, cell, eps)
    e1, e2, sc = np.zeros(1), np.zeros(1), np.zeros(1)
    args = [np.ascontiguousarray(a) if a is not None else None for a in (src, kw.get("charges"), kw.get("forces"))]
    st = ref.L.ref_periodicity_residual(R.h, 50, n, args[0].ctypes.data,
                                        args[1].ctypes.data if args[1] is not None else None,
                                        args[2].ctypes.data if args[2] is not None else None, None, None, 1, 8,
                                        e1.ctypes.data, e2.ctypes.data, sc.ctypes.data)
    assert st == 0
    assert abs(rep["scale"] - sc[0]) <= 1e-12 * sc[0]
