"""Seeded synthetic workloads: deterministic, in the closed cell,
neutral where the kernel requires it, the right sizes."""
import numpy as np
import pytest


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_inputs_valid(pw, name):
    from paper_2111_01083_b200 import configs

    n = {"c1": 1000, "c2": 5000, "c3": 5000, "c4": 20000}[name]
    a = configs.generate(name, n_src=n)
    b = configs.generate(name, n_src=n)
    assert np.array_equal(a.sources, b.sources)
    c = a.config
    d, xi, eta = c.cell[:3]
    x2 = a.sources[:, 1] / eta
    x1 = (a.sources[:, 0] - xi * x2) / d
    assert np.all(np.abs(x1) <= 0.5) and np.all(np.abs(x2) <= 0.5)
    strength = a.charges if c.strength == "charge" else a.forces
    assert strength.shape[0] == n
    if c.neutral:
        tot = np.abs(strength).sum()
        assert np.all(np.abs(strength.sum(axis=0)) <= 1e-12 * tot)
    if c.separate_targets:
        assert a.targets is not a.sources and a.targets.shape == a.sources.shape
    else:
        assert a.targets is a.sources
    assert len(np.unique(a.sample)) == len(a.sample) == min(c.oracle_sample, n)


def test_c4_clusters(pw):
    from paper_2111_01083_b200 import configs

    a = configs.generate("c4", n_src=50000)
    # 16 Gaussian clusters of sigma 0.02: most points within 3 sigma of a centre
    from paper_2111_01083_b200.configs import uniform_points

    centres = uniform_points(a.config.seed + 104729, 16, 1.0, 0.0, 1.0)
    dx = a.sources[:, None, 0] - centres[None, :, 0]
    dx = dx - np.round(dx)
    dy = a.sources[:, None, 1] - centres[None, :, 1]
    dist = np.min(np.hypot(dx, dy), axis=1)
    assert np.mean(dist < 0.06) > 0.95
    assert np.all(np.abs(a.sources) <= 0.5)


def test_full_sizes_match_baseline(pw):
    from paper_2111_01083_b200 import configs

    assert [configs.CONFIGS[k].n_src for k in ("c1", "c2", "c3", "c4", "c5")] == [1000, 100000, 1000000, 1000000,
                                                                                 10000000]
    assert [configs.CONFIGS[k].eps for k in ("c1", "c2", "c3", "c4", "c5")] == [1e-10, 1e-10, 1e-8, 1e-10, 1e-8]


def test_reference_arm_draws_the_same_bytes(pw):
    """bench.py's reference arm draws its inputs from the reference's own Rng in oracle/_ref
    (or the C restatement), never from the product library: same bytes for every config."""
    import workloads
    from oracle import pyoracle
    from paper_2111_01083_b200 import configs

    for name in ("c1", "c2", "c3", "c4", "c5"):
        a = configs.generate(name, n_src=3000)
        b = workloads.generate(name, n_src=3000, rng=pyoracle.rng_uniform)
        assert np.array_equal(a.sources, b.sources) and np.array_equal(a.targets, b.targets)
        assert np.array_equal(a.sample, b.sample)
        sa = a.charges if a.charges is not None else a.forces
        sb = b.charges if b.charges is not None else b.forces
        assert np.array_equal(sa, sb)
    if pyoracle.ref_available():
        assert np.array_equal(pyoracle.Ref().rng_uniform(77, 5000), pyoracle.Port().rng_uniform(77, 5000))


def test_workload_ordinals_match_the_api(pw):
    """workloads.py restates periwave::Pde / Periodicity as plain ints (cell.hpp:9,
    kernels.hpp:7): they must be the product enums' values, or every config changes cell."""
    import workloads

    assert (workloads.POISSON, workloads.MODHELMHOLTZ, workloads.STOKES) == (
        pw.Pde.Poisson, pw.Pde.ModHelmholtz, pw.Pde.Stokes)
    assert (workloads.SINGLY, workloads.DOUBLY) == (pw.Periodicity.Singly, pw.Periodicity.Doubly)
    per = {k: pw.Periodicity(c.cell[3]) for k, c in workloads.CONFIGS.items()}
    assert per == {"c1": pw.Periodicity.Doubly, "c2": pw.Periodicity.Doubly, "c3": pw.Periodicity.Doubly,
                   "c4": pw.Periodicity.Singly, "c5": pw.Periodicity.Doubly}
