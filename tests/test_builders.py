"""Host periodizer builders (the plane-wave mode/coefficient tables the device plan
uploads) against the compiled reference, element by element."""
import numpy as np
import pytest

CASES = [
    (0, 0.0, (1.0, 0.0, 1.0, 2), 1e-10),    # c1
    (1, 10.0, (1.0, 0.3, 0.8, 2), 1e-10),   # c2
    (2, 0.0, (1.0, 0.0, 1.0, 2), 1e-8),     # c3
    (0, 0.0, (1.0, 0.0, 1.0, 1), 1e-10),    # c4
    (1, 1.0, (100.0, 0.0, 1.0, 2), 1e-8),   # c5
    (3, 1.5, (1.0, 0.2, 0.9, 2), 1e-10),
    (3, 0.7, (1.0, 0.1, 2.0, 1), 1e-6),
    (1, 1.0, (1.0, 0.0, 1.0 / 12.0, 2), 1e-12),
    (0, 0.0, (1.0, -0.9, 0.3, 2), 1e-9),
    (2, 0.0, (1.0, 0.45, 3.0, 1), 1e-6),
]


def _compare(mine, theirs):
    assert len(mine) == len(theirs)
    for a, b in zip(mine, theirs):
        assert (a.axis, a.dir, a.has_m0) == (b.axis, b.dir, b.has_m0)
        for f in ("phase", "decay_t", "decay_s", "shift_t", "shift_s"):
            x, y = getattr(a, f), getattr(b, f)
            assert x.shape == y.shape
            assert np.array_equal(x, y), f
        for t1, t2 in zip(a.tables, b.tables):
            if t2.size and t1.size:
                assert np.max(np.abs(t1 - t2)) <= 1e-15 * np.max(np.abs(t2))
        assert np.allclose(a.m0, b.m0, rtol=1e-15, atol=0)


@pytest.mark.parametrize("case", CASES)
def test_tables_match_reference(pw, ref, case):
    pde, beta, cell, eps = case
    c = pw.make_unit_cell(cell[0], cell[1], cell[2], pw.Periodicity(cell[3]))
    assert c.m0 == ref.unit_cell_m0(cell)
    P = pw.make_periodizer(pw.Pde(pde), beta, c, eps)
    R = ref.make_periodizer(pde, beta, cell, eps)
    assert P.rank() == R.rank()
    assert P.info()["requires_neutrality"] == R.requires_neutrality()
    for kind in range(4):
        _compare(P.parts(kind), R.parts(kind))


@pytest.mark.parametrize("pde,beta,l", [(0, 0.0, 1), (0, 0.0, 3), (1, 1.5, 1), (1, 10.0, 1), (1, 2.0, 4)])
def test_multipole_tables_match_reference(pw, ref, pde, beta, l):
    for cell in ((1.0, 0.0, 1.0, 2), (1.0, 0.3, 0.8, 2), (1.0, 0.0, 1.5, 1)):
        c = pw.make_unit_cell(cell[0], cell[1], cell[2], pw.Periodicity(cell[3]))
        P = pw.make_multipole_periodizer(pw.Pde(pde), beta, l, c, 1e-10)
        R = ref.make_multipole_periodizer(pde, beta, l, cell, 1e-10)
        assert P.rank() == R.rank()
        _compare(P.parts(0), R.parts(0))


def test_dlp_tables_match_reference(pw, ref):
    for cell in ((1.0, 0.0, 1.0, 2), (1.0, 0.35, 0.8, 2), (1.0, 0.2, 2.0, 1)):
        c = pw.make_unit_cell(cell[0], cell[1], cell[2], pw.Periodicity(cell[3]))
        P = pw.make_stokes_dlp_periodizer(c, 1e-8)
        R = ref.make_stokes_dlp_periodizer(cell, 1e-8)
        assert P.rank() == R.rank()
        _compare(P.parts(3), R.parts(3))


def test_truncation_order_known_values(pw, ref):
    # proj/tests/test_periodize.cpp:104-122 known values 5/3/46/5206 are for these cells
    for cell, eps in (((1.0, 0.0, 1.0, 2), 1e-12), ((1.0, 0.0, 1.0, 2), 1e-6), ((1.0, 0.0, 0.1, 2), 1e-12),
                      ((1.0, 0.0, 0.001, 2), 1e-12), ((100.0, 0.0, 1.0, 2), 1e-8)):
        c = pw.make_unit_cell(cell[0], cell[1], cell[2], pw.Periodicity(cell[3]))
        assert pw.truncation_order(c, eps) == ref.truncation_order(cell, eps)
    c = pw.make_unit_cell(1.0, 0.0, 1.0)
    assert pw.truncation_order(c, 1e-12) == 5


def test_paper_appendix_a_ranks(pw):
    """ranks 1360 / 214 / 676 (+676 pressure) / 1216 / 1354."""
    want = {(0, (1.0, 0.0, 1.0, 2), 1e-10, 0.0): 1360, (1, (1.0, 0.3, 0.8, 2), 1e-10, 10.0): 214,
            (2, (1.0, 0.0, 1.0, 2), 1e-8, 0.0): 1352, (0, (1.0, 0.0, 1.0, 1), 1e-10, 0.0): 1216,
            (1, (100.0, 0.0, 1.0, 2), 1e-8, 1.0): 1354}
    for (pde, cell, eps, beta), r in want.items():
        c = pw.make_unit_cell(cell[0], cell[1], cell[2], pw.Periodicity(cell[3]))
        assert pw.make_periodizer(pw.Pde(pde), beta, c, eps).rank() == r


def test_tables_roundtrip_through_the_abi(pw, ref):
    """Reference tables injected through pwb_periodizer_add_part come back unchanged."""
    R = ref.make_periodizer(2, 0.0, (1.0, 0.3, 0.8, 2), 1e-8)
    c = pw.make_unit_cell(1.0, 0.3, 0.8)
    P = pw.Periodizer.from_tables(pw.Pde.Stokes, 0.0, c, 1e-8, R.all_parts(), requires_neutrality=True)
    assert P.rank() == R.rank()
    for kind in range(4):
        _compare(P.parts(kind), R.parts(kind))
