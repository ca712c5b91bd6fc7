"""The `periwave-b200` command-line tool: the reference CLI's
`apply` / `validate` contract (proj/tools/periwave_cli.cpp:151-361), driven end to end
the way proj/tests/test_cli.cpp drives the reference binary.

CPU tests cover argument/record errors (they exit before any device work); the
GPU tests cover the outputs against the reference through oracle/_ref."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, rel_l2

CLI = os.path.join(ROOT, "paper_2111_01083_b200", "bin", "periwave-b200")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        pytest.fail("CLI not built: run __graft_entry__.build() (make -C paper_2111_01083_b200)")
    return CLI


def run(cli, *args, cwd=None):
    p = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600, cwd=cwd)
    return p.returncode, p.stdout + p.stderr


# ------------------------------------------------------------------ errors (CPU)
def test_malformed_record_reports_file_and_line(cli, tmp_path):
    bad, tgt = tmp_path / "bad.txt", tmp_path / "t.txt"
    bad.write_text("0.1 0.2 oops\n")
    tgt.write_text("0.0 0.0\n")
    code, log = run(cli, "apply", "--pde", "poisson", "--eps", "1e-8", bad, tgt)
    assert code == 2 and "bad.txt:1" in log


def test_inconsistent_columns_report_line(cli, tmp_path):
    bad, tgt = tmp_path / "bad.txt", tmp_path / "t.txt"
    bad.write_text("# header\n0.1 0.2 1.0\n0.3 0.4 1.0 2.0\n")
    tgt.write_text("0.0 0.0\n")
    code, log = run(cli, "apply", "--pde", "poisson", "--eps", "1e-8", bad, tgt)
    assert code == 2 and "bad.txt:3" in log and "inconsistent column count" in log


def test_bad_target_record(cli, tmp_path):
    src, tgt = tmp_path / "s.txt", tmp_path / "t.txt"
    src.write_text("0.1 0.2 1.0\n")
    tgt.write_text("\n0.0 0.0 3.0\n")
    code, log = run(cli, "apply", "--pde", "poisson", "--eps", "1e-8", src, tgt)
    assert code == 2 and "t.txt:2" in log and "expected 'x y'" in log


@pytest.mark.parametrize("args,needle", [
    (["--eps", "1e-20"], "--eps must lie in"),
    (["--eps", "1e-2"], "--eps must lie in"),
    (["--pde", "helmholtz"], "--pde"),
    (["--accel", "fast"], "--accel"),
    (["--cell", "1,0"], "--cell"),
    (["--cell", "1,0,1", "--aspect", "2"], "excludes"),
    (["--bogus", "1"], "unknown option"),
])
def test_bad_configs_exit_2(cli, tmp_path, args, needle):
    src, tgt = tmp_path / "s.txt", tmp_path / "t.txt"
    src.write_text("0.1 0.2 1.0\n")
    tgt.write_text("0.0 0.0\n")
    code, log = run(cli, "apply", *args, src, tgt)
    assert code == 2 and needle in log, log


def test_kernel_record_mismatch(cli, tmp_path):
    src, tgt = tmp_path / "s.txt", tmp_path / "t.txt"
    tgt.write_text("0.0 0.0\n")
    src.write_text("0.1 0.2 1.0 2.0\n")
    code, log = run(cli, "apply", "--pde", "poisson", "--eps", "1e-8", src, tgt)
    assert code == 2 and "scalar kernels take 'x y q'" in log
    src.write_text("0.1 0.2 1.0\n")
    code, log = run(cli, "apply", "--pde", "stokes", "--eps", "1e-8", src, tgt)
    assert code == 2 and "vector kernels take" in log
    src.write_text("0.1 0.2 1.0 2.0 1.0 0.0\n")
    code, log = run(cli, "apply", "--pde", "mstokes", "--beta", "1", "--eps", "1e-8", src, tgt)
    assert code == 2 and "Stokes-only" in log


def test_missing_file(cli, tmp_path):
    tgt = tmp_path / "t.txt"
    tgt.write_text("0.0 0.0\n")
    code, log = run(cli, "apply", tmp_path / "nope.txt", tgt)
    assert code == 2 and "cannot open" in log


# ------------------------------------------------------------------ outputs (GPU)
def _read_fields(path, cols):
    txt = open(path).read().split()
    return np.array([float(t) for t in txt]).reshape(-1, cols)


@pytest.mark.gpu
def test_validate_gates_residual_and_writes_report(cli, gpu, tmp_path):
    rep = tmp_path / "report.json"
    code, log = run(cli, "validate", "--pde", "mhelm", "--beta", "1", "--eps", "1e-9", "--aspect", "1,4",
                    "--n-src", "300", "--samples", "80", "--seed", "7", "--out", rep)
    assert code == 0, log
    r = json.loads(rep.read_text())
    assert r["pass"] is True and r["failures"] == []
    assert r["pde"] == "mhelm" and r["beta"] == 1.0 and r["eps"] == 1e-9
    assert len(r["rows"]) == 2
    for row in r["rows"]:
        assert row["rank"] > 0
        assert row["residuals"]["rel"] <= 5e-9
        assert {"per", "near", "total", "free"} <= set(row["timings"])
        assert row["cell"]["d"] == 1.0


@pytest.mark.gpu
def test_apply_reproduces_validate_dump_bitwise(cli, gpu, tmp_path):
    src, fld, tgt = tmp_path / "sources.txt", tmp_path / "fields.txt", tmp_path / "targets.txt"
    common = ["--pde", "mhelm", "--beta", "1", "--eps", "1e-9", "--aspect", "1", "--accel", "direct", "--seed", "11"]
    code, log = run(cli, "validate", *common, "--n-src", "150", "--samples", "40", "--dump-sources", src,
                    "--dump-fields", fld)
    assert code == 0, log
    rows = [ln.split() for ln in src.read_text().splitlines()]
    tgt.write_text("".join(f"{x} {y}\n" for x, y, _ in rows))
    out, out2 = tmp_path / "a.txt", tmp_path / "b.txt"
    assert run(cli, "apply", *common, src, tgt, "--out", out)[0] == 0
    a, b = fld.read_text(), out.read_text()
    assert a and a == b
    assert run(cli, "apply", *common, src, tgt, "--out", out2)[0] == 0
    assert out2.read_text() == b


@pytest.mark.gpu
def test_validate_sources_follow_reference_rng(cli, gpu, pw, tmp_path):
    """--dump-sources holds the reference generator's stream (cli.cpp:108-132) byte for byte."""
    src = tmp_path / "s.txt"
    code, log = run(cli, "validate", "--pde", "poisson", "--eps", "1e-8", "--n-src", "64", "--samples", "20",
                    "--seed", "5", "--dump-sources", src)
    assert code == 0, log
    u = pw.rng_uniform(5, 3 * 64)
    x1, x2 = u[0:128:2] - 0.5, u[1:128:2] - 0.5
    q = -1.0 + 2.0 * u[128:]
    q = q - (q / 64).sum()  # neutralised like the reference (mean accumulated as q/n)
    want = "".join("%.17g %.17g %.17g\n" % (1.0 * a + 0.0 * b, 0.0 * a + 1.0 * b, c) for a, b, c in zip(x1, x2, q))
    got = src.read_text().splitlines()
    assert len(got) == 64
    g = np.array([[float(t) for t in ln.split()] for ln in got])
    w = np.array([[float(t) for t in ln.split()] for ln in want.splitlines()])
    np.testing.assert_array_equal(g[:, :2], w[:, :2])
    assert np.max(np.abs(g[:, 2] - w[:, 2])) <= 1e-15


@pytest.mark.gpu
def test_empty_targets_produce_empty_output(cli, gpu, tmp_path):
    src, tgt, out = tmp_path / "one.txt", tmp_path / "none.txt", tmp_path / "o.txt"
    src.write_text("0.1 0.2 1.0\n-0.1 -0.2 -1.0\n")
    tgt.write_text("# no targets\n")
    code, log = run(cli, "apply", "--pde", "poisson", "--eps", "1e-8", src, tgt, "--out", out)
    assert code == 0, log
    assert out.read_text() == ""


@pytest.mark.gpu
@pytest.mark.parametrize("pde,beta,cols,pressure,per", [
    ("poisson", 0.0, 3, False, 2),
    ("mhelm", 2.0, 3, False, 1),
    ("stokes", 0.0, 4, True, 2),
    ("mstokes", 1.5, 4, False, 2),
    ("stokes", 0.0, 6, False, 2),
])
def test_apply_matches_reference_and_wraps(cli, gpu, ref, tmp_path, pde, beta, cols, pressure, per):
    """apply on records against the reference's total_field; targets given one lattice
    step outside the cell evaluate at their wrapped images (cli.cpp:134-142) and are
    echoed as given."""
    rng = np.random.default_rng(101 + cols)
    n, m = 120, 40
    cell = (1.0, 0.0, 1.0, per)
    x = rng.uniform(-0.49, 0.49, (n, 2))
    t = rng.uniform(-0.49, 0.49, (m, 2))
    shifted = t.copy()
    shifted[::2, 0] += 1.0  # one period in e1
    if cols == 3:
        w = rng.uniform(-1, 1, (n, 1))
        if pde == "poisson":
            w -= w.mean()
    elif cols == 4:
        w = rng.uniform(-1, 1, (n, 2))
        if pde == "stokes":
            w -= w.mean(axis=0)
    else:
        f = rng.uniform(-1, 1, (n, 2))
        f -= f.mean(axis=0)  # the double-layer periodizer also requires neutral densities
        ang = rng.uniform(0, 2 * np.pi, n)
        w = np.concatenate([f, np.stack([np.cos(ang), np.sin(ang)], 1)], 1)
    src, tgt, out = tmp_path / "s.txt", tmp_path / "t.txt", tmp_path / "o.txt"
    src.write_text("".join(" ".join("%.17g" % v for v in row) + "\n" for row in np.concatenate([x, w], 1)))
    tgt.write_text("".join("%.17g %.17g\n" % (a, b) for a, b in shifted))
    args = ["apply", "--pde", pde, "--beta", beta, "--eps", "1e-10", "--periodicity", per, src, tgt, "--out", out]
    if pressure:
        args.append("--pressure")
    code, log = run(cli, *args)
    assert code == 0, log
    ncol = 3 if cols == 3 else (5 if pressure else 4)
    got = _read_fields(out, ncol)
    np.testing.assert_array_equal(got[:, :2], shifted)  # echoed as given (bit-exact through %.17g)

    pdes = {"poisson": 0, "mhelm": 1, "stokes": 2, "mstokes": 3}
    if cols == 6:
        R = ref.make_stokes_dlp_periodizer(cell, 1e-10)
        want = R.apply(0, x, t, forces=w[:, :2], normals=w[:, 2:], path=1)
    else:
        R = ref.make_periodizer(pdes[pde], beta, cell, 1e-10)
        kw = dict(charges=w[:, 0]) if cols == 3 else dict(forces=w)
        want = R.apply(0, x, t, path=1, with_pressure=pressure, **kw)
    gauge = pde in ("poisson", "stokes")
    if cols == 3:
        assert rel_l2(got[:, 2], want["scalar"], gauge=gauge) <= 1e-9
    else:
        assert rel_l2(got[:, 2:4], want["velocity"], gauge=gauge) <= 1e-9
        if pressure:
            assert rel_l2(got[:, 4], want["pressure"], gauge=True) <= 1e-9
