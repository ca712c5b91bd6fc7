"""Sharded passes on one GPU, run one after another (no kernel waits on another):
the pieces a multi-GPU rank runs compose to the single-call result."""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("binning", [True, False])
@pytest.mark.parametrize("name,n,pressure", [("c4", 40000, False), ("c3", 33000, True), ("c5", 34000, False)])
def test_symmetric_items_compose_bitwise(pw, gpu, monkeypatch, name, n, pressure, binning):
    """Work items split across 2 or 3 simulated ranks add up (int64) to the single call,
    bitwise. Screened kernels (c5) bin on both paths: every rank sorts the same points the
    same way and adds its sorted-order accumulator back in input order (engine.cu
    sym_partial); PWB_NO_BINNING=1 runs both in input order."""
    import torch

    from paper_2111_01083_b200 import configs, dist as pdist

    if not binning:
        monkeypatch.setenv("PWB_NO_BINNING", "1")
    inp = configs.generate(name, n_src=n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    kw = "charges" if c.strength == "charge" else "forces"
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges if kw == "charges" else inp.forces).cuda()
    opt = pw.ApplyOptions(with_pressure=pressure)
    # n above the symmetric-tile threshold (32768), so the single call takes the same tile
    whole = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, **{kw: q}), opt)
    items, nout = pw.near_sym_items(pz, n, opt)
    for world in (2, 3):
        acc = torch.zeros(n * nout * 3, dtype=torch.int64, device="cuda")
        ks = set()
        for r in range(world):
            lo, hi = pdist.contiguous(items, world, r)
            part = torch.zeros_like(acc)
            k, status = pw.near_sym_partial(pz, pw.ParticleSystem(sources=src, targets=src, **{kw: q}), part, lo, hi,
                                            opt)
            assert status == 0
            ks.add(k)
            acc += part  # the int64 reduce-scatter operand
        assert len(ks) == 1  # every rank scales identically
        got = pw.FieldResult()
        key = "scalar" if kw == "charges" else "velocity"
        setattr(got, key, torch.zeros_like(getattr(whole, key)))
        if pressure:
            got.pressure = torch.zeros_like(whole.pressure)
        pw.fixed_to_field(pz, acc, n, got, opt, like=src, scale_exp=ks.pop())
        assert torch.equal(getattr(got, key), getattr(whole, key))
        if pressure:
            assert torch.equal(got.pressure, whole.pressure)


@pytest.mark.parametrize("name,n", [("c5", 60000), ("c4", 40000)])
def test_balanced_split_covers_items_and_composes(pw, gpu, name, n):
    """pwb_near_sym_split: monotone bounds from 0 to the item count, identical on repeated
    calls (every rank must compute the same split), and the per-rank partials over those
    ranges add up bitwise to the single call. Screened kernels (c5) split by estimated cost,
    the others (c4) by count."""
    import torch

    from paper_2111_01083_b200 import configs

    inp = configs.generate(name, n_src=n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges).cuda()
    opt = pw.ApplyOptions()
    s = pw.ParticleSystem(sources=src, targets=src, charges=q)
    items, nout = pw.near_sym_items(pz, n, opt)
    whole = pw.near_field(pz, s, opt)
    for world in (3, 8):
        b = pw.near_sym_split(pz, s, world, opt)
        assert b == pw.near_sym_split(pz, s, world, opt)
        assert b[0] == 0 and b[-1] == items and all(x <= y for x, y in zip(b, b[1:]))
        if name == "c4":
            assert b == [items * r // world for r in range(world + 1)]
        acc = torch.zeros(n * nout * 3, dtype=torch.int64, device="cuda")
        for r in range(world):
            part = torch.zeros_like(acc)
            k, status = pw.near_sym_partial(pz, s, part, b[r], b[r + 1], opt)
            assert status == 0
            acc += part
        got = pw.FieldResult()
        got.scalar = torch.zeros_like(whole.scalar)
        pw.fixed_to_field(pz, acc, n, got, opt, like=src, scale_exp=k)
        assert torch.equal(got.scalar, whole.scalar)


def test_sharded_total_field_matches_single_call(pw, gpu):
    """dist.sharded_total_field with a single-process Comm per simulated rank; the
    all-reduce / reduce-scatter are done by summing the per-rank buffers here."""
    import torch

    from paper_2111_01083_b200 import configs, dist as pdist

    inp = configs.generate("c4", n_src=20001)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges).cuda()
    opt = pw.ApplyOptions()
    ref = pw.total_field(pz, pw.ParticleSystem(sources=src, targets=src, charges=q), opt)
    n, world = 20001, 3
    be = pdist.CudaBackend(pw, pz, opt, src, q, "charges")
    coeff = be.coeff_buffer()
    for r in range(world):
        part = be.coeff_buffer()
        be.far_source(*pdist.contiguous(n, world, r), part)
        coeff += part
    items, nout = be.near_items()
    chunk = pdist.target_chunk(n, world)
    acc = be.accumulator(chunk * world * nout * 3)
    for r in range(world):
        part = be.accumulator(chunk * world * nout * 3)
        k, status = be.near_partial(*pdist.contiguous(items, world, r), part)
        assert status == 0
        acc += part
    outs = []
    for r in range(world):
        lo, hi = pdist.target_slice(n, world, r)
        out = be.far_target(coeff, lo, hi)
        assert out.accelerated == ref.accelerated
        be.fixed_to_out(acc[r * chunk * nout * 3:(r + 1) * chunk * nout * 3], hi - lo, out, k)
        outs.append(out.scalar)
    got = torch.cat(outs).cpu().numpy()
    assert rel_l2(got, ref.scalar.cpu().numpy(), gauge=True) <= 1e-13


def test_split_rejects_bad_world_sizes(pw, gpu):
    import torch

    from paper_2111_01083_b200 import configs

    inp = configs.generate("c5", n_src=5000)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    s = pw.ParticleSystem(sources=src, targets=src, charges=torch.from_numpy(inp.charges).cuda())
    for w in (0, 65):
        with pytest.raises(pw.PeriwaveError) as e:
            pw.near_sym_split(pz, s, w)
        assert e.value.code == pw.ErrorCode.Unsupported
    assert pw.near_sym_split(pz, s, 1) == [0, pw.near_sym_items(pz, 5000)[0]]


@pytest.mark.parametrize("name,n", [("c4", 40000), ("c3", 33000), ("c5", 34000)])
@pytest.mark.parametrize("scale", [1e-15, 1e15, 2.0 ** -600])
def test_symmetric_tile_scales_with_the_strengths(pw, gpu, name, n, scale):
    """The fixed-point accumulator's scale follows max|strength| (near_sym_impl.cuh fx_add):
    strengths times 1e-15, 1e15 or 2^-600 give the unscaled field times the same factor,
    to fp64 accuracy (the reference sums in plain fp64, apply.cpp:532-540). Powers of two
    scale exactly: bitwise."""
    import torch

    from paper_2111_01083_b200 import configs

    inp = configs.generate(name, n_src=n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    kw = "charges" if c.strength == "charge" else "forces"
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges if kw == "charges" else inp.forces).cuda()
    key = "scalar" if kw == "charges" else "velocity"
    base = getattr(pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, **{kw: q})), key)
    got = getattr(pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, **{kw: q * scale})), key) / scale
    if scale == 2.0 ** -600:
        assert torch.equal(got, base)
    else:
        # q * 1e-15 rounds each strength (1 ulp); Stokes velocities cancel a little: 1e-13
        assert rel_l2(got.cpu().numpy(), base.cpu().numpy()) <= 1e-13


def test_symmetric_tile_nonfinite_strength_falls_back(pw, gpu):
    """A non-finite strength overflows the fixed point; the engine redoes the near field in
    fp64 on the one-sided tile, so the output carries the NaN/inf like the reference's sum."""
    import torch

    from paper_2111_01083_b200 import configs

    inp = configs.generate("c5", n_src=40000)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges).cuda()
    q[123] = float("inf")
    u = pw.near_field(pz, pw.ParticleSystem(sources=src, targets=src, charges=q)).scalar.cpu().numpy()
    assert not np.all(np.isfinite(u))
    assert np.isinf(u[123]) or np.isnan(u[123])


def test_sym_partial_reports_coincidence_without_raising(pw, gpu):
    """pwb_near_sym_partial returns status bit 0 for a non-identity coincidence (the caller
    combines the ranks' status words before the reduce-scatter, dist.py); only the item
    range holding the pair reports it."""
    import torch

    from paper_2111_01083_b200 import configs

    n = 40000
    inp = configs.generate("c4", n_src=n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    pts = inp.sources.copy()
    pts[0] = (-0.5, 0.1)
    pts[-1] = (0.5, 0.1)  # the image of point 0 under the shift (d, 0)
    src = torch.from_numpy(pts).cuda()
    s = pw.ParticleSystem(sources=src, targets=src, charges=torch.from_numpy(inp.charges).cuda())
    items, nout = pw.near_sym_items(pz, n)
    seen = []
    for lo, hi in ((0, items // 2), (items // 2, items)):
        acc = torch.zeros(n * nout * 3, dtype=torch.int64, device="cuda")
        seen.append(pw.near_sym_partial(pz, s, acc, lo, hi)[1])
    assert sorted(seen) == [0, pw.SYM_COINCIDENT]
    with pytest.raises(pw.PeriwaveError) as e:
        pw.near_field(pz, s)
    assert e.value.code == pw.ErrorCode.CoincidentSourceTarget
