"""Multi-rank host logic of the sharded total_field (paper_2111_01083_b200/dist.py) on
CPU: world_size 2 over gloo, with a NumPy stand-in for the device passes that follows
the same decomposition (source slices + coefficient all-reduce for the far field;
triangle work items + int64 fixed-point reduce-scatter for the symmetric near field).
Checks: every target slice and work item is covered once, the two-rank result equals
the one-rank result (near part bitwise), and both match the direct sums."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

TILE, CHUNK = 4, 2


def _fx_exponent(maxabs, n):
    """Mirror of pw_engine.cuh fx_exponent: 2^e > max|q|, 2^lg >= n, k = 24 - e - lg."""
    if maxabs == 0.0 or not np.isfinite(maxabs):
        return 0
    e = int(np.frexp(maxabs)[1])  # maxabs < 2^e (frexp mantissa in [0.5, 1))
    lg = int(n - 1).bit_length() if n > 1 else 0
    return int(np.clip(24 - e - lg, -960, 960))


def _fx_split(v):
    a = np.trunc(v * 2.0 ** -22)
    r1 = v - a * 2.0 ** 22
    b = np.trunc(r1 * 2.0 ** 20)
    r2 = r1 - b * 2.0 ** -20
    c = np.rint(r2 * 2.0 ** 62)
    return np.stack([a, b, c], -1).astype(np.int64)


def _fx_value(acc):
    a, b, c = acc[..., 0].astype(np.float64), acc[..., 1].astype(np.float64), acc[..., 2].astype(np.float64)
    return a * 2.0 ** 22 + (b * 2.0 ** -20 + c * 2.0 ** -62)


class NumpyBackend:
    """CPU stand-in: direct plane-wave sums over the product's own tables and the
    image-summed Laplace pair kernel."""

    def __init__(self, pw, pz, src, q):
        import torch

        self.torch = torch
        self.src, self.q, self.n = src, q, len(src)
        self.parts = pz.parts(pw.PART_SCALAR)
        from oracle.pyoracle import near_shifts

        info = pz.info()
        c = info["cell"]
        self.shifts, self.ident = near_shifts((c.d, c.xi, c.eta, int(c.periodicity)))
        self.nmodes = sum(p.size for p in self.parts)

    def _mode_factors(self, pts, target):
        out = []
        for p in self.parts:
            w = pts[:, 1] if p.axis == 0 else pts[:, 0]
            s = pts[:, 0] if p.axis == 0 else pts[:, 1]
            if target:
                f = np.exp(p.decay_t[None, :] * (w[:, None] - p.shift_t[None, :])) * np.exp(1j * p.phase * s[:, None])
            else:
                f = np.exp(p.decay_s[None, :] * (w[:, None] - p.shift_s[None, :])) * np.exp(-1j * p.phase * s[:, None])
            out.append(f)
        return np.concatenate(out, axis=1)

    def coeff_buffer(self):
        return self.torch.zeros(2 * self.nmodes + 1, dtype=self.torch.float64)

    def far_source(self, lo, hi, coeff):
        S = self._mode_factors(self.src[lo:hi], False)
        raw = S.T @ self.q[lo:hi]
        moment = np.sum(self.src[lo:hi, 1] * self.q[lo:hi])
        coeff[:] = self.torch.from_numpy(np.concatenate([raw.real, raw.imag, [moment]]))

    def far_target(self, coeff, lo, hi):
        c = coeff.numpy()
        raw = c[:self.nmodes] + 1j * c[self.nmodes:2 * self.nmodes]
        diag = np.concatenate([p.tables[0][0::2] + 1j * p.tables[0][1::2] for p in self.parts])
        T = self._mode_factors(self.src[lo:hi], True)
        u = T @ (diag * raw)
        m0 = sum(p.m0[0] for p in self.parts if p.has_m0)
        u = u + m0 * self.src[lo:hi, 1] * c[-1]
        from types import SimpleNamespace

        return SimpleNamespace(scalar=self.torch.from_numpy(np.ascontiguousarray(u.real)), velocity=None)

    def _items(self):
        nb = (self.n + TILE - 1) // TILE
        items = []
        for I in range(nb):
            for J0 in range(I, nb, CHUNK):
                items.append((I, J0, min(nb, J0 + CHUNK)))
        return items

    def near_items(self):
        return len(self._items()), 1

    def accumulator(self, n):
        return self.torch.zeros(n, dtype=self.torch.int64)

    def _G(self, t, s, identity_skip):
        g = 0.0
        for k, (sx, sy) in enumerate(self.shifts):
            rx, ry = (t[0] - s[0]) - sx, (t[1] - s[1]) - sy
            if rx == 0.0 and ry == 0.0:  # apply.cpp:538-545: skip in the identity image, else flag
                if not (identity_skip and k == self.ident):
                    self.status |= 1
                continue
            g += -np.log(rx * rx + ry * ry) / (4 * np.pi)
        return g

    def small_ints(self, vals):
        return self.torch.tensor(vals, dtype=self.torch.int64)

    def near_partial(self, lo, hi, acc):
        """Same contract as pwb_near_sym_partial: (scale_exp, status), no raise."""
        self.status = 0
        k = _fx_exponent(float(np.max(np.abs(self.q))), self.n)
        sc = 2.0 ** k
        a = acc.numpy().reshape(-1, 1, 3)
        for I, J0, J1 in self._items()[lo:hi]:
            rows = range(I * TILE, min(self.n, (I + 1) * TILE))
            racc = {l: 0.0 for l in rows}
            for J in range(J0, J1):
                cols = range(J * TILE, min(self.n, (J + 1) * TILE))
                cacc = {j: 0.0 for j in cols}
                for l in rows:
                    for j in cols:
                        if J == I:
                            racc[l] += self.q[j] * self._G(self.src[l], self.src[j], True)
                        elif True:
                            g = self._G(self.src[l], self.src[j], False)
                            racc[l] += self.q[j] * g
                            cacc[j] += self.q[l] * g
                if J != I:
                    for j, v in cacc.items():
                        a[j, 0] += _fx_split(np.float64(v) * sc)
            for l, v in racc.items():
                a[l, 0] += _fx_split(np.float64(v) * sc)
        return k, self.status

    def fixed_to_out(self, acc, n, out, scale_exp):
        v = _fx_value(acc.numpy().reshape(-1, 3)[:n]) * 2.0 ** -scale_exp
        out.scalar += self.torch.from_numpy(v)

    def near_targets(self, lo, hi, out):
        raise AssertionError("symmetric path expected")


def _system(pw, coincident=False, scale=1.0):
    rng = np.random.default_rng(5)
    n = 37  # not a multiple of the world size or the tile
    src = np.ascontiguousarray(np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n)], 1))
    if coincident:  # the last point is the first one's image under the shift (d, 0): the pair
        src[0, 0], src[-1] = -0.5, (0.5, src[0, 1])  # lies in the last row tile, one rank's items only
    q = rng.uniform(-1, 1, n) * scale
    q -= q.mean()
    cell = pw.make_unit_cell(1.0, 0.0, 1.0)
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, cell, 1e-6)
    return pz, src, q


def _worker(rank, world, port, outdir, uneven=False, coincident=False, scale=1.0):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import dist as pdist

    pz, src, q = _system(pw, coincident, scale)
    be = NumpyBackend(pw, pz, src, q)
    if uneven:  # a cost-balanced split (CudaBackend.near_split) need not be even: 80 / 20
        items = be.near_items()[0]
        be.near_split = lambda w: [0, (4 * items) // 5, items]
    plan = pdist.ShardPlan(len(src), len(src), world, rank)
    try:
        out, (lo, hi) = pdist.sharded_total_field(be, pdist.Comm(world), plan, symmetric=True)
    except pw.PeriwaveError as e:  # every rank must raise the same error (no hang)
        with open(os.path.join(outdir, f"err{rank}.txt"), "w") as f:
            f.write(e.code.name)
        dist.barrier()
        dist.destroy_process_group()
        return
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.concatenate([[lo, hi], out.scalar.numpy()]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partitions_cover_everything():
    from paper_2111_01083_b200 import dist as pdist

    for n in (0, 1, 7, 37, 1000):
        for world in (1, 2, 3, 8):
            got = []
            for r in range(world):
                lo, hi = pdist.contiguous(n, world, r)
                got.extend(range(lo, hi))
            assert got == list(range(n))
            got = []
            for r in range(world):
                lo, hi = pdist.target_slice(n, world, r)
                assert hi - lo <= pdist.target_chunk(n, world)
                got.extend(range(lo, hi))
            assert got == list(range(n))


def test_item_counts_match_the_device_decomposition(pw):
    cell = pw.make_unit_cell(1.0, 0.0, 1.0, pw.Periodicity.Singly)
    pz = pw.make_periodizer(pw.Pde.Poisson, 0.0, cell, 1e-10)
    for n, want in ((1, 1), (512, 1), (513, 2), (4095, None), (4096, None), (1000000, None)):
        items, nout = pw.near_sym_items(pz, n)
        if n < 4096:
            # Laplace image-loop tile: 512-point row tiles (4 targets x 128 threads), 128-point
            # column tiles, 32 column tiles (4096 sources) per item; row tile I starts at column tile 4 I
            nb, ncb, r, chunk = (n + 511) // 512, (n + 127) // 128, 4, 32
        else:
            # product-form tile (singly periodic, d a power of two, binned from 4096 points):
            # 1024-point row tiles (8 targets x 128 threads), 256-point column tiles, 4 per item
            nb, ncb, r, chunk = (n + 1023) // 1024, (n + 255) // 256, 4, 4
        assert items == sum((ncb - r * i + chunk - 1) // chunk for i in range(nb))
        assert nout == 1
        if want is not None:
            assert items == want
    # any period takes the product-form tile's decomposition (unscaled form when d is not a power of two)
    pz15 = pw.make_periodizer(pw.Pde.Poisson, 0.0, pw.make_unit_cell(1.5, 0.0, 1.0, pw.Periodicity.Singly), 1e-10)
    n = 1000000
    nb, ncb = (n + 1023) // 1024, (n + 255) // 256
    assert pw.near_sym_items(pz15, n)[0] == sum((ncb - 4 * i + 3) // 4 for i in range(nb))
    # the full precision tier (eps < 1e-11) keeps the image-loop tile
    pzf = pw.make_periodizer(pw.Pde.Poisson, 0.0, cell, 1e-12)
    nb, ncb = (n + 511) // 512, (n + 127) // 128
    assert pw.near_sym_items(pzf, n)[0] == sum((ncb - 4 * i + 31) // 32 for i in range(nb))
    st = pw.make_periodizer(pw.Pde.Stokes, 0.0, pw.make_unit_cell(1.0, 0.0, 1.0), 1e-8)
    assert pw.near_sym_items(st, 300, pw.ApplyOptions(with_pressure=True))[1] == 3


def test_two_ranks_gloo_equal_one_rank(pw, port, tmp_path):
    import torch.multiprocessing as mp

    from paper_2111_01083_b200 import dist as pdist

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    parts = [np.load(tmp_path / f"r{r}.npy") for r in range(world)]
    two = np.concatenate([p[2:] for p in parts])
    assert [(int(p[0]), int(p[1])) for p in parts] == [pdist.target_slice(37, 2, r) for r in range(2)]

    pz, src, q = _system(pw)
    be = NumpyBackend(pw, pz, src, q)
    one, _ = pdist.sharded_total_field(be, pdist.Comm(1), pdist.ShardPlan(37, 37, 1, 0), symmetric=True)
    one = one.scalar.numpy()
    # the Poisson far field carries ~1e9 weights on the lambda -> 0 modes, so a different
    # summation order of the all-reduce moves the gauge constant: compare mean-removed
    d = (two - two.mean()) - (one - one.mean())
    assert np.max(np.abs(d)) <= 1e-13 * np.max(np.abs(one))
    # against the direct sums: C restatement near images + the NumPy far field
    from oracle.pyoracle import near_shifts

    shifts, ident = near_shifts((1.0, 0.0, 1.0, 2))
    near, _ = port.near(port.LAPLACE, src, src, shifts, ident, q=q)
    coeff = be.coeff_buffer()
    be.far_source(0, 37, coeff)
    far = be.far_target(coeff, 0, 37).scalar.numpy()
    want = near[:, 0] + far
    assert np.max(np.abs(one - want)) <= 1e-12 * np.max(np.abs(want))
    # the near part alone is exact integer arithmetic: two ranks == one rank bitwise
    be2 = NumpyBackend(pw, pz, src, q)
    items, _ = be2.near_items()
    full = be2.accumulator(37 * 3)
    be2.near_partial(0, items, full)
    halves = be2.accumulator(37 * 3)
    for r in range(2):
        lo, hi = pdist.contiguous(items, 2, r)
        part = be2.accumulator(37 * 3)
        be2.near_partial(lo, hi, part)
        halves += part
    assert np.array_equal(full.numpy(), halves.numpy())


def test_two_ranks_gloo_uneven_item_split(pw, port, tmp_path):
    """dist.sharded_total_field honours the backend's item bounds (pwb_near_sym_split's
    cost-balanced ranges are uneven by count); the result equals the even split's."""
    import torch.multiprocessing as mp

    from paper_2111_01083_b200 import dist as pdist

    world = 2
    outs = {}
    for uneven in (False, True):
        d = tmp_path / ("u" if uneven else "e")
        d.mkdir()
        mp.start_processes(_worker, args=(world, _free_port(), str(d), uneven), nprocs=world, join=True,
                           start_method="spawn")
        outs[uneven] = np.concatenate([np.load(d / f"r{r}.npy")[2:] for r in range(world)])
    a, b = outs[False], outs[True]
    assert np.max(np.abs((a - a.mean()) - (b - b.mean()))) <= 1e-13 * np.max(np.abs(a))


def test_two_ranks_coincidence_raises_on_every_rank(pw, port, tmp_path):
    """A coincident pair lives in one rank's item range only; the status all-reduce makes
    every rank raise CoincidentSourceTarget (apply.cpp:544-545) instead of the owner
    raising while its peer blocks in the reduce-scatter."""
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), False, True), nprocs=world, join=True,
                       start_method="spawn")
    assert [(tmp_path / f"err{r}.txt").read_text() for r in range(world)] == ["CoincidentSourceTarget"] * 2
    # exactly one rank's item range holds the pair
    pz, src, q = _system(pw, coincident=True)
    be = NumpyBackend(pw, pz, src, q)
    items, _ = be.near_items()
    from paper_2111_01083_b200 import dist as pdist

    seen = [be.near_partial(*pdist.contiguous(items, 2, r), be.accumulator(37 * 3))[1] for r in range(2)]
    assert sorted(seen) == [0, 1]


@pytest.mark.parametrize("scale", [1e-15, 1e15])
def test_two_ranks_scaled_strengths(pw, port, tmp_path, scale):
    """The fixed-point scale follows the strengths: results scale exactly with them."""
    import torch.multiprocessing as mp

    world = 2
    outs = {}
    for sc in (1.0, scale):
        d = tmp_path / f"s{sc:g}"
        d.mkdir()
        mp.start_processes(_worker, args=(world, _free_port(), str(d), False, False, sc), nprocs=world, join=True,
                           start_method="spawn")
        outs[sc] = np.concatenate([np.load(d / f"r{r}.npy")[2:] for r in range(world)])
    a, b = outs[1.0], outs[scale] / scale
    assert np.max(np.abs((a - a.mean()) - (b - b.mean()))) <= 1e-12 * np.max(np.abs(a))
