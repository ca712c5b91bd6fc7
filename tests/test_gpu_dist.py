"""Two real processes running dist.sharded_total_field on the B200 kernels (CudaBackend).

Both ranks sit on cuda:0 and talk over gloo (one GPU per box here); the kernels of one
rank never wait on the other's, only the host-side collectives meet. What this proves is
the sharded code path with world > 1 end to end through the C-ABI: the near field (int64
fixed-point partials + reduce-scatter) is bitwise the single call's, the far field (fp64
all-reduce of the plane-wave coefficients) agrees to 1e-13 after gauge removal, a
coincidence in one rank's item range raises on both ranks, and the separate-target path
(c2) is target-sharded with no near exchange.
"""
import os
import socket

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(name, n, coincident=False):
    from paper_2111_01083_b200 import configs

    inp = configs.generate(name, n_src=n)
    if coincident:  # a source on the (1, 0) image of another, far down the list: one rank's items hold the pair
        y = inp.sources[5, 1]
        inp.sources[5] = (-0.5, y)
        inp.sources[n - 3] = (0.5, y)
    return inp


def _worker(rank, world, port, outdir, name, n, coincident):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import dist as pdist

    import datetime

    torch.cuda.set_device(0)
    # a rank that dies must not leave its peer in a collective for gloo's 30-minute default
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=180))
    try:
        inp = _inputs(name, n, coincident)
        c = inp.config
        pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
        kw = "charges" if c.strength == "charge" else "forces"
        src = torch.from_numpy(inp.sources).cuda()
        q = torch.from_numpy(inp.charges if kw == "charges" else inp.forces).cuda()
        symmetric = not c.separate_targets
        tgt = None if symmetric else torch.from_numpy(np.ascontiguousarray(inp.targets)).cuda()
        opt = pw.ApplyOptions(with_gradient=c.gradient)
        plan = pdist.ShardPlan(n, len(inp.targets), world, rank)
        comm = pdist.Comm(world)
        be = pdist.CudaBackend(pw, pz, opt, src, q, kw, tgt)
        try:
            out, (lo, hi) = pdist.sharded_total_field(be, comm, plan, symmetric)
        except pw.PeriwaveError as e:
            with open(os.path.join(outdir, f"err{rank}.txt"), "w") as f:
                f.write(e.code.name)
            return

        class NearOnly(pdist.CudaBackend):
            def far_source(self, lo_, hi_, coeff):
                pass

            def far_target(self, coeff, lo_, hi_):
                r = super().far_target(coeff, lo_, hi_)
                for key in ("scalar", "velocity", "gradient"):
                    t = getattr(r, key, None)
                    if t is not None:
                        t.zero_()
                return r

        near, _ = pdist.sharded_total_field(NearOnly(pw, pz, opt, src, q, kw, tgt), comm, plan, symmetric)
        key = "scalar" if kw == "charges" else "velocity"
        res = {"lo": lo, "hi": hi, "total": getattr(out, key).cpu().numpy(), "near": getattr(near, key).cpu().numpy()}
        if c.gradient:
            res["grad"] = out.gradient.cpu().numpy()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), **res)
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _run(tmp_path, name, n, world=2, coincident=False):
    import torch.multiprocessing as mp

    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), name, n, coincident), nprocs=world,
                       join=True, start_method="spawn")


@pytest.mark.parametrize("name,n", [("c4", 40000), ("c3", 33000), ("c5", 34000)])
def test_two_processes_match_the_single_call(pw, gpu, tmp_path, name, n):
    import torch

    from paper_2111_01083_b200 import dist as pdist

    _run(tmp_path, name, n)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    assert [(int(p["lo"]), int(p["hi"])) for p in parts] == [pdist.target_slice(n, 2, r) for r in range(2)]
    total = np.concatenate([p["total"] for p in parts])
    near = np.concatenate([p["near"] for p in parts])

    inp = _inputs(name, n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    kw = "charges" if c.strength == "charge" else "forces"
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges if kw == "charges" else inp.forces).cuda()
    s = pw.ParticleSystem(sources=src, targets=src, **{kw: q})
    key = "scalar" if kw == "charges" else "velocity"
    # n >= 32768: the single call takes the same symmetric fixed-point tile -> bitwise
    one_near = getattr(pw.near_field(pz, s, pw.ApplyOptions()), key).cpu().numpy()
    assert np.array_equal(near, one_near)
    one = getattr(pw.total_field(pz, s, pw.ApplyOptions()), key).cpu().numpy()
    assert rel_l2(total, one, gauge=True) <= 1e-13


def test_two_processes_separate_targets(pw, gpu, tmp_path):
    """c2 shape (separate targets, gradient): target-sharded near field, no near exchange."""
    import torch

    n = 6000
    _run(tmp_path, "c2", n)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    inp = _inputs("c2", n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    s = pw.ParticleSystem(sources=torch.from_numpy(inp.sources).cuda(), charges=torch.from_numpy(inp.charges).cuda(),
                          targets=torch.from_numpy(np.ascontiguousarray(inp.targets)).cuda())
    one = pw.total_field(pz, s, pw.ApplyOptions(with_gradient=True))
    assert rel_l2(np.concatenate([p["total"] for p in parts]), one.scalar.cpu().numpy()) <= 1e-13
    assert rel_l2(np.concatenate([p["grad"] for p in parts]), one.gradient.cpu().numpy()) <= 1e-13


def test_two_processes_coincidence_raises_on_both_ranks(pw, gpu, tmp_path):
    _run(tmp_path, "c4", 40000, coincident=True)
    assert [(tmp_path / f"err{r}.txt").read_text() for r in range(2)] == ["CoincidentSourceTarget"] * 2
