"""Multi-GPU total_field: one process per GPU, NCCL through torch.distributed.

The path shards with exactly two exchange steps:

* far field -- the plane-wave coefficient buffer is linear in the sources: every rank
  runs S2PW on a contiguous source slice, one all-reduce (fp64, sum) of <= ~0.3 MB
  forms the global buffer, then every rank evaluates PW2T on its target slice;
* near field, targets == sources -- the unordered (target, source) pairs are cut into
  work items (pwb_near_sym_items); every rank runs a contiguous item range into its
  own int64 fixed-point accumulator over ALL targets, one reduce-scatter (int64 sum,
  exact and order-independent) hands each rank the accumulator of its target slice.
  Before it, one tiny all-reduce (MAX) of the ranks' status words: a coincidence any
  rank found raises the reference's CoincidentSourceTarget on every rank.
  With separate targets the near field is target-sharded with no exchange.

Outputs stay sharded: rank r owns targets [r*chunk, min(n, (r+1)*chunk)),
chunk = ceil(n / world). The host logic is backend-agnostic (`Backend`), so it is
tested on CPU with gloo (tests/test_dist_gloo.py) and run on B200s with `CudaBackend`.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


def contiguous(n: int, world: int, rank: int):
    """Balanced contiguous split of range(n): (lo, hi) for `rank`."""
    return (n * rank) // world, (n * (rank + 1)) // world


def target_chunk(n: int, world: int) -> int:
    return max(1, math.ceil(n / world))


def target_slice(n: int, world: int, rank: int):
    c = target_chunk(n, world)
    lo = min(n, rank * c)
    return lo, min(n, lo + c)


def _host_staged(op, t):
    """gloo reduces host tensors: a device tensor goes through a host copy (NCCL and host
    tensors are reduced in place)."""
    import torch.distributed as dist

    if t.device.type == "cpu" or dist.get_backend() == "nccl":
        op(t)
        return t
    h = t.cpu()
    op(h)
    t.copy_(h)
    return t


class Comm:
    """all_reduce / reduce_scatter (sum) over the default process group; world 1 is local."""

    def __init__(self, world: int):
        self.world = world

    def allreduce(self, t):
        if self.world > 1:
            import torch.distributed as dist

            _host_staged(dist.all_reduce, t)
        return t

    def allreduce_max(self, t):
        if self.world > 1:
            import torch.distributed as dist

            _host_staged(lambda x: dist.all_reduce(x, op=dist.ReduceOp.MAX), t)
        return t

    def reduce_scatter(self, inp, out):
        """out = (sum over ranks of inp)[rank * len(out) : (rank + 1) * len(out)]."""
        if self.world == 1:
            out.copy_(inp[: out.numel()])
            return out
        import torch.distributed as dist

        if dist.get_backend() == "nccl":
            dist.reduce_scatter_tensor(out, inp)
        else:  # gloo has no reduce-scatter: all-reduce (on the host) then keep the own slice
            tmp = inp.cpu() if inp.device.type != "cpu" else inp.clone()
            dist.all_reduce(tmp)
            r = dist.get_rank()
            out.copy_(tmp[r * out.numel():(r + 1) * out.numel()])
        return out


@dataclass
class ShardPlan:
    n_src: int
    n_tgt: int
    world: int
    rank: int

    @property
    def sources(self):
        return contiguous(self.n_src, self.world, self.rank)

    @property
    def targets(self):
        return target_slice(self.n_tgt, self.world, self.rank)

    @property
    def chunk(self):
        return target_chunk(self.n_tgt, self.world)


def sharded_total_field(backend, comm: Comm, plan: ShardPlan, symmetric: bool):
    """One rank's share of total_field; returns (local output, (t_lo, t_hi))."""
    s_lo, s_hi = plan.sources
    t_lo, t_hi = plan.targets
    coeff = backend.coeff_buffer()
    backend.far_source(s_lo, s_hi, coeff)
    comm.allreduce(coeff)
    out = backend.far_target(coeff, t_lo, t_hi)
    if symmetric:
        items, nout = backend.near_items()
        # balanced item ranges: by estimated cost for the screened kernels (identical on
        # every rank: the same points give the same bounds), by count otherwise
        split = getattr(backend, "near_split", None)
        if split is not None:
            bounds = split(plan.world)
            i_lo, i_hi = bounds[plan.rank], bounds[plan.rank + 1]
        else:
            i_lo, i_hi = contiguous(items, plan.world, plan.rank)
        acc = backend.accumulator(plan.chunk * plan.world * nout * 3)
        scale_exp, status = backend.near_partial(i_lo, i_hi, acc)
        # agree on the status before the reduce-scatter: a coincidence seen by one rank
        # raises CoincidentSourceTarget on every rank (no peer left blocked in the
        # collective); the fixed-point scale must be the same everywhere (it is derived
        # from the global strengths) -- max(k) == -max(-k) checks it
        flags = comm.allreduce_max(backend.small_ints([status, scale_exp, -scale_exp]))
        status, k_hi, k_lo = (int(v) for v in flags.tolist())
        from . import raise_sym_status

        raise_sym_status(status)
        if k_hi != -k_lo:
            raise RuntimeError(f"ranks disagree on the fixed-point scale ({-k_lo}..{k_hi}): "
                               "every rank must hold the same strengths")
        mine = backend.accumulator(plan.chunk * nout * 3)
        comm.reduce_scatter(acc, mine)
        backend.fixed_to_out(mine, t_hi - t_lo, out, scale_exp)
    else:
        backend.near_targets(t_lo, t_hi, out)
    return out, (t_lo, t_hi)


class CudaBackend:
    """The B200 kernels through the C-ABI, device-resident inputs (torch tensors)."""

    def __init__(self, pw, pz, opt, sources, strength, strength_name, targets=None):
        import torch

        self.pw, self.pz, self.opt = pw, pz, opt
        self.src, self.q, self.kw = sources, strength, strength_name
        self.tgt = sources if targets is None else targets
        self.ns, self.nt = sources.shape[0], self.tgt.shape[0]
        self.torch = torch
        self.dev = sources.device

    def coeff_buffer(self):
        n = self.pw.far_coeff_size(self.pz, self.opt, self.ns, self.nt)
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def far_source(self, lo, hi, coeff):
        sys_ = self.pw.ParticleSystem(sources=self.src[lo:hi], **{self.kw: self.q[lo:hi]})
        self.pw.far_source_pass(self.pz, sys_, coeff, self.opt, self.ns, self.nt)

    def far_target(self, coeff, lo, hi):
        sys_ = self.pw.ParticleSystem(sources=self.src, targets=self.tgt[lo:hi], **{self.kw: self.q})
        return self.pw.far_target_pass(self.pz, sys_, coeff, self.opt, None, self.ns, self.nt)

    def near_items(self):
        return self.pw.near_sym_items(self.pz, self.ns, self.opt)

    def accumulator(self, n):
        return self.torch.zeros(n, dtype=self.torch.int64, device=self.dev)

    def small_ints(self, vals):
        return self.torch.tensor(vals, dtype=self.torch.int64, device=self.dev)

    def near_partial(self, lo, hi, acc):
        """-> (scale_exp, status) of pwb_near_sym_partial."""
        sys_ = self.pw.ParticleSystem(sources=self.src, targets=self.src, **{self.kw: self.q})
        return self.pw.near_sym_partial(self.pz, sys_, acc, lo, hi, self.opt)

    def near_split(self, world):
        sys_ = self.pw.ParticleSystem(sources=self.src, targets=self.src, **{self.kw: self.q})
        return self.pw.near_sym_split(self.pz, sys_, world, self.opt)

    def fixed_to_out(self, acc, n, out, scale_exp):
        ref = out.scalar if out.scalar is not None else out.velocity
        self.pw.fixed_to_field(self.pz, acc, n, out, self.opt, like=ref, scale_exp=scale_exp)

    def near_targets(self, lo, hi, out):
        sys_ = self.pw.ParticleSystem(sources=self.src, targets=self.tgt[lo:hi], **{self.kw: self.q})
        self.pw.near_field(self.pz, sys_, self.opt, out)
