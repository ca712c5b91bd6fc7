"""One warm total_field of a config on cuda:0 (for ncu captures of the hot kernels).

    python tools/profile_step.py c4 [--sym 0|1] [--n N] [--strip W]

--strip W (c5): the N points drawn uniform in x in [-W/2, W/2] of c5's 100 x 1 cell, i.e. c5's
density (1e5 per unit area: N = 1e5 W) and tile geometry on a slice the profiler can replay.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c4", nargs="?")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--sym", type=int, default=1)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--strip", type=float, default=None)
    args = ap.parse_args()
    import torch

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs

    inp = configs.generate(args.config, n_src=args.n)
    c = inp.config
    if args.strip:
        import numpy as np

        n = len(inp.sources)
        u = configs.rng_uniform(c.seed + 31, 2 * n)
        inp.sources = np.ascontiguousarray(np.stack([(u[0::2] - 0.5) * args.strip, u[1::2] - 0.5], axis=1))
        inp.targets = inp.sources
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    tgt = src if (args.sym and not c.separate_targets) else torch.from_numpy(inp.targets.copy()).cuda()
    kw = {"charges" if c.strength == "charge" else "forces":
          torch.from_numpy(inp.charges if c.strength == "charge" else inp.forces).cuda()}
    s = pw.ParticleSystem(sources=src, targets=tgt, **kw)
    for _ in range(args.reps):
        r = pw.total_field(pz, s, pw.ApplyOptions(with_gradient=c.gradient))
    torch.cuda.synchronize()
    import ctypes

    fd, nd = ctypes.c_double(), ctypes.c_double()
    pw.lib().pwb_last_phase_ms(pz.handle, -1, ctypes.byref(fd), ctypes.byref(nd))
    print("ok", args.config, len(inp.sources), f"near_ms={nd.value:.2f} far_ms={fd.value:.2f}",
          float((r.scalar if r.scalar is not None else r.velocity).abs().sum()))


if __name__ == "__main__":
    main()
