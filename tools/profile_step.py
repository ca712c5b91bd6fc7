"""One warm total_field of a config on cuda:0 (for ncu captures of the hot kernels).

    python tools/profile_step.py c4 [--sym 0|1] [--n N]
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
    args = ap.parse_args()
    import torch

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs

    inp = configs.generate(args.config, n_src=args.n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    tgt = src if (args.sym and not c.separate_targets) else torch.from_numpy(inp.targets.copy()).cuda()
    kw = {"charges" if c.strength == "charge" else "forces":
          torch.from_numpy(inp.charges if c.strength == "charge" else inp.forces).cuda()}
    s = pw.ParticleSystem(sources=src, targets=tgt, **kw)
    for _ in range(args.reps):
        r = pw.total_field(pz, s, pw.ApplyOptions(with_gradient=c.gradient))
    torch.cuda.synchronize()
    print("ok", args.config, float((r.scalar if r.scalar is not None else r.velocity).abs().sum()))


if __name__ == "__main__":
    main()
