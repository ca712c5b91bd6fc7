"""Wider parity check at full size: the GPU's full symmetric total_field of c3 / c4 (all
targets, the bench's path) against the compiled reference (oracle/_ref, Direct path, all
host threads) at a fresh seeded sample of targets, larger than the golden subsample.

    python tools/parity_wide.py [--targets 8192] [--configs c4 c3] > profiles/r1b_parity_wide.json

Test infrastructure: the reference is the checker here, never the thing measured."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--targets", type=int, default=8192)
    ap.add_argument("--configs", nargs="+", default=["c4", "c3"])
    args = ap.parse_args()
    import torch

    import paper_2111_01083_b200 as pw
    from conftest import rel_l2
    from oracle import pyoracle
    from paper_2111_01083_b200 import configs

    R = pyoracle.Ref()
    threads = os.cpu_count() or 1
    out = {}
    for name in args.configs:
        inp = configs.generate(name)
        c = inp.config
        pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
        kw = dict(charges=inp.charges) if c.strength == "charge" else dict(forces=inp.forces)
        src = torch.from_numpy(inp.sources).cuda()
        kwd = {k: torch.from_numpy(v).cuda() for k, v in kw.items()}
        r = pw.total_field(pz, pw.ParticleSystem(sources=src, targets=src, **kwd), pw.ApplyOptions())
        key = "scalar" if c.strength == "charge" else "velocity"
        got = getattr(r, key).cpu().numpy()
        rng = np.random.default_rng(20261020 + int(name[1]))
        idx = np.sort(rng.choice(len(inp.sources), args.targets, replace=False))
        rp = R.make_periodizer(int(c.pde), c.beta, tuple(float(v) for v in c.cell[:3]) + (int(c.cell[3]),), c.eps)
        want = rp.apply(0, inp.sources, np.ascontiguousarray(inp.sources[idx]), path=1, threads=threads, **kw)[key]
        gauge = c.pde in (pw.Pde.Poisson, pw.Pde.Stokes)
        err = rel_l2(got[idx], want, gauge)
        out[name] = {"eps": c.eps, "bar": 10 * c.eps, "n_src": len(inp.sources), "targets_checked": args.targets,
                     "seed": 20261020 + int(name[1]), "gpu_path": "total_field, Auto, symmetric tile (all targets)",
                     "reference_path": "oracle/_ref total_field, Direct, %d threads" % threads,
                     "rel_l2": err, "accelerated": bool(r.accelerated)}
        print(name, json.dumps(out[name]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
