"""Relative l2 errors of the GPU path against the committed golden fixtures, per config.

    python tools/parity_report.py > profiles/r1b_parity.json

The same comparisons as tests/test_gpu_golden.py (the compiled reference's Direct
total_field at each config's seeded target subsample, all sources at full N; gauge-removed
for Poisson potentials and Stokes velocities), printed as numbers instead of asserted:
the subsample run (separate targets, one-sided tiles) and, for targets == sources, the full
symmetric run read at the subsample (the bench's path). c5 at full size is
tools/run_c5_full.py."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    import paper_2111_01083_b200 as pw
    from conftest import rel_l2
    from paper_2111_01083_b200 import configs

    out = {}
    for name in ("c1", "c2", "c3", "c4", "c5"):
        g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz")))
        inp = configs.generate(name)
        c = inp.config
        pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
        kw = dict(charges=inp.charges) if c.strength == "charge" else dict(forces=inp.forces)
        gauge = c.pde in (pw.Pde.Poisson, pw.Pde.Stokes)
        tgt = np.ascontiguousarray(inp.targets[g["sample"]])
        r = pw.total_field(pz, pw.ParticleSystem(sources=inp.sources, targets=tgt, **kw),
                           pw.ApplyOptions(path=pw.ApplyPath.Direct, with_gradient=c.gradient))
        got = r.scalar if c.strength == "charge" else r.velocity
        row = {"eps": c.eps, "bar": 10 * c.eps, "n_src": len(inp.sources), "subsample": len(tgt),
               "subsample_vs_reference_direct": rel_l2(got, g["direct"], gauge)}
        if c.gradient:
            row["gradient_vs_reference_multipole"] = rel_l2(r.gradient, g["gradient"])
        if "accelerated" in g:
            row["subsample_vs_reference_accelerated"] = rel_l2(got, g["accelerated"], gauge)
        if not c.separate_targets and name != "c5":
            src = torch.from_numpy(inp.sources).cuda()
            kwd = {k: torch.from_numpy(v).cuda() for k, v in kw.items()}
            rf = pw.total_field(pz, pw.ParticleSystem(sources=src, targets=src, **kwd), pw.ApplyOptions())
            full = (rf.scalar if c.strength == "charge" else rf.velocity).cpu().numpy()
            row["full_symmetric_auto_vs_reference_direct"] = rel_l2(full[g["sample"]], g["direct"], gauge)
        out[name] = row
        print(name, json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
