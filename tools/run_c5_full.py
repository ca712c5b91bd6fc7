"""One full-size c5 total_field (1e7 points, targets == sources) on cuda:0, timed, and checked
against the golden oracle subsample (tests/golden/c5.npz, 10*eps gauge-free bar).

    python tools/run_c5_full.py [--n N]

c5 is a parity configuration (9e14 pair-images); this records what the
full problem costs on one B200 rather than extrapolating it."""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=None)
    args = ap.parse_args()
    import torch

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs

    inp = configs.generate("c5", n_src=args.n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges).cuda()
    sysd = pw.ParticleSystem(sources=src, targets=src, charges=q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = pw.total_field(pz, sysd, pw.ApplyOptions())
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    fd, nd = ctypes.c_double(), ctypes.c_double()
    pw.lib().pwb_last_phase_ms(pz.handle, -1, ctypes.byref(fd), ctypes.byref(nd))
    out = {"config": "c5", "n": len(inp.sources), "wall_s": wall, "far_ms": fd.value, "near_ms": nd.value,
           "accelerated": bool(r.accelerated)}
    if args.n is None:
        g = np.load(os.path.join(ROOT, "tests", "golden", "c5.npz"))
        got = r.scalar.cpu().numpy()[g["sample"]]
        for key in ("direct", "accelerated"):
            if key in g:
                want = g[key]
                out[f"rel_l2_vs_{key}"] = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        out["bar"] = 10 * c.eps
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
