"""Near-field time with inputs in generator order vs spatially sorted order.

    python tools/sort_experiment.py c2 [--n N]

Prints the near-phase milliseconds (library events) for both orders; used to decide
whether the engine should bin points before the near tile (K0 branch divergence)."""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def morton_order(pts, bits=8):
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    g = np.clip(((pts - lo) / np.maximum(hi - lo, 1e-300) * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros(len(pts), dtype=np.int64)
    for b in range(bits):
        key |= ((g[:, 0] >> b) & 1) << (2 * b)
        key |= ((g[:, 1] >> b) & 1) << (2 * b + 1)
    return np.argsort(key, kind="stable")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c2", nargs="?")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs

    inp = configs.generate(args.config, n_src=args.n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    kwn = "charges" if c.strength == "charge" else "forces"
    w = inp.charges if kwn == "charges" else inp.forces
    sep = c.separate_targets
    for label in ("generator", "morton"):
        src, ww, tgt = inp.sources, w, inp.targets
        if label == "morton":
            ps = morton_order(src)
            src, ww = src[ps], w[ps]
            tgt = tgt[morton_order(tgt)] if sep else src
        s_d = torch.from_numpy(np.ascontiguousarray(src)).cuda()
        t_d = torch.from_numpy(np.ascontiguousarray(tgt)).cuda() if sep else s_d
        sysd = pw.ParticleSystem(sources=s_d, targets=t_d, **{kwn: torch.from_numpy(np.ascontiguousarray(ww)).cuda()})
        opt = pw.ApplyOptions(with_gradient=c.gradient)
        times = []
        for _ in range(args.reps):
            pw.total_field(pz, sysd, opt)
            torch.cuda.synchronize()
            fd, nd = ctypes.c_double(), ctypes.c_double()
            pw.lib().pwb_last_phase_ms(pz.handle, -1, ctypes.byref(fd), ctypes.byref(nd))
            times.append(nd.value)
        print(f"{args.config} n={len(src)} {label}: near ms {min(times):.2f} (all {[round(t, 2) for t in times]})",
              flush=True)


if __name__ == "__main__":
    main()
