"""Generate the golden fixtures in tests/golden/ from the compiled reference (oracle/_ref).

TEST INFRASTRUCTURE. Run in the build container (the GPU box has no /root/reference,
but these fixtures travel with the repo):

    python tests/golden/make_golden.py [c1 c2 ...]

For every BASELINE.json config the full-size inputs are regenerated from their seeds
(paper_2111_01083_b200/configs.py, the reference's own Rng stream); the reference's
total_field runs on the oracle target subsample with all sources, on
the Direct path (the oracle of record) and, where Auto resolves to Accelerated, also on
the Auto path. Targets are independent, so the subsample values equal the full run's.
c2's gradient comes from the reference's l = 1 modified-Helmholtz multipole periodizer:
grad u = -(beta/2pi) (Re, Im) of its complex field.
Bessel evaluations use the fast GSL-shaped shim (oracle/shim/bessel_shim.cpp), pinned to
<= 2e-15 against std::cyl_bessel_k in tests/test_oracle_pins.py.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from paper_2111_01083_b200 import configs  # noqa: E402


def main(names):
    ref = pyoracle.Ref()
    threads = os.cpu_count() or 1
    for name in names:
        t0 = time.time()
        inp = configs.generate(name)
        c = inp.config
        cell = tuple(float(v) for v in c.cell[:3]) + (int(c.cell[3]),)
        R = ref.make_periodizer(int(c.pde), c.beta, cell, c.eps)
        tgt = np.ascontiguousarray(inp.targets[inp.sample])
        kw = dict(charges=inp.charges) if c.strength == "charge" else dict(forces=inp.forces)
        key = "scalar" if c.strength == "charge" else "velocity"
        out = {"sample": inp.sample.astype(np.int64)}
        direct = R.apply(0, inp.sources, tgt, path=1, threads=threads, **kw)
        out["direct"] = direct[key]
        auto_path = R.choose_path(len(inp.sources), len(inp.targets))
        meta = {"config": name, "n_src": len(inp.sources), "n_tgt": len(inp.targets), "eps": c.eps,
                "rank": R.rank(), "auto_path_full": ["Auto", "Direct", "Accelerated"][auto_path],
                "threads": threads, "generator": "paper_2111_01083_b200/configs.py", "seed": c.seed}
        if auto_path == 2:
            # the subsample run decides its own path from (n_src, n_sample); force the full-size choice
            acc = R.apply(0, inp.sources, tgt, path=2, threads=threads, **kw)
            out["accelerated"] = acc[key]
            meta["accelerated_flag"] = bool(acc["accelerated"])
        if c.gradient:
            M = ref.make_multipole_periodizer(int(c.pde), c.beta, 1, cell, c.eps)
            coef = np.stack([inp.charges, np.zeros_like(inp.charges)], -1)
            cs = M.apply(0, inp.sources, tgt, coefficients=coef, path=1, threads=threads)["complex"]
            out["gradient"] = -(c.beta / (2 * np.pi)) * cs
        meta["seconds"] = time.time() - t0
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(name, meta, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
