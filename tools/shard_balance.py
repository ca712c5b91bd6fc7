"""Per-rank near-field time of the multi-GPU split, measured on one GPU.

    python tools/shard_balance.py c5 --n 1000000 [--worlds 2 4 8]

For each world size W the symmetric work items are split as a W-rank job would split them
(pwb_near_sym_split: cost-balanced for the screened kernels; PWB_COUNT_SPLIT=1 forces the
even split by count) and every rank's item range is run alone on this GPU with CUDA events
around it. max/mean over the ranks is the load imbalance the W-GPU job would see in its
dominant phase (the exchange is one int64 reduce-scatter, < 0.1 % of the step).
Prints one JSON line per W."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c5", nargs="?")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    args = ap.parse_args()
    import torch

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs

    inp = configs.generate(args.config, n_src=args.n)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    kw = "charges" if c.strength == "charge" else "forces"
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges if kw == "charges" else inp.forces).cuda()
    opt = pw.ApplyOptions(with_gradient=c.gradient)
    s = pw.ParticleSystem(sources=src, targets=src, **{kw: q})
    n = src.shape[0]
    items, nout = pw.near_sym_items(pz, n, opt)
    acc = torch.zeros(n * nout * 3, dtype=torch.int64, device="cuda")

    def timed(lo, hi):
        acc.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pw.near_sym_partial(pz, s, acc, lo, hi, opt)  # -> (scale_exp, status)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    timed(0, items)  # warm (plan, binning buffers)
    whole = timed(0, items)
    for w in args.worlds:
        bounds = pw.near_sym_split(pz, s, w, opt)
        ts = [timed(bounds[r], bounds[r + 1]) for r in range(w)]
        mean = sum(ts) / w
        print(json.dumps({"config": args.config, "n": n, "world": w,
                          "split": "count" if os.environ.get("PWB_COUNT_SPLIT") else "balanced",
                          "whole_ms": round(whole, 2), "rank_ms": [round(t, 2) for t in ts],
                          "max_over_mean": round(max(ts) / mean, 4),
                          "near_efficiency": round(whole / w / max(ts), 4)}), flush=True)


if __name__ == "__main__":
    main()
