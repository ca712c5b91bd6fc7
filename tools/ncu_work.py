"""Evaluated fp64 work of one near launch from an ncu --set full capture (raw page CSV).

    python tools/ncu_work.py CONFIG RAW_CSV --n-src N [--n-tgt M] [--symmetric 0|1] [--update]

Reads the executed thread-level fp64 instruction counts (DFMA, DADD, DMUL; predicated-on
lanes only), the launch duration and the DRAM bytes of the captured kernel and prints the
per-launch and per-pair-group figures. --update writes them into profiles/work_model.json,
which bench.py turns into the hardware roofline fraction of the live run:

    achieved = (2 DFMA + DADD + DMUL per pair-group) x pair-groups / near time

A pair-group is one (target, source) pair over all near images: n_src (n_src + 1) / 2 for
the symmetric tile (each unordered pair once, the self pairs included), n_src n_tgt for the
one-sided tile.
"""
from __future__ import annotations

import argparse
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODEL = os.path.join(ROOT, "profiles", "work_model.json")


def read_raw(path):
    rows = list(csv.reader(open(path)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append({k: (u, v) for k, u, v in zip(head, units, r)})
    return out


def num(rec, key):
    u, v = rec[key]
    return float(v.replace(",", ""))


def to_bytes(rec, key):
    u, v = rec[key]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * scale


def to_seconds(rec, key):
    u, v = rec[key]
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3}.get(u, 1e-9)
    return float(v.replace(",", "")) * scale


def work(rec):
    cyc = num(rec, "smsp__cycles_elapsed.avg")
    ins = {op: num(rec, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") * cyc
           for op in ("dfma", "dadd", "dmul")}
    return {
        "kernel": rec["Kernel Name"][1],
        "launch_s": to_seconds(rec, "gpu__time_duration.sum"),
        "thread_instr": ins,
        "fp64_flops": 2 * ins["dfma"] + ins["dadd"] + ins["dmul"],
        "fp64_instr": sum(ins.values()),
        "dram_bytes": to_bytes(rec, "dram__bytes_read.sum") + to_bytes(rec, "dram__bytes_write.sum"),
        "fp64_pipe_pct": num(rec, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("raw")
    ap.add_argument("--n-src", type=int, required=True)
    ap.add_argument("--n-tgt", type=int, default=None)
    ap.add_argument("--symmetric", type=int, default=1)
    ap.add_argument("--update", action="store_true")
    args = ap.parse_args()
    recs = read_raw(args.raw)
    w = work(max(recs, key=lambda r: to_seconds(r, "gpu__time_duration.sum")))
    ns = args.n_src
    nt = args.n_tgt or ns
    groups = ns * (ns + 1) / 2 if args.symmetric else float(ns) * nt
    entry = {
        "capture": os.path.relpath(args.raw, ROOT), "n_src": ns, "n_tgt": nt, "symmetric": bool(args.symmetric),
        "pair_groups": groups, "kernel": w["kernel"], "launch_ms": w["launch_s"] * 1e3,
        "fp64_thread_instr": w["thread_instr"], "fp64_flops_per_launch": w["fp64_flops"],
        "fp64_flops_per_group": w["fp64_flops"] / groups, "fp64_instr_per_group": w["fp64_instr"] / groups,
        "dram_bytes_per_launch": w["dram_bytes"], "fp64_pipe_pct": w["fp64_pipe_pct"],
    }
    print(json.dumps(entry, indent=1))
    if args.update:
        model = json.load(open(MODEL)) if os.path.exists(MODEL) else {}
        model[args.config] = entry
        with open(MODEL, "w") as f:
            json.dump(model, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main()
