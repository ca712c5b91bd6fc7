"""Instruction mix of the innermost hot loop of a kernel in the built library.

    python tools/sass_loop_stats.py 'SymLaplaceILb1EEELi3ELi1'  [--lib path] [--marker MUFU]

Finds the kernel(s) whose mangled name matches the regex, locates the smallest
backward-branch loop containing >= --min-markers marker instructions (default
MUFU.RCP64H: one per pair-group in the log-based tiles) and prints the opcode
counts and the fp64-pipe instructions per marker. Static analysis only (cuobjdump).
"""
import argparse
import os
import re
import subprocess
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FP64 = ("DFMA", "DADD", "DMUL")


def functions(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*);", line)
        if m and cur:
            body.append((int(m.group(1), 16), m.group(3), m.group(4)))
    if cur:
        yield cur, body


def hot_loop(ins, marker, min_markers):
    best = None
    for a, op, rest in ins:
        if not op.startswith("BRA"):
            continue
        m = re.search(r"0x([0-9a-f]+)", rest)
        if not m or int(m.group(1), 16) >= a:
            continue
        tgt = int(m.group(1), 16)
        body = [x for x in ins if tgt <= x[0] <= a]
        nm = sum(1 for x in body if x[1].startswith(marker))
        if nm >= min_markers and (best is None or len(body) < len(best)):
            best = body
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("pattern")
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2111_01083_b200", "libperiwave_b200.so"))
    ap.add_argument("--marker", default="MUFU.RCP64H")
    ap.add_argument("--min-markers", type=int, default=4)
    args = ap.parse_args()
    for name, ins in functions(args.lib):
        if not re.search(args.pattern, name):
            continue
        loop = hot_loop(ins, args.marker, args.min_markers)
        if loop is None:
            print(name, ": no loop with", args.marker)
            continue
        c = Counter(x[1].split(".")[0] for x in loop)
        nm = sum(1 for x in loop if x[1].startswith(args.marker))
        fp = sum(c[k] for k in FP64)
        print(f"{name}\n  loop {len(loop)} instr, {nm} x {args.marker}, fp64 {fp} "
              f"({fp / nm:.2f} per marker), all {len(loop) / nm:.2f} per marker")
        print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main()
