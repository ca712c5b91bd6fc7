#!/usr/bin/env python
"""Benchmark: targets/s of the periodic evaluation on BASELINE.json's headline workload.

Workload (default c4, the config the metric "targets/sec at N=1e6, eps=1e-10" is quoted on):
singly periodic Laplace, 1x1 cell, N=1e6 sources from 16 Gaussian clusters, targets =
sources, eps = 1e-10, fp64. One step = one total_field (far plane-wave apply + fused near
images) over all targets, inputs resident in HBM.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c4]

N > 1 (torchrun, one rank per GPU, NCCL): targets are split in contiguous slices (strong
scaling: the job is fixed), every rank holds all sources for the near images, the S2PW
source sums run on a source slice per rank and meet in one ncclAllReduce(fp64, sum) of the
plane-wave coefficient buffer. Time = CUDA events on the launch stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "targets/sec at N=1e6, eps=1e-10, fp64, 1/2/4/8 B200; % of FP64 roofline"
# SURVEY.md §8(d) algorithmic flops per near pair (one image of one (target, source))
F_PAIR = {"c1": 29, "c2": 153, "c3": 48, "c4": 29, "c5": 94}
F_FAR = {"c1": 70, "c2": 70, "c3": 86, "c4": 70, "c5": 70}
# fp64-pipe instructions per (target, source) pair-group of the symmetric tile (all images),
# counted in the SASS of the fast inner loop (cuobjdump; profiles/r1_c4_near_sym_ncu.md)
# (tools/sass_loop_stats.py), per log tier (coarse: 256-entry table log when eps >= 1e-10):
# the reduced tier runs when eps >= 1e-11 unless
# PWB_FULL_PRECISION is set (pw_math.cuh log_pos_k)
FP64_INSTR_PER_GROUP = {("c4", "full"): 29.25, ("c4", "reduced"): 18.25, ("c4", "coarse"): 17.25,
                        ("c3", "full"): 103.0, ("c3", "reduced"): 83.0, ("c3", "coarse"): 82.0}
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r1_traffic.json")


def near_kernel_name(config, symmetric):
    """The dominant near launch of a config (engine.cu Plan::near, near.cu / near_sym.cu)."""
    fam = {"c1": ("SymLaplace", "Laplace", "3,3"), "c2": ("SymModHelm<grad>", "ModHelmGrad", "5,3"),
           "c3": ("SymStokes", "Stokes<no pressure>", "3,3"), "c4": ("SymLaplace", "Laplace", "3,1"),
           "c5": ("SymModHelm", "ModHelm", "3,3")}[config]
    binned = " on Morton-binned inputs" if config in ("c2", "c5") else ""
    if symmetric:
        return f"near_sym_kernel<{fam[0]},{fam[2]}> (fused near images, each unordered pair once){binned}"
    return f"near_tile_kernel<{fam[1]},{fam[2]}> (fused near images){binned}"


def measured_traffic(config, n):
    """dram bytes per launch of the dominant kernel from the committed ncu capture (same config, same N)."""
    try:
        with open(TRAFFIC_FILE) as f:
            t = json.load(f).get(config)
    except (OSError, ValueError):
        return None
    return t["bytes"] if t and t.get("n") == n else None
WORKLOAD = {
    "c1": "c1: doubly periodic Poisson, square cell, N=1000 uniform, targets=sources, eps=1e-10",
    "c2": "c2: doubly periodic mod. Helmholtz beta=10, cell (1,0.3,0.8), 1e5 src / 1e5 tgt, eps=1e-10, u+grad u",
    "c3": "c3: doubly periodic Stokes, square cell, N=1e6 uniform, targets=sources, eps=1e-8",
    "c4": "c4: singly periodic Poisson, 1x1 cell, N=1e6 from 16 Gaussian clusters (sigma 0.02), targets=sources,"
          " eps=1e-10",
    "c5": "c5: doubly periodic mod. Helmholtz beta=1, cell 100x1, N=1e7 uniform, targets=sources, eps=1e-8",
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        sm = [num(s[0]) for s in self.samples if num(s[0])]
        mx = [num(s[1]) for s in self.samples if num(s[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------- CPU reference arm
def reference_sample_times(inp, sizes, threads):
    """oracle/_ref total_field (Auto path, the reference's default) on target subsamples."""
    from oracle import pyoracle

    c = inp.config
    R = pyoracle.Ref().make_periodizer(int(c.pde), c.beta, tuple(float(v) for v in c.cell[:3]) + (int(c.cell[3]),),
                                       c.eps)
    kw = dict(charges=inp.charges) if c.strength == "charge" else dict(forces=inp.forces)
    out = []
    for s in sizes:
        tgt = inp.targets[inp.sample[:s]] if s <= len(inp.sample) else inp.targets[:s]
        t0 = time.perf_counter()
        R.apply(0, inp.sources, tgt, path=0, threads=threads, **kw)
        out.append((s, time.perf_counter() - t0))
    return out


def port_sample_times(inp, sizes, threads):
    """Fallback when oracle/_ref is absent: the C restatement, near images + direct far."""
    from oracle import pyoracle
    import paper_2111_01083_b200 as pw

    c = inp.config
    port = pyoracle.Port()
    shifts, ident = pyoracle.near_shifts(tuple(float(v) for v in c.cell[:3]) + (int(c.cell[3]),))
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    parts = pz.parts(pw.PART_SCALAR) if c.strength == "charge" else pz.parts(pw.PART_BLOCK)
    kind = {pw.Pde.Poisson: port.LAPLACE, pw.Pde.ModHelmholtz: port.MODHELM, pw.Pde.Stokes: port.STOKES}[c.pde]
    out = []
    for s in sizes:
        tgt = inp.targets[inp.sample[:s]] if s <= len(inp.sample) else inp.targets[:s]
        t0 = time.perf_counter()
        port.near(kind, inp.sources, tgt, shifts, ident, q=inp.charges, vec=inp.forces, beta=c.beta, threads=threads)
        port.far(parts, inp.sources, tgt, charges=inp.charges, forces=inp.forces, threads=threads)
        out.append((s, time.perf_counter() - t0))
    return out


def cpu_rate(inp, sizes, threads):
    """Fit t(N_T) = a + b N_T on the samples, extrapolate to the full target count."""
    from oracle import pyoracle

    if pyoracle.ref_available():
        kind, samples = "reference", reference_sample_times(inp, sizes, threads)
    else:
        kind, samples = "port", port_sample_times(inp, sizes, threads)
    (s1, t1), (s2, t2) = samples[0], samples[-1]
    b = (t2 - t1) / (s2 - s1) if s2 != s1 else t2 / s2
    a = max(0.0, t1 - b * s1)
    nt = len(inp.targets)
    t_full = a + b * nt
    return {"value": nt / t_full, "unit": "targets/s", "cores": threads, "kind": kind,
            "sample": f"all {len(inp.sources)} sources, target subsamples {sizes} timed "
                      f"({', '.join(f'{t:.2f}s' for _, t in samples)}); t(N_T)=a+b*N_T extrapolated to "
                      f"N_T={nt} (a={a:.3f}s, b={b:.3e}s)",
            "extrapolated_seconds": t_full}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2111_01083_b200 import configs

    from oracle import pyoracle

    inp = configs.generate(args.config)
    threads = os.cpu_count() or 1
    s = args.cpu_sample
    timer = reference_sample_times if pyoracle.ref_available() else port_sample_times
    kind = "reference" if pyoracle.ref_available() else "port"
    t_all0 = time.perf_counter()
    for _ in range(args.warmup):  # one bounded sample per warm-up step
        timer(inp, [s // 2], threads)
    # timed steps alternate target subsamples S and 2S; t(N_T) = a + b N_T from the medians
    runs = {s: [], 2 * s: []}
    for k in range(args.steps):
        size = s if k % 2 == 0 else 2 * s
        runs[size].extend(t for _, t in timer(inp, [size], threads))
    if not runs[2 * s]:
        runs[2 * s].extend(t for _, t in timer(inp, [2 * s], threads))
    wall = time.perf_counter() - t_all0
    t1, t2 = statistics.median(runs[s]), statistics.median(runs[2 * s])
    b = max((t2 - t1) / s, 1e-30)
    a = max(0.0, t1 - b * s)
    nt = len(inp.targets)
    value = nt / (a + b * nt)
    cb = {"value": value, "unit": "targets/s", "cores": threads, "kind": kind,
          "sample": f"each step: all {len(inp.sources)} sources, a seeded target subsample of {s} or {2 * s} "
                    f"(median {t1:.2f}s / {t2:.2f}s); t(N_T)=a+b*N_T extrapolated to N_T={nt} "
                    f"(a={a:.3f}s, b={b:.3e}s)",
          "extrapolated_seconds": a + b * nt}
    line = {"metric": METRIC, "value": value, "unit": "targets/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(1, args.steps + args.warmup),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md §8(d))", "impl": "reference",
            "config": {"workload": WORKLOAD[args.config], "n_src": len(inp.sources), "n_tgt": len(inp.targets),
                       "path": "auto (reference default)"},
            "cpu_baseline": cb, "e2e": {"value": value, "unit": "targets/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOAD))
    ap.add_argument("--cpu-sample", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs

    ws, rank, local = dist_env()
    # PWB_BENCH_SHARDED=1 runs the multi-GPU code path (NCCL process group, sharded far and
    # near passes, collectives) even at world size 1, to exercise it on a single-GPU box
    sharded = ws > 1 or os.environ.get("PWB_BENCH_SHARDED") == "1"
    if sharded:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()

    inp = configs.generate(args.config)
    c = inp.config
    cell = pw.make_unit_cell(c.cell[0], c.cell[1], c.cell[2], c.cell[3])
    t_b0 = time.perf_counter()
    pz = pw.make_periodizer(c.pde, c.beta, cell, c.eps)  # host builder (reported apart)
    build_ms = (time.perf_counter() - t_b0) * 1e3
    ns, nt = len(inp.sources), len(inp.targets)
    from paper_2111_01083_b200.dist import target_slice

    t_lo, t_hi = target_slice(nt, ws, rank)  # rank's targets (outputs stay sharded)
    kw_name = "charges" if c.strength == "charge" else "forces"
    strength = inp.charges if c.strength == "charge" else inp.forces

    src_d = torch.from_numpy(inp.sources).to(dev)
    str_d = torch.from_numpy(strength).to(dev)
    # targets = sources (c1, c3, c4, c5): hand the library the same array so the symmetric
    # near tile (each unordered pair once) applies; shards and separate targets are copies
    same = not sharded and not c.separate_targets
    tgt_d = src_d if same else torch.from_numpy(np.ascontiguousarray(inp.targets[t_lo:t_hi])).to(dev)
    opt = pw.ApplyOptions(path=pw.ApplyPath.Auto, with_gradient=c.gradient, stream=stream.cuda_stream)
    full = pw.ParticleSystem(sources=src_d, targets=tgt_d, **{kw_name: str_d})
    out = pw.FieldResult()
    from paper_2111_01083_b200 import dist as pdist

    symmetric = not c.separate_targets
    if sharded:
        tgt_all = None if symmetric else torch.from_numpy(np.ascontiguousarray(inp.targets)).to(dev)
        backend = pdist.CudaBackend(pw, pz, opt, src_d, str_d, kw_name, tgt_all)
        plan = pdist.ShardPlan(ns, nt, ws, rank)
        comm = pdist.Comm(ws)

    def step():
        nonlocal out
        if not sharded:
            out = pw.total_field(pz, full, opt)
            return
        # S2PW on my source slice + allreduce(fp64) of the coefficients; PW2T on my target
        # slice; symmetric near items + reduce-scatter(int64) of the fixed-point sums
        out, _ = pdist.sharded_total_field(backend, comm, plan, symmetric)

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)  # > 126 MB L2
    torch.cuda.synchronize()
    t_f0 = time.perf_counter()
    first_ms = None
    for k in range(args.warmup):
        step()
        if k == 0:  # first call: plan upload (mode tables, NUFFT setup, cuFFT plans) + one step
            torch.cuda.synchronize()
            first_ms = (time.perf_counter() - t_f0) * 1e3
    torch.cuda.synchronize()

    fd, nd = ctypes_doubles()
    launches0 = launch_count(pw)
    near_ms = []
    step_ms = []
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local if ws > 1 else 0) as clocks:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush between timed iterations (not timed)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            pw.lib().pwb_last_phase_ms(pz.handle, -1, fd, nd)
            near_ms.append(nd._obj.value)
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    launches = (launch_count(pw) - launches0) / args.steps
    t_step = sum(step_ms) / args.steps
    t_near = sum(near_ms) / args.steps
    if sharded:
        tt = torch.tensor([t_step, t_near], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_near = float(tt[0]), float(tt[1])

    # ---- end to end through the public API from pinned host memory (H2D + compute + D2H)
    src_h = torch.from_numpy(inp.sources).pin_memory()
    str_h = torch.from_numpy(strength).pin_memory()
    tgt_h = src_h if same else torch.from_numpy(np.ascontiguousarray(inp.targets[t_lo:t_hi])).pin_memory()
    tgt_all_h = None if not c.separate_targets else torch.from_numpy(np.ascontiguousarray(inp.targets)).pin_memory()
    e2e_ms = []
    host_sys = pw.ParticleSystem(sources=src_h, targets=tgt_h, **{kw_name: str_h})
    for k in range(args.e2e_steps + 1):
        if sharded:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if not sharded:
            r = pw.total_field(pz, host_sys, opt)  # library stages H2D / D2H on `stream`
        else:
            s_d = src_h.to(dev, non_blocking=True)
            q_d = str_h.to(dev, non_blocking=True)
            t_d = None if symmetric else tgt_all_h.to(dev, non_blocking=True)
            be = pdist.CudaBackend(pw, pz, opt, s_d, q_d, kw_name, t_d)
            rr, _ = pdist.sharded_total_field(be, comm, plan, symmetric)
            host_out = (rr.scalar if rr.scalar is not None else rr.velocity).to("cpu", non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        if k > 0:  # first one warms the staging buffers
            e2e_ms.append(e0.elapsed_time(e1))
    t_e2e = sum(e2e_ms) / len(e2e_ms)
    if sharded:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt[0])
    nout = 1 if c.strength == "charge" else 2
    # bytes of the tensors copied per e2e step: sources + strengths (+ targets when separate)
    h2d = 8 * (2 * ns + (1 if c.strength == "charge" else 2) * ns) + (16 * nt if c.separate_targets else 0)
    d2h = 8 * nout * (t_hi - t_lo) + (16 * (t_hi - t_lo) if c.gradient else 0)

    # ---- roofline of the dominant kernel (fused near-image P2P tile)
    import ctypes

    peak = ctypes.c_double(0.0)
    pw.lib().pwb_fp64_peak_probe(-1, ctypes.byref(peak))
    nimg = len(pw.near_translations(cell))
    # pairs handled by this rank's near launch (symmetric items split evenly across ranks)
    pairs = nimg * ns * nt / ws if (symmetric and sharded) else nimg * ns * (t_hi - t_lo)
    flops_near = pairs * F_PAIR[args.config]
    achieved = flops_near / (t_near * 1e-3) / 1e12
    rank_far = pz.rank()
    far_flops = rank_far * (ns + nt) * F_FAR[args.config]
    # hardware view: issued fp64 instructions of the fused symmetric tile (static SASS count per
    # (target, source) pair-group covering all images, profiles/r1_c4_near_sym_ncu.md) over the
    # DFMA instruction peak (peak TFLOP/s / 2)
    pipe_frac = None
    tier = "reduced" if (c.eps >= 1e-11 and not os.environ.get("PWB_FULL_PRECISION")) else "full"
    if tier == "reduced" and c.eps >= 1e-10 and not os.environ.get("PWB_NO_COARSE"):
        tier = "coarse"  # 256-entry table log (engine.cu a.coarse_log)
    if same and (args.config, tier) in FP64_INSTR_PER_GROUP and not sharded:
        groups = ns * (ns + 1) / 2.0
        pipe_frac = groups * FP64_INSTR_PER_GROUP[(args.config, tier)] / (t_near * 1e-3) / (peak.value * 1e12 / 2.0)

    line = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_rate(inp, [args.cpu_sample, 2 * args.cpu_sample], os.cpu_count() or 1)
            except Exception as e:  # reported, not fatal
                cpu = {"value": None, "unit": "targets/s", "cores": os.cpu_count(), "kind": "unavailable",
                       "sample": f"failed: {e}"}
        value = nt / (t_step * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": "targets/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": {"workload": WORKLOAD[args.config], "n_src": ns, "n_tgt": nt, "eps": c.eps,
                       "path": "auto", "rank": rank_far, "near_images": nimg,
                       "l2": "256 MB flush buffer written between timed iterations (inputs 24-40 MB < L2)",
                       "parallelism": f"targets split {ws}-way, S2PW sources split {ws}-way + NCCL allreduce"
                       if sharded else "single GPU"},
            "e2e": {"value": nt / (t_e2e * 1e-3), "unit": "targets/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                         "frac": achieved / peak.value if peak.value else None,
                         "traffic": measured_traffic(args.config, ns) if not sharded else None,
                         "log_tier": tier,
                         "kernel": near_kernel_name(args.config, same and (ns >= 32768 or sharded)),
                         "near_ms_per_launch": t_near, "far_ms": t_step - t_near,
                         "fp64_pipe_frac": pipe_frac,
                         "note": "frac > 1: the fused symmetric tile evaluates each unordered (target, source)"
                                 " pair once with one log for all images; the survey model charges 29 flop per"
                                 " image per ordered pair. fp64_pipe_frac is the hardware efficiency"
                                 " (issued DFMA-pipe instructions / DFMA peak); ncu cross-check in profiles/",
                         "algorithmic_flops_per_launch": flops_near,
                         "flop_model": f"SURVEY.md §8(d): {F_PAIR[args.config]} flop per (image, target, source) "
                                       f"pair x {nimg} images x {ns} x {t_hi - t_lo}; far {far_flops:.3e} flop "
                                       f"(rank {rank_far}) not in the kernel figure",
                         "peak_source": "measured on this box: best-of DFMA-chain burst (pwb_fp64_peak_probe); "
                                        "MEASURED_PEAKS.json has no fp64 entry; spec 37.2 TFLOP/s"},
            "clocks": clocks.summary(),
            "host_setup": {"periodizer_build_ms": build_ms, "first_call_ms": first_ms,
                           "note": "host periodizer build (own C++ builder) and the first total_field "
                                   "(plan upload + one step), both outside the timed region"},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def ctypes_doubles():
    import ctypes

    a, b = ctypes.c_double(0.0), ctypes.c_double(0.0)
    return ctypes.byref(a), ctypes.byref(b)


def launch_count(pw):
    import ctypes

    n = ctypes.c_long(0)
    pw.lib().pwb_launch_count(ctypes.byref(n))
    return n.value


if __name__ == "__main__":
    sys.exit(main())
