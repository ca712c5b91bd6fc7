#!/usr/bin/env python
"""Benchmark: targets/s of the periodic evaluation on BASELINE.json's headline workload.

Workload (default c4, the config the metric "targets/sec at N=1e6, eps=1e-10" is quoted on):
singly periodic Laplace, 1x1 cell, N=1e6 sources from 16 Gaussian clusters, targets =
sources, eps = 1e-10, fp64. One step = one total_field (far plane-wave apply + fused near
images) over all targets, inputs resident in HBM.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c4]
                  [--dist-backend nccl|gloo]

N > 1: one rank per GPU. Under torchrun (WORLD_SIZE set) the ranks are the launcher's;
without it bench.py re-executes itself under torch.distributed.run with N ranks, and
refuses (exit 2) when fewer than N GPUs are visible unless --dist-backend gloo asks for N
ranks sharing the visible GPUs (a functional check of the sharded path, not a scaling
number). The job is fixed (strong scaling): the S2PW source sums run on a source slice per
rank and meet in one all-reduce (fp64, sum) of the plane-wave coefficient buffer, PW2T runs
on the rank's target slice, the symmetric near pairs are split into per-rank work-item
ranges whose int64 fixed-point accumulators meet in one reduce-scatter (dist.py). Time =
CUDA events on the launch stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "targets/sec at N=1e6, eps=1e-10, fp64, 1/2/4/8 B200; % of FP64 roofline"
# SURVEY.md §8(d) model flops per near pair (one image of one ordered (target, source)) and
# per far mode per point: the model's charge, reported as `model_speedup` beside the roofline
F_PAIR = {"c1": 29, "c2": 153, "c3": 48, "c4": 29, "c5": 94}
F_FAR = {"c1": 70, "c2": 70, "c3": 86, "c4": 70, "c5": 70}
# evaluated fp64 work of the dominant near launch per config, from committed ncu captures
# of the same kernels (tools/ncu_work.py -> profiles/work_model.json)
WORK_MODEL = os.path.join(ROOT, "profiles", "work_model.json")
WORKLOAD = {
    "c1": "c1: doubly periodic Poisson, square cell, N=1000 uniform, targets=sources, eps=1e-10",
    "c2": "c2: doubly periodic mod. Helmholtz beta=10, cell (1,0.3,0.8), 1e5 src / 1e5 tgt, eps=1e-10, u+grad u",
    "c3": "c3: doubly periodic Stokes, square cell, N=1e6 uniform, targets=sources, eps=1e-8",
    "c4": "c4: singly periodic Poisson, 1x1 cell, N=1e6 from 16 Gaussian clusters (sigma 0.02), targets=sources,"
          " eps=1e-10",
    "c5": "c5: doubly periodic mod. Helmholtz beta=1, cell 100x1, N=1e7 uniform, targets=sources, eps=1e-8",
}
L2_POLICY = "GPU arm: 256 MB buffer written between timed iterations (> 126 MB L2; inputs 24-40 MB)"


def bench_config(name, inp):
    """The `config` object of both arms (identical dicts: same workload, same sizes)."""
    c = inp.config
    return {"workload": WORKLOAD[name], "n_src": int(len(inp.sources)), "n_tgt": int(len(inp.targets)),
            "eps": c.eps, "path": "auto", "l2": L2_POLICY}


def host_cpu():
    """Model and core counts of this host (lscpu), and the threads this process may use."""
    info = {"threads_available": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = dict(line.split(":", 1) for line in out.splitlines() if ":" in line)
        kv = {k.strip(): v.strip() for k, v in kv.items()}
        sockets = int(kv.get("Socket(s)", "0") or 0)
        per = int(kv.get("Core(s) per socket", "0") or 0)
        info.update({"model": kv.get("Model name"), "sockets": sockets, "cores_per_socket": per,
                     "physical_cores": sockets * per if sockets and per else None,
                     "threads_per_core": int(kv.get("Thread(s) per core", "0") or 0) or None,
                     "logical_cpus": int(kv.get("CPU(s)", "0") or 0) or None})
    except Exception as e:  # reported, not fatal
        info["lscpu"] = f"unavailable: {e}"
    return info


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def visible_gpus():
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        n = sum(1 for line in out.splitlines() if line.startswith("GPU "))
    except Exception:
        n = 0
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd is not None:
        n = min(n, len([v for v in cvd.split(",") if v.strip()]))
    return n


def self_launch(args):
    """--gpus N without a launcher: re-run this script under torch.distributed.run, N ranks."""
    n = args.gpus
    have = visible_gpus()
    if args.impl != "reference" and args.dist_backend == "nccl" and have < n:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have} "
              f"(--dist-backend gloo runs {n} ranks on the visible GPUs as a functional check)", file=sys.stderr)
        return 2
    env = dict(os.environ)
    if args.dist_backend == "nccl":
        env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines show the rank count
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


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
def reference_inputs(name):
    """The workload drawn from the reference's own Rng (oracle/_ref, else the C restatement):
    the reference arm never maps the product library."""
    import workloads
    from oracle import pyoracle

    return workloads.generate(name, rng=pyoracle.rng_uniform)


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
    """Only when oracle/_ref was not built: the C restatement (near images + direct far).
    Its mode tables come from the product's builder, so this fallback does load the product
    library (outside the timed calls); the GPU box always has oracle/_ref."""
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


def cpu_sampler():
    from oracle import pyoracle

    return ("reference", reference_sample_times) if pyoracle.ref_available() else ("port", port_sample_times)


def extrapolate(inp, s, t1, t2):
    """t(N_T) = a + b N_T through the medians at N_T = s and 2s, evaluated at the full N_T."""
    b = max((t2 - t1) / s, 1e-30)
    a = max(0.0, t1 - b * s)
    nt = len(inp.targets)
    return a, b, a + b * nt


def cpu_rate(inp, sample, threads):
    """Bounded CPU baseline on rank 0: target subsamples S and 2S (all sources), extrapolated."""
    kind, timer = cpu_sampler()
    (_, t1), (_, t2) = timer(inp, [sample, 2 * sample], threads)
    a, b, t_full = extrapolate(inp, sample, t1, t2)
    nt = len(inp.targets)
    return {"value": nt / t_full, "unit": "targets/s", "cores": threads, "kind": kind,
            "sample": f"all {len(inp.sources)} sources, target subsamples of {sample} and {2 * sample} "
                      f"({t1:.2f}s, {t2:.2f}s); t(N_T)=a+b*N_T extrapolated to N_T={nt} (a={a:.3f}s, b={b:.3e}s)",
            "extrapolated_seconds": t_full, "host": host_cpu()}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    inp = reference_inputs(args.config)
    threads = len(os.sched_getaffinity(0))
    s = args.cpu_sample
    kind, timer = cpu_sampler()
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
    a, b, t_full = extrapolate(inp, s, t1, t2)
    nt = len(inp.targets)
    value = nt / t_full
    cb = {"value": value, "unit": "targets/s", "cores": threads, "kind": kind,
          "sample": f"each step: all {len(inp.sources)} sources, a seeded target subsample of {s} or {2 * s} "
                    f"(median {t1:.2f}s / {t2:.2f}s); t(N_T)=a+b*N_T extrapolated to N_T={nt} "
                    f"(a={a:.3f}s, b={b:.3e}s)",
          "extrapolated_seconds": t_full, "host": host_cpu()}
    line = {"metric": METRIC, "value": value, "unit": "targets/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(1, args.steps + args.warmup),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SURVEY.md §8(d))", "impl": "reference",
            "config": bench_config(args.config, inp),
            "parallelism": f"{threads} host threads (the reference's parallel_for, util.hpp:61-79)",
            "cpu_baseline": cb, "e2e": {"value": value, "unit": "targets/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm
def near_kernel_name(config, symmetric):
    """The dominant near launch of a config (engine.cu Plan::near, near.cu / near_sym.cu)."""
    fam = {"c1": ("SymLaplace", "Laplace", "3,3"), "c2": ("SymModHelm<grad>", "ModHelmGrad", "5,3"),
           "c3": ("SymStokes", "Stokes<no pressure>", "3,3"), "c4": ("SymLaplace", "Laplace", "3,1"),
           "c5": ("SymModHelm", "ModHelm", "3,3")}[config]
    binned = " on Morton-binned inputs" if config in ("c2", "c5") else ""
    if symmetric:
        return f"near_sym_kernel<{fam[0]},{fam[2]}> (fused near images, each unordered pair once){binned}"
    return f"near_tile_kernel<{fam[1]},{fam[2]}> (fused near images){binned}"


def roofline(config, ns, nt, sym_tile, ws, t_near_ms, peak_tf, nimg):
    """Hardware roofline of the dominant near launch from its evaluated fp64 work.

    The executed fp64 flops per pair-group (2 DFMA + DADD + DMUL, predicated-on lanes) come
    from the committed ncu capture of the same kernel (profiles/work_model.json, written by
    tools/ncu_work.py); the live near time comes from CUDA events on the launch stream. A
    pair-group is one (target, source) pair over all near images; each rank evaluates 1/ws of
    them. frac <= 1 by construction (it is an executed-work fraction of the fp64 peak)."""
    try:
        with open(WORK_MODEL) as f:
            m = json.load(f).get(config)
    except (OSError, ValueError):
        m = None
    groups = ns * (ns + 1) / 2.0 if sym_tile else float(ns) * nt
    t = t_near_ms * 1e-3
    model_flops = F_PAIR[config] * nimg * float(ns) * nt / ws
    out = {"bound": "fp64", "peak": peak_tf, "unit": "TFLOP/s", "near_ms_per_launch": t_near_ms,
           "model_speedup": model_flops / t / (peak_tf * 1e12) if peak_tf else None,
           "model_note": f"SURVEY.md §8(d) charges {F_PAIR[config]} flop per (image, target, source) x {nimg} "
                         f"images x {ns} x {nt}: the ratio of that model to the fp64 peak over the near time. "
                         "It exceeds 1 because the fused symmetric tile evaluates each unordered pair once with "
                         "one log for all images; it is not a roofline"}
    if not m or bool(m.get("symmetric")) != bool(sym_tile):
        out.update({"achieved": None, "frac": None, "traffic": None,
                    "work_source": f"no ncu capture of this kernel for {config} in profiles/work_model.json"})
        return out
    flops = m["fp64_flops_per_group"] * groups / ws
    instr = m["fp64_instr_per_group"] * groups / ws
    achieved = flops / t / 1e12
    same_n = m["n_src"] == ns and m["n_tgt"] == nt
    out.update({
        "achieved": achieved, "frac": achieved / peak_tf if peak_tf else None,
        "fp64_pipe_frac": instr / t / (peak_tf * 1e12 / 2.0) if peak_tf else None,
        "traffic": m["dram_bytes_per_launch"] if same_n and ws == 1 else None,
        "fp64_flops_per_pair_group": m["fp64_flops_per_group"],
        "fp64_instr_per_pair_group": m["fp64_instr_per_group"],
        "pair_groups_per_launch": groups / ws,
        "kernel": m["kernel"],
        "work_source": f"{m['capture']} (ncu --set full, n_src={m['n_src']}, n_tgt={m['n_tgt']}, "
                       f"{m['launch_ms']:.1f} ms cold; tools/ncu_work.py)",
    })
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOAD))
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--cpu-sample", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    launched = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not launched:
        return self_launch(args)
    ws, rank, local = dist_env()
    if launched and ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started {ws} ranks", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs
    from paper_2111_01083_b200 import dist as pdist

    ngpu = torch.cuda.device_count()
    if ngpu < 1:
        print("bench.py: no CUDA device visible", file=sys.stderr)
        return 2
    local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    if args.dist_backend == "nccl" and local_ws > ngpu:
        print(f"bench.py: {local_ws} ranks on this node need {local_ws} GPUs, {ngpu} visible "
              "(--dist-backend gloo shares them)", file=sys.stderr)
        return 2
    # PWB_BENCH_SHARDED=1 runs the multi-GPU code path (process group, sharded far and near
    # passes, collectives) even at world size 1
    sharded = ws > 1 or os.environ.get("PWB_BENCH_SHARDED") == "1"
    dev_index = local % ngpu
    torch.cuda.set_device(dev_index)
    if sharded:
        import datetime

        tmo = datetime.timedelta(seconds=600)  # a dead rank fails the job instead of hanging it
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index), timeout=tmo)
        else:
            dist.init_process_group("gloo", timeout=tmo)
    dev = torch.device("cuda", dev_index)
    stream = torch.cuda.current_stream()

    inp = configs.generate(args.config)
    c = inp.config
    cell = pw.make_unit_cell(c.cell[0], c.cell[1], c.cell[2], c.cell[3])
    t_b0 = time.perf_counter()
    pz = pw.make_periodizer(c.pde, c.beta, cell, c.eps)  # host builder (reported apart)
    build_ms = (time.perf_counter() - t_b0) * 1e3
    ns, nt = len(inp.sources), len(inp.targets)
    t_lo, t_hi = pdist.target_slice(nt, ws, rank)  # rank's targets (outputs stay sharded)
    kw_name = "charges" if c.strength == "charge" else "forces"
    strength = inp.charges if c.strength == "charge" else inp.forces

    src_d = torch.from_numpy(inp.sources).to(dev)
    str_d = torch.from_numpy(strength).to(dev)
    symmetric = not c.separate_targets
    # targets = sources (c1, c3, c4, c5): hand the library the same array so the symmetric
    # near tile (each unordered pair once) applies; shards and separate targets are copies
    same = not sharded and symmetric
    tgt_d = src_d if same else torch.from_numpy(np.ascontiguousarray(inp.targets[t_lo:t_hi])).to(dev)
    opt = pw.ApplyOptions(path=pw.ApplyPath.Auto, with_gradient=c.gradient, stream=stream.cuda_stream)
    full = pw.ParticleSystem(sources=src_d, targets=tgt_d, **{kw_name: str_d})
    out = pw.FieldResult()
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
    with ClockSampler(dev_index) as clocks:
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
    res = out.scalar if out.scalar is not None else out.velocity
    # gauge-free digest (Poisson / Stokes fields are defined up to a constant per component,
    # and the far field's reduction order moves that constant): per component sum, sum of
    # squares, count -> centered l2
    res2 = res.reshape(res.shape[0], -1)
    digest = [float(v) for v in torch.cat([res2.sum(0), (res2 * res2).sum(0)]).tolist()] + [float(res2.shape[0])]
    per_rank = [{"rank": 0, "device": dev_index, "step_ms": t_step, "near_ms": t_near, "far_ms": t_step - t_near}]
    if sharded:
        tt = torch.zeros(ws, 3, dtype=torch.float64, device=dev)
        tt[rank] = torch.tensor([t_step, t_near, dev_index], dtype=torch.float64)
        comm.allreduce(tt)
        per_rank = [{"rank": r, "device": int(tt[r, 2]), "step_ms": float(tt[r, 0]), "near_ms": float(tt[r, 1]),
                     "far_ms": float(tt[r, 0] - tt[r, 1])} for r in range(ws)]
        t_step, t_near = float(tt[:, 0].max()), float(tt[:, 1].max())
        dg = torch.tensor(digest, dtype=torch.float64, device=dev)
        comm.allreduce(dg)
        digest = [float(v) for v in dg.tolist()]

    # ---- end to end through the public API from pinned host memory (H2D + compute + D2H)
    src_h = torch.from_numpy(inp.sources).pin_memory()
    str_h = torch.from_numpy(strength).pin_memory()
    tgt_h = src_h if same else torch.from_numpy(np.ascontiguousarray(inp.targets[t_lo:t_hi])).pin_memory()
    tgt_all_h = None if symmetric else torch.from_numpy(np.ascontiguousarray(inp.targets)).pin_memory()
    e2e_ms = []
    host_sys = pw.ParticleSystem(sources=src_h, targets=tgt_h, **{kw_name: str_h})
    for k in range(args.e2e_steps + 1):
        if sharded:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if not sharded:
            pw.total_field(pz, host_sys, opt)  # library stages H2D / D2H on `stream`
        else:
            s_d = src_h.to(dev, non_blocking=True)
            q_d = str_h.to(dev, non_blocking=True)
            t_d = None if symmetric else tgt_all_h.to(dev, non_blocking=True)
            be = pdist.CudaBackend(pw, pz, opt, s_d, q_d, kw_name, t_d)
            rr, _ = pdist.sharded_total_field(be, comm, plan, symmetric)
            (rr.scalar if rr.scalar is not None else rr.velocity).to("cpu", non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        if k > 0:  # first one warms the staging buffers
            e2e_ms.append(e0.elapsed_time(e1))
    t_e2e = sum(e2e_ms) / len(e2e_ms)
    if sharded:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        comm.allreduce_max(tt)
        t_e2e = float(tt[0])
    nout = 1 if c.strength == "charge" else 2
    # bytes of the tensors copied per e2e step: sources + strengths (+ targets when separate)
    h2d = 8 * (2 * ns + (1 if c.strength == "charge" else 2) * ns) + (16 * nt if c.separate_targets else 0)
    d2h = 8 * nout * (t_hi - t_lo) + (16 * (t_hi - t_lo) if c.gradient else 0)

    # ---- roofline of the dominant kernel (fused near-image P2P tile)
    import ctypes

    peak = ctypes.c_double(0.0)
    if sharded:  # one rank at a time: ranks sharing a GPU must not halve each other's probe
        for r in range(ws):
            dist.barrier()
            if r == rank:
                pw.lib().pwb_fp64_peak_probe(-1, ctypes.byref(peak))
        dist.barrier()
    else:
        pw.lib().pwb_fp64_peak_probe(-1, ctypes.byref(peak))
    nimg = len(pw.near_translations(cell))
    sym_tile = symmetric and (sharded or ns >= 32768)
    roof = roofline(args.config, ns, nt, sym_tile, ws, t_near, peak.value, nimg)
    roof["kernel"] = roof.get("kernel") or near_kernel_name(args.config, sym_tile)
    roof["far_ms"] = t_step - t_near
    roof["peak_source"] = ("measured on this box: best-of DFMA-chain burst (pwb_fp64_peak_probe); "
                           "MEASURED_PEAKS.json has no fp64 entry; spec 37.2 TFLOP/s")
    shared = sharded and ws > min(ws, ngpu)

    line = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_rate(reference_inputs(args.config), args.cpu_sample, len(os.sched_getaffinity(0)))
            except Exception as e:  # reported, not fatal
                cpu = {"value": None, "unit": "targets/s", "cores": len(os.sched_getaffinity(0)),
                       "kind": "unavailable", "sample": f"failed: {e}"}
        value = nt / (t_step * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": "targets/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": bench_config(args.config, inp),
            "parallelism": (f"{ws} ranks ({args.dist_backend}): targets split {ws}-way, S2PW sources split "
                            f"{ws}-way + all-reduce, symmetric near items split + int64 reduce-scatter"
                            if sharded else "single GPU"),
            "plan": {"far_rank": pz.rank(), "near_images": nimg, "symmetric_tile": sym_tile},
            "devices": {"ranks": ws, "distinct_gpus": min(ws, ngpu) if sharded else 1,
                        "backend": args.dist_backend if sharded else None, "ranks_share_gpus": shared,
                        "note": "ranks share GPUs (--dist-backend gloo): a functional run of the sharded "
                                "path, not a scaling number" if shared else None},
            "per_rank": per_rank,
            "output_digest": output_digest(digest),
            "e2e": {"value": nt / (t_e2e * 1e-3), "unit": "targets/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": roof,
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


def output_digest(d):
    """[sum_c..., sumsq_c..., n] over all ranks -> per-component mean and centered l2 norm
    (sqrt(sum (u - mean)^2)): comparable across rank counts for every kernel."""
    k = (len(d) - 1) // 2
    n = d[-1]
    return {"targets": int(n), "mean": [d[c] / n for c in range(k)],
            "centered_l2": [max(0.0, d[k + c] - d[c] * d[c] / n) ** 0.5 for c in range(k)]}


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
