"""Where a small call's time goes (c1: N = 1000): per call, on cuda:0,

  * api_us         pw.total_field (Python wrapper + C-ABI), wall clock, synchronised
  * capi_us        pwb_total_field with prebuilt ctypes structs (no Python marshalling)
  * capi_event_us  CUDA-event time of the same C-ABI call on its stream

    python tools/call_overhead.py [--config c1] [--calls 300]
"""
import argparse
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--calls", type=int, default=300)
    args = ap.parse_args()
    import torch

    import paper_2111_01083_b200 as pw
    from paper_2111_01083_b200 import configs

    inp = configs.generate(args.config)
    c = inp.config
    pz = pw.make_periodizer(c.pde, c.beta, pw.make_unit_cell(*c.cell[:3], c.cell[3]), c.eps)
    src = torch.from_numpy(inp.sources).cuda()
    q = torch.from_numpy(inp.charges).cuda()
    stream = torch.cuda.current_stream()
    opt = pw.ApplyOptions(stream=stream.cuda_stream)
    s = pw.ParticleSystem(sources=src, targets=src, charges=q)
    for _ in range(5):
        pw.total_field(pz, s, opt)
    torch.cuda.synchronize()

    t0 = time.perf_counter()
    for _ in range(args.calls):
        pw.total_field(pz, s, opt)
    torch.cuda.synchronize()
    api = (time.perf_counter() - t0) / args.calls * 1e6

    cs, _ = s._c()
    co = opt._c()
    out = torch.empty(len(inp.sources), dtype=torch.float64, device="cuda")
    cf = pw._Field()
    cf.scalar = out.data_ptr()
    cf.memory = pw.MEM_DEVICE
    fn = pw.lib().pwb_total_field
    t0 = time.perf_counter()
    for _ in range(args.calls):
        fn(pz.handle, ctypes.byref(cs), ctypes.byref(co), ctypes.byref(cf))
    torch.cuda.synchronize()
    capi = (time.perf_counter() - t0) / args.calls * 1e6

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gpu = 0.0
    for _ in range(args.calls):
        e0.record(stream)
        fn(pz.handle, ctypes.byref(cs), ctypes.byref(co), ctypes.byref(cf))
        e1.record(stream)
        e1.synchronize()
        gpu += e0.elapsed_time(e1) * 1e3
    gpu /= args.calls
    print({"config": args.config, "n": len(inp.sources), "api_us": round(api, 2), "capi_us": round(capi, 2),
           "capi_event_us": round(gpu, 2)})


if __name__ == "__main__":
    main()
