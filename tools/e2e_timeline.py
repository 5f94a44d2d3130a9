"""Device timeline (CUPTI, all streams) of bench.py's end-to-end steps
(qt_create from pinned host memory + qt_multiply_async + qt_read_back_async)
on config 5 at P = 1: every kernel and copy with its stream, start and
duration, and the host time of each API call — to see what serialises.

  python tools/e2e_timeline.py [steps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from torch.profiler import ProfilerActivity, profile

import qtgen
from paper_1501_07800_b200 import qtmm


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    ctx = qtmm.Context(0, stream=stream)
    Am = qtgen.config(5)["A"]
    brow = torch.from_numpy(Am.brow).pin_memory()
    bcol = torch.from_numpy(Am.bcol).pin_memory()
    vals = torch.from_numpy(Am.vals).pin_memory()
    outs = [None, None]
    host = []

    def step(i):
        t0 = time.perf_counter()
        A = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, 32, brow, bcol, vals)
        t1 = time.perf_counter()
        C, st = A.multiply(A, wait=False)
        t2 = time.perf_counter()
        nb = C.nblocks
        o = outs[i % 2]
        if o is None or o[0].shape[0] != nb:
            o = (torch.empty(nb, dtype=torch.int32).pin_memory(), torch.empty(nb, dtype=torch.int32).pin_memory(),
                 torch.empty((nb, 32, 32), dtype=torch.float64).pin_memory())
            outs[i % 2] = o
        C.to_blocks(o, wait=False)
        t3 = time.perf_counter()
        A.close()
        C.close()
        t4 = time.perf_counter()
        host.append((t0, t1 - t0, t2 - t1, t3 - t2, t4 - t3))

    for i in range(2):
        step(i)
    ctx.synchronize()
    host.clear()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        T0 = time.perf_counter()
        for i in range(steps):
            step(i)
        ctx.synchronize()
        T1 = time.perf_counter()
    path = "/tmp/e2e_trace.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    dev = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    dev.sort(key=lambda e: e["ts"])
    t0 = dev[0]["ts"] if dev else 0
    print(f"wall {1e3 * (T1 - T0) / steps:.2f} ms per step")
    for e in dev:
        name = e["name"][:60]
        extra = ""
        if e.get("cat") == "gpu_memcpy":
            b = e.get("args", {}).get("bytes", 0)
            extra = f" {b / 1e6:.1f} MB {b / max(e['dur'], 1) / 1e3:.1f} GB/s"
        print(f"  stream {e.get('tid')!s:>4} t={e['ts'] - t0:10.1f} dur {e['dur']:9.1f}  {name}{extra}")
    for h in host:
        print(f"  host: create {1e3 * h[1]:.2f} ms, multiply {1e3 * h[2]:.2f} ms, read-back enqueue {1e3 * h[3]:.2f} ms,"
              f" close {1e3 * h[4]:.2f} ms")


if __name__ == "__main__":
    main()
