"""Device timeline of a few qt_multiply calls (CUPTI via torch.profiler):
every kernel and memcpy/memset with its duration and the idle gap before it,
to see where the fixed per-call cost of small products goes.

  python tools/timeline.py leaf32_0.01 cfg1 cfg3
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import qtgen
from paper_1501_07800_b200 import qtmm


def leaf(ctx, bs, fill, dtype=np.float64):
    n, nb = 4096, 4096 // bs
    rng = np.random.default_rng(int(1000 * fill) + bs)
    mats = []
    for _ in range(2):
        m = rng.random((nb, nb)) < fill
        br, bc = np.nonzero(m)
        v = rng.uniform(-1, 1, size=(len(br), bs, bs)).astype(dtype)
        mats.append(qtmm.Matrix.from_blocks(ctx, n, n, bs, br.astype(np.int32), bc.astype(np.int32), v))
    return mats


def cfg(ctx, k):
    c = qtgen.config(k)
    A = qtmm.Matrix.from_blocks(ctx, c["A"].n, c["A"].leaf_dim, 32, c["A"].brow, c["A"].bcol, c["A"].vals)
    if c["same"]:
        return A, A
    B = qtmm.Matrix.from_blocks(ctx, c["B"].n, c["B"].leaf_dim, 32, c["B"].brow, c["B"].bcol, c["B"].vals)
    return A, B


def show(name, A, B, stream, wait, calls=3):
    for _ in range(5):
        C, _ = A.multiply(B, wait=wait)
        C.close()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(calls):
            C, _ = A.multiply(B, wait=wait)
            C.close()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    print(f"== {name} ({'blocking' if wait else 'async'}), {calls} calls")
    prev = None
    t0 = ev[0].time_range.start if ev else 0
    for e in ev:
        gap = 0 if prev is None else e.time_range.start - prev
        print(f"  t={e.time_range.start - t0:9.1f} us  gap {gap:7.1f}  dur {e.time_range.elapsed_us():8.1f}  {e.name[:90]}")
        prev = e.time_range.end
    if ev:
        span = ev[-1].time_range.end - t0
        busy = sum(e.time_range.elapsed_us() for e in ev)
        print(f"  span {span:.1f} us, busy {busy:.1f} us, per call {span / calls:.1f} us")


def main():
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    ctx = qtmm.Context(0, stream=stream)
    for w in sys.argv[1:] or ["leaf32_0.01", "cfg1"]:
        if w.startswith("leaf"):
            bs, fill = w[4:].split("_")
            A, B = leaf(ctx, int(bs), float(fill))
        else:
            A, B = cfg(ctx, int(w[3:]))
        for wait in (True, False):
            show(w, A, B, stream, wait)


if __name__ == "__main__":
    main()
