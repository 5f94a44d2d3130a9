"""Host-side cost of one blocking qt_multiply on small products: wall time of
the Python call, of the raw ctypes call, of C.close(), and one QT_TRACE line
(host marks inside multiply_local).

  python tools/host_cost.py leaf32_0.01 cfg1
"""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch

from paper_1501_07800_b200 import qtmm
from timeline import cfg, leaf


def main():
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    ctx = qtmm.Context(0, stream=stream)
    lib = qtmm._lib
    for w in sys.argv[1:] or ["leaf32_0.01", "cfg1"]:
        if w.startswith("leaf"):
            bs, fill = w[4:].split("_")
            A, B = leaf(ctx, int(bs), float(fill))
        else:
            A, B = cfg(ctx, int(w[3:]))
        for _ in range(20):
            C, _ = A.multiply(B)
            C.close()
        tm, tc, toff = [], [], []
        for _ in range(200):
            t0 = time.perf_counter()
            C, _ = A.multiply(B)
            t1 = time.perf_counter()
            C.close()
            t2 = time.perf_counter()
            tm.append(t1 - t0)
            tc.append(t2 - t1)
        ctx.set_timing(False)
        for _ in range(200):
            t0 = time.perf_counter()
            C, _ = A.multiply(B)
            toff.append(time.perf_counter() - t0)
            C.close()
        ctx.set_timing(True)
        raw = []
        h = ctypes.c_void_p()
        stt = qtmm.Stats()
        for _ in range(200):
            t0 = time.perf_counter()
            lib.qt_multiply(A._h, B._h, ctypes.byref(h), ctypes.byref(stt))
            t1 = time.perf_counter()
            lib.qt_destroy(h)
            raw.append(t1 - t0)
        med = lambda v: round(1e6 * statistics.median(v), 1)
        print(f"{w}: multiply {med(tm)} us (timing off {med(toff)} us), close {med(tc)} us, "
              f"raw ctypes qt_multiply {med(raw)} us", flush=True)


if __name__ == "__main__":
    main()
