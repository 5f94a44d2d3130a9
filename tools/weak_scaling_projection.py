"""Projected weak scaling of config 5 (the bench workload) from one GPU: for
P = 1, 2, 4, 8 every rank g's multiply runs as a virtual rank
(qt_multiply_virtual: rank g's A strip times B_ext, where B_ext = its local
rows plus exactly the rows the exchange would bring) and is timed on the
device; the projected step is the slowest rank's time.  The payload exchange
itself (NCCL over NVLink, overlapped with the local tiles on P GPUs) is not
part of it: its bytes are reported beside the time, and 34 MB at NVLink's
~700 GB/s is ~50 us.  A projection, not a multi-GPU measurement.

  python tools/weak_scaling_projection.py > profiles/r02_weak_scaling_projection.jsonl
  python tools/weak_scaling_projection.py cfg4   # strong scaling of config 4 (one fixed
                                                 # matrix split into P strips by qt_plan_strips)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch

import qtgen
from paper_1501_07800_b200 import qtmm

FLOP = 2 * 32 ** 3


def main():
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    ctx = qtmm.Context(0, stream=stream)
    os.environ["QT_OVERLAP"] = "0"  # one numeric launch per rank (nothing to overlap on one GPU)
    strong = len(sys.argv) > 1 and sys.argv[1] == "cfg4"
    base = None
    M4 = qtgen.config(4)["A"] if strong else None
    for P in (1, 2, 4, 8):
        M = M4 if strong else qtgen.config(5, P=P)["A"]
        A = qtmm.Matrix.from_blocks(ctx, M.n, M.leaf_dim, 32, M.brow, M.bcol, M.vals)
        if strong:  # product-balanced strips at leaf rows (the library's planner)
            b, _ = qtmm.plan_strips(M.n, 32, P, (M.brow, M.bcol), M.brow, align_rows=M.leaf_dim // 32)
            bounds = [int(x) for x in b]
        else:
            bounds = [g * (M.nbr // P) for g in range(P)] + [M.nbr]
        ranks = []
        for g in range(P):
            for _ in range(2):
                C, st = A.multiply_virtual(A, P, g, bounds) if P > 1 else A.multiply(A)
                C.close()
            sts = []
            for _ in range(5):
                C, st = A.multiply_virtual(A, P, g, bounds) if P > 1 else A.multiply(A)
                sts.append(st)
                C.close()
            ms = statistics.median(s.ms_symbolic + s.ms_numeric for s in sts)
            ranks.append({"rank": g, "ms": round(ms, 4), "block_products": st.block_products,
                          "bytes_recv_payload": st.bytes_recv_payload})
        A.close()
        t = max(r["ms"] for r in ranks)
        prods = sum(r["block_products"] for r in ranks)
        value = prods * FLOP / (t * 1e-3) / 1e9
        if base is None:
            base = value
        print(json.dumps({"config": ("cfg4 strong scaling" if strong else "cfg5 weak scaling")
                          + ", projected from virtual ranks", "P": P, "bounds": bounds,
                          "projected_gflops": round(value, 1), "per_gpu_gflops": round(value / P, 1),
                          "efficiency_vs_P1": round(value / (base * P), 4), "slowest_rank_ms": t,
                          "speedup_vs_P1": round(value / base, 3),
                          "block_products": prods,
                          "bytes_recv_max": max(r["bytes_recv_payload"] for r in ranks),
                          "ranks": ranks}), flush=True)
    os.environ.pop("QT_OVERLAP", None)


if __name__ == "__main__":
    main()
