"""Diagnostics: one small block-size-16 product (the leaf sweep's N=4096, fill 0.01) repeated."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_07800_b200 import qtmm  # noqa: E402

fill = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
torch.cuda.set_device(0)
st = torch.cuda.Stream()
ctx = qtmm.Context(0, stream=st)
n = 4096
nb = n // bs
rng = np.random.default_rng(10 + bs)
mats = []
for _ in range(2):
    m = rng.random((nb, nb)) < fill
    br, bc = np.nonzero(m)
    v = rng.uniform(-1, 1, size=(len(br), bs, bs))
    mats.append(qtmm.Matrix.from_blocks(ctx, n, n, bs, br.astype(np.int32), bc.astype(np.int32), v))
A, B = mats
for i in range(30):
    C, s = A.multiply(B)
    C.close()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
for i in range(50):
    C, s = A.multiply(B)
    C.close()
e1.record(st)
torch.cuda.synchronize()
print(f"bs {bs} fill {fill}: {e0.elapsed_time(e1) / 50:.4f} ms per multiply, products {s.block_products}, "
      f"sym {s.ms_symbolic:.4f} num {s.ms_numeric:.4f} total {s.ms_total:.4f}")
