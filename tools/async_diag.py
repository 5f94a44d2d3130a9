import sys, time, os
sys.path.insert(0, '/root/repo')
import torch, qtgen
from paper_1501_07800_b200 import qtmm
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
ctx = qtmm.Context(0, stream=stream)
c = qtgen.config(1)
A = qtmm.Matrix.from_blocks(ctx, c["A"].n, c["A"].leaf_dim, 32, c["A"].brow, c["A"].bcol, c["A"].vals)
B = qtmm.Matrix.from_blocks(ctx, c["B"].n, c["B"].leaf_dim, 32, c["B"].brow, c["B"].bcol, c["B"].vals)
for _ in range(50):
    C, st = A.multiply(B, wait=False); C.close()
torch.cuda.synchronize()
N = 400
t0 = time.perf_counter()
for _ in range(N):
    C, st = A.multiply(B, wait=False); C.close()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6*(t1-t0)/N:.1f} us/call, total {1e6*(t2-t0)/N:.1f} us/call")
import ctypes
t0 = time.perf_counter()
h = ctypes.c_void_p(); stt = qtmm.Stats()
lib = qtmm._lib
for _ in range(N):
    lib.qt_multiply_async(A._h, B._h, ctypes.byref(h), ctypes.byref(stt)); lib.qt_destroy(h)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"raw ctypes: host {1e6*(t1-t0)/N:.1f} us/call, total {1e6*(t2-t0)/N:.1f} us/call")
