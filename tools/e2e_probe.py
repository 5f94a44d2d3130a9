import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import qtgen
from paper_1501_07800_b200 import qtmm
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
ctx = qtmm.Context(0, stream=stream)
Am = qtgen.config(2)["A"]
brow = torch.from_numpy(Am.brow).pin_memory(); bcol = torch.from_numpy(Am.bcol).pin_memory(); vals = torch.from_numpy(Am.vals).pin_memory()
outs = [None, None]
def step(i, wait):
    t0 = time.perf_counter()
    A = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, 32, brow, bcol, vals)
    t1 = time.perf_counter()
    C, st = A.multiply(A, wait=wait)
    t2 = time.perf_counter()
    nb = C.nblocks
    o = outs[i % 2]
    if o is None:
        o = (torch.empty(nb, dtype=torch.int32).pin_memory(), torch.empty(nb, dtype=torch.int32).pin_memory(), torch.empty((nb, 32, 32), dtype=torch.float64).pin_memory())
        outs[i % 2] = o
    C.to_blocks(o, wait=wait)
    t3 = time.perf_counter()
    A.close(); C.close()
    return t1 - t0, t2 - t1, t3 - t2
for wait in (True, False):
    for i in range(3): step(i, wait)
    ctx.synchronize()
    T = time.perf_counter()
    r = [step(i, wait) for i in range(5)]
    ctx.synchronize()
    T = time.perf_counter() - T
    print("wait" if wait else "async", "per step %.2f ms" % (T / 5 * 1e3), "create %.2f multiply %.2f readback %.2f" % tuple(np.mean(r, 0) * 1e3))
# raw copy rates
d = torch.empty(vals.numel(), dtype=torch.float64, device='cuda')
torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(vals.view(-1), non_blocking=True); torch.cuda.synchronize(); h2d=time.perf_counter()-t
o = outs[0][2].view(-1)
dd = torch.empty(o.numel(), dtype=torch.float64, device='cuda')
torch.cuda.synchronize(); t=time.perf_counter(); o.copy_(dd, non_blocking=True); torch.cuda.synchronize(); d2h=time.perf_counter()-t
print("H2D %.1f GB/s (%.2f ms)  D2H %.1f GB/s (%.2f ms)" % (vals.numel()*8/h2d/1e9, h2d*1e3, o.numel()*8/d2h/1e9, d2h*1e3))
