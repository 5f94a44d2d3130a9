#!/usr/bin/env python
"""Benchmark: effective FP64 GFLOP/s of C = A*A (block-sparse quadtree multiply)
at N GPUs, plus bytes received per GPU (BASELINE.json metric).

Workload: BASELINE config 5 at every N — the weak-scaling
banded matrix N = 16384*P, a_ij != 0 iff |i-j| <= 1024, uniform[-1,1], leaf
2048, block 32, C = A*A (FP64), P = N; rank g generates and owns block rows
[512g, 512(g+1)) (counter-based generator: no data moves to set up).  N = 1
is the same matrix as config 2 (which has leaf 1024; it is reported as the
extra key "cfg2").  1/2/4/8 GPUs are therefore one weak-scaling series.
A step = one qt_multiply (symbolic BFS + [exchange] + numeric kernel) on
device-resident inputs.  value = total nonzero block products * 2*32^3 /
max-over-ranks device time.  Inputs (A 264 MB + C 507 MB per GPU) exceed the
126 MB L2, so no explicit flush is done between steps.

Launch: `python bench.py --gpus N` with N > 1 and no torchrun environment
re-launches itself under torch.distributed.run (one rank per GPU, NCCL);
under torchrun WORLD_SIZE must equal --gpus (exit 2 otherwise).

`--impl reference` times the oracle (plain CPU block-CSR multiply, the
reference arm of this tier) on a bounded sample of the same workload.
`--dry-run` exercises the launcher and the rank plumbing (gloo, no GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import qtgen  # noqa: E402  (seeded inputs only)

BS = 32
FLOP_PER_PRODUCT = 2 * BS ** 3
METRIC = "effective FP64 GFLOP/s (nonzero block products)"
UNIT = "GFLOP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="qtmm", choices=["qtmm", "reference"])
    ap.add_argument("--dtype", default="f64", choices=["f64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--no-symm", action="store_true")
    ap.add_argument("--no-cfg2", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher + rank plumbing only (gloo, CPU): no GPU work, value null")
    return ap.parse_args()


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args) -> int:
    """--gpus N > 1 without a torchrun environment: run N ranks of this script
    under torch.distributed.run (one process per GPU, rendezvous on
    127.0.0.1); rank 0 prints the JSON line.  Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(P: int, rank: int):
    """Inputs of this rank: (config dict, description).  Config 5 at every P
    (P = 1 is config 2's matrix with leaf 2048)."""
    c = qtgen.config(5, P=P, rank=rank)
    desc = (f"cfg5 weak-scaling banded C=A*A N=16384*{P} d=1024 (bandwidth 2049) leaf 2048 bs 32 FP64"
            + (", row strips" if P > 1 else ""))
    return c, desc


def oracle_workload(P: int):
    """The rows the cpu_baseline / reference legs sample: rank 0's strip of
    config 5 (plus the B rows its products read), i.e. the same matrix rows
    rank 0 multiplies."""
    if P == 1:
        return qtgen.config(5, P=1, rank=0)
    return qtgen.config(5, P=P, rows=(0, 512 + 32))


def aggregate(dist, vals, device, world: int):
    """All-gather a small float64 vector from every rank -> [world, len] numpy
    (CUDA tensor under NCCL, CPU tensor under gloo)."""
    import torch
    if world == 1:
        return np.asarray([vals], dtype=np.float64)
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    gl = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gl, t)
    return torch.stack(gl).cpu().numpy()


def row_bounds(nbr: int, P: int):
    """Equal block-row strips (config 5: 512 block rows = 16384 rows per GPU)."""
    per = nbr // P
    return [g * per for g in range(P)] + [nbr]


# ----------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- oracle legs


def oracle_sample(c: dict, target_s: float = 12.0, row_cap: int | None = None):
    """Time the oracle (as it stands) on block rows of the same workload,
    starting in the middle of the generated rows and never past `row_cap`
    (rows whose products read B rows that were not generated).
    Returns (GFLOP/s, threads, description, seconds)."""
    import oracle
    A = c["A"]
    nbr = A.nbr
    Bm = c["B"]
    # products of block row I = sum over K in row I of A of |row K of B|
    rowcnt = np.bincount(Bm.brow, minlength=nbr)
    prod_row = np.bincount(A.brow, weights=rowcnt[A.bcol], minlength=nbr).astype(np.int64)
    nt = oracle.default_threads()
    a = (A.brow, A.bcol, A.vals)
    b = (Bm.brow, Bm.bcol, Bm.vals)
    lo = int(A.brow.min()) if A.nb else 0
    hi = min(int(A.brow.max()) + 1 if A.nb else 0, row_cap if row_cap is not None else nbr)
    mid = lo + (hi - 1 - lo) // 2 if A.nb else 0
    rows = max(1, min(max(nt, 4), hi - mid))
    t0 = time.perf_counter()
    oracle.spgemm(nbr, BS, a, b, nthreads=nt, rows=(mid, mid + rows))
    dt = time.perf_counter() - t0
    rate = prod_row[mid:mid + rows].sum() / max(dt, 1e-9)
    want = int(target_s * rate)
    r1 = mid
    acc = 0
    while r1 < hi and acc < want:
        acc += prod_row[r1]
        r1 += 1
    r1 = max(r1, mid + 1)
    t0 = time.perf_counter()
    oracle.spgemm(nbr, BS, a, b, nthreads=nt, rows=(mid, r1))
    dt = time.perf_counter() - t0
    prods = int(prod_row[mid:r1].sum())
    gf = prods * FLOP_PER_PRODUCT / dt / 1e9
    return gf, nt, f"block rows [{mid},{r1}) of the workload's C ({prods} block products)", dt


def cpu_info():
    """The host the oracle ran on (print the CPU model and the compile flags)."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "oracle_flags": "gcc -O2 -ffp-contract=off, pthreads"}


def oracle_cap(P: int):
    """Last block row (exclusive) the oracle may sample from oracle_workload(P):
    at P > 1 the rows generated beyond rank 0's strip only serve as B rows."""
    return None if P == 1 else 512


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    P = args.gpus
    c = oracle_workload(P)
    desc = (workload(1, 0)[1] if P == 1 else
            f"cfg5 weak-scaling banded C=A*A N=16384*{P} d=1024 leaf 2048 bs 32 FP64 (rank 0's rows)")
    per_step_s = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    times, rates = [], []
    nt = 1
    sample = ""
    for i in range(args.warmup + args.steps):
        gf, nt, sample, dt = oracle_sample(c, target_s=per_step_s, row_cap=oracle_cap(P))
        if i >= args.warmup:
            rates.append(gf)
            times.append(dt)
    v = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": P,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.median(times), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (qtgen counter-based generator)",
        "config": {"workload": desc, "sample": sample},
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": nt, "kind": "oracle",
                         "sample": sample, **cpu_info()},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- product leg


def dry_run(args, rank: int, world: int):
    """Launcher and rank plumbing without a GPU (CPU test of the N > 1 path):
    gloo process group, this rank's workload strip, the max/sum aggregation
    and the JSON line shape; value is null (nothing is multiplied)."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    c, desc = workload(world, rank)
    Am = c["A"]
    bounds = row_bounds(Am.nbr, world)
    allv = aggregate(dist, [float(rank), float(Am.nb), float(Am.brow.min()), float(Am.brow.max())],
                     "cpu", world)
    if rank == 0:
        line = {"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "dry_run": True,
                "config": {"workload": desc, "row_bounds": bounds,
                           "blocks_per_rank": [int(x) for x in allv[:, 1]],
                           "rows_per_rank": [[int(x), int(y)] for x, y in allv[:, 2:4]]},
                "ranks_seen": [int(x) for x in allv[:, 0]]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def timed_steps(stream, step, steps, barrier):
    """K steps between a barrier + synchronize on both sides; CUDA events on
    the library's stream.  Returns (ms per step, [qt_stats])."""
    import torch
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stats = []
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(steps):
        stats.append(step())
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    return ev0.elapsed_time(ev1) / steps, stats


def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
        return
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: one rank per GPU is required\n")
        sys.exit(2)
    if args.dry_run:
        dry_run(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    P = world
    if torch.cuda.device_count() < (local + 1):
        sys.stderr.write(f"bench.py: rank {rank} needs cuda:{local}, {torch.cuda.device_count()} visible\n")
        sys.exit(2)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    from paper_1501_07800_b200 import qtmm

    stream = torch.cuda.Stream(dev)
    ctx = qtmm.Context(dev, stream=stream)
    cinfo = ctx.info()
    if cinfo["comm_ranks"] != P:
        sys.stderr.write(f"bench.py: the library communicator has {cinfo['comm_ranks']} ranks, expected {P}\n")
        sys.exit(2)
    c, desc = workload(P, rank)
    Am = c["A"]
    bounds = row_bounds(Am.nbr, P) if P > 1 else None
    # device-resident inputs
    A = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, BS, Am.brow, Am.bcol, Am.vals, row_bounds=bounds)

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        C, st = A.multiply(A)
        C.close()
        return st

    for _ in range(max(3, args.warmup)):
        st = step()
    # FP64 peak for the roofline denominator (MEASURED_PEAKS.json has no FP64 entry)
    # (the best of three 100 ms runs: a single run varies by ~1.5 %)
    peak_dmma = max(ctx.fp64_peak("dmma", 100.0) for _ in range(3))
    sampler = ClockSampler(dev)
    sampler.start()
    l0 = ctx.kernel_launches
    ms, stats = timed_steps(stream, step, args.steps, barrier)
    clocks = sampler.stop()
    launches = ctx.kernel_launches - l0
    products = stats[-1].block_products
    ms_num = statistics.mean(s.ms_numeric for s in stats)
    ms_sym = statistics.mean(s.ms_symbolic for s in stats)
    ms_exch = statistics.mean(s.ms_exchange for s in stats)
    ms_pay = statistics.mean(s.ms_payload for s in stats)
    recv = stats[-1].bytes_recv_payload
    recv_meta = stats[-1].bytes_recv_meta
    allv = aggregate(dist, [ms, float(products), float(recv), float(recv_meta), float(launches), ms_num,
                            float(stats[-1].blocks_recv), ms_exch, ms_pay], "cuda", world)
    ms_max = float(allv[:, 0].max())
    total_products = float(allv[:, 1].sum())
    recv_all = allv[:, 2]
    meta_all = allv[:, 3]
    launches_total = int(allv[:, 4].sum())
    value = total_products * FLOP_PER_PRODUCT / (ms_max * 1e-3) / 1e9
    # dominant kernel: the numeric kernel, timed with events on its stream (qt_stats)
    flops_launch = products * FLOP_PER_PRODUCT
    achieved = flops_launch / (ms_num * 1e-3) / 1e12

    cfg2 = None
    if P == 1 and not args.no_cfg2:
        cfg2 = measure_cfg2(qtmm, ctx, stream, args)
    symm = None
    if P == 1 and not args.no_symm:
        symm = measure_symm(qtmm, ctx, stream, args)

    fp32 = None
    if not args.no_fp32:
        fp32 = measure_fp32(qtmm, ctx, stream, Am, bounds, args, world, dist, barrier)

    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(qtmm, ctx, stream, Am, bounds, args, world, dist, barrier)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        gf, nt, sample, _ = oracle_sample(oracle_workload(P), target_s=12.0, row_cap=oracle_cap(P))
        cpu = {"value": round(gf, 3), "unit": UNIT, "cores": nt, "kind": "oracle",
               "sample": sample + (" (rank 0's strip)" if P > 1 else ""), **cpu_info()}

    if rank == 0:
        # SpSUMMA: 2 m k sqrt(p) elements per process with m = nonzeros per
        # row (2d+1) and k = 16384 rows per process (the paper's weak-scaling setup)
        m_nnz_row = 2 * 1024 + 1
        k = 16384
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": P,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (qtgen counter-based generator, uniform[-1,1])",
            "config": {"workload": desc, "n": Am.n, "leaf_dim": Am.leaf_dim, "block": BS,
                       "global_block_products": int(total_products),
                       "block_products_per_rank": [int(x) for x in allv[:, 1]],
                       "l2": "no flush: inputs larger than L2 (A 264 MB + C 507 MB per GPU > 126 MB)",
                       "parallelism": f"row strips x{P} (NCCL, {cinfo['comm_ranks']}-rank communicator)"
                       if P > 1 else "single GPU"},
            "roofline": {"bound": "tensor", "kernel": "k_numeric_f64 (DMMA m8n8k4 f64)",
                         "achieved": round(achieved, 3), "peak": round(peak_dmma / 1e12, 3),
                         "unit": "TFLOP/s", "frac": round(achieved / (peak_dmma / 1e12), 4),
                         "traffic": traffic_from_profiles(P),
                         "peak_source": "live DMMA microbenchmark in this run (qt_fp64_peak, best of 3 x 100 ms); "
                                        "MEASURED_PEAKS.json has no FP64 entry; nominal 37.2 TF "
                                        "= 148 SM x 64 FMA x 2 x 1.965 GHz",
                         "ms_numeric": round(ms_num, 4), "ms_symbolic": round(ms_sym, 4),
                         "ms_numeric_per_rank": [round(float(x), 4) for x in allv[:, 5]],
                         "ms_call_median": round(statistics.median(s.ms_total for s in stats), 4),
                         "ms_call_min": round(min(s.ms_total for s in stats), 4),
                         "ms_exchange": round(ms_exch, 4),
                         "ms_exchange_max": round(float(allv[:, 7].max()), 4),
                         "ms_payload_overlapped": round(ms_pay, 4),
                         "ms_payload_max": round(float(allv[:, 8].max()), 4),
                         "tiles_overlapped_after": [int(stats[-1].tiles_overlapped), int(stats[-1].tiles_after)],
                         "numeric_share": round(ms_num / ms_max, 4)},
            "bytes_recv_per_gpu": {"max": int(recv_all.max()), "avg": float(recv_all.mean()),
                                   "min": int(recv_all.min()), "per_rank": [int(x) for x in recv_all],
                                   "meta_max": int(meta_all.max()),
                                   "blocks_recv_per_rank": [int(x) for x in allv[:, 6]],
                                   "unit": "bytes (FP64 payload)",
                                   "spsumma_comparator": 2 * m_nnz_row * k * (P ** 0.5) * 8,
                                   "spsumma_note": "2mk*sqrt(p)*8 B per process (P:726-728), m=2049, k=16384; "
                                                   "a formula, not measured (at P=1 nothing moves)"},
            "nccl": cinfo,
            "cpu_baseline": cpu,
            "cfg2": cfg2,
            "fp32_variant": fp32,
            "symm_square": symm,
            "e2e": e2e,
            "gpu_launches": launches_total,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    A.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def measure_cfg2(qtmm, ctx, stream, args):
    """BASELINE config 2 (the N=1 matrix with leaf 1024 instead of 2048): the
    same step timed on its own, reported beside the config-5 headline."""
    c = qtgen.config(2)["A"]
    A = qtmm.Matrix.from_blocks(ctx, c.n, c.leaf_dim, BS, c.brow, c.bcol, c.vals)

    def step():
        C, st = A.multiply(A)
        C.close()
        return st

    for _ in range(3):
        step()
    ms, sts = timed_steps(stream, step, args.steps, lambda: None)
    A.close()
    prods = sts[-1].block_products
    ms_num = statistics.mean(s.ms_numeric for s in sts)
    return {"workload": "cfg2 banded C=A*A N=16384 d=1024 leaf 1024 bs 32 FP64",
            "value": round(prods * FLOP_PER_PRODUCT / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
            "ms_per_step": round(ms, 4), "ms_numeric": round(ms_num, 4),
            "ms_symbolic": round(statistics.mean(s.ms_symbolic for s in sts), 4),
            "block_products": int(prods)}


def measure_fp32(qtmm, ctx, stream, Am, bounds, args, world, dist, barrier):
    """BASELINE config 5's FP32 variant: the same matrix rounded to FP32, same
    step, the tcgen05 3xTF32 kernel (secondary dtype; reported beside the FP64
    headline, not instead of it)."""
    import torch
    A32 = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, BS, Am.brow, Am.bcol,
                                  Am.vals.astype(np.float32), row_bounds=bounds)
    for _ in range(3):
        C, st = A32.multiply(A32)
        C.close()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sts = []
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    e0.record(stream)
    for _ in range(args.steps):
        C, st = A32.multiply(A32)
        sts.append(st)
        C.close()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms_num = statistics.mean(x.ms_numeric for x in sts)
    prods = sts[-1].block_products
    a = aggregate(dist, [ms, float(prods), float(sts[-1].bytes_recv_payload)], "cuda", world)
    A32.close()
    value = a[:, 1].sum() * FLOP_PER_PRODUCT / (a[:, 0].max() * 1e-3) / 1e9
    achieved = prods * FLOP_PER_PRODUCT / (ms_num * 1e-3) / 1e12
    peaks = measured_peaks()
    bf16 = peaks.get("bf16_tflops")
    # 3xTF32: three kind::tf32 MMAs per product; TF32 = bf16 x (1.1 / 2.25) (nominal dense ratio)
    peak = bf16 * (1.1 / 2.25) / 3.0 if bf16 else None
    return {"value": round(value, 1), "unit": UNIT + " (FP32, 3xTF32 on tcgen05)",
            "ms_per_step": round(float(a[:, 0].max()), 4), "dtype": "f32",
            "bytes_recv_per_gpu_max": int(a[:, 2].max()),
            "roofline": {"bound": "tensor", "kernel": "k_numeric_f32 (tcgen05.mma kind::tf32, 3 MMAs/product)",
                         "achieved": round(achieved, 2), "peak": round(peak, 1) if peak else None,
                         "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if peak else None,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops x (1.1/2.25 nominal tf32/bf16) / 3",
                         "ms_numeric": round(ms_num, 4)},
            # the 3xTF32 kernel draws ~990 W: the board's power cap lowers the SM clock (sw_power_cap)
            "clocks": clocks}


def measure_symm(qtmm, ctx, stream, args):
    """The symmetric square (§3.3) of the same banded workload with symmetric
    values, upper block triangle stored: its own effective GFLOP/s (over the
    block products it performs) and its speedup over the full multiply of the
    expanded matrix (the paper reports ~2x)."""
    import torch
    full = qtgen.config(2, symmetric=True)["A"]
    U = qtgen.upper(full)
    A = qtmm.Matrix.from_blocks(ctx, full.n, full.leaf_dim, BS, full.brow, full.bcol, full.vals)
    Au = qtmm.Matrix.from_blocks(ctx, U.n, U.leaf_dim, BS, U.brow, U.bcol, U.vals)
    res = {}
    for label, fn in (("full", lambda: A.multiply(A)), ("symm", lambda: Au.symm_square())):
        for _ in range(3):
            C, st = fn()
            C.close()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            C, st = fn()
            C.close()
        e1.record(stream)
        torch.cuda.synchronize()
        res[label] = (e0.elapsed_time(e1) / args.steps, st.block_products)
    A.close()
    Au.close()
    ms, prods = res["symm"]
    return {"value": round(prods * FLOP_PER_PRODUCT / (ms * 1e-3) / 1e9, 1), "unit": UNIT,
            "ms_per_step": round(ms, 4), "block_products": int(prods),
            "full_multiply_ms": round(res["full"][0], 4),
            "speedup_vs_full": round(res["full"][0] / ms, 3),
            "workload": "cfg2 matrix with symmetric values, upper block triangle stored"}


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0, "_source": "fallback (B200_PROFILING.md)"}


def traffic_from_profiles(P: int):
    """DRAM bytes per launch of the numeric kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("cfg5_P1" if P == 1 else "cfg5_interior")
    except Exception:
        return None


def measure_e2e(qtmm, ctx, stream, Am, bounds, args, world, dist, barrier):
    """Same metric through the public API with HOST buffers: every step copies
    A (pinned host) to the device inside qt_create (on the context's H2D
    stream), multiplies with qt_multiply_async (returns once the numeric kernel
    is enqueued) and reads C back to pinned host memory with
    qt_read_back_async (device-to-host copies on the copy stream): step i+1's
    H2D overlaps step i's numeric kernel and D2H (PCIe is full duplex); the
    timed region ends after qt_ctx_synchronize, i.e. after the last step's C
    is in host memory."""
    import torch
    brow = torch.from_numpy(Am.brow).pin_memory()
    bcol = torch.from_numpy(Am.bcol).pin_memory()
    vals = torch.from_numpy(Am.vals).pin_memory()
    outs = [None, None]  # double-buffered pinned results (step i writes outs[i % 2])
    # (a stream of steps, as many as the device-resident leg times (at most
    # 50, ~0.5 s): the first step's H2D and multiply fill the pipeline, after
    # which the steps are bound by the D2H of C)
    steps = max(2, min(args.steps, 50))

    def step(i):
        A = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, BS, brow, bcol, vals, row_bounds=bounds)
        C, st = A.multiply(A, wait=False)
        nb = C.nblocks
        o = outs[i % 2]
        if o is None or o[0].shape[0] != nb:
            o = (torch.empty(nb, dtype=torch.int32).pin_memory(),
                 torch.empty(nb, dtype=torch.int32).pin_memory(),
                 torch.empty((nb, BS, BS), dtype=torch.float64).pin_memory())
            outs[i % 2] = o
        C.to_blocks(o, wait=False)
        A.close()
        C.close()
        return st, nb

    for i in range(2):
        step(i)
    ctx.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        st, nb = step(i)
    ctx.synchronize()  # the last step's C is in host memory
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    a = aggregate(dist, [ms, float(st.block_products)], "cuda", world)
    ms, prods = float(a[:, 0].max()), float(a[:, 1].sum())
    h2d = Am.brow.nbytes + Am.bcol.nbytes + Am.vals.nbytes
    d2h = nb * (8 + BS * BS * 8)
    return {"value": round(prods * FLOP_PER_PRODUCT / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
            "ms_per_step": round(ms, 3), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "qt_create(host pinned, H2D stream) + qt_multiply_async + qt_read_back_async(host pinned, "
                   "copy stream), steps pipelined, qt_ctx_synchronize at the end"}


if __name__ == "__main__":
    main()
