"""The N>1 path's host logic on CPU with torch.distributed (gloo), world size 2
and 4: bench.py's rank aggregation and row strips, partition-independent input
generation, and the row-strip request/response protocol of DESIGN.md §7 (the
one qt_dist.cu implements over NCCL) run over gloo with the oracle doing the
arithmetic — every rank gets exactly the rows its C strip needs, the
gathered C equals the single-process product bit for bit, and the bytes
received equal oracle.exchange_plan."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_entry, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = []
    while not q.empty():
        results.append(q.get())
    for p in procs:
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    errs = [r for r in results if isinstance(r, str)]
    assert not errs, errs[0]
    return results


def _entry(rank, world, port, fn, args, q):
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = fn(rank, world, *args)
        q.put(("ok", rank, out))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        q.put(traceback.format_exc())
        raise


# --------------------------------------------------------------------- bench plumbing


def _bench_aggregate(rank, world):
    import bench
    a = bench.aggregate(dist, [1.0 + rank, 10.0 * rank], "cpu", world)
    assert a.shape == (world, 2)
    assert a[:, 0].max() == world and a[:, 1].sum() == 10.0 * sum(range(world))
    b = bench.row_bounds(512 * world, world)
    assert b[0] == 0 and b[-1] == 512 * world and all(b[g + 1] - b[g] == 512 for g in range(world))
    return True


@pytest.mark.parametrize("world", [2])
def test_bench_aggregation_gloo(world):
    assert len(_run(world, _bench_aggregate)) == world


# --------------------------------------------------------------------- inputs per rank


def _gen_rows(rank, world):
    import qtgen
    c = qtgen.config(5, P=world, rank=rank, small=True)
    A = c["A"]
    obj = [None] * world
    dist.all_gather_object(obj, (A.brow, A.bcol, A.vals))
    if rank == 0:
        full = qtgen.config(5, P=world, small=True)["A"]
        br = np.concatenate([o[0] for o in obj])
        bc = np.concatenate([o[1] for o in obj])
        v = np.concatenate([o[2] for o in obj])
        assert np.array_equal(br, full.brow) and np.array_equal(bc, full.bcol)
        assert np.array_equal(v, full.vals)
    return True


@pytest.mark.parametrize("world", [2, 4])
def test_generation_is_partition_independent(world):
    _run(world, _gen_rows)


# --------------------------------------------------------------------- exchange protocol


def _protocol(rank, world, cfg_idx):
    import oracle
    import qtgen
    bs = 32
    if cfg_idx == 5:
        full = qtgen.config(5, P=world, small=True)
    else:
        full = qtgen.config(cfg_idx, small=True)
    Af, Bf = full["A"], full["B"]
    nbr = Af.nbr
    per = nbr // world
    bounds = [g * per for g in range(world)] + [nbr]
    lo, hi = bounds[rank], bounds[rank + 1]
    mine = lambda M: (M.brow >= lo) & (M.brow < hi)
    ma, mb = mine(Af), mine(Bf)
    A = (Af.brow[ma], Af.bcol[ma], Af.vals[ma])           # local strip of A
    B = (Bf.brow[mb], Bf.bcol[mb], Bf.vals[mb])           # local strip of B
    # 1. rows needed from others, sorted, split by owner
    need = np.unique(A[1])
    need = need[(need < lo) | (need >= hi)].astype(np.int32)
    my_counts = np.array([((need >= bounds[q]) & (need < bounds[q + 1])).sum() for q in range(world)],
                         np.int64)
    # 0. P x P request matrix
    M = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(M, torch.from_numpy(my_counts))
    M = torch.stack(M).numpy()
    # 1. request lists (send to owners, receive from requesters)
    reqs = []
    for q in range(world):
        if q == rank:
            continue
        seg = need[(need >= bounds[q]) & (need < bounds[q + 1])]
        if len(seg):
            reqs.append(dist.isend(torch.from_numpy(seg.copy()), q))
    incoming = {}
    for r in range(world):
        if r != rank and M[r, rank] > 0:
            buf = torch.zeros(int(M[r, rank]), dtype=torch.int32)
            dist.recv(buf, r)
            incoming[r] = buf.numpy()
    for w in reqs:
        w.wait()
    # 2./3. owner replies: per row block counts, then columns + values
    rowcnt = np.bincount(B[0] - lo, minlength=hi - lo)
    order = np.lexsort((B[1], B[0]))
    Bs = (B[0][order], B[1][order], B[2][order])
    ptr = np.concatenate([[0], np.cumsum(rowcnt)])
    sends = []
    for r, rows in incoming.items():
        cnt = rowcnt[rows - lo].astype(np.int32)
        idx = np.concatenate([np.arange(ptr[k - lo], ptr[k - lo + 1]) for k in rows]).astype(np.int64)
        sends.append(dist.isend(torch.from_numpy(cnt), r))
        sends.append(dist.isend(torch.from_numpy(Bs[1][idx].astype(np.int32)), r))
        sends.append(dist.isend(torch.from_numpy(np.ascontiguousarray(Bs[2][idx])), r))
    got_r, got_c, got_v = [], [], []
    recv_meta = 0
    for q in range(world):
        if q == rank or my_counts[q] == 0:
            continue
        seg = need[(need >= bounds[q]) & (need < bounds[q + 1])]
        cnt = torch.zeros(len(seg), dtype=torch.int32)
        dist.recv(cnt, q)
        nb = int(cnt.sum())
        cols = torch.zeros(nb, dtype=torch.int32)
        vals = torch.zeros((nb, bs, bs), dtype=torch.float64)
        dist.recv(cols, q)
        dist.recv(vals, q)
        got_r.append(np.repeat(seg, cnt.numpy()))
        got_c.append(cols.numpy())
        got_v.append(vals.numpy())
        recv_meta += 4 * len(seg) + 4 * nb
    for w in sends:
        w.wait()
    nrecv = sum(len(x) for x in got_c)
    Bx = (np.concatenate([B[0]] + got_r), np.concatenate([B[1]] + got_c),
          np.concatenate([B[2]] + got_v) if got_v else B[2])
    # local product of the strip (oracle arithmetic)
    C = oracle.spgemm(nbr, bs, A, Bx, nthreads=2)
    plan = oracle.exchange_plan(bounds, (Af.brow, Af.bcol), (Bf.brow, Bf.bcol), bs * bs * 8)[rank]
    assert nrecv == plan["blocks_received"]
    assert nrecv * bs * bs * 8 == plan["payload_bytes"]
    assert recv_meta == plan["meta_bytes"]
    obj = [None] * world
    dist.all_gather_object(obj, C)
    if rank == 0:
        ref = oracle.spgemm(nbr, bs, (Af.brow, Af.bcol, Af.vals), (Bf.brow, Bf.bcol, Bf.vals), nthreads=2)
        r = np.concatenate([o[0] for o in obj])
        c = np.concatenate([o[1] for o in obj])
        v = np.concatenate([o[2] for o in obj])
        assert np.array_equal(r, ref[0]) and np.array_equal(c, ref[1])
        assert np.array_equal(v, ref[2])   # bitwise: every C block computed wholly on one rank
    return nrecv


@pytest.mark.parametrize("world,cfg", [(2, 5), (4, 5), (2, 3), (2, 4)])
def test_row_strip_protocol_gloo(world, cfg):
    res = _run(world, _protocol, cfg)
    assert len(res) == world


# --------------------------------------------------------------------- bench launcher


def _bench(*argv, env=None):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(root, "bench.py"), *argv], capture_output=True,
                          text=True, env=e, timeout=240)


def test_bench_relaunches_n_ranks_gloo_dry_run():
    """`bench.py --gpus 2` with no torchrun environment launches 2 ranks itself
    (torch.distributed.run, 127.0.0.1) and rank 0 prints one line with n_gpus 2
    and both ranks' config-5 strips (dry run: gloo, no GPU)."""
    import json
    r = _bench("--gpus", "2", "--dry-run", "--steps", "2")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks_seen"] == [0, 1]
    assert d["config"]["row_bounds"] == [0, 512, 1024]
    assert d["config"]["rows_per_rank"] == [[0, 511], [512, 1023]]
    # config 5 at P=2: both ranks are edge ranks with 512 rows and a 33-block half-band
    assert d["config"]["blocks_per_rank"][0] == d["config"]["blocks_per_rank"][1] > 0


def test_bench_rejects_world_mismatch():
    r = _bench("--gpus", "2", "--dry-run", env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
