"""The real multi-GPU path: one process per GPU, the library's own NCCL
communicator (NcclTransport, qt_dist.cu), config 5 at P = 2 (the weak-scaling
run, BASELINE.json configs[4]).  Needs >= 2 GPUs; skipped otherwise (gpurun
and the driver's round-end tiers have one GPU: there the same code path runs
on the loopback transport, tests/test_gpu_parity.py).

Checked per rank against the oracle: sampled C rows bit-exact (integer
variant), the bytes received = oracle.exchange_plan (the paper's "data
received by each process"), the communicator's rank count; and
`bench.py --gpus 2` launching its own ranks prints one line with n_gpus 2."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


needs2 = pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (one process per GPU over NCCL)")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q):
    import traceback
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        import torch
        import torch.distributed as dist
        import oracle
        import qtgen
        from paper_1501_07800_b200 import qtmm
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
        ctx = qtmm.Context(rank, stream=torch.cuda.Stream(rank))
        info = ctx.info()
        assert info == {"rank": rank, "world": world, "comm_ranks": world, "transport": "nccl"}, info
        P = world
        bounds = [512 * g for g in range(P + 1)]
        lo, hi = bounds[rank], bounds[rank + 1]
        mine = qtgen.config(5, "int", P=P, rank=rank)["A"]
        A = qtmm.Matrix.from_blocks(ctx, mine.n, mine.leaf_dim, 32, mine.brow, mine.bcol, mine.vals,
                                    row_bounds=bounds)
        C, st = A.multiply(A)
        got = C.to_blocks()
        # the oracle side: rank's strip with its halo rows (the rows its products read)
        halo = qtgen.config(5, "int", P=P, rows=(max(0, lo - 32), min(512 * P, hi + 32)))["A"]
        t = (halo.brow, halo.bcol, halo.vals)
        plan = oracle.exchange_plan(bounds, (halo.brow, halo.bcol), (halo.brow, halo.bcol), 8192)[rank]
        assert st.bytes_recv_payload == plan["payload_bytes"], (st.bytes_recv_payload, plan)
        assert st.bytes_recv_meta == plan["meta_bytes"]
        for rlo, rhi in ((lo, lo + 3), (lo + 254, lo + 258), (hi - 3, hi)):
            ref = oracle.spgemm(512 * P, 32, t, t, rows=(rlo, rhi))
            m = (got[0] >= rlo) & (got[0] < rhi)
            assert np.array_equal(got[0][m], ref[0]) and np.array_equal(got[1][m], ref[1])
            assert np.array_equal(got[2][m], ref[2])
        q.put(("ok", rank, int(st.bytes_recv_payload)))
        C.close()
        A.close()
        ctx.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        q.put(("err", rank, traceback.format_exc()))
        raise


@needs2
def test_nccl_two_ranks_cfg5_vs_oracle():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = []
    while not q.empty():
        res.append(q.get())
    errs = [r for r in res if r[0] == "err"]
    assert not errs, errs[0][2]
    assert all(p.exitcode == 0 for p in procs)
    # P = 2: both ranks are edge ranks, 17.0 MB each
    assert sorted(r[2] for r in res) == [17039360, 17039360]


@needs2
def test_bench_two_gpus_self_launch():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--no-e2e", "--no-fp32", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900,
                       env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["nccl"]["comm_ranks"] == 2 and d["nccl"]["transport"] == "nccl"
    assert d["bytes_recv_per_gpu"]["max"] == 17039360
    assert d["config"]["global_block_products"] == 4212000


def test_nccl_binding_one_rank():
    """Runs on one GPU: the library loads NCCL (dlopen), builds a one-rank
    communicator from a fresh unique id (ncclCommInitRank), reports it
    (ncclCommCount) and tears it down; a multiply on that context equals the
    oracle (integer values: exact)."""
    import torch
    import oracle
    import qtgen
    from paper_1501_07800_b200 import build
    build.build()
    from paper_1501_07800_b200 import qtmm
    torch.cuda.init()
    ctx = qtmm.Context(0, stream=torch.cuda.Stream(0), nccl_self=True)
    try:
        assert ctx.info() == {"rank": 0, "world": 1, "comm_ranks": 1, "transport": "nccl"}
        c = qtgen.config(1, "int")
        A = qtmm.Matrix.from_blocks(ctx, 512, 128, 32, c["A"].brow, c["A"].bcol, c["A"].vals)
        B = qtmm.Matrix.from_blocks(ctx, 512, 128, 32, c["B"].brow, c["B"].bcol, c["B"].vals)
        C, st = A.multiply(B)
        got = C.to_blocks()
        ref = oracle.spgemm(16, 32, (c["A"].brow, c["A"].bcol, c["A"].vals), (c["B"].brow, c["B"].bcol, c["B"].vals))
        assert all(np.array_equal(x, y) for x, y in zip(got, ref))
        assert st.bytes_recv_payload == 0
        for M in (A, B, C):
            M.close()
    finally:
        ctx.close()
