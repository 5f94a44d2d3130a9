"""Per-config device timing of qt_multiply (all BASELINE configs that fit one
GPU), with the numeric-kernel share.  Not part of the bench contract: a
development tool whose output is summarised in profiles/."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import qtgen  # noqa: E402
from paper_1501_07800_b200 import qtmm  # noqa: E402

FLOP = 2 * 32 ** 3


def run_sym(ctx, stream, name, full, steps=20):
    """Symmetric square of the upper triangle vs the full multiply of the same matrix."""
    U = qtgen.upper(full)
    A = qtmm.Matrix.from_blocks(ctx, full.n, full.leaf_dim, 32, full.brow, full.bcol, full.vals)
    Au = qtmm.Matrix.from_blocks(ctx, U.n, U.leaf_dim, 32, U.brow, U.bcol, U.vals)
    out = {}
    for label, fn in (("full", lambda: A.multiply(A)), ("symm", lambda: Au.symm_square())):
        for _ in range(3):
            C, st = fn()
            C.close()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sts = []
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            C, st = fn()
            sts.append(st)
            C.close()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out[label] = {"ms_step": round(ms, 4), "block_products": sts[-1].block_products,
                      "c_blocks": sts[-1].c_blocks,
                      "ms_numeric": round(statistics.mean(s.ms_numeric for s in sts), 4),
                      "tflops_numeric": round(sts[-1].block_products * FLOP /
                                              statistics.mean(s.ms_numeric for s in sts) / 1e9, 2)}
    out["speedup"] = round(out["full"]["ms_step"] / out["symm"]["ms_step"], 3)
    print(json.dumps({"config": name, **out}), flush=True)


def run_sym16(ctx, stream, steps=10):
    """The paper's S^2 shape at block size 16 (reading C-28): a
    symmetric banded pattern of 16-blocks (half-width 48 blocks, fill 0.5),
    N = 16384; symmetric square of the upper triangle vs the full multiply."""
    rng = np.random.default_rng(1007)
    nbr, w = 1024, 48
    I, J = np.meshgrid(np.arange(nbr), np.arange(nbr), indexing="ij")
    m = np.triu((np.abs(I - J) <= w) & (rng.random((nbr, nbr)) < 0.5))
    np.fill_diagonal(m, True)
    ur, uc = np.nonzero(m)
    uv = rng.uniform(-1, 1, size=(len(ur), 16, 16))
    d = ur == uc
    uv[d] = (uv[d] + uv[d].transpose(0, 2, 1)) / 2
    off = ~d
    fr = np.concatenate([ur, uc[off]]).astype(np.int32)
    fc = np.concatenate([uc, ur[off]]).astype(np.int32)
    fv = np.concatenate([uv, uv[off].transpose(0, 2, 1)])
    A = qtmm.Matrix.from_blocks(ctx, nbr * 16, 2048, 16, fr, fc, fv)
    Au = qtmm.Matrix.from_blocks(ctx, nbr * 16, 2048, 16, ur.astype(np.int32), uc.astype(np.int32), uv)
    out = {}
    for label, fn in (("full", lambda: A.multiply(A)), ("symm", lambda: Au.symm_square())):
        for _ in range(3):
            C, st = fn()
            C.close()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sts = []
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            C, st = fn()
            sts.append(st)
            C.close()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out[label] = {"ms_step": round(ms, 4), "block_products_16": sts[-1].block_products,
                      "c_blocks_16": sts[-1].c_blocks,
                      "ms_symbolic": round(statistics.mean(s.ms_symbolic for s in sts), 4),
                      "ms_numeric": round(statistics.mean(s.ms_numeric for s in sts), 4),
                      "gflops_effective_16": round(sts[-1].block_products * 2 * 16 ** 3 / ms / 1e6, 1)}
    out["speedup"] = round(out["full"]["ms_step"] / out["symm"]["ms_step"], 3)
    print(json.dumps({"config": "S^2 bs16 banded N=16384 (w=48 blocks, fill 0.5): symm_square vs full", **out}),
          flush=True)


def run(ctx, stream, name, c, steps=20):
    Am = c["A"]
    A = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, 32, Am.brow, Am.bcol, Am.vals)
    if c["same"]:
        B = A
    else:
        Bm = c["B"]
        B = qtmm.Matrix.from_blocks(ctx, Bm.n, Bm.leaf_dim, 32, Bm.brow, Bm.bcol, Bm.vals)
    for _ in range(3):
        C, st = A.multiply(B)
        C.close()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sts = []
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        C, st = A.multiply(B)
        sts.append(st)
        C.close()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st = sts[-1]
    num = statistics.mean(s.ms_numeric for s in sts)
    sym = statistics.mean(s.ms_symbolic for s in sts)
    out = {"config": name, "block_products": st.block_products, "c_blocks": st.c_blocks,
           "A_blocks": Am.nb, "ms_step": round(ms, 4), "ms_numeric": round(num, 4),
           "ms_symbolic": round(sym, 4), "gflops_effective": round(st.block_products * FLOP / ms / 1e6, 1),
           "tflops_numeric": round(st.block_products * FLOP / num / 1e9, 2),
           "level_tasks": st.as_dict()["level_tasks"]}
    print(json.dumps(out), flush=True)
    return out


def run_virtual(ctx, stream, name, M, P, ranks, steps=10):
    """Rank g of a P-rank multiply on one GPU (virtual ranks): numeric time with
    the exchange overlap on (two launches: local-only tiles, then the tiles
    behind the payload) and off (one launch).  The difference is what the
    split costs; the payload time it can hide is only measurable with P GPUs."""
    A = qtmm.Matrix.from_blocks(ctx, M.n, M.leaf_dim, 32, M.brow, M.bcol, M.vals)
    bounds = [g * (M.nbr // P) for g in range(P)] + [M.nbr]
    for g in ranks:
        out = {"config": name, "P": P, "rank": g}
        for ov in ("0", "1"):
            os.environ["QT_OVERLAP"] = ov
            for _ in range(2):
                C, st = A.multiply_virtual(A, P, g, bounds)
                C.close()
            sts = []
            for _ in range(steps):
                C, st = A.multiply_virtual(A, P, g, bounds)
                sts.append(st)
                C.close()
            num = statistics.median(s.ms_numeric for s in sts)
            out["overlap_" + ov] = {"ms_numeric": round(num, 4),
                                    "ms_symbolic": round(statistics.median(s.ms_symbolic for s in sts), 4),
                                    "tflops_numeric": round(st.block_products * FLOP / num / 1e9, 2),
                                    "tiles_overlapped": st.tiles_overlapped, "tiles_after": st.tiles_after}
        out["block_products"] = st.block_products
        out["bytes_recv_payload"] = st.bytes_recv_payload
        print(json.dumps(out), flush=True)
    os.environ.pop("QT_OVERLAP", None)


def run_virtual_sym(ctx, stream, name, full, P, ranks, steps=5):
    """Rank g of the P-rank symmetric square (virtual ranks) vs rank g of the
    full multiply of the expanded matrix: received bytes, products, times."""
    U = qtgen.upper(full)
    A = qtmm.Matrix.from_blocks(ctx, full.n, full.leaf_dim, 32, full.brow, full.bcol, full.vals)
    Au = qtmm.Matrix.from_blocks(ctx, U.n, U.leaf_dim, 32, U.brow, U.bcol, U.vals)
    bounds = [g * (full.nbr // P) for g in range(P)] + [full.nbr]
    for g in ranks:
        out = {"config": name, "P": P, "rank": g}
        for label, fn in (("full", lambda: A.multiply_virtual(A, P, g, bounds)),
                          ("symm", lambda: Au.symm_square_virtual(P, g, bounds))):
            for _ in range(2):
                C, st = fn()
                C.close()
            sts = []
            for _ in range(steps):
                C, st = fn()
                sts.append(st)
                C.close()
            out[label] = {"block_products": st.block_products, "bytes_recv_payload": st.bytes_recv_payload,
                          "bytes_recv_meta": st.bytes_recv_meta,
                          "ms_symbolic": round(statistics.median(s.ms_symbolic for s in sts), 4),
                          "ms_numeric": round(statistics.median(s.ms_numeric for s in sts), 4)}
        out["payload_ratio"] = round(out["symm"]["bytes_recv_payload"] / max(1, out["full"]["bytes_recv_payload"]), 4)
        print(json.dumps(out), flush=True)


def run_graph(ctx, stream, name, c, reps=1000, per_graph=10):
    """Numeric pass only, re-run through a plan captured into a CUDA graph
    (config 1 is launch-latency bound; its kernel time is taken
    from graph-replayed iterations).  per_graph executes per captured graph."""
    Am = c["A"]
    A = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, 32, Am.brow, Am.bcol, Am.vals)
    B = A if c["same"] else qtmm.Matrix.from_blocks(ctx, c["B"].n, c["B"].leaf_dim, 32, c["B"].brow, c["B"].bcol,
                                                    c["B"].vals)
    plan, C, st = A.multiply_plan(B)
    for _ in range(3):
        plan.execute()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(per_graph):
            plan.execute()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    n = max(1, reps // per_graph)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(n):
            g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (n * per_graph)
    print(json.dumps({"config": name + " (numeric pass via plan, CUDA-graph replay)", "block_products": st.block_products,
                      "us_per_execute": round(us, 2),
                      "tflops_numeric": round(st.block_products * FLOP / (us * 1e-6) / 1e12, 2),
                      "executes": n * per_graph, "per_call_ms_numeric": round(st.ms_numeric, 4)}), flush=True)
    plan.close()


def leaf_sweep(ctx, stream):
    """The paper's leaf benchmark shape (Figs. leafmat_bench_double /
    _single): C = A*B at N = 4096 as ONE leaf, blocks of size bs placed
    uniformly at random with a given fill factor (A and B independent),
    FP64 and FP32; device time of qt_multiply, effective GFLOP/s over nonzero
    block products (2 bs^3 each).  Block size 16 runs as quadrants of the
    32-blocks (reading C-27): only its 16-block products are counted."""
    n = 4096
    dts = [d for d in (np.float64, np.float32) if os.environ.get("QT_SWEEP_DT", "f64,f32").find(
        "f64" if d == np.float64 else "f32") >= 0]
    bss = [int(x) for x in os.environ.get("QT_SWEEP_BS", "16,32,64").split(",")]
    for dtype in dts:
        for bs in bss:
            nb = n // bs
            for fill in (0.01, 0.02, 0.05, 0.1, 0.2, 0.5, 1.0):
                rng = np.random.default_rng(int(1000 * fill) + bs)
                mats = []
                for _ in range(2):
                    m = rng.random((nb, nb)) < fill
                    br, bc = np.nonzero(m)
                    v = rng.uniform(-1, 1, size=(len(br), bs, bs)).astype(dtype)
                    mats.append(qtmm.Matrix.from_blocks(ctx, n, n, bs, br.astype(np.int32), bc.astype(np.int32), v))
                A, B = mats
                for _ in range(3):
                    C, st = A.multiply(B)
                    C.close()
                steps = 10

                def timed(wait, timing=True):
                    ctx.set_timing(timing)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record(stream)
                    for _ in range(steps):
                        C, st = A.multiply(B, wait=wait)
                        C.close()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ctx.set_timing(True)
                    return e0.elapsed_time(e1) / steps, st

                ms, st = timed(True)
                ms_off, _ = timed(True, timing=False)  # qt_ctx_set_timing(0): no event records / queries
                ms_async, _ = timed(False)  # qt_multiply_async, calls pipelined
                flop = st.block_products * 2.0 * bs ** 3
                print(json.dumps({"config": "leaf sweep N=4096 (one leaf)", "dtype": "f64" if dtype == np.float64 else "f32",
                                  "bs": bs, "fill": fill, "block_products": st.block_products,
                                  "ms_step": round(ms, 4), "gflops_effective": round(flop / ms / 1e6, 1),
                                  "ms_step_timing_off": round(ms_off, 4),
                                  "gflops_timing_off": round(flop / ms_off / 1e6, 1),
                                  "ms_step_async": round(ms_async, 4),
                                  "gflops_async": round(flop / ms_async / 1e6, 1)}), flush=True)
                A.close()
                B.close()


def main():
    which = sys.argv[1:] or ["1", "2", "3", "4", "5"]
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    ctx = qtmm.Context(0, stream=stream)
    peak = ctx.fp64_peak("dmma", 200.0)
    print(json.dumps({"dmma_peak_tflops": round(peak / 1e12, 3),
                      "dfma_peak_tflops": round(ctx.fp64_peak("dfma", 200.0) / 1e12, 3)}), flush=True)
    for w in which:
        if w == "leafsweep":
            leaf_sweep(ctx, stream)
        elif w == "1":
            run(ctx, stream, "cfg1 dense N=512", qtgen.config(1), steps=200)
        elif w == "1off":  # config 1, blocking calls with the context's timing off (no event records)
            c = qtgen.config(1)
            A = qtmm.Matrix.from_blocks(ctx, c["A"].n, c["A"].leaf_dim, 32, c["A"].brow, c["A"].bcol, c["A"].vals)
            B = qtmm.Matrix.from_blocks(ctx, c["B"].n, c["B"].leaf_dim, 32, c["B"].brow, c["B"].bcol, c["B"].vals)
            ctx.set_timing(False)
            for _ in range(20):
                C, st = A.multiply(B)
                C.close()
            steps = 400
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                C, st = A.multiply(B)
                C.close()
            e1.record(stream)
            torch.cuda.synchronize()
            ctx.set_timing(True)
            ms = e0.elapsed_time(e1) / steps
            print(json.dumps({"config": "cfg1 dense N=512, blocking qt_multiply, timing off", "ms_step": round(ms, 4),
                              "block_products": st.block_products,
                              "gflops_effective": round(st.block_products * FLOP / ms / 1e6, 1)}), flush=True)
        elif w == "1async":  # config 1 through qt_multiply_async (sync-free: back-to-back on the device)
            c = qtgen.config(1)
            A = qtmm.Matrix.from_blocks(ctx, c["A"].n, c["A"].leaf_dim, 32, c["A"].brow, c["A"].bcol, c["A"].vals)
            B = qtmm.Matrix.from_blocks(ctx, c["B"].n, c["B"].leaf_dim, 32, c["B"].brow, c["B"].bcol, c["B"].vals)
            for _ in range(20):
                C, st = A.multiply(B, wait=False)
                C.close()
            steps = 400
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                C, st = A.multiply(B, wait=False)
                C.close()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            print(json.dumps({"config": "cfg1 dense N=512, qt_multiply_async (pipelined)", "ms_step": round(ms, 4),
                              "block_products": st.block_products,
                              "gflops_effective": round(st.block_products * FLOP / ms / 1e6, 1)}), flush=True)
        elif w == "2":
            run(ctx, stream, "cfg2 banded N=16384", qtgen.config(2))
        elif w == "3":
            run(ctx, stream, "cfg3 random N=32768 p=0.01", qtgen.config(3))
        elif w == "4":
            run(ctx, stream, "cfg4 ES-like N=98304", qtgen.config(4), steps=10)
        elif w == "5":
            run(ctx, stream, "cfg5 P=1 banded N=16384 leaf 2048", qtgen.config(5, P=1))
        elif w == "5f32":
            c = qtgen.config(5, P=1)
            M = c["A"]
            M32 = qtgen.BlockMatrix(M.n, M.leaf_dim, 32, M.brow, M.bcol, M.vals.astype(np.float32))
            out = run(ctx, stream, "cfg5 P=1 banded N=16384 leaf 2048 FP32 (3xTF32 tcgen05)",
                      {"A": M32, "B": M32, "same": True})
            if len(sys.argv) > 1 and "--err" in sys.argv:
                pass
        elif w == "dense4096f32":
            br, bc = qtgen.pattern_dense(128)
            v = qtgen.block_values(br, bc, 32, 1).astype(np.float32)
            M = qtgen.BlockMatrix(4096, 1024, 32, br, bc, v)
            run(ctx, stream, "dense N=4096 FP32 (supplementary)", {"A": M, "B": M, "same": True})
        elif w == "err5f32":
            import oracle
            c = qtgen.config(5, P=1)
            M = c["A"]
            v32 = M.vals.astype(np.float32)
            A = qtmm.Matrix.from_blocks(ctx, M.n, M.leaf_dim, 32, M.brow, M.bcol, v32)
            r, cc, v = (A @ A).to_blocks()
            ref = oracle.spgemm(M.nbr, 32, (M.brow, M.bcol, v32.astype(np.float64)),
                                (M.brow, M.bcol, v32.astype(np.float64)), rows=(200, 232))
            m = (r >= 200) & (r < 232)
            d = v[m].astype(np.float64) - ref[2]
            print(json.dumps({"cfg5_fp32_rel_fro_err_rows_200_232": float(np.linalg.norm(d) / np.linalg.norm(ref[2])),
                              "max_abs_err": float(np.abs(d).max())}), flush=True)
        elif w == "sym2":
            run_sym(ctx, stream, "cfg2 banded symmetric: symm_square vs full", qtgen.config(2, symmetric=True)["A"])
        elif w == "sym5f32":
            M = qtgen.config(5, P=1, symmetric=True)["A"]
            run_sym(ctx, stream, "cfg5 banded symmetric FP32: symm_square vs full",
                    qtgen.BlockMatrix(M.n, M.leaf_dim, 32, M.brow, M.bcol, M.vals.astype(np.float32)))
        elif w == "sym16":
            run_sym16(ctx, stream)
        elif w == "sym4":
            run_sym(ctx, stream, "cfg4 ES-like symmetric (S^2): symm_square vs full",
                    qtgen.config(4, symmetric=True)["A"], steps=5)
        elif w == "scr4":
            import oracle  # noqa: F401  (not used: error measured against the unscreened product)
            c = qtgen.config(4)
            Am = c["A"]
            A = qtmm.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, 32, Am.brow, Am.bcol, Am.vals)
            C0, st0 = A.multiply(A)
            r0, c0, v0 = C0.to_blocks()
            for tau in (0.5, 2.0, 8.0):
                for _ in range(2):
                    C, st = A.multiply_screened(A, tau)
                    C.close()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(5):
                    C, st = A.multiply_screened(A, tau)
                    if _ < 4:
                        C.close()
                e1.record(stream)
                torch.cuda.synchronize()
                r, cc, v = C.to_blocks()
                # error vs the full product (blocks missing from C count as zero)
                idx = {(int(a), int(b)): t for t, (a, b) in enumerate(zip(r, cc))}
                err2 = 0.0
                for t in range(len(r0)):
                    k = (int(r0[t]), int(c0[t]))
                    d = v0[t] - (v[idx[k]] if k in idx else 0.0)
                    err2 += float((d * d).sum())
                print(json.dumps({"config": f"cfg4 screened tau={tau}", "ms_step": round(e0.elapsed_time(e1) / 5, 4),
                                  "block_products": st.block_products, "full_products": st0.block_products,
                                  "c_blocks": st.c_blocks, "rel_fro_err_vs_full": (err2 ** 0.5) / float(np.linalg.norm(v0))}),
                      flush=True)
        elif w == "virt8":
            run_virtual(ctx, stream, "cfg5 P=8 banded (virtual ranks)", qtgen.config(5, P=8)["A"], 8, [0, 3])
        elif w == "virt8r3":  # interior rank 3 of P=8, one numeric launch per multiply (ncu traffic)
            M = qtgen.config(5, P=8, rows=(3 * 512 - 32, 4 * 512 + 32))["A"]
            A = qtmm.Matrix.from_blocks(ctx, M.n, M.leaf_dim, 32, M.brow, M.bcol, M.vals)
            os.environ["QT_OVERLAP"] = "0"
            for _ in range(4):
                C, st = A.multiply_virtual(A, 8, 3, [512 * g for g in range(9)])
                C.close()
            print(json.dumps({"config": "cfg5 P=8 rank 3 (virtual, overlap off)", "block_products": st.block_products,
                              "ms_numeric": round(st.ms_numeric, 4), "bytes_recv_payload": st.bytes_recv_payload}))
            os.environ.pop("QT_OVERLAP", None)
        elif w == "virt8f32":
            M = qtgen.config(5, P=8)["A"]
            run_virtual(ctx, stream, "cfg5 P=8 banded FP32 (virtual ranks)",
                        qtgen.BlockMatrix(M.n, M.leaf_dim, 32, M.brow, M.bcol, M.vals.astype(np.float32)), 8, [3])
        elif w == "virt4cfg4":
            run_virtual(ctx, stream, "cfg4 ES-like P=4 (virtual ranks)", qtgen.config(4)["A"], 4, [1], steps=5)
        elif w == "virtsym8":
            run_virtual_sym(ctx, stream, "cfg5 P=8 banded symmetric (virtual ranks)",
                            qtgen.config(5, P=8, symmetric=True)["A"], 8, [0, 3])
        elif w == "virtsym4cfg4":
            run_virtual_sym(ctx, stream, "cfg4 ES-like symmetric P=4 (virtual ranks)",
                            qtgen.config(4, symmetric=True)["A"], 4, [0, 1])
        elif w == "graph1":
            run_graph(ctx, stream, "cfg1 dense N=512", qtgen.config(1))
        elif w == "graph2":
            run_graph(ctx, stream, "cfg2 banded N=16384", qtgen.config(2), reps=50, per_graph=5)
        elif w == "dense4096":
            br, bc = qtgen.pattern_dense(128)
            v = qtgen.block_values(br, bc, 32, 1)
            M = qtgen.BlockMatrix(4096, 1024, 32, br, bc, v)
            run(ctx, stream, "dense N=4096 (supplementary)", {"A": M, "B": M, "same": True})


if __name__ == "__main__":
    main()
