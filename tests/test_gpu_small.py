"""Small products: the symbolic pass's dense start and the timing switch.
Needs a B200.

Dense start (qt_symbolic.cu, k_bfs_small): for plain and transposed products
the tasks of level l0 <= 4 are read off the operands' dense top-level node
maps instead of l0 BFS transitions.  The recursion of §3.2
registers at level l exactly the pairs (op(A)_l(I,K), op(B)_l(K,J)) of
non-NIL nodes, so the per-level task counts C_l, the C nodes per
level and the product itself must equal the oracle's whatever the depth of
the tree relative to l0 (trees of 1..9 levels below the root here).

Timing off (qt_ctx_set_timing): same results, zero timings."""
import numpy as np
import pytest

import oracle
import qtgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qt():
    from paper_1501_07800_b200 import build
    build.build()
    from paper_1501_07800_b200 import qtmm
    return qtmm


@pytest.fixture(scope="module")
def ctx(qt):
    import torch
    torch.cuda.init()
    return qt.Context(0)


def rand_bm(rng, nbr, p, bs=32, leaf=128, dtype=np.float64):
    m = rng.random((nbr, nbr)) < p
    m[rng.integers(0, nbr), rng.integers(0, nbr)] = True
    br, bc = np.nonzero(m)
    v = rng.integers(-4, 5, size=(len(br), bs, bs)).astype(dtype)
    return qtgen.BlockMatrix(nbr * bs, leaf, bs, br.astype(np.int32), bc.astype(np.int32), v)


def mk(qt, ctx, M):
    return qt.Matrix.from_blocks(ctx, M.n, M.leaf_dim, M.bs, M.brow, M.bcol, M.vals)


def c_nodes_per_level(L, a_rc, b_rc):
    """C nodes with at least one task at level l: (I,J) with some K such that
    A_l(I,K) and B_l(K,J) are both non-NIL (patterns coarsened to 2^l)."""
    out = []
    for l in range(L + 1):
        s, m = L - l, 1 << l
        a = np.zeros((m, m), bool)
        b = np.zeros((m, m), bool)
        a[np.asarray(a_rc[0]) >> s, np.asarray(a_rc[1]) >> s] = True
        b[np.asarray(b_rc[0]) >> s, np.asarray(b_rc[1]) >> s] = True
        out.append(int(((a.astype(np.int64) @ b.astype(np.int64)) > 0).sum()))
    return out


@pytest.mark.parametrize("nbr,p", [(2, 0.9), (3, 0.5), (9, 0.3), (17, 0.1), (40, 0.05), (100, 0.02),
                                   (300, 0.004)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_dense_start_levels_and_values(qt, ctx, nbr, p, ta, tb):
    rng = np.random.default_rng(1000 * nbr + 2 * ta + tb)
    Am, Bm = rand_bm(rng, nbr, p), rand_bm(rng, nbr, p)
    C, st = mk(qt, ctx, Am).multiply_ex(mk(qt, ctx, Bm), ta, tb)
    got = C.to_blocks()
    ref = oracle.spgemm_t(nbr, 32, (Am.brow, Am.bcol, Am.vals), (Bm.brow, Bm.bcol, Bm.vals), ta, tb)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    assert np.array_equal(got[2], ref[2])
    L, _ = oracle.tree_levels(Am.n, 32, 128)
    ar = (Am.bcol, Am.brow) if ta else (Am.brow, Am.bcol)
    br = (Bm.bcol, Bm.brow) if tb else (Bm.brow, Bm.bcol)
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts(L, ar, br)
    assert list(st.level_c_nodes[: L]) == c_nodes_per_level(L, ar, br)[:L]
    assert st.level_c_nodes[L] == len(ref[0])


def test_dense_start_async_chain(qt, ctx):
    """qt_multiply_async products (sync-free) as operands: their dense maps are
    built with their levels on first use."""
    rng = np.random.default_rng(5)
    Am, Bm = rand_bm(rng, 60, 0.05), rand_bm(rng, 60, 0.05)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    C1, _ = A.multiply(B, wait=False)
    C2, st = C1.multiply(A, wait=False)
    ra = (Am.brow, Am.bcol, Am.vals)
    r1 = oracle.spgemm(60, 32, ra, (Bm.brow, Bm.bcol, Bm.vals))
    r2 = oracle.spgemm(60, 32, r1, ra)
    got = C2.to_blocks()
    assert np.array_equal(got[0], r2[0]) and np.array_equal(got[1], r2[1]) and np.array_equal(got[2], r2[2])


@pytest.mark.parametrize("case", ["f64", "f32", "bs16", "bs64"])
def test_timing_off_same_results(qt, ctx, case):
    rng = np.random.default_rng(9)
    bs = {"bs16": 16, "bs64": 64}.get(case, 32)
    dt = np.float32 if case == "f32" else np.float64
    Am = rand_bm(rng, 24, 0.2, bs=bs, leaf=4 * bs, dtype=dt)
    Bm = rand_bm(rng, 24, 0.2, bs=bs, leaf=4 * bs, dtype=dt)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    C_on, s_on = A.multiply(B)
    ctx.set_timing(False)
    try:
        C_off, s_off = A.multiply(B)
        got = C_off.to_blocks()  # (the call returned with its work complete)
    finally:
        ctx.set_timing(True)
    ref = C_on.to_blocks()
    assert all(np.array_equal(x, y) for x, y in zip(got, ref))
    assert s_off.ms_symbolic == 0 and s_off.ms_numeric == 0 and s_off.ms_total == 0
    assert s_on.ms_total > 0
    assert s_off.block_products == s_on.block_products and s_off.c_blocks == s_on.c_blocks
    assert list(s_off.level_tasks) == list(s_on.level_tasks)


def test_huge_sparse_grid(qt, ctx):
    """A 2^15 x 2^15 block grid (n = 1 048 576) holding a few hundred blocks:
    16 quadtree levels, per-level histograms of 512 KiB read back in chunks of
    the mapped staging buffer (read_small), a deep BFS over nearly empty
    levels.  Pattern, values, per-level task counts vs the oracle."""
    rng = np.random.default_rng(15)
    nbr = 1 << 15
    mats = []
    for _ in range(2):
        # blocks clustered on a few block rows / columns so that products exist
        rows = rng.integers(0, 64, size=300) * 512 + rng.integers(0, 4, size=300)
        cols = rng.integers(0, 64, size=300) * 512 + rng.integers(0, 4, size=300)
        key = np.unique(rows.astype(np.int64) * nbr + cols)
        br, bc = (key // nbr).astype(np.int32), (key % nbr).astype(np.int32)
        v = rng.integers(-4, 5, size=(len(br), 32, 32)).astype(np.float64)
        mats.append(qtgen.BlockMatrix(nbr * 32, 1024, 32, br, bc, v))
    Am, Bm = mats
    C, st = mk(qt, ctx, Am).multiply(mk(qt, ctx, Bm))
    ref = oracle.spgemm(nbr, 32, (Am.brow, Am.bcol, Am.vals), (Bm.brow, Bm.bcol, Bm.vals))
    got = C.to_blocks()
    assert len(ref[0]) > 0
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]) and np.array_equal(got[2], ref[2])
    L, _ = oracle.tree_levels(Am.n, 32, 1024)
    assert L == 15
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts(L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
