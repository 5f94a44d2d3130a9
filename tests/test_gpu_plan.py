"""Plans (qt_multiply_plan / qt_plan_execute / qt_update_values): the numeric
pass re-run on new values of the same patterns.  Needs a B200.

The re-executed C must be bitwise the C of a fresh qt_multiply on the new
values (same kernel, same summation order) and equal the oracle's product of
the new values (integers: exact); a CUDA-graph replay of qt_plan_execute gives
the same result (the call only enqueues kernels on the context stream)."""
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


def rand_bm(rng, nbr, p, bs, leaf, dtype, kind="int"):
    m = rng.random((nbr, nbr)) < p
    br, bc = np.nonzero(m)
    v = (rng.integers(-4, 5, size=(len(br), bs, bs)) if kind == "int"
         else rng.uniform(-1, 1, size=(len(br), bs, bs))).astype(dtype)
    return qtgen.BlockMatrix(nbr * bs, leaf, bs, br.astype(np.int32), bc.astype(np.int32), v)


def mk(qt, ctx, M):
    return qt.Matrix.from_blocks(ctx, M.n, M.leaf_dim, M.bs, M.brow, M.bcol, M.vals)


def sorted_vals(M, vals):
    o = np.lexsort((M.bcol, M.brow))
    return np.ascontiguousarray(vals[o]), (M.brow[o], M.bcol[o])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True)])
def test_plan_update_execute_bitwise(qt, ctx, dtype, ta, tb):
    rng = np.random.default_rng(500 + 2 * ta + tb + (dtype == np.float32))
    nbr = 27
    Am = rand_bm(rng, nbr, 0.25, 32, 128, dtype)
    Bm = rand_bm(rng, nbr, 0.25, 32, 128, dtype)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    plan, C, st = A.multiply_plan(B, ta, tb)
    ref0 = oracle.spgemm_t(nbr, 32, (Am.brow, Am.bcol, Am.vals.astype(np.float64)),
                           (Bm.brow, Bm.bcol, Bm.vals.astype(np.float64)), ta, tb)
    got0 = C.to_blocks()
    assert np.array_equal(got0[0], ref0[0]) and np.array_equal(got0[2].astype(np.float64), ref0[2])
    for it in range(2):
        # new values, same patterns, given in read-back order
        va = rng.integers(-4, 5, size=Am.vals.shape).astype(dtype)
        vb = rng.integers(-4, 5, size=Bm.vals.shape).astype(dtype)
        va_s, (ar, ac) = sorted_vals(Am, va)
        vb_s, (br, bc) = sorted_vals(Bm, vb)
        A.update_values(va_s)
        B.update_values(vb_s)
        plan.execute()
        got = C.to_blocks()
        fresh = A.multiply_ex(B, ta, tb)[0].to_blocks()
        assert all(np.array_equal(x, y) for x, y in zip(got, fresh))
        ref = oracle.spgemm_t(nbr, 32, (ar, ac, va_s.astype(np.float64)), (br, bc, vb_s.astype(np.float64)), ta, tb)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[2].astype(np.float64), ref[2])
    plan.close()


def test_plan_cuda_graph_replay(qt):
    import torch
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    c = qt.Context(0, stream=s)
    rng = np.random.default_rng(77)
    nbr = 16
    Am = rand_bm(rng, nbr, 1.0, 32, 128, np.float64, "uniform")
    A = mk(qt, c, Am)
    plan, C, _ = A.multiply_plan(A)
    ref = C.to_blocks()
    va = rng.uniform(-1, 1, size=Am.vals.shape)
    va_s, _ = sorted_vals(Am, va)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.execute()
    A.update_values(va_s)
    g.replay()
    torch.cuda.synchronize()
    got = C.to_blocks()
    fresh = (A @ A).to_blocks()
    assert all(np.array_equal(x, y) for x, y in zip(got, fresh))
    assert not np.array_equal(got[2], ref[2])
    plan.close()
    for m in (C, A):       # (matrices before their context)
        m.close()
    c.close()


def test_plan_block_size_64_and_16_execute(qt, ctx):
    rng = np.random.default_rng(78)
    for bs, nbr in ((64, 9), (16, 30)):
        Mm = rand_bm(rng, nbr, 0.3, bs, max(bs, 32) * 2, np.float64)
        M = mk(qt, ctx, Mm)
        plan, C, _ = M.multiply_plan(M)
        ref = C.to_blocks()
        plan.execute()                               # same values: the same C
        got = C.to_blocks()
        assert all(np.array_equal(x, y) for x, y in zip(got, ref))
        with pytest.raises(qt.QtError) as e:
            M.update_values(Mm.vals)
        assert e.value.name == "QT_EBS"
        plan.close()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_symm_square_plan(qt, ctx, dtype):
    """Purification-style S^2 with a fixed pattern: update U's values, execute
    the plan, compare with a fresh symmetric square and the oracle (exact)."""
    rng = np.random.default_rng(900 + (dtype == np.float32))
    nbr = 20
    m = np.triu(rng.random((nbr, nbr)) < 0.3)
    np.fill_diagonal(m, True)
    br, bc = np.nonzero(m)

    def vals():
        v = rng.integers(-4, 5, size=(len(br), 32, 32)).astype(dtype)
        for t in range(len(br)):
            if br[t] == bc[t]:
                v[t] = np.triu(v[t]) + np.triu(v[t], 1).T
        return v

    U = qt.Matrix.from_blocks(ctx, nbr * 32, 128, 32, br.astype(np.int32), bc.astype(np.int32), vals())
    plan, C, _ = U.symm_square_plan()
    for _ in range(2):
        v = vals()                      # (br, bc) from np.nonzero: already in (brow, bcol) order
        U.update_values(v)
        plan.execute()
        got = C.to_blocks()
        fresh = U.symm_square()[0].to_blocks()
        assert all(np.array_equal(x, y) for x, y in zip(got, fresh))
        ref = oracle.symm_square(nbr, 32, (br.astype(np.int32), bc.astype(np.int32), v.astype(np.float64)))
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[2].astype(np.float64), ref[2])
    plan.close()


def test_async_small_products_pipeline(qt, ctx):
    """Sync-free qt_multiply_async (small products): products returned before
    their block count is known (c_blocks -1) are resolved on first use — as
    operands of the next multiply, by to_blocks, by close — including more
    products in flight than the context's 32-slot count ring; every result
    equals the oracle's (integer values: exact)."""
    import oracle
    rng = np.random.default_rng(77)
    nbr = 12
    mats = []
    for _ in range(2):
        m = rng.random((nbr, nbr)) < 0.4
        br, bc = np.nonzero(m)
        v = rng.integers(-2, 3, size=(len(br), 32, 32)).astype(np.float64)
        mats.append((br.astype(np.int32), bc.astype(np.int32), v))
    A = qt.Matrix.from_blocks(ctx, nbr * 32, 64, 32, *mats[0])
    B = qt.Matrix.from_blocks(ctx, nbr * 32, 64, 32, *mats[1])
    ref_ab = oracle.spgemm(nbr, 32, mats[0], mats[1])
    # a chain: C1 = A B, C2 = C1 A, C3 = C2 B (each operand still pending)
    C1, s1 = A.multiply(B, wait=False)
    assert s1.c_blocks == -1 and s1.block_products > 0
    C2, _ = C1.multiply(A, wait=False)
    C3, _ = C2.multiply(B, wait=False)
    ref2 = oracle.spgemm(nbr, 32, ref_ab, mats[0])
    ref3 = oracle.spgemm(nbr, 32, ref2, mats[1])
    for C, ref in ((C1, ref_ab), (C2, ref2), (C3, ref3)):
        r, c, v = C.to_blocks()
        assert np.array_equal(r, ref[0]) and np.array_equal(c, ref[1]) and np.array_equal(v, ref[2])
        assert C.nblocks == len(ref[0])
    # 80 products in flight (the ring wraps), half of them destroyed unread
    outs = [A.multiply(B, wait=False)[0] for _ in range(80)]
    for i, C in enumerate(outs):
        if i % 2:
            C.close()
    for i, C in enumerate(outs):
        if not i % 2:
            r, c, v = C.to_blocks()
            assert np.array_equal(v, ref_ab[2])
            C.close()
