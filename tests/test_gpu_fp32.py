"""FP32 path (tcgen05 kind::tf32, 3xTF32) parity with the oracle.  Needs a B200.

Reading C-9: inputs are the FP32-rounded values; the oracle computes the
double product of those rounded inputs; the bar is relative Frobenius error
<= 1e-5 (BASELINE north star), and bit-exact results on small-integer inputs
(pin P-12: every partial sum is an integer < 2^24, exact in FP32 and in the
3xTF32 split)."""
import numpy as np
import pytest

import oracle
import qtgen

pytestmark = pytest.mark.gpu
REL_FRO_F32 = 1e-5


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


def f32(M: qtgen.BlockMatrix):
    return qtgen.BlockMatrix(M.n, M.leaf_dim, M.bs, M.brow, M.bcol, M.vals.astype(np.float32))


def mk(qt, ctx, M):
    return qt.Matrix.from_blocks(ctx, M.n, M.leaf_dim, M.bs, M.brow, M.bcol, M.vals)


def ref64(M):
    return (M.brow, M.bcol, M.vals.astype(np.float64))


def random_bm(rng, nbr, p, kind, leaf):
    mask = rng.random((nbr, nbr)) < p
    br, bc = np.nonzero(mask)
    if kind == "int":
        v = rng.integers(-4, 5, size=(len(br), 32, 32)).astype(np.float32)
    else:
        v = rng.uniform(-1, 1, size=(len(br), 32, 32)).astype(np.float32)
    return qtgen.BlockMatrix(nbr * 32, leaf, 32, br.astype(np.int32), bc.astype(np.int32), v)


def check(got, ref, kind):
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    assert got[2].dtype == np.float32
    if kind == "int":
        assert np.array_equal(got[2].astype(np.float64), ref[2])
    else:
        d = got[2].astype(np.float64) - ref[2]
        rel = np.linalg.norm(d) / np.linalg.norm(ref[2])
        assert rel <= REL_FRO_F32, rel


def test_fp32_hand_example_embedded(qt, ctx):
    a = np.zeros((1, 32, 32), np.float32)
    b = np.zeros((1, 32, 32), np.float32)
    a[0, :2, :2] = [[1, 2], [3, 4]]
    b[0, :2, :2] = [[5, 6], [7, 8]]
    z = np.zeros(1, np.int32)
    A = qt.Matrix.from_blocks(ctx, 32, 32, 32, z, z, a)
    B = qt.Matrix.from_blocks(ctx, 32, 32, 32, z, z, b)
    r, c, v = (A @ B).to_blocks()
    assert list(r) == [0] and list(c) == [0]
    assert np.array_equal(v[0, :2, :2], np.array([[19, 22], [43, 50]], np.float32))
    assert np.all(v[0, 2:, :] == 0) and np.all(v[0, :, 2:] == 0)


def test_fp32_roundtrip_layout(qt, ctx):
    rng = np.random.default_rng(2)
    M = random_bm(rng, 9, 0.5, "uniform", 64)
    r, c, v = mk(qt, ctx, M).to_blocks()
    o = np.lexsort((M.bcol, M.brow))
    assert np.array_equal(v, M.vals[o])


@pytest.mark.parametrize("nbr,p,leaf", [(1, 1.0, 32), (4, 1.0, 32), (5, 0.6, 64), (16, 0.3, 128),
                                        (37, 0.2, 256), (64, 0.05, 512)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
@pytest.mark.parametrize("route", ["tcgen05", "auto", "fp64"])
def test_fp32_random_patterns(qt, ctx, monkeypatch, nbr, p, leaf, kind, route):
    """FP32 products on the tcgen05 kernel (QT_F32_DENSITY=0), on the FP64
    kernel over FP64 copies (reading C-30; QT_F32_DENSITY=2 forces it) and
    with the library's density rule: all equal the oracle's double product of
    the FP32 inputs (integers bit-exact, uniform within 1e-5)."""
    monkeypatch.setenv("QT_F32_DENSITY", {"tcgen05": "0", "fp64": "2", "auto": "0.2"}[route])
    rng = np.random.default_rng(nbr * 11 + (kind == "int"))
    Am = random_bm(rng, nbr, p, kind, leaf)
    Bm = random_bm(rng, nbr, p, kind, leaf)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    C, st = A.multiply(B)
    got = C.to_blocks()
    ref = oracle.spgemm(nbr, 32, ref64(Am), ref64(Bm))
    check(got, ref, kind)
    # qt_multiply_async takes the same route (sync-free for small products)
    Ca, _ = A.multiply(B, wait=False)
    check(Ca.to_blocks(), ref, kind)
    L, _ = oracle.tree_levels(Am.n, 32, leaf)
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts(
        L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))


@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_fp32_cfg1(qt, ctx, kind):
    c = qtgen.config(1, kind)
    Am, Bm = f32(c["A"]), f32(c["B"])
    got = (mk(qt, ctx, Am) @ mk(qt, ctx, Bm)).to_blocks()
    check(got, oracle.spgemm(16, 32, ref64(Am), ref64(Bm)), kind)


@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_fp32_cfg5_small_full_oracle(qt, ctx, kind):
    c = qtgen.config(5, kind, P=2, small=True)
    Am = f32(c["A"])
    A = mk(qt, ctx, Am)
    got = (A @ A).to_blocks()
    check(got, oracle.spgemm(Am.nbr, 32, ref64(Am), ref64(Am)), kind)


@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_fp32_cfg5_full_size_sampled(qt, ctx, kind):
    """BASELINE config 5's FP32 variant at full size (P = 1): integer inputs
    bit-exact (|partial sums| <= 33 280 < 2^24, pin P-12), uniform within 1e-5."""
    c = qtgen.config(5, kind, P=1)
    Am = f32(c["A"])
    A = mk(qt, ctx, Am)
    C, st = A.multiply(A)
    got = C.to_blocks()
    assert st.block_products == 2048800 and st.c_blocks == 61888
    for lo, hi in [(0, 6), (300, 306), (506, 512)]:
        ref = oracle.spgemm(Am.nbr, 32, ref64(Am), ref64(Am), rows=(lo, hi))
        m = (got[0] >= lo) & (got[0] < hi)
        check((got[0][m], got[1][m], got[2][m]), ref, kind)


def test_fp32_cfg5_virtual_rank_full_size_int(qt, ctx):
    """FP32 config 5 at P = 4, interior rank 1 (virtual ranks): sampled rows
    bit-exact against the oracle, bytes = the exchange plan at 4 KiB per block."""
    P, g = 4, 1
    lo, hi = 512 * g, 512 * (g + 1)
    c = qtgen.config(5, "int", P=P, rows=(lo - 32, hi + 32))
    Am = f32(c["A"])
    A = mk(qt, ctx, Am)
    bounds = [512 * q for q in range(P + 1)]
    Cg, st = A.multiply_virtual(A, P, g, bounds)
    plan = oracle.exchange_plan(bounds, (Am.brow, Am.bcol), (Am.brow, Am.bcol), 4096)[g]
    assert st.bytes_recv_payload == plan["payload_bytes"]
    got = Cg.to_blocks()
    for rlo, rhi in ((lo, lo + 3), (hi - 3, hi)):
        ref = oracle.spgemm(512 * P, 32, ref64(Am), ref64(Am), rows=(rlo, rhi))
        m = (got[0] >= rlo) & (got[0] < rhi)
        check((got[0][m], got[1][m], got[2][m]), ref, "int")


def test_fp32_cfg4_small(qt, ctx):
    c = qtgen.config(4, small=True)
    Am = f32(c["A"])
    A = mk(qt, ctx, Am)
    check((A @ A).to_blocks(), oracle.spgemm(Am.nbr, 32, ref64(Am), ref64(Am)), "uniform")


def test_fp32_run_to_run_bitwise(qt, ctx):
    c = qtgen.config(5, P=2, small=True)
    A = mk(qt, ctx, f32(c["A"]))
    v0 = (A @ A).to_blocks()[2]
    for _ in range(2):
        assert np.array_equal((A @ A).to_blocks()[2], v0)


@pytest.mark.parametrize("P", [2, 4])
def test_fp32_virtual_ranks_bitwise(qt, ctx, P):
    c = qtgen.config(5, P=P, small=True)
    Am = f32(c["A"])
    A = mk(qt, ctx, Am)
    full = (A @ A).to_blocks()
    per = Am.nbr // P
    bounds = [g * per for g in range(P + 1)]
    plan = oracle.exchange_plan(bounds, (Am.brow, Am.bcol), (Am.brow, Am.bcol), 4096)
    for g in range(P):
        Cg, st = A.multiply_virtual(A, P, g, bounds)
        r, cc, v = Cg.to_blocks()
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(v, full[2][m])
        assert st.bytes_recv_payload == plan[g]["payload_bytes"]   # FP32 halves the payload



@pytest.mark.parametrize("ta,tb", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_fp32_transposed_products(qt, ctx, ta, tb, kind):
    rng = np.random.default_rng(91 + 3 * ta + 7 * tb + (kind == "int"))
    nbr = 21
    Am = random_bm(rng, nbr, 0.3, kind, 128)
    Bm = random_bm(rng, nbr, 0.3, kind, 128)
    got = mk(qt, ctx, Am).multiply_ex(mk(qt, ctx, Bm), ta, tb)[0].to_blocks()
    ref = oracle.spgemm_t(nbr, 32, ref64(Am), ref64(Bm), ta, tb)
    check(got, ref, kind)


def _sym_upper_f32(rng, nbr, p, kind, leaf):
    mask = np.triu(rng.random((nbr, nbr)) < p)
    np.fill_diagonal(mask, rng.random(nbr) < 0.7)
    br, bc = np.nonzero(mask)
    v = (rng.integers(-4, 5, size=(len(br), 32, 32)) if kind == "int"
         else rng.uniform(-1, 1, size=(len(br), 32, 32))).astype(np.float32)
    for t in range(len(br)):
        if br[t] == bc[t]:
            v[t] = np.triu(v[t]) + np.triu(v[t], 1).T
    return qtgen.BlockMatrix(nbr * 32, leaf, 32, br.astype(np.int32), bc.astype(np.int32), v)


@pytest.mark.parametrize("nbr,p,leaf", [(4, 1.0, 64), (13, 0.4, 128), (40, 0.12, 256)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_fp32_symm_square(qt, ctx, nbr, p, leaf, kind):
    """FP32 symmetric square (upper block triangle stored) on the
    tcgen05 kernel: blocks of U read transposed are staged from a transposed
    copy of the pool; C's upper triangle equals the oracle's (double product
    of the FP32 inputs, expanded symmetric matrix) bit-exactly on integers and
    within 1e-5 relative Frobenius on uniform values."""
    rng = np.random.default_rng(700 + nbr + (kind == "int"))
    Um = _sym_upper_f32(rng, nbr, p, kind, leaf)
    C, st = mk(qt, ctx, Um).symm_square()
    got = C.to_blocks()
    ref = oracle.symm_square(nbr, 32, ref64(Um))
    check(got, ref, kind)
    L, _ = oracle.tree_levels(Um.n, 32, leaf)
    assert st.block_products == oracle.level_task_counts_sym(L, (Um.brow, Um.bcol))[-1]


def test_fp32_symm_square_cfg5_small(qt, ctx):
    c = qtgen.config(5, P=1, small=True, symmetric=True)
    full = f32(c["A"])
    U = qtgen.upper(full)
    C, _ = mk(qt, ctx, U).symm_square()
    got = C.to_blocks()
    ref = oracle.symm_square(full.nbr, 32, ref64(U))
    check(got, ref, "uniform")


# ----------------------------------------- norm-screened product in FP32 (f4; reading C-29)


@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_fp32_screened_multiply(qt, ctx, kind):
    """FP32 screened product: the FP64 screened multiply of the (exactly
    converted) FP32 values, C rounded to FP32.  Pattern = oracle.spgemm(tau=)
    on the same values; integers bit-exact, uniform within 1e-5."""
    rng = np.random.default_rng(71 + (kind == "int"))
    nbr = 24
    mats = []
    for _ in range(2):
        m = rng.random((nbr, nbr)) < 0.3
        br, bc = np.nonzero(m)
        v = (rng.integers(-4, 5, size=(len(br), 32, 32)) if kind == "int"
             else rng.uniform(-1, 1, size=(len(br), 32, 32)))
        v = v * rng.integers(1, 9, size=(len(br), 1, 1))
        mats.append(qtgen.BlockMatrix(nbr * 32, 128, 32, br.astype(np.int32), bc.astype(np.int32),
                                      v.astype(np.float32)))
    Am, Bm = mats
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    na = np.sqrt(oracle.block_norm2(Am.vals.astype(np.float64)))
    nb = np.sqrt(oracle.block_norm2(Bm.vals.astype(np.float64)))
    prods = np.unique(np.outer(na, nb).ravel())
    mids = (prods[1:] + prods[:-1]) / 2
    for tau in [0.0, float(mids[len(mids) // 3]), float(mids[2 * len(mids) // 3])]:
        C, st = A.multiply_screened(B, tau)
        got = C.to_blocks()
        ref = oracle.spgemm(nbr, 32, ref64(Am), ref64(Bm), tau=tau)
        check(got, ref, kind)
