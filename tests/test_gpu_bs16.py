"""Block size 16 ("a block size around 16-64", the
paper's S^2 runs use block size 16; reading C-27).  Needs a B200.

16x16 blocks are held as the quadrants of the kernels' 32x32 blocks with an
occupancy mask; C's 16-block pattern is the symbolic product one level below
the 32-blocks.  Every result is compared with the oracle run at bs = 16 (its
own plain block-CSR multiply at that block size): pattern identical,
integer-valued inputs bit-exact, uniform inputs within the FP64 gate and the
Higham bound; per-level task counts (16-block level included) equal the
oracle's coarsening counts."""
import numpy as np
import pytest

import oracle
import qtgen

pytestmark = pytest.mark.gpu
REL_FRO_F64 = 1e-12


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


def random_bm16(rng, nbr, p, kind, leaf, dtype=np.float64, mask=None):
    m = rng.random((nbr, nbr)) < p if mask is None else mask
    br, bc = np.nonzero(m)
    v = (rng.integers(-4, 5, size=(len(br), 16, 16)) if kind == "int"
         else rng.uniform(-1, 1, size=(len(br), 16, 16))).astype(dtype)
    return qtgen.BlockMatrix(nbr * 16, leaf, 16, br.astype(np.int32), bc.astype(np.int32), v)


def mk(qt, ctx, M):
    return qt.Matrix.from_blocks(ctx, M.n, M.leaf_dim, 16, M.brow, M.bcol, M.vals)


def tup(M):
    return (M.brow, M.bcol, M.vals.astype(np.float64))


def check(got, ref, A, B, nbr, kind):
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    if kind == "int":
        assert np.array_equal(got[2].astype(np.float64), ref[2])
    elif len(ref[0]):
        d = got[2] - ref[2]
        assert np.linalg.norm(d) <= REL_FRO_F64 * np.linalg.norm(ref[2])
        _, _, bound = oracle.higham_bound(nbr, 16, A, B, nbr * 16)
        assert np.all(np.abs(d) <= bound + 1e-300)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_bs16_roundtrip(qt, ctx, dtype):
    rng = np.random.default_rng(16)
    M = random_bm16(rng, 14, 0.35, "uniform", 64, dtype)
    perm = rng.permutation(M.nb)
    A = qt.Matrix.from_blocks(ctx, M.n, 64, 16, M.brow[perm], M.bcol[perm], M.vals[perm])
    info = A.info()
    assert info["bs"] == 16 and A.nblocks == M.nb and info["global_nblocks"] == M.nb
    r, c, v = A.to_blocks()
    o = np.lexsort((M.bcol, M.brow))
    assert np.array_equal(r, M.brow[o]) and np.array_equal(c, M.bcol[o]) and np.array_equal(v, M.vals[o])


def test_bs16_errors(qt, ctx):
    v = np.ones((2, 16, 16))
    with pytest.raises(qt.QtError) as e:
        qt.Matrix.from_blocks(ctx, 128, 64, 16, np.array([3, 3], np.int32), np.array([5, 5], np.int32), v)
    assert e.value.name == "QT_EDUP" and "brow=3, bcol=5" in str(e.value)
    with pytest.raises(qt.QtError) as e:
        qt.Matrix.from_blocks(ctx, 128, 64, 16, np.array([0, 8], np.int32), np.array([0, 1], np.int32), v)
    assert e.value.name == "QT_ERANGE" and "brow=8" in str(e.value)
    with pytest.raises(qt.QtError) as e:      # n must be a multiple of 32 (reading C-27)
        qt.Matrix.from_blocks(ctx, 48, 32, 16, np.array([0], np.int32), np.array([0], np.int32), v[:1])
    assert e.value.name == "QT_EINVAL"
    # symmetric square: the (1,0) 16-block of a diagonal 32-container is below the diagonal
    U = qt.Matrix.from_blocks(ctx, 128, 64, 16, np.array([0, 5], np.int32), np.array([1, 4], np.int32), v)
    with pytest.raises(qt.QtError) as e:
        U.symm_square()
    assert e.value.name == "QT_EINVAL" and "brow=5, bcol=4" in str(e.value)
    U = qt.Matrix.from_blocks(ctx, 128, 64, 16, np.array([0, 6], np.int32), np.array([1, 1], np.int32), v)
    with pytest.raises(qt.QtError) as e:
        U.symm_square()
    assert e.value.name == "QT_EINVAL" and "brow=6, bcol=1" in str(e.value)


@pytest.mark.parametrize("nbr,p,leaf", [(2, 1.0, 32), (8, 1.0, 64), (14, 0.5, 64), (38, 0.15, 128),
                                        (64, 0.04, 256)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_bs16_multiply(qt, ctx, nbr, p, leaf, kind):
    rng = np.random.default_rng(1600 + nbr + (kind == "int"))
    Am = random_bm16(rng, nbr, p, kind, leaf)
    Bm = random_bm16(rng, nbr, p, kind, leaf)
    C, st = mk(qt, ctx, Am).multiply(mk(qt, ctx, Bm))
    got = C.to_blocks()
    ref = oracle.spgemm(nbr, 16, tup(Am), tup(Bm))
    check(got, ref, tup(Am), tup(Bm), nbr, kind)
    assert C.nblocks == len(ref[0]) and st.c_blocks == len(ref[0])
    L, _ = oracle.tree_levels(Am.n, 16, leaf)
    counts = oracle.level_task_counts(L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    if nbr >= 8:      # (smaller grids: the containers' quadtree has one level more than the oracle's)
        assert st.nlevels == L + 1
        assert list(st.level_tasks[: L + 1]) == counts
        assert C.level_nodes() == oracle.level_node_counts(L, (ref[0], ref[1]))
    assert st.block_products == counts[-1]


def test_bs16_quadrants_that_never_meet(qt, ctx):
    # A holds only (even, even) 16-blocks, B only (odd, odd): every 32-level
    # container pair exists but no 16-block product does -> C is empty
    nbr = 16
    ev = np.zeros((nbr, nbr), bool)
    ev[0::2, 0::2] = True
    od = np.zeros((nbr, nbr), bool)
    od[1::2, 1::2] = True
    rng = np.random.default_rng(5)
    Am = random_bm16(rng, nbr, 0, "int", 64, mask=ev)
    Bm = random_bm16(rng, nbr, 0, "int", 64, mask=od)
    C, st = mk(qt, ctx, Am).multiply(mk(qt, ctx, Bm))
    assert C.nblocks == 0 and st.block_products == 0 and st.c_blocks == 0
    assert len(C.to_blocks()[0]) == 0
    # mixed: half the containers' products vanish at 16-granularity
    Bm2 = random_bm16(rng, nbr, 0, "int", 64, mask=ev | od)
    C2, st2 = mk(qt, ctx, Am).multiply(mk(qt, ctx, Bm2))
    ref = oracle.spgemm(nbr, 16, tup(Am), tup(Bm2))
    check(C2.to_blocks(), ref, tup(Am), tup(Bm2), nbr, "int")


def test_bs16_chain_and_transposes_fp32(qt, ctx):
    rng = np.random.default_rng(161)
    nbr = 22
    Am = random_bm16(rng, nbr, 0.2, "int", 64, np.float32)
    Bm = random_bm16(rng, nbr, 0.2, "int", 64, np.float32)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    for ta, tb in [(False, False), (True, False), (False, True), (True, True)]:
        got = A.multiply_ex(B, ta, tb)[0].to_blocks()
        ref = oracle.spgemm_t(nbr, 16, tup(Am), tup(Bm), ta, tb)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
        assert np.array_equal(got[2].astype(np.float64), ref[2])
    # a product used as an operand again: its masks drive the next product
    C = A @ B
    got = (C @ A).to_blocks()
    c_ref = oracle.spgemm(nbr, 16, tup(Am), tup(Bm))
    ref = oracle.spgemm(nbr, 16, c_ref, tup(Am))
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[2].astype(np.float64), ref[2])


@pytest.mark.parametrize("tau", [0.0, 2.0, 9.0])
def test_bs16_truncate(qt, ctx, tau):
    rng = np.random.default_rng(162)
    M = random_bm16(rng, 20, 0.4, "uniform", 64)
    M.vals *= rng.uniform(0, 1, size=(M.nb, 1, 1)) ** 4
    A = mk(qt, ctx, M)
    T = A.truncate(tau)
    r, c, v = T.to_blocks()
    rr, rc, rv = oracle.truncate(M.brow, M.bcol, M.vals, tau)
    assert np.array_equal(r, rr) and np.array_equal(c, rc) and np.array_equal(v, rv)
    assert T.nblocks == len(rr)
    # the truncated matrix multiplies as its listed blocks
    got = (T @ T).to_blocks()
    ref = oracle.spgemm(20, 16, (rr, rc, rv), (rr, rc, rv))
    check(got, ref, (rr, rc, rv), (rr, rc, rv), 20, "uniform")


@pytest.mark.parametrize("P,bounds", [(2, [0, 16, 40]), (3, [0, 6, 22, 40])])
def test_bs16_virtual_ranks(qt, ctx, P, bounds):
    rng = np.random.default_rng(163 + P)
    M = random_bm16(rng, 40, 0.12, "uniform", 128)
    A = mk(qt, ctx, M)
    full = (A @ A).to_blocks()
    # the exchange moves 32-blocks (containers): the plan on the container pattern
    cont = np.unique((M.brow // 2).astype(np.int64) * 1000 + M.bcol // 2)
    cr, cc = cont // 1000, cont % 1000
    plan = oracle.exchange_plan([b // 2 for b in bounds], (cr, cc), (cr, cc), 8192)
    for g in range(P):
        Cg, st = A.multiply_virtual(A, P, g, bounds)
        r, c, v = Cg.to_blocks()
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(c, full[1][m]) and np.array_equal(v, full[2][m])
        assert st.bytes_recv_payload == plan[g]["payload_bytes"]
        assert st.bytes_recv_meta == plan[g]["meta_bytes"] + plan[g]["blocks_received"]   # + 1 mask byte per block
    with pytest.raises(qt.QtError) as e:
        A.multiply_virtual(A, 2, 0, [0, 15, 40])
    assert e.value.name == "QT_EINVAL"


def test_bs16_loopback_two_ranks(qt, ctx):
    import threading
    import torch
    rng = np.random.default_rng(164)
    M = random_bm16(rng, 48, 0.1, "int", 128)
    full = (mk(qt, ctx, M) @ mk(qt, ctx, M)).to_blocks()
    bounds = [0, 20, 48]
    hub = qt.LoopbackHub(2)
    out, errs = [None] * 2, []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            c = qt.Context(0, stream=s, loopback=(hub, g, 2))
            m = (M.brow >= bounds[g]) & (M.brow < bounds[g + 1])
            A = qt.Matrix.from_blocks(c, M.n, M.leaf_dim, 16, M.brow[m], M.bcol[m], M.vals[m], row_bounds=bounds)
            C, st = A.multiply(A)
            T = C.truncate(50.0)
            out[g] = (C.to_blocks(), C.info(), T.to_blocks())
            for x in (T, C, A):
                x.close()
            c.close()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank_fn, args=(g,)) for g in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    hub.close()
    assert not errs, errs
    tr = oracle.truncate(*full, 50.0)
    for g in range(2):
        (r, c, v), info, (tr_r, tr_c, tr_v) = out[g]
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(v, full[2][m])
        assert (info["row_lo"], info["row_hi"]) == (bounds[g], bounds[g + 1])
        mt = (tr[0] >= bounds[g]) & (tr[0] < bounds[g + 1])
        assert np.array_equal(tr_r, tr[0][mt]) and np.array_equal(tr_c, tr[1][mt])


def random_upper16(rng, nbr, p, kind, leaf, dtype=np.float64):
    """Upper block triangle at 16-block granularity, symmetric diagonal blocks."""
    m = np.triu(rng.random((nbr, nbr)) < p)
    M = random_bm16(rng, nbr, p, kind, leaf, dtype, mask=m)
    for t in range(M.nb):
        if M.brow[t] == M.bcol[t]:
            M.vals[t] = np.triu(M.vals[t]) + np.triu(M.vals[t], 1).T
    return M


@pytest.mark.parametrize("nbr,p,leaf", [(2, 1.0, 32), (8, 1.0, 64), (14, 0.5, 64), (38, 0.15, 128),
                                        (64, 0.05, 256)])
@pytest.mark.parametrize("kind,dtype", [("int", np.float64), ("uniform", np.float64), ("int", np.float32)])
def test_bs16_symm_square(qt, ctx, nbr, p, leaf, kind, dtype):
    """Reading C-28: C = A^2 from A's upper 16-block triangle; the oracle
    expands U to the full symmetric matrix and multiplies at bs 16.  The
    16-block products counted are those of C's upper triangle (brute-force
    coarsening count, oracle.level_task_counts_sym), i.e. the (1,0) quadrants
    of diagonal containers are neither stored nor counted."""
    rng = np.random.default_rng(1700 + nbr + 3 * (kind == "int") + 7 * (dtype == np.float32))
    Um = random_upper16(rng, nbr, p, kind, leaf, dtype)
    U = mk(qt, ctx, Um)
    C, st = U.symm_square()
    got = C.to_blocks()
    ref = oracle.symm_square(nbr, 16, tup(Um))
    assert np.all(got[0] <= got[1])
    if kind == "int":
        check(got, ref, None, None, nbr, "int")
    else:
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
        full = oracle.expand_symmetric(*tup(Um))
        d = got[2] - ref[2]
        assert np.linalg.norm(d) <= REL_FRO_F64 * np.linalg.norm(ref[2])
        br, bc, bound = oracle.higham_bound(nbr, 16, full, full, nbr * 16)
        assert np.all(np.abs(d) <= bound[br <= bc] + 1e-300)   # (bound of the full product, upper blocks)
    assert C.nblocks == len(ref[0]) and st.c_blocks == len(ref[0])
    L, _ = oracle.tree_levels(Um.n, 16, leaf)
    assert st.block_products == oracle.level_task_counts_sym(L, (Um.brow, Um.bcol))[-1]
    # the stored U is untouched (the diagonal completion works on a copy)
    r, c, v = U.to_blocks()
    o = np.lexsort((Um.bcol, Um.brow))
    assert np.array_equal(v, Um.vals[o])
    # C is again upper-triangular bs-16 storage: square it once more
    C2 = C.symm_square()[0].to_blocks()
    ref2 = oracle.symm_square(nbr, 16, ref)
    assert np.array_equal(C2[0], ref2[0]) and np.array_equal(C2[1], ref2[1])
    if kind == "int" and dtype == np.float64:     # (|C^2| < 2^53: exact)
        assert np.array_equal(C2[2], ref2[2])


def test_bs16_symm_square_matches_full_multiply(qt, ctx):
    """The symmetric square equals the upper triangle of the full multiply of
    the expanded matrix computed by the library itself (integer values: exact),
    and needs fewer 16-block products."""
    rng = np.random.default_rng(1777)
    nbr = 96
    Um = random_upper16(rng, nbr, 0.08, "int", 256)
    fr, fc, fv = oracle.expand_symmetric(Um.brow, Um.bcol, Um.vals)
    F = qt.Matrix.from_blocks(ctx, Um.n, 256, 16, fr, fc, fv)
    Cf, sf = F.multiply(F)
    r, c, v = Cf.to_blocks()
    keep = r <= c
    Cs, ss = mk(qt, ctx, Um).symm_square()
    gr, gc, gv = Cs.to_blocks()
    assert np.array_equal(gr, r[keep]) and np.array_equal(gc, c[keep]) and np.array_equal(gv, v[keep])
    assert ss.block_products < 0.6 * sf.block_products


def _containers(M):
    k = np.unique(np.stack([M.brow // 2, M.bcol // 2], 1), axis=0)
    return k[:, 0], k[:, 1]


@pytest.mark.parametrize("P,bounds", [(2, [0, 16, 40]), (3, [0, 6, 22, 40]), (4, [0, 0, 10, 30, 40])])
def test_bs16_symm_square_virtual_ranks(qt, ctx, P, bounds):
    """Rank g of the P-rank symmetric square at block size 16 (C-26 at
    container granularity, C-28): its rows equal the single-rank result's,
    bitwise; the containers received are oracle.exchange_plan_symm's on the
    container pattern (8 KiB each) plus one mask byte per container."""
    rng = np.random.default_rng(1790 + P)
    Um = random_upper16(rng, 40, 0.15, "uniform", 128)
    U = mk(qt, ctx, Um)
    full = U.symm_square()[0].to_blocks()
    plan = oracle.exchange_plan_symm([b // 2 for b in bounds], _containers(Um), 8192)
    for g in range(P):
        Cg, st = U.symm_square_virtual(P, g, bounds)
        r, c, v = Cg.to_blocks()
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(c, full[1][m]) and np.array_equal(v, full[2][m])
        assert st.bytes_recv_payload == plan[g]["payload_bytes"]
        assert st.bytes_recv_meta == plan[g]["meta_bytes"] + plan[g]["blocks_received"]
    with pytest.raises(qt.QtError) as e:
        U.symm_square_virtual(2, 0, [0, 15, 40])
    assert e.value.name == "QT_EINVAL"


def test_bs16_symm_square_loopback_two_ranks(qt, ctx):
    import threading
    import torch
    rng = np.random.default_rng(1795)
    Um = random_upper16(rng, 48, 0.12, "int", 128)
    full = mk(qt, ctx, Um).symm_square()[0].to_blocks()
    bounds = [0, 20, 48]
    plan = oracle.exchange_plan_symm([b // 2 for b in bounds], _containers(Um), 8192)
    hub = qt.LoopbackHub(2)
    out, errs = [None] * 2, []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            c = qt.Context(0, stream=torch.cuda.Stream(), loopback=(hub, g, 2))
            m = (Um.brow >= bounds[g]) & (Um.brow < bounds[g + 1])
            A = qt.Matrix.from_blocks(c, Um.n, Um.leaf_dim, 16, Um.brow[m], Um.bcol[m], Um.vals[m],
                                      row_bounds=bounds)
            C, st = A.symm_square()
            out[g] = (C.to_blocks(), st.bytes_recv_payload, st.bytes_recv_meta)
            C.close()
            A.close()
            c.close()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank_fn, args=(g,)) for g in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    hub.close()
    assert not errs, errs
    ref = oracle.symm_square(48, 16, tup(Um))
    assert np.array_equal(full[0], ref[0]) and np.array_equal(full[2], ref[2])
    for g in range(2):
        (r, c, v), pay, meta = out[g]
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(c, full[1][m]) and np.array_equal(v, full[2][m])
        assert pay == plan[g]["payload_bytes"]
        assert meta == plan[g]["meta_bytes"] + plan[g]["blocks_received"]


# ----------------------------------------- norm-screened product at block size 16 (f4)


def _taus16(Am, Bm):
    na = np.sqrt(oracle.block_norm2(Am.vals.astype(np.float64)))
    nb = np.sqrt(oracle.block_norm2(Bm.vals.astype(np.float64)))
    prods = np.unique(np.outer(na, nb).ravel())
    mids = (prods[1:] + prods[:-1]) / 2
    return [0.0] + [float(mids[int(len(mids) * f)]) for f in (0.2, 0.5, 0.8)]


def _screened_count(Am, Bm, tau):
    """16-block products with ||A_IK||^2 ||B_KJ||^2 >= tau^2 (the oracle's test)."""
    na2 = oracle.block_norm2(Am.vals.astype(np.float64))
    nb2 = oracle.block_norm2(Bm.vals.astype(np.float64))
    n = 0
    by_row = {}
    for q in range(Bm.nb):
        by_row.setdefault(int(Bm.brow[q]), []).append(q)
    for p in range(Am.nb):
        for q in by_row.get(int(Am.bcol[p]), []):
            n += na2[p] * nb2[q] >= tau * tau
    return n


@pytest.mark.parametrize("nbr,p,leaf", [(14, 0.5, 64), (38, 0.15, 128)])
@pytest.mark.parametrize("kind,dtype", [("int", np.float64), ("uniform", np.float64), ("int", np.float32)])
def test_bs16_screened_multiply(qt, ctx, nbr, p, leaf, kind, dtype):
    """qt_multiply_screened at block size 16: each 16-block product is kept iff
    ||A_IK||_F ||B_KJ||_F >= tau (16-block norms, squared and summed row-major
    as the oracle does).  Pattern and values equal oracle.spgemm(tau=) at bs 16,
    block_products equals the number of surviving 16-block products, and
    ||C - C~||_F <= sum of the skipped products' norm bounds."""
    rng = np.random.default_rng(500 + nbr + (kind == "int") + (dtype == np.float32))
    Am = random_bm16(rng, nbr, p, kind, leaf, dtype)
    Bm = random_bm16(rng, nbr, p, kind, leaf, dtype)
    Am.vals *= rng.integers(1, 9, size=(Am.nb, 1, 1)).astype(dtype)     # varied 16-block norms
    Bm.vals *= rng.integers(1, 9, size=(Bm.nb, 1, 1)).astype(dtype)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    full = oracle.spgemm(nbr, 16, tup(Am), tup(Bm))
    for tau in _taus16(Am, Bm):
        C, st = A.multiply_screened(B, tau)
        got = C.to_blocks()
        ref = oracle.spgemm(nbr, 16, tup(Am), tup(Bm), tau=tau)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
        if kind == "int":
            assert np.array_equal(got[2].astype(np.float64), ref[2])
        elif len(ref[0]):
            assert np.linalg.norm(got[2] - ref[2]) <= REL_FRO_F64 * np.linalg.norm(ref[2])
        assert st.block_products == _screened_count(Am, Bm, tau)
        if tau == 0.0:
            assert np.array_equal(got[0], full[0]) and np.array_equal(got[1], full[1])


def test_bs16_screened_eslike_small(qt, ctx):
    """Config 4's recipe (small) split into 16-blocks, screened at two taus:
    uniform values within the FP64 gate of the oracle's screened product."""
    c = qtgen.config(4, small=True)["A"]
    # each 32-block -> four 16-blocks
    br = np.repeat(2 * c.brow, 4) + np.tile([0, 0, 1, 1], c.nb)
    bc = np.repeat(2 * c.bcol, 4) + np.tile([0, 1, 0, 1], c.nb)
    v = c.vals.reshape(c.nb, 2, 16, 2, 16).transpose(0, 1, 3, 2, 4).reshape(4 * c.nb, 16, 16)
    M = qtgen.BlockMatrix(c.n, c.leaf_dim, 16, br.astype(np.int32), bc.astype(np.int32), np.ascontiguousarray(v))
    A = mk(qt, ctx, M)
    for tau in [1e-3, 5e-2]:
        C, st = A.multiply_screened(A, tau)
        got = C.to_blocks()
        ref = oracle.spgemm(M.nbr, 16, tup(M), tup(M), tau=tau)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
        assert np.linalg.norm(got[2] - ref[2]) <= REL_FRO_F64 * np.linalg.norm(ref[2])
