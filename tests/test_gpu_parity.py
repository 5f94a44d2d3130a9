"""Parity of the CUDA path (through the C ABI) with the oracle.  Needs a B200.

Bars: block patterns and integer-valued results
bit-exact; uniform[-1,1] FP64 results within relative Frobenius error 1e-12
and inside the elementwise Higham bound 2*gamma_K*(|A||B|) (pin P-9).
"""
import json
import os

import numpy as np
import pytest

import oracle
import qtgen

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
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


def mk(qt, ctx, M: qtgen.BlockMatrix):
    return qt.Matrix.from_blocks(ctx, M.n, M.leaf_dim, M.bs, M.brow, M.bcol, M.vals)


def as_tuple(M: qtgen.BlockMatrix):
    return (M.brow, M.bcol, M.vals)


def assert_same_pattern(got, ref):
    assert got[0].shape == ref[0].shape, (got[0].shape, ref[0].shape)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])


def assert_close_f64(got, ref, A, B, nbr, bs, k_terms):
    assert_same_pattern(got, ref)
    d = got[2] - ref[2]
    nr = np.linalg.norm(ref[2])
    rel = np.linalg.norm(d) / (nr if nr > 0 else 1.0)
    assert rel <= REL_FRO_F64, rel
    _, _, bound = oracle.higham_bound(nbr, bs, A, B, k_terms)
    assert np.all(np.abs(d) <= bound + 1e-300)


def random_bm(rng, nbr, bs, p, kind, leaf):
    mask = rng.random((nbr, nbr)) < p
    br, bc = np.nonzero(mask)
    if kind == "int":
        v = rng.integers(-4, 5, size=(len(br), bs, bs)).astype(np.float64)
    else:
        v = rng.uniform(-1, 1, size=(len(br), bs, bs))
    return qtgen.BlockMatrix(nbr * bs, leaf, bs, br.astype(np.int32), bc.astype(np.int32), v)


# ----------------------------------------------------------------- small cases


def test_hand_example_embedded(qt, ctx):
    g = json.load(open(os.path.join(GOLD, "spec_hand_example.json")))
    a = np.zeros((1, 32, 32))
    b = np.zeros((1, 32, 32))
    a[0, :2, :2] = g["A"]
    b[0, :2, :2] = g["B"]
    z = np.zeros(1, np.int32)
    A = qt.Matrix.from_blocks(ctx, 32, 32, 32, z, z, a)
    B = qt.Matrix.from_blocks(ctx, 32, 32, 32, z, z, b)
    C, st = A.multiply(B)
    r, c, v = C.to_blocks()
    assert list(r) == [0] and list(c) == [0]
    assert np.array_equal(v[0, :2, :2], np.array(g["C"], float))
    assert np.all(v[0, 2:, :] == 0) and np.all(v[0, :, 2:] == 0)
    assert st.block_products == 1


def test_create_read_back_roundtrip(qt, ctx):
    rng = np.random.default_rng(0)
    M = random_bm(rng, 13, 32, 0.4, "uniform", 128)
    perm = rng.permutation(M.nb)
    A = qt.Matrix.from_blocks(ctx, M.n, M.leaf_dim, 32, M.brow[perm], M.bcol[perm], M.vals[perm])
    r, c, v = A.to_blocks()
    o = np.lexsort((M.bcol, M.brow))
    assert np.array_equal(r, M.brow[o]) and np.array_equal(c, M.bcol[o])
    assert np.array_equal(v, M.vals[o])


@pytest.mark.parametrize("nbr,p,leaf", [(1, 1.0, 32), (2, 1.0, 32), (5, 0.5, 64), (16, 0.3, 128),
                                        (37, 0.2, 256), (64, 0.05, 512), (100, 0.08, 1024)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_random_patterns(qt, ctx, nbr, p, leaf, kind):
    rng = np.random.default_rng(nbr * 7 + (kind == "int"))
    Am = random_bm(rng, nbr, 32, p, kind, leaf)
    Bm = random_bm(rng, nbr, 32, p, kind, leaf)
    C, st = mk(qt, ctx, Am).multiply(mk(qt, ctx, Bm))
    got = C.to_blocks()
    ref = oracle.spgemm(nbr, 32, as_tuple(Am), as_tuple(Bm))
    if kind == "int":
        assert_same_pattern(got, ref)
        assert np.array_equal(got[2], ref[2])
    else:
        assert_close_f64(got, ref, as_tuple(Am), as_tuple(Bm), nbr, 32, nbr * 32)
    L, _ = oracle.tree_levels(Am.n, 32, leaf)
    assert st.nlevels == L + 1
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts(
        L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    assert st.c_blocks == len(ref[0])
    # C's quadtree = the tree spanned by its blocks
    assert C.level_nodes() == oracle.level_node_counts(L, (ref[0], ref[1]))


def test_identity_both_sides(qt, ctx):
    rng = np.random.default_rng(3)
    Am = random_bm(rng, 24, 32, 0.3, "uniform", 256)
    eye = qtgen.BlockMatrix(Am.n, 256, 32, np.arange(24, dtype=np.int32), np.arange(24, dtype=np.int32),
                            np.repeat(np.eye(32)[None], 24, axis=0))
    A, I = mk(qt, ctx, Am), mk(qt, ctx, eye)
    o = np.lexsort((Am.bcol, Am.brow))
    for X, Y in [(A, I), (I, A)]:
        r, c, v = (X @ Y).to_blocks()
        assert np.array_equal(r, Am.brow[o]) and np.array_equal(c, Am.bcol[o])
        assert np.array_equal(v, Am.vals[o])


@pytest.mark.parametrize("n,d", [(2048, 128), (4096, 100)])
def test_banded_all_ones_closed_form(qt, ctx, n, d):
    bs = 32
    nbr = n // bs
    br, bc = qtgen.pattern_banded(nbr, qtgen.band_blocks(d, bs))
    v = qtgen.block_values(br, bc, bs, 0, "ones", band_d=d)
    A = qt.Matrix.from_blocks(ctx, n, 512, bs, br, bc, v)
    r, c, w = (A @ A).to_blocks()
    D = qtgen.band_blocks(d, bs)
    assert np.all(np.abs(r - c) <= 2 * D)
    i = r[:, None, None].astype(np.int64) * bs + np.arange(bs)[None, :, None]
    j = c[:, None, None].astype(np.int64) * bs + np.arange(bs)[None, None, :]
    lo = np.maximum(np.maximum(i, j) - d, 0)
    hi = np.minimum(np.minimum(i, j) + d, n - 1)
    ref = np.where(np.abs(i - j) <= 2 * d, np.maximum(hi - lo + 1, 0), 0)
    assert np.array_equal(w, ref.astype(float))


def test_empty_operands(qt, ctx):
    z = np.zeros(0, np.int32)
    E = qt.Matrix.from_blocks(ctx, 256, 64, 32, z, z, np.zeros((0, 32, 32)))
    rng = np.random.default_rng(1)
    Am = random_bm(rng, 8, 32, 0.5, "int", 64)
    A = mk(qt, ctx, Am)
    for X, Y in [(E, A), (A, E), (E, E)]:
        C, st = X.multiply(Y)
        assert C.nblocks == 0 and st.block_products == 0
        r, c, v = C.to_blocks()
        assert r.shape[0] == 0


def test_disjoint_k_gives_empty(qt, ctx):
    # A has only block column 0, B only block row 1: every product is NIL
    A = qt.Matrix.from_blocks(ctx, 64, 32, 32, np.array([0, 1], np.int32), np.array([0, 0], np.int32),
                              np.ones((2, 32, 32)))
    B = qt.Matrix.from_blocks(ctx, 64, 32, 32, np.array([1], np.int32), np.array([1], np.int32),
                              np.ones((1, 32, 32)))
    C, st = A.multiply(B)
    assert C.nblocks == 0 and st.block_products == 0
    assert C.level_nodes() == [0, 0]  # 2x2 blocks: levels 0 (root) and 1 (blocks)


def test_errors(qt, ctx):
    one = np.ones((1, 32, 32))
    with pytest.raises(qt.QtError) as e:
        qt.Matrix.from_blocks(ctx, 64, 32, 32, np.array([2], np.int32), np.array([0], np.int32), one)
    assert e.value.name == "QT_ERANGE" and "brow=2" in str(e.value)
    with pytest.raises(qt.QtError) as e:
        qt.Matrix.from_blocks(ctx, 64, 32, 32, np.array([1, 1], np.int32), np.array([0, 0], np.int32),
                              np.ones((2, 32, 32)))
    assert e.value.name == "QT_EDUP" and "brow=1, bcol=0" in str(e.value)
    with pytest.raises(qt.QtError) as e:
        qt.Matrix.from_blocks(ctx, 48, 32, 32, np.array([0], np.int32), np.array([0], np.int32), one)
    assert e.value.name == "QT_EINVAL"
    with pytest.raises(qt.QtError) as e:
        qt.Matrix.from_blocks(ctx, 64, 96, 32, np.array([0], np.int32), np.array([0], np.int32), one)
    assert e.value.name == "QT_EINVAL"
    z = np.array([0], np.int32)
    A = qt.Matrix.from_blocks(ctx, 64, 32, 32, z, z, one)
    B = qt.Matrix.from_blocks(ctx, 128, 32, 32, z, z, one)
    with pytest.raises(qt.QtError) as e:
        A @ B
    assert e.value.name == "QT_EDIM"
    B = qt.Matrix.from_blocks(ctx, 64, 64, 32, z, z, one)
    with pytest.raises(qt.QtError) as e:
        A @ B
    assert e.value.name == "QT_EBS"
    B = qt.Matrix.from_blocks(ctx, 64, 32, 32, z, z, one.astype(np.float32))
    with pytest.raises(qt.QtError) as e:
        A @ B
    assert e.value.name == "QT_EDTYPE"


def test_run_to_run_bitwise(qt, ctx):
    c = qtgen.config(2, small=True)
    A = mk(qt, ctx, c["A"])
    v0 = (A @ A).to_blocks()[2]
    for _ in range(3):
        assert np.array_equal((A @ A).to_blocks()[2], v0)


def test_leaf_dim_invariance(qt, ctx):
    c = qtgen.config(2, small=True)
    M = c["A"]
    outs = []
    for leaf in (32, 256, 2048):
        A = qt.Matrix.from_blocks(ctx, M.n, leaf, 32, M.brow, M.bcol, M.vals)
        outs.append((A @ A).to_blocks())
    for o in outs[1:]:
        assert_same_pattern(o, outs[0])
        assert np.array_equal(o[2], outs[0][2])


# ----------------------------------------------------------------- configs


def test_cfg1_dense_int_bitexact_and_uniform(qt, ctx):
    for kind in ("int", "uniform"):
        c = qtgen.config(1, kind)
        A, B = mk(qt, ctx, c["A"]), mk(qt, ctx, c["B"])
        C, st = A.multiply(B)
        got = C.to_blocks()
        ref = oracle.spgemm(16, 32, as_tuple(c["A"]), as_tuple(c["B"]))
        assert st.block_products == 4096
        assert list(st.level_tasks[:5]) == [1, 8, 64, 512, 4096]
        if kind == "int":
            assert_same_pattern(got, ref)
            assert np.array_equal(got[2], ref[2])
        else:
            assert_close_f64(got, ref, as_tuple(c["A"]), as_tuple(c["B"]), 16, 32, 512)


def _sampled_rows_check(qt, ctx, c, rows, kind):
    Am, Bm = c["A"], c["B"]
    A = mk(qt, ctx, Am)
    B = A if c["same"] else mk(qt, ctx, Bm)
    C, st = A.multiply(B)
    nbr = Am.nbr
    L, _ = oracle.tree_levels(Am.n, 32, Am.leaf_dim)
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts(
        L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    got = C.to_blocks()
    pr, pc = oracle.pattern_product(nbr, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    assert_same_pattern(got, (pr, pc))
    sel = np.zeros(len(got[0]), bool)
    for lo, hi in rows:
        sel |= (got[0] >= lo) & (got[0] < hi)
        ref = oracle.spgemm(nbr, 32, as_tuple(Am), as_tuple(Bm), rows=(lo, hi))
        m = (got[0] >= lo) & (got[0] < hi)
        g = (got[0][m], got[1][m], got[2][m])
        if kind == "int":
            assert_same_pattern(g, ref)
            assert np.array_equal(g[2], ref[2])
        else:
            assert_same_pattern(g, ref)
            d = g[2] - ref[2]
            assert np.linalg.norm(d) <= REL_FRO_F64 * np.linalg.norm(ref[2])
            _, _, bound = oracle.higham_bound(nbr, 32, as_tuple(Am), as_tuple(Bm), nbr * 32,
                                              rows=(lo, hi))
            assert np.all(np.abs(d) <= bound + 1e-300)
    return st


@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_cfg2_banded_full_size_sampled(qt, ctx, kind):
    c = qtgen.config(2, kind)
    st = _sampled_rows_check(qt, ctx, c, [(0, 8), (250, 262), (504, 512)], kind)
    assert st.block_products == 2048800 and st.c_blocks == 61888


@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_cfg3_random_full_size_sampled(qt, ctx, kind):
    """Config 3 at full size: full pattern = the boolean product; sampled
    block rows bit-exact (integer variant) / within the FP64 bar (uniform)."""
    c = qtgen.config(3, kind)
    _sampled_rows_check(qt, ctx, c, [(0, 16), (500, 520), (1000, 1024)], kind)


@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_cfg4_eslike_full_size_sampled(qt, ctx, kind):
    """Config 4 at full size (3072 atoms): full pattern and per-level task
    counts vs the oracle; sampled atom rows bit-exact on integer values."""
    c = qtgen.config(4, kind)
    _sampled_rows_check(qt, ctx, c, [(0, 4), (1500, 1504), (3068, 3072)], kind)


def test_cfg1_2_3_4_int_every_config_once(qt, ctx):
    """The integer variants of configs 1-4 in one place (north star: bit-exact
    on small-integer inputs for all five configs; config 5 is checked per
    rank in test_virtual_ranks_cfg5_full_size_int_values)."""
    for idx in (1, 2, 3, 4):
        c = qtgen.config(idx, "int")
        nbr = c["A"].nbr
        _sampled_rows_check(qt, ctx, c, [(nbr // 2 - 2, nbr // 2 + 2)], "int")


def test_cfg4_small_full_oracle(qt, ctx):
    c = qtgen.config(4, small=True)
    Am = c["A"]
    A = mk(qt, ctx, Am)
    got = (A @ A).to_blocks()
    ref = oracle.spgemm(Am.nbr, 32, as_tuple(Am), as_tuple(Am))
    assert_close_f64(got, ref, as_tuple(Am), as_tuple(Am), Am.nbr, 32, Am.nbr * 32)


# ----------------------------------------------------------------- virtual ranks (multi-GPU path)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_virtual_ranks_bitwise_and_bytes(qt, ctx, P):
    c = qtgen.config(5, P=P, small=True)
    Am = c["A"]
    A = mk(qt, ctx, Am)
    full = (A @ A).to_blocks()
    per = Am.nbr // P
    bounds = [g * per for g in range(P + 1)]
    plan = oracle.exchange_plan(bounds, (Am.brow, Am.bcol), (Am.brow, Am.bcol), 8192)
    for g in range(P):
        Cg, st = A.multiply_virtual(A, P, g, bounds)
        r, cc, v = Cg.to_blocks()
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(cc, full[1][m])
        assert np.array_equal(v, full[2][m])                  # P-10: bitwise across P
        assert st.bytes_recv_payload == plan[g]["payload_bytes"]
        assert st.bytes_recv_meta == plan[g]["meta_bytes"]
        assert st.blocks_recv == plan[g]["blocks_received"]


def test_virtual_single_rank_moves_nothing(qt, ctx):
    c = qtgen.config(2, small=True)
    A = mk(qt, ctx, c["A"])
    C, st = A.multiply_virtual(A, 1, 0, [0, c["A"].nbr])
    assert st.bytes_recv_payload == 0 and st.bytes_recv_meta == 0


# ----------------------------------------------------------------- truncate


@pytest.mark.parametrize("tau", [0.0, 0.5, 3.0, 20.0])
def test_truncate_matches_oracle(qt, ctx, tau):
    rng = np.random.default_rng(17)
    Mm = random_bm(rng, 20, 32, 0.4, "uniform", 128)
    Mm.vals *= rng.uniform(0, 1, size=(Mm.nb, 1, 1)) ** 4
    A = mk(qt, ctx, Mm)
    r, c, v = A.truncate(tau).to_blocks()
    rr, rc, rv = oracle.truncate(Mm.brow, Mm.bcol, Mm.vals, tau)
    assert np.array_equal(r, rr) and np.array_equal(c, rc) and np.array_equal(v, rv)


# ----------------------------------------------------------------- loopback ranks (the NCCL code path)


def _loopback_run(qt, P, c, bounds):
    import threading
    import torch
    Am = c["A"]
    hub = qt.LoopbackHub(P)
    out = [None] * P
    errs = []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            ctx = qt.Context(0, stream=s, loopback=(hub, g, P))
            m = (Am.brow >= bounds[g]) & (Am.brow < bounds[g + 1])
            A = qt.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, 32, Am.brow[m], Am.bcol[m], Am.vals[m],
                                      row_bounds=bounds)
            C, st = A.multiply(A)
            out[g] = (C.to_blocks(), st.as_dict(), A.info(), C.info())
            C.close()
            A.close()
            ctx.close()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank_fn, args=(g,)) for g in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    hub.close()
    assert not errs, errs
    return out


@pytest.mark.parametrize("P", [2, 4])
def test_loopback_ranks_nccl_path(qt, ctx, P):
    """Rank threads on the loopback transport run the NCCL code path; each
    rank's rows equal the oracle's (integer inputs: exact) and the
    single-rank product's (bitwise, pin P-10)."""
    c = qtgen.config(5, "int", P=P, small=True)
    Am = c["A"]
    full = (mk(qt, ctx, Am) @ mk(qt, ctx, Am)).to_blocks()
    ref = oracle.spgemm(Am.nbr, 32, as_tuple(Am), as_tuple(Am))
    assert_same_pattern(full, ref)
    assert np.array_equal(full[2], ref[2])
    per = Am.nbr // P
    bounds = [g * per for g in range(P)] + [Am.nbr]
    plan = oracle.exchange_plan(bounds, (Am.brow, Am.bcol), (Am.brow, Am.bcol), 8192)
    out = _loopback_run(qt, P, c, bounds)
    for g in range(P):
        (r, cc, v), st, ainfo, cinfo = out[g]
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(cc, full[1][m])
        assert np.array_equal(v, full[2][m])                  # bitwise across P
        assert st["bytes_recv_payload"] == plan[g]["payload_bytes"]
        assert st["bytes_recv_meta"] == plan[g]["meta_bytes"]
        assert ainfo["global_nblocks"] == Am.nb
        assert (cinfo["row_lo"], cinfo["row_hi"]) == (bounds[g], bounds[g + 1])
    # what each rank sent = what the others received from it
    sent = sum(o[1]["bytes_sent_payload"] for o in out)
    assert sent == sum(p["payload_bytes"] for p in plan)


def test_loopback_cfg4_small_two_ranks(qt, ctx):
    c = qtgen.config(4, "int", small=True)
    Am = c["A"]
    full = oracle.spgemm(Am.nbr, 32, as_tuple(Am), as_tuple(Am))
    bounds = [0, Am.nbr // 3, Am.nbr]   # uneven strips
    out = _loopback_run(qt, 2, c, bounds)
    for g in range(2):
        (r, cc, v), st, _, _ = out[g]
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(v, full[2][m])


@pytest.mark.parametrize("P,tau", [(2, 5.0), (3, 40.0), (2, 0.0)])
def test_loopback_truncate_matches_single_rank(qt, ctx, P, tau):
    import threading
    import torch
    rng = np.random.default_rng(23)
    Mm = random_bm(rng, 24, 32, 0.4, "uniform", 128)
    Mm.vals *= rng.uniform(0, 1, size=(Mm.nb, 1, 1)) ** 4
    ref = oracle.truncate(Mm.brow, Mm.bcol, Mm.vals, tau)
    single = mk(qt, ctx, Mm).truncate(tau).to_blocks()
    assert np.array_equal(single[0], ref[0]) and np.array_equal(single[2], ref[2])
    bounds = [g * 24 // P for g in range(P)] + [24]
    hub = qt.LoopbackHub(P)
    out, errs = [None] * P, []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            c = qt.Context(0, stream=torch.cuda.Stream(), loopback=(hub, g, P))
            m = (Mm.brow >= bounds[g]) & (Mm.brow < bounds[g + 1])
            A = qt.Matrix.from_blocks(c, Mm.n, 128, 32, Mm.brow[m], Mm.bcol[m], Mm.vals[m], row_bounds=bounds)
            T = A.truncate(tau)
            out[g] = (T.to_blocks(), T.info())
            T.close()
            A.close()
            c.close()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank_fn, args=(g,)) for g in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    hub.close()
    assert not errs, errs
    r = np.concatenate([o[0][0] for o in out])
    c_ = np.concatenate([o[0][1] for o in out])
    v = np.concatenate([o[0][2] for o in out])
    assert np.array_equal(r, ref[0]) and np.array_equal(c_, ref[1]) and np.array_equal(v, ref[2])
    assert all(o[1]["global_nblocks"] == len(ref[0]) for o in out)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_virtual_ranks_cfg5_full_size_int_values(qt, ctx, P):
    """Config 5 at full size, integer variant, every rank of P = 2/4/8 (the
    weak-scaling run): rank g's C rows are bit-exact against the oracle on
    sampled block rows (its first, middle and last rows, which read the halo
    received from both neighbours), and the bytes it receives equal the
    oracle's exchange plan.  Each rank's strip is generated with its halo
    rows only (the rows its products read)."""
    nbr = 512 * P
    bounds = [512 * q for q in range(P + 1)]
    for g in range(P):
        lo, hi = 512 * g, 512 * (g + 1)
        c = qtgen.config(5, "int", P=P, rows=(max(0, lo - 32), min(nbr, hi + 32)))
        Am = c["A"]
        A = mk(qt, ctx, Am)
        Cg, st = A.multiply_virtual(A, P, g, bounds)
        plan = oracle.exchange_plan(bounds, (Am.brow, Am.bcol), (Am.brow, Am.bcol), 8192)[g]
        assert st.bytes_recv_payload == plan["payload_bytes"]
        got = Cg.to_blocks()
        assert got[0].min() >= lo and got[0].max() < hi
        for rlo, rhi in ((lo, lo + 3), (lo + 254, lo + 258), (hi - 3, hi)):
            ref = oracle.spgemm(nbr, 32, as_tuple(Am), as_tuple(Am), rows=(rlo, rhi))
            m = (got[0] >= rlo) & (got[0] < rhi)
            assert_same_pattern((got[0][m], got[1][m]), ref)
            assert np.array_equal(got[2][m], ref[2])
        A.close()
        Cg.close()


@pytest.mark.parametrize("P,g,expect", [(2, 0, 17039360), (4, 1, 34078720), (8, 5, 34078720)])
def test_virtual_rank_bytes_cfg5_full_size(qt, ctx, P, g, expect):
    """Config 5 at full size (N = 16384*P): the bytes rank g receives in the
    weak-scaling run — the paper's central quantity — equal the
    oracle's exchange plan (34.1 MB per interior GPU, flat in P; 17.0 MB at P=2).
    Only rank g's strip and its halo rows are generated (nothing else is read)."""
    nbr = 512 * P
    lo, hi = 512 * g, 512 * (g + 1)
    c = qtgen.config(5, P=P, rows=(max(0, lo - 32), min(nbr, hi + 32)))
    Am = c["A"]
    A = mk(qt, ctx, Am)
    bounds = [512 * q for q in range(P + 1)]
    Cg, st = A.multiply_virtual(A, P, g, bounds)
    plan = oracle.exchange_plan(bounds, (Am.brow, Am.bcol), (Am.brow, Am.bcol), 8192)[g]
    assert st.bytes_recv_payload == plan["payload_bytes"] == expect
    assert st.bytes_recv_meta == plan["meta_bytes"]
    # the strip's product is complete: interior rows have the full 2*64+1 C blocks
    rows = Cg.to_blocks()[0]
    assert rows.min() >= lo and rows.max() < hi
    counts = np.bincount(rows - lo, minlength=hi - lo)
    assert counts.max() == 129



# ----------------------------------------------------------------- transposed task types


@pytest.mark.parametrize("ta,tb", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
@pytest.mark.parametrize("nbr,p", [(5, 0.6), (37, 0.2)])
def test_transposed_products(qt, ctx, ta, tb, kind, nbr, p):
    rng = np.random.default_rng(nbr + 3 * ta + 7 * tb + (kind == "int"))
    Am = random_bm(rng, nbr, 32, p, kind, 128)
    Bm = random_bm(rng, nbr, 32, p, kind, 128)
    C, st = mk(qt, ctx, Am).multiply_ex(mk(qt, ctx, Bm), ta, tb)
    got = C.to_blocks()
    ref = oracle.spgemm_t(nbr, 32, as_tuple(Am), as_tuple(Bm), ta, tb)
    if kind == "int":
        assert_same_pattern(got, ref)
        assert np.array_equal(got[2], ref[2])
    else:
        a = oracle.transpose(*as_tuple(Am)) if ta else as_tuple(Am)
        b = oracle.transpose(*as_tuple(Bm)) if tb else as_tuple(Bm)
        assert_close_f64(got, ref, a, b, nbr, 32, nbr * 32)
    L, _ = oracle.tree_levels(Am.n, 32, 128)
    ar = (Am.bcol, Am.brow) if ta else (Am.brow, Am.bcol)
    br = (Bm.bcol, Bm.brow) if tb else (Bm.brow, Bm.bcol)
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts(L, ar, br)


def test_transposed_aat_banded(qt, ctx):
    c = qtgen.config(2, "int", small=True)
    A = mk(qt, ctx, c["A"])
    got = A.multiply_ex(A, False, True)[0].to_blocks()   # A A^T
    ref = oracle.spgemm_t(c["A"].nbr, 32, as_tuple(c["A"]), as_tuple(c["A"]), False, True)
    assert_same_pattern(got, ref)
    assert np.array_equal(got[2], ref[2])


# ----------------------------------------------------------------- symmetric square (§3.3)


def random_sym_upper(rng, nbr, p, kind, leaf):
    mask = np.triu(rng.random((nbr, nbr)) < p)
    np.fill_diagonal(mask, rng.random(nbr) < 0.7)
    br, bc = np.nonzero(mask)
    v = (rng.integers(-4, 5, size=(len(br), 32, 32)).astype(np.float64) if kind == "int"
         else rng.uniform(-1, 1, size=(len(br), 32, 32)))
    for t in range(len(br)):
        if br[t] == bc[t]:
            v[t] = np.triu(v[t]) + np.triu(v[t], 1).T
    return qtgen.BlockMatrix(nbr * 32, leaf, 32, br.astype(np.int32), bc.astype(np.int32), v)


@pytest.mark.parametrize("nbr,p,leaf", [(1, 1.0, 32), (4, 1.0, 64), (7, 0.5, 64), (24, 0.25, 256),
                                        (61, 0.08, 512)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_symm_square(qt, ctx, nbr, p, leaf, kind):
    rng = np.random.default_rng(100 + nbr + (kind == "int"))
    Um = random_sym_upper(rng, nbr, p, kind, leaf)
    C, st = mk(qt, ctx, Um).symm_square()
    got = C.to_blocks()
    ref = oracle.symm_square(nbr, 32, as_tuple(Um))
    if kind == "int":
        assert_same_pattern(got, ref)
        assert np.array_equal(got[2], ref[2])
    else:
        full = oracle.expand_symmetric(*as_tuple(Um))
        assert_same_pattern(got, ref)
        d = got[2] - ref[2]
        assert np.linalg.norm(d) <= REL_FRO_F64 * np.linalg.norm(ref[2])
        br_, bc_, bound = oracle.higham_bound(nbr, 32, full, full, nbr * 32)
        assert np.all(np.abs(d) <= bound[br_ <= bc_] + 1e-300)
    L, _ = oracle.tree_levels(Um.n, 32, leaf)
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts_sym(L, (Um.brow, Um.bcol))
    assert st.block_products == oracle.level_task_counts_sym(L, (Um.brow, Um.bcol))[-1]


def test_symm_square_banded_cfg2_small_and_half_work(qt, ctx):
    c = qtgen.config(2, "int", small=True, symmetric=True)
    full = c["A"]
    U = qtgen.upper(full)
    A = mk(qt, ctx, full)
    Cf, stf = A.multiply(A)
    Cs, sts = mk(qt, ctx, U).symm_square()
    got = Cs.to_blocks()
    r, cc, v = Cf.to_blocks()
    k = r <= cc
    assert np.array_equal(got[0], r[k]) and np.array_equal(got[1], cc[k])
    assert np.array_equal(got[2], v[k])              # integers: exact, same as the full multiply
    # about half the work (ratio in [0.4, 0.6]; diagonal C blocks are computed whole)
    assert 0.4 <= sts.block_products / stf.block_products <= 0.6


def test_symm_square_rejects_lower_blocks(qt, ctx):
    A = qt.Matrix.from_blocks(ctx, 64, 32, 32, np.array([1], np.int32), np.array([0], np.int32),
                              np.ones((1, 32, 32)))
    with pytest.raises(qt.QtError) as e:
        A.symm_square()
    assert e.value.name == "QT_EINVAL" and "brow=1, bcol=0" in str(e.value)


# ----------------------------------------------------------------- block size 64


def random_bm64(rng, nbr, p, kind, leaf, dtype=np.float64):
    mask = rng.random((nbr, nbr)) < p
    br, bc = np.nonzero(mask)
    v = (rng.integers(-4, 5, size=(len(br), 64, 64)) if kind == "int"
         else rng.uniform(-1, 1, size=(len(br), 64, 64))).astype(dtype)
    return qtgen.BlockMatrix(nbr * 64, leaf, 64, br.astype(np.int32), bc.astype(np.int32), v)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_bs64_roundtrip(qt, ctx, dtype):
    rng = np.random.default_rng(64)
    M = random_bm64(rng, 9, 0.4, "uniform", 128, dtype)
    perm = rng.permutation(M.nb)
    A = qt.Matrix.from_blocks(ctx, M.n, 128, 64, M.brow[perm], M.bcol[perm], M.vals[perm])
    assert A.info()["bs"] == 64 and A.nblocks == M.nb
    r, c, v = A.to_blocks()
    o = np.lexsort((M.bcol, M.brow))
    assert np.array_equal(r, M.brow[o]) and np.array_equal(c, M.bcol[o]) and np.array_equal(v, M.vals[o])


@pytest.mark.parametrize("nbr,p", [(1, 1.0), (3, 0.7), (19, 0.2)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_bs64_multiply(qt, ctx, nbr, p, kind):
    rng = np.random.default_rng(640 + nbr + (kind == "int"))
    Am = random_bm64(rng, nbr, p, kind, 256)
    Bm = random_bm64(rng, nbr, p, kind, 256)
    C, st = mk(qt, ctx, Am).multiply(mk(qt, ctx, Bm))
    got = C.to_blocks()
    ref = oracle.spgemm(nbr, 64, as_tuple(Am), as_tuple(Bm))
    assert_same_pattern(got, ref)
    if kind == "int":
        assert np.array_equal(got[2], ref[2])
    else:
        assert np.linalg.norm(got[2] - ref[2]) <= REL_FRO_F64 * np.linalg.norm(ref[2])
        _, _, bound = oracle.higham_bound(nbr, 64, as_tuple(Am), as_tuple(Bm), nbr * 64)
        assert np.all(np.abs(got[2] - ref[2]) <= bound + 1e-300)
    L, _ = oracle.tree_levels(Am.n, 64, 256)
    assert st.nlevels == L + 1
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts(L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    assert st.block_products == oracle.level_task_counts(L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))[-1]
    assert C.level_nodes() == oracle.level_node_counts(L, (ref[0], ref[1]))


def test_bs64_fp32_and_transposed(qt, ctx):
    rng = np.random.default_rng(6464)
    Am = random_bm64(rng, 11, 0.3, "int", 128, np.float32)
    Bm = random_bm64(rng, 11, 0.3, "int", 128, np.float32)
    for ta, tb in [(False, False), (True, False), (False, True)]:
        got = mk(qt, ctx, Am).multiply_ex(mk(qt, ctx, Bm), ta, tb)[0].to_blocks()
        ref = oracle.spgemm_t(11, 64, (Am.brow, Am.bcol, Am.vals.astype(np.float64)),
                              (Bm.brow, Bm.bcol, Bm.vals.astype(np.float64)), ta, tb)
        assert_same_pattern(got, ref)
        assert np.array_equal(got[2].astype(np.float64), ref[2])


def test_bs64_symm_square(qt, ctx):
    rng = np.random.default_rng(77)
    nbr = 12
    mask = np.triu(rng.random((nbr, nbr)) < 0.35)
    np.fill_diagonal(mask, True)
    br, bc = np.nonzero(mask)
    v = rng.integers(-4, 5, size=(len(br), 64, 64)).astype(np.float64)
    for t in range(len(br)):
        if br[t] == bc[t]:
            v[t] = np.triu(v[t]) + np.triu(v[t], 1).T
    U = (br.astype(np.int32), bc.astype(np.int32), v)
    A = qt.Matrix.from_blocks(ctx, nbr * 64, 256, 64, *U)
    C, st = A.symm_square()
    got = C.to_blocks()
    ref = oracle.symm_square(nbr, 64, U)
    assert_same_pattern(got, ref)
    assert np.array_equal(got[2], ref[2])
    L, _ = oracle.tree_levels(nbr * 64, 64, 256)
    assert st.block_products == oracle.level_task_counts_sym(L, U[:2])[-1]


def test_bs64_truncate_and_virtual(qt, ctx):
    rng = np.random.default_rng(90)
    M = random_bm64(rng, 16, 0.4, "uniform", 128)
    M.vals *= rng.uniform(0, 1, size=(M.nb, 1, 1)) ** 4
    A = mk(qt, ctx, M)
    r, c, v = A.truncate(10.0).to_blocks()
    rr, rc, rv = oracle.truncate(M.brow, M.bcol, M.vals, 10.0)
    assert np.array_equal(r, rr) and np.array_equal(c, rc) and np.array_equal(v, rv)
    full = (A @ A).to_blocks()
    bounds = [0, 5, 16]
    for g in range(2):
        Cg, st = A.multiply_virtual(A, 2, g, bounds)
        rg, cg, vg = Cg.to_blocks()
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(rg, full[0][m]) and np.array_equal(vg, full[2][m])
        plan = oracle.exchange_plan(bounds, (M.brow, M.bcol), (M.brow, M.bcol), 64 * 64 * 8)[g]
        assert st.bytes_recv_payload == plan["payload_bytes"]


# ----------------------------------------------------------------- norm-screened product


def _taus(Am, Bm):
    na = np.sqrt(oracle.block_norm2(Am.vals))
    nb = np.sqrt(oracle.block_norm2(Bm.vals))
    prods = np.unique(np.outer(na, nb).ravel())
    mids = (prods[1:] + prods[:-1]) / 2
    return [0.0] + [float(mids[int(len(mids) * f)]) for f in (0.1, 0.5, 0.9)]


@pytest.mark.parametrize("nbr,p", [(9, 0.5), (40, 0.15)])
@pytest.mark.parametrize("kind", ["int", "uniform"])
def test_screened_multiply(qt, ctx, nbr, p, kind):
    rng = np.random.default_rng(300 + nbr + (kind == "int"))
    Am = random_bm(rng, nbr, 32, p, kind, 128)
    Bm = random_bm(rng, nbr, 32, p, kind, 128)
    Am.vals *= rng.integers(1, 9, size=(Am.nb, 1, 1))     # varied block norms
    Bm.vals *= rng.integers(1, 9, size=(Bm.nb, 1, 1))
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    for tau in _taus(Am, Bm):
        C, st = A.multiply_screened(B, tau)
        got = C.to_blocks()
        ref = oracle.spgemm(nbr, 32, as_tuple(Am), as_tuple(Bm), tau=tau)
        assert_same_pattern(got, ref)
        if kind == "int":
            assert np.array_equal(got[2], ref[2])
        elif len(ref[0]):
            assert np.linalg.norm(got[2] - ref[2]) <= REL_FRO_F64 * np.linalg.norm(ref[2])
        assert st.block_products <= oracle.level_task_counts(
            oracle.tree_levels(Am.n, 32, 128)[0], (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))[-1]


def test_screened_eslike_small(qt, ctx):
    c = qtgen.config(4, small=True)
    Am = c["A"]
    A = mk(qt, ctx, Am)
    for tau in [1e-3, 1e-1]:
        C, st = A.multiply_screened(A, tau)
        got = C.to_blocks()
        ref = oracle.spgemm(Am.nbr, 32, as_tuple(Am), as_tuple(Am), tau=tau)
        assert_same_pattern(got, ref)
        assert np.linalg.norm(got[2] - ref[2]) <= REL_FRO_F64 * np.linalg.norm(ref[2])


# ---------------------------------------------- persistent BFS (large levels)

def _arrow_bm(rng, nbr, bs, kind, leaf):
    """Dense first block row and column plus the diagonal: level groups of very
    different sizes (one C node with ~nbr tasks, the rest with 1-2)."""
    mask = np.eye(nbr, dtype=bool)
    mask[0, :] = True
    mask[:, 0] = True
    mask |= rng.random((nbr, nbr)) < 0.01
    br, bc = np.nonzero(mask)
    if kind == "int":
        v = rng.integers(-4, 5, size=(len(br), bs, bs)).astype(np.float64)
    else:
        v = rng.uniform(-1, 1, size=(len(br), bs, bs))
    return qtgen.BlockMatrix(nbr * bs, leaf, bs, br.astype(np.int32), bc.astype(np.int32), v)


@pytest.mark.parametrize("nbr", [200, 700])
def test_bfs_skewed_group_sizes(qt, ctx, nbr):
    """The large-level kernel splits work by task counts and walks groups with
    W-lane sub-warps chosen from the mean group size: an arrow pattern puts a
    huge group next to thousands of tiny ones."""
    rng = np.random.default_rng(900 + nbr)
    Am = _arrow_bm(rng, nbr, 32, "int", 256)
    Bm = _arrow_bm(rng, nbr, 32, "int", 256)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    C, st = A.multiply(B)
    got = C.to_blocks()
    ref = oracle.spgemm(nbr, 32, as_tuple(Am), as_tuple(Bm))
    assert_same_pattern(got, ref)
    assert np.array_equal(got[2], ref[2])
    L = oracle.tree_levels(Am.n, 32, 256)[0]
    want = oracle.level_task_counts(L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    assert list(st.level_tasks[:len(want)]) == list(want)


def test_bfs_deep_sparse_levels(qt, ctx):
    """Random p = 0.002 on a 2048 x 2048 block grid (12 levels): almost every
    group at the lower levels has one task (W = 1 sub-warps) and several
    levels run in the persistent kernel."""
    rng = np.random.default_rng(77)
    nbr = 2048
    Am = random_bm(rng, nbr, 32, 0.002, "int", 2048)
    Bm = random_bm(rng, nbr, 32, 0.002, "int", 2048)
    A, B = mk(qt, ctx, Am), mk(qt, ctx, Bm)
    C, st = A.multiply(B)
    r, c, v = C.to_blocks()
    pat = oracle.pattern_product(nbr, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    assert np.array_equal(r, pat[0]) and np.array_equal(c, pat[1])
    L = oracle.tree_levels(Am.n, 32, 2048)[0]
    want = oracle.level_task_counts(L, (Am.brow, Am.bcol), (Bm.brow, Bm.bcol))
    assert list(st.level_tasks[:len(want)]) == list(want)
    # values on a sample of block rows
    lo, hi = 1000, 1040
    ref = oracle.spgemm(nbr, 32, as_tuple(Am), as_tuple(Bm), rows=(lo, hi))
    m = (r >= lo) & (r < hi)
    assert np.array_equal(r[m], ref[0]) and np.array_equal(c[m], ref[1])
    assert np.array_equal(v[m], ref[2])


def test_screened_everything_pruned(qt, ctx):
    """tau above every block-product norm: the BFS prunes at an upper level
    and the large levels see empty frontiers; C is the empty matrix."""
    rng = np.random.default_rng(31)
    Am = random_bm(rng, 300, 32, 0.05, "uniform", 256)
    A = mk(qt, ctx, Am)
    C, st = A.multiply_screened(A, 1e6)
    r, c, v = C.to_blocks()
    assert len(r) == 0 and st.block_products == 0


# ------------------------------------------ f1 / f4 at the full BASELINE size

def test_symm_square_cfg4_full_size_sampled(qt, ctx):
    """The paper's S^2 operation at config 4's full size (3072 atoms, symmetric
    values, upper triangle stored): C's pattern is the upper triangle of the
    full boolean product, sampled block rows match the oracle's product of
    the expanded matrix, and the work is half the full multiply's."""
    c = qtgen.config(4, symmetric=True)
    full = c["A"]
    U = qtgen.upper(full)
    C, st = mk(qt, ctx, U).symm_square()
    r, cc, v = C.to_blocks()
    nbr = full.nbr
    pr, pc = oracle.pattern_product(nbr, (full.brow, full.bcol), (full.brow, full.bcol))
    up = pr <= pc
    assert np.array_equal(r, pr[up]) and np.array_equal(cc, pc[up])
    L, _ = oracle.tree_levels(U.n, 32, U.leaf_dim)
    assert list(st.level_tasks[: L + 1]) == oracle.level_task_counts_sym(L, (U.brow, U.bcol))
    full_products = oracle.level_task_counts(L, (full.brow, full.bcol), (full.brow, full.bcol))[-1]
    assert 0.45 <= st.block_products / full_products <= 0.55
    for lo, hi in [(0, 4), (1500, 1504), (3064, 3072)]:
        ref = oracle.spgemm(nbr, 32, as_tuple(full), as_tuple(full), rows=(lo, hi))
        k = ref[0] <= ref[1]
        m = (r >= lo) & (r < hi)
        assert np.array_equal(r[m], ref[0][k]) and np.array_equal(cc[m], ref[1][k])
        d = v[m] - ref[2][k]
        assert np.linalg.norm(d) <= REL_FRO_F64 * np.linalg.norm(ref[2][k])


def test_screened_cfg4_full_size_sampled(qt, ctx):
    """Norm-screened product at config 4's full size (tau = 2): the pattern and
    sampled block rows equal the oracle's screened product, and the skipped
    products obey the error bound ||C - C~||_F <= sum of skipped ||A_IK|| ||B_KJ||."""
    c = qtgen.config(4)
    Am = c["A"]
    A = mk(qt, ctx, Am)
    tau = 2.0
    C, st = A.multiply_screened(A, tau)
    r, cc, v = C.to_blocks()
    nbr = Am.nbr
    for lo, hi in [(0, 4), (1500, 1504), (3068, 3072)]:
        ref = oracle.spgemm(nbr, 32, as_tuple(Am), as_tuple(Am), rows=(lo, hi), tau=tau)
        m = (r >= lo) & (r < hi)
        assert np.array_equal(r[m], ref[0]) and np.array_equal(cc[m], ref[1])
        assert np.linalg.norm(v[m] - ref[2]) <= REL_FRO_F64 * np.linalg.norm(ref[2])
    C0, st0 = A.multiply(A)
    assert st.block_products < st0.block_products


def test_read_back_async_matches_sync(qt, ctx):
    """qt_read_back_async: unpack on the context stream, device-to-host copies
    on the copy stream; after qt_ctx_synchronize the pinned host buffers hold
    exactly what qt_read_back returns, even when C is destroyed right after
    the call and its memory is reused by the next multiply."""
    import torch
    rng = np.random.default_rng(55)
    Am = random_bm(rng, 96, 32, 0.2, "uniform", 256)
    A = mk(qt, ctx, Am)
    refs, outs = [], []
    for _ in range(3):
        C, _ = A.multiply(A)
        ref = C.to_blocks()
        nb = len(ref[0])
        o = (torch.empty(nb, dtype=torch.int32).pin_memory(), torch.empty(nb, dtype=torch.int32).pin_memory(),
             torch.empty((nb, 32, 32), dtype=torch.float64).pin_memory())
        C.to_blocks(o, wait=False)
        C.close()
        refs.append(ref)
        outs.append(o)
        D, _ = A.multiply(A)      # reuses C's memory while the copies may still run
        D.close()
    ctx.synchronize()
    for ref, o in zip(refs, outs):
        assert np.array_equal(o[0].numpy(), ref[0]) and np.array_equal(o[1].numpy(), ref[1])
        assert np.array_equal(o[2].numpy(), ref[2])


def test_multiply_async_pipeline(qt, ctx):
    """qt_create from pinned host memory (H2D stream) + qt_multiply_async +
    qt_read_back_async, three steps issued back to back with A and C destroyed
    right after use: after qt_ctx_synchronize every step's host result equals
    the synchronous multiply's, and the stats other than timings are filled."""
    import torch
    rng = np.random.default_rng(56)
    mats = [random_bm(rng, 80, 32, 0.25, "uniform", 256) for _ in range(3)]
    refs = []
    for Am in mats:
        A = mk(qt, ctx, Am)
        C, st_ref = A.multiply(A)
        refs.append((C.to_blocks(), st_ref.block_products))
    outs, stats = [], []
    for Am, (ref, _) in zip(mats, refs):
        br = torch.from_numpy(Am.brow).pin_memory()
        bc = torch.from_numpy(Am.bcol).pin_memory()
        v = torch.from_numpy(Am.vals).pin_memory()
        A = qt.Matrix.from_blocks(ctx, Am.n, Am.leaf_dim, 32, br, bc, v)
        C, st = A.multiply(A, wait=False)
        A.close()
        nb = len(ref[0])
        o = (torch.empty(nb, dtype=torch.int32).pin_memory(), torch.empty(nb, dtype=torch.int32).pin_memory(),
             torch.empty((nb, 32, 32), dtype=torch.float64).pin_memory())
        C.to_blocks(o, wait=False)
        C.close()
        outs.append(o)
        stats.append(st)
    ctx.synchronize()
    for (ref, prods), o, st in zip(refs, outs, stats):
        assert st.block_products == prods
        assert np.array_equal(o[0].numpy(), ref[0]) and np.array_equal(o[1].numpy(), ref[1])
        assert np.array_equal(o[2].numpy(), ref[2])
