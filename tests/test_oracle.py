"""Pins of the oracle against what the paper and mathematics fix (no GPU).

Every check here compares ``oracle`` with something other than itself:
a value printed in SPEC/PAPER (tests/golden/, cited), a closed form, a library
routine on a case that reduces to it (numpy dense matmul, scipy sparse
product), brute force on tiny inputs, or an invariant.  Pins P-n refer to
SURVEY.md §8(c).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import qtgen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _dense_to_blocks(M, bs):
    n = M.shape[0]
    nbr = n // bs
    br, bc, v = [], [], []
    for I in range(nbr):
        for J in range(nbr):
            blk = M[I * bs:(I + 1) * bs, J * bs:(J + 1) * bs]
            if np.any(blk != 0):
                br.append(I), bc.append(J), v.append(blk.copy())
    if not br:
        return np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, bs, bs))
    return np.array(br, np.int32), np.array(bc, np.int32), np.array(v)


def _blocks_to_dense(nbr, bs, br, bc, v):
    out = np.zeros((nbr * bs, nbr * bs))
    for t in range(len(br)):
        out[br[t] * bs:(br[t] + 1) * bs, bc[t] * bs:(bc[t] + 1) * bs] = v[t]
    return out


def _random_block_matrix(rng, nbr, bs, p, kind="int"):
    mask = rng.random((nbr, nbr)) < p
    br, bc = np.nonzero(mask)
    if kind == "int":
        v = rng.integers(-4, 5, size=(len(br), bs, bs)).astype(np.float64)
    else:
        v = rng.uniform(-1, 1, size=(len(br), bs, bs))
    return br.astype(np.int32), bc.astype(np.int32), v


# --------------------------------------------------------------------- P-1


def test_hand_example_spec_s218():
    g = _gold("spec_hand_example.json")
    A, B = np.array(g["A"], float), np.array(g["B"], float)
    a = _dense_to_blocks(A, 1)
    b = _dense_to_blocks(B, 1)
    r, c, v = oracle.spgemm(2, 1, a, b, nthreads=1)
    C = _blocks_to_dense(2, 1, r, c, v)
    assert np.array_equal(C, np.array(g["C"], float))
    assert np.array_equal(oracle.dense_mm(A, B), np.array(g["C"], float))


# --------------------------------------------------------------------- P-2 / P-6


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
@pytest.mark.parametrize("p", [0.15, 0.5, 1.0])
def test_bruteforce_integer_exact(seed, p):
    rng = np.random.default_rng(seed)
    nbr, bs = 8, 4
    a = _random_block_matrix(rng, nbr, bs, p)
    b = _random_block_matrix(rng, nbr, bs, p)
    r, c, v = oracle.spgemm(nbr, bs, a, b, nthreads=3)
    # values: numpy's dense product of integer-valued doubles is exact here
    Ad = _blocks_to_dense(nbr, bs, *a)
    Bd = _blocks_to_dense(nbr, bs, *b)
    ref = Ad @ Bd
    assert np.array_equal(_blocks_to_dense(nbr, bs, r, c, v), ref)
    assert np.array_equal(oracle.dense_mm(Ad, Bd), ref)
    # pattern: the structural (boolean) product, independent scipy routine
    pr, pc = oracle.pattern_product(nbr, a[:2], b[:2])
    assert np.array_equal(r, pr) and np.array_equal(c, pc)
    # output sorted by (brow, bcol)
    key = r.astype(np.int64) * nbr + c
    assert np.all(np.diff(key) > 0)


def test_uniform_close_to_library_product():
    rng = np.random.default_rng(7)
    nbr, bs = 12, 8
    a = _random_block_matrix(rng, nbr, bs, 0.4, "uniform")
    b = _random_block_matrix(rng, nbr, bs, 0.4, "uniform")
    r, c, v = oracle.spgemm(nbr, bs, a, b)
    ref = _blocks_to_dense(nbr, bs, *a) @ _blocks_to_dense(nbr, bs, *b)
    got = _blocks_to_dense(nbr, bs, r, c, v)
    assert np.linalg.norm(got - ref) <= 1e-14 * np.linalg.norm(ref)


def test_structural_zero_blocks_kept():
    # reading C-1: a C block whose value cancels to zero is still in the pattern
    bs = 2
    a = (np.array([0, 0], np.int32), np.array([0, 1], np.int32),
         np.array([np.eye(2), np.eye(2)]))
    b = (np.array([0, 1], np.int32), np.array([1, 1], np.int32),
         np.array([np.eye(2), -np.eye(2)]))
    r, c, v = oracle.spgemm(2, bs, a, b)
    assert list(zip(r.tolist(), c.tolist())) == [(0, 1)]
    assert np.all(v == 0)


def test_empty_operands():
    e = (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 4, 4)))
    rng = np.random.default_rng(1)
    a = _random_block_matrix(rng, 4, 4, 0.5)
    for x, y in [(e, a), (a, e), (e, e)]:
        r, c, v = oracle.spgemm(4, 4, x, y)
        assert r.shape[0] == 0 and v.shape[0] == 0


def test_thread_count_invariance_uniform():
    rng = np.random.default_rng(3)
    nbr, bs = 16, 8
    a = _random_block_matrix(rng, nbr, bs, 0.3, "uniform")
    b = _random_block_matrix(rng, nbr, bs, 0.3, "uniform")
    r1, c1, v1 = oracle.spgemm(nbr, bs, a, b, nthreads=1)
    r5, c5, v5 = oracle.spgemm(nbr, bs, a, b, nthreads=5)
    assert np.array_equal(r1, r5) and np.array_equal(c1, c5)
    assert np.array_equal(v1, v5)  # bitwise


def test_row_range_sample():
    rng = np.random.default_rng(4)
    nbr, bs = 16, 4
    a = _random_block_matrix(rng, nbr, bs, 0.3)
    b = _random_block_matrix(rng, nbr, bs, 0.3)
    r, c, v = oracle.spgemm(nbr, bs, a, b)
    rs, cs, vs = oracle.spgemm(nbr, bs, a, b, rows=(5, 9))
    sel = (r >= 5) & (r < 9)
    assert np.array_equal(rs, r[sel]) and np.array_equal(cs, c[sel]) and np.array_equal(vs, v[sel])


# --------------------------------------------------------------------- P-3


def test_identity_both_sides():
    rng = np.random.default_rng(5)
    nbr, bs = 10, 8
    a = _random_block_matrix(rng, nbr, bs, 0.3, "uniform")
    eye = (np.arange(nbr, dtype=np.int32), np.arange(nbr, dtype=np.int32),
           np.repeat(np.eye(bs)[None], nbr, axis=0))
    for x, y in [(a, eye), (eye, a)]:
        r, c, v = oracle.spgemm(nbr, bs, x, y)
        o = np.lexsort((a[1], a[0]))
        assert np.array_equal(r, a[0][o]) and np.array_equal(c, a[1][o])
        assert np.array_equal(v, a[2][o])  # one nonzero term + exact zeros


# --------------------------------------------------------------------- P-4 / P-5


def _banded_ones(n, d, bs):
    nbr = n // bs
    br, bc = qtgen.pattern_banded(nbr, qtgen.band_blocks(d, bs))
    v = qtgen.block_values(br, bc, bs, 0, "ones", band_d=d)
    return br, bc, v


@pytest.mark.parametrize("n,d,bs", [(64, 3, 4), (96, 7, 8), (256, 16, 16), (128, 5, 4)])
def test_banded_closed_form_and_closure(n, d, bs):
    a = _banded_ones(n, d, bs)
    r, c, v = oracle.spgemm(n // bs, bs, a, a)
    C = _blocks_to_dense(n // bs, bs, r, c, v)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    lo = np.maximum(np.maximum(i, j) - d, 0)
    hi = np.minimum(np.minimum(i, j) + d, n - 1)
    ref = np.where(np.abs(i - j) <= 2 * d, np.maximum(hi - lo + 1, 0), 0)
    assert np.array_equal(C, ref.astype(float))
    # block band closure: C block band = 2 * input block band (bs | d+1 aside)
    D = qtgen.band_blocks(d, bs)
    assert np.all(np.abs(r - c) <= 2 * D)


def test_dense_all_ones():
    n, bs = 64, 8
    nbr = n // bs
    br, bc = qtgen.pattern_dense(nbr)
    v = np.ones((len(br), bs, bs))
    r, c, w = oracle.spgemm(nbr, bs, (br, bc, v), (br, bc, v))
    assert len(r) == nbr * nbr and np.all(w == n)


# --------------------------------------------------------------------- level counts (P-8)


def test_tree_levels_configs():
    assert oracle.tree_levels(512, 32, 128) == (4, 2)        # cfg1
    assert oracle.tree_levels(16384, 32, 1024) == (9, 4)     # cfg2
    assert oracle.tree_levels(32768, 32, 2048) == (10, 4)    # cfg3
    assert oracle.tree_levels(98304, 32, 4096) == (12, 5)    # cfg4 (padded to 4096 blocks)
    assert oracle.tree_levels(4, 1, 2) == (2, 1)
    assert oracle.tree_levels(32, 32, 32) == (0, 0)          # single block: the root is the block
    assert oracle.tree_levels(64, 32, 32) == (1, 1)          # 2x2 blocks
    assert oracle.tree_levels(96, 32, 64) == (2, 1)          # 3x3 blocks padded to 4x4 (C-3)
    assert oracle.tree_levels(128, 32, 64) == (2, 1)


def test_single_block_level_counts():
    """A 1x1-block product is one task at the single level (the root = the block)."""
    assert oracle.level_task_counts(0, ([0], [0]), ([0], [0])) == [1]
    assert oracle.level_node_counts(0, ([0], [0])) == [1]
    # 2x2 blocks, A = diag, B = dense: root task, then 4 block products
    assert oracle.level_task_counts(1, ([0, 1], [0, 1]), ([0, 0, 1, 1], [0, 1, 0, 1])) == [1, 4]


def test_dense_two_level_spec_s90():
    g = _gold("task_count_examples.json")
    br, bc = qtgen.pattern_dense(4)
    L, leaf = oracle.tree_levels(4, 1, 2)
    counts = oracle.level_task_counts(L, (br, bc), (br, bc))
    assert counts[: leaf + 1] == g["dense_two_level"]["levels"]


@pytest.mark.parametrize("L", [2, 3, 5])
def test_dense_counts_are_8_pow_l(L):
    br, bc = qtgen.pattern_dense(1 << L)
    assert oracle.level_task_counts(L, (br, bc), (br, bc)) == [8 ** l for l in range(L + 1)]


def _banded_level_closed_form(L, D):
    out = []
    for l in range(L + 1):
        s = L - l
        Dl = (D + (1 << s) - 1) >> s
        m = 1 << l
        K = np.arange(m)
        rK = np.minimum(K + Dl, m - 1) - np.maximum(K - Dl, 0) + 1
        out.append(int((rK * rK).sum()))
    return out


@pytest.mark.parametrize("L,D", [(6, 1), (6, 4), (9, 32), (7, 0)])
def test_banded_counts_closed_form_and_paper_bound(L, D):
    br, bc = qtgen.pattern_banded(1 << L, D)
    got = oracle.level_task_counts(L, (br, bc), (br, bc))
    assert got == _banded_level_closed_form(L, D)
    if D >= 1 and (D & (D - 1)) == 0:
        # P:578-587 Eq. eq:no_of_mmul_tasks_at_level_banded with d = D = 2^k
        k = D.bit_length() - 1
        for l in range(L + 1):
            dl = 1 if l < L - k else 2 ** (l - (L - k))
            assert got[l] < 2 ** l * (2 * dl + 1) ** 2
        # P:594-598 total bound
        N = 1 << L
        assert sum(got) < (4 + 4 / 7) * D * D * N + (5 + 1 / 3) * D * N + 2 * N + 9 / D * N


def test_cfg2_counts_survey_p7_p8():
    # cfg2: N=16384, bs 32, d=1024 -> block band 32, 512x512 blocks, L=9
    c = qtgen.config(2)
    A = c["A"]
    assert A.nb == 32224
    got = oracle.level_task_counts(9, (A.brow, A.bcol), (A.brow, A.bcol))
    assert got == _banded_level_closed_form(9, 32)
    assert got == [1, 8, 26, 62, 134, 750, 4884, 34952, 263824, 2048800]
    pr, pc = oracle.pattern_product(512, (A.brow, A.bcol), (A.brow, A.bcol))
    assert len(pr) == 61888 and np.all(np.abs(pr - pc) <= 64)


@pytest.mark.parametrize("P,total", [(2, 4212000), (4, 8538400), (8, 17191200)])
def test_cfg5_products_survey_p7(P, total):
    """Config 5 (N = 16384 P, half-bandwidth 1024 -> block band 32): the block
    products of C = A·A over all ranks (SURVEY P-7), from the banded closed
    form of the per-level counts on the padded quadtree."""
    nbr = 512 * P
    br, bc = qtgen.pattern_banded(nbr, qtgen.band_blocks(1024, 32))
    L, _ = oracle.tree_levels(nbr * 32, 32, 2048)
    got = oracle.level_task_counts(L, (br, bc), (br, bc))
    assert got[-1] == total
    # the paper's banded bound per level, 2^l (2 d_l + 1)^2 with d_l the band at level l
    for l, c in enumerate(got):
        d_l = -(-32 // (1 << (L - l)))
        assert c <= (1 << l) * (2 * d_l + 1) ** 2


def test_cfg4_overlap_growth_survey_p14():
    """Config 4 (3-D overlap pattern): task counts at least double from level
    to level below the root (the paper's overlap-matrix argument, P:634-635;
    SURVEY P-14), measured on the block pattern of the generator."""
    pos = qtgen.es_geometry()
    ar, ac, _ = qtgen.pattern_es(pos, 7.0)
    L, leaf = oracle.tree_levels(len(pos) * 32, 32, 4096)
    got = oracle.level_task_counts(L, (ar, ac), (ar, ac))
    assert (L, leaf) == (12, 5) and got[0] == 1
    assert all(got[l] >= 2 * got[l - 1] for l in range(1, L + 1)), got
    assert 6.0e6 < got[-1] < 6.6e6          # ~6.3 M block products (C-15 reading)


def _random_expectation(L, delta, l):
    # P:517-519 Eq. eq:no_of_mmul_tasks_at_level_random
    n_l = 4 ** (L - l)
    return 8 ** l * (1 - (1 - delta) ** n_l) ** 2


def test_random_formula_golden_example():
    g = _gold("task_count_examples.json")["random_formula_example"]
    assert _random_expectation(g["L"], g["delta"], g["l"]) == pytest.approx(g["C_l"])


def test_random_counts_match_paper_expectation():
    L, delta = 7, 0.05
    nbr = 1 << L
    seeds = [(21, 22), (23, 24), (25, 26), (27, 28)]
    acc = np.zeros(L + 1)
    for sa, sb in seeds:
        a = qtgen.pattern_random(nbr, delta, sa)
        b = qtgen.pattern_random(nbr, delta, sb)
        got = oracle.level_task_counts(L, a, b)
        for l in range(L + 1):
            assert got[l] <= 8 ** l                        # P:540-543 Eq. eq:bound_random_A
        acc += np.array(got)
    acc /= len(seeds)
    for l in range(L + 1):
        e = _random_expectation(L, delta, l)
        assert acc[l] == pytest.approx(e, rel=0.12)
        assert acc[l] <= 1.12 * 16 ** L * delta ** 2 / 2 ** l   # P:548-552 Eq. eq:bound_random_B


def test_node_counts_dense_and_banded():
    br, bc = qtgen.pattern_dense(8)
    assert oracle.level_node_counts(3, (br, bc)) == [1, 4, 16, 64]
    br, bc = qtgen.pattern_banded(8, 0)
    assert oracle.level_node_counts(3, (br, bc)) == [1, 2, 4, 8]


# --------------------------------------------------------------------- exchange plan (P-11)


def test_exchange_plan_single_rank_zero():
    c = qtgen.config(2, small=True)
    A = c["A"]
    plan = oracle.exchange_plan([0, A.nbr], (A.brow, A.bcol), (A.brow, A.bcol), 8192)
    assert plan[0]["payload_bytes"] == 0 and plan[0]["meta_bytes"] == 0


@pytest.mark.parametrize("P", [2, 4, 8])
def test_exchange_plan_banded_closed_form(P):
    # config 5: 512 block rows per rank, block band D = 32, 65 blocks per full row
    nbr, D, per = 512 * P, 32, 512
    br, bc = qtgen.pattern_banded(nbr, D)
    bounds = [g * per for g in range(P + 1)]
    plan = oracle.exchange_plan(bounds, (br, bc), (br, bc), 8192)
    for g in range(P):
        nb_neighbors = (g > 0) + (g < P - 1)
        # each halo row K is a full interior row: 2D+1 = 65 blocks
        assert plan[g]["rows_requested"] == D * nb_neighbors
        assert plan[g]["blocks_received"] == D * nb_neighbors * (2 * D + 1)
        assert plan[g]["payload_bytes"] == D * nb_neighbors * (2 * D + 1) * 8192
        assert sum(plan[g]["blocks_from"]) == plan[g]["blocks_received"]
        assert plan[g]["blocks_from"][g] == 0
    mx = max(p["payload_bytes"] for p in plan)
    assert mx == (34078720 if P > 2 else 17039360)   # 34.1 MB / 17.0 MB


def test_spsumma_golden():
    g = _gold("spsumma_example.json")
    assert oracle.spsumma_volume(g["m"], g["N"], g["p"]) == g["elements"]
    assert oracle.spsumma_volume(5, 100, 1) == 2 * 5 * 100


# --------------------------------------------------------------------- truncate (P-13)


def test_truncate_spec_examples():
    bs = 1
    br = np.array([0, 1], np.int32)
    bc = np.array([0, 1], np.int32)
    v = np.array([[[3.0]], [[4.0]]])
    r, c, w = oracle.truncate(br, bc, v, 3.5)
    assert list(zip(r.tolist(), c.tolist())) == [(1, 1)] and w[0, 0, 0] == 4.0
    r, c, w = oracle.truncate(br, bc, v, 0.0)
    assert len(r) == 2


def test_truncate_error_bound_and_maximality():
    rng = np.random.default_rng(9)
    br, bc, v = _random_block_matrix(rng, 12, 4, 0.5, "uniform")
    v = v * rng.uniform(0, 1, size=(len(br), 1, 1)) ** 3
    nrm = np.sqrt((v ** 2).sum(axis=(1, 2)))
    for tau in [0.0, 0.1, 0.5, 1.0, 3.0]:
        r, c, w = oracle.truncate(br, bc, v, tau)
        kept = set(zip(r.tolist(), c.tolist()))
        dropped = [t for t in range(len(br)) if (br[t], bc[t]) not in kept]
        err2 = sum(nrm[t] ** 2 for t in dropped)
        assert err2 < tau * tau or (tau == 0 and not dropped)
        # maximal prefix: the smallest kept block would push the error to >= tau
        if len(r):
            smallest = min(nrm[t] for t in range(len(br)) if (br[t], bc[t]) in kept)
            assert err2 + smallest ** 2 >= tau * tau
            assert smallest >= max([nrm[t] for t in dropped], default=0.0)


# --------------------------------------------------------------------- P-9


def test_higham_bound_holds_against_extended_precision():
    rng = np.random.default_rng(11)
    nbr, bs = 6, 8
    a = _random_block_matrix(rng, nbr, bs, 0.6, "uniform")
    b = _random_block_matrix(rng, nbr, bs, 0.6, "uniform")
    r, c, v = oracle.spgemm(nbr, bs, a, b)
    Ad = _blocks_to_dense(nbr, bs, *a).astype(np.longdouble)
    Bd = _blocks_to_dense(nbr, bs, *b).astype(np.longdouble)
    exact = Ad @ Bd
    br_, bc_, bound = oracle.higham_bound(nbr, bs, a, b, k_terms=nbr * bs)
    got = _blocks_to_dense(nbr, bs, r, c, v)
    ex = np.asarray(exact, dtype=np.float64)
    B = _blocks_to_dense(nbr, bs, br_, bc_, bound)
    err = np.abs(got.astype(np.longdouble) - exact).astype(np.float64)
    assert np.all(err <= B + 1e-300)
    assert np.max(err) > 0 or np.array_equal(got, ex)
    assert oracle.gamma(2080, 2.0 ** -53) == pytest.approx(2080 * 2.0 ** -53, rel=1e-10)


# --------------------------------------------------------------------- transposed task types


@pytest.mark.parametrize("ta,tb", [(True, False), (False, True), (True, True)])
def test_transposed_products_vs_dense_library(ta, tb):
    rng = np.random.default_rng(31 + 2 * ta + tb)
    nbr, bs = 7, 4
    a = _random_block_matrix(rng, nbr, bs, 0.4)
    b = _random_block_matrix(rng, nbr, bs, 0.4)
    r, c, v = oracle.spgemm_t(nbr, bs, a, b, ta, tb)
    Ad = _blocks_to_dense(nbr, bs, *a)
    Bd = _blocks_to_dense(nbr, bs, *b)
    ref = (Ad.T if ta else Ad) @ (Bd.T if tb else Bd)
    assert np.array_equal(_blocks_to_dense(nbr, bs, r, c, v), ref)
    pr, pc = oracle.pattern_product(nbr, (a[1], a[0]) if ta else a[:2], (b[1], b[0]) if tb else b[:2])
    assert np.array_equal(r, pr) and np.array_equal(c, pc)


def test_transpose_identity_ab_t():
    # (A B)^T = B^T A^T, both sides from the oracle's own routine on exact integers
    rng = np.random.default_rng(5)
    nbr, bs = 6, 4
    a = _random_block_matrix(rng, nbr, bs, 0.5)
    b = _random_block_matrix(rng, nbr, bs, 0.5)
    ab = oracle.spgemm(nbr, bs, a, b)
    btat = oracle.spgemm_t(nbr, bs, b, a, True, True)
    t = oracle.transpose(*ab)
    o = np.lexsort((t[1], t[0]))
    assert np.array_equal(t[0][o], btat[0]) and np.array_equal(t[2][o], btat[2])


# --------------------------------------------------------------------- symmetric square (§3.3)


def test_symm_square_spec_example():
    g = _gold("spec_symm_square_example.json")
    u = g["upper_A"]
    U = (np.array(u["brow"], np.int32), np.array(u["bcol"], np.int32),
         np.array(u["vals"], float).reshape(-1, 1, 1))
    r, c, v = oracle.symm_square(2, 1, U)
    e = g["upper_C"]
    assert r.tolist() == e["brow"] and c.tolist() == e["bcol"]
    assert v.ravel().tolist() == e["vals"]


def _random_symmetric_upper(rng, nbr, bs, p, kind="int"):
    mask = np.triu(rng.random((nbr, nbr)) < p)
    br, bc = np.nonzero(mask)
    v = (rng.integers(-4, 5, size=(len(br), bs, bs)).astype(float) if kind == "int"
         else rng.uniform(-1, 1, size=(len(br), bs, bs)))
    for t in range(len(br)):
        if br[t] == bc[t]:
            v[t] = np.triu(v[t]) + np.triu(v[t], 1).T   # symmetric diagonal block
    return br.astype(np.int32), bc.astype(np.int32), v


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_symm_square_vs_dense_library_and_half_work(seed):
    rng = np.random.default_rng(seed)
    nbr, bs = 16, 4                       # N = 64
    U = _random_symmetric_upper(rng, nbr, bs, 0.3)
    full = oracle.expand_symmetric(*U)
    D = _blocks_to_dense(nbr, bs, *full)
    assert np.array_equal(D, D.T)
    ref = D @ D
    r, c, v = oracle.symm_square(nbr, bs, U)
    assert np.all(r <= c)
    got = _blocks_to_dense(nbr, bs, r, c, v)
    for t in range(len(r)):
        I, J = r[t], c[t]
        assert np.array_equal(got[I * bs:(I + 1) * bs, J * bs:(J + 1) * bs],
                              ref[I * bs:(I + 1) * bs, J * bs:(J + 1) * bs])
    # every nonzero upper block of the product is present (structural pattern)
    pr, pc = oracle.pattern_product(nbr, full[:2], full[:2])
    k = pr <= pc
    assert np.array_equal(r, pr[k]) and np.array_equal(c, pc[k])
    # work: about half of the full multiply's block products ([0.4, 0.6])
    L, _ = oracle.tree_levels(nbr * bs, bs, bs)
    half = oracle.level_task_counts_sym(L, U[:2])[-1]
    whole = oracle.level_task_counts(L, full[:2], full[:2])[-1]
    assert 0.4 <= half / whole <= 0.6


def test_symm_square_identity():
    nbr, bs = 8, 4
    I = (np.arange(nbr, dtype=np.int32), np.arange(nbr, dtype=np.int32),
         np.repeat(np.eye(bs)[None], nbr, axis=0))
    r, c, v = oracle.symm_square(nbr, bs, I)
    assert np.array_equal(r, I[0]) and np.array_equal(c, I[1]) and np.array_equal(v, I[2])


def test_symm_level_counts_dense_closed_form():
    # dense symmetric pattern: at level l, pairs I <= J: m(m+1)/2, times m values of K
    L = 4
    nbr = 1 << L
    r, c = np.nonzero(np.triu(np.ones((nbr, nbr), bool)))
    got = oracle.level_task_counts_sym(L, (r, c))
    assert got == [(1 << l) * (1 << l) * ((1 << l) + 1) // 2 for l in range(L + 1)]


# --------------------------------------------------------------------- norm-screened product (f4)


def _scaled_int_matrix(rng, nbr, bs, p):
    br, bc, v = _random_block_matrix(rng, nbr, bs, p)
    v = v * rng.integers(1, 9, size=(len(br), 1, 1))     # varied block norms, still integers
    return br, bc, v


def _separating_taus(a, b):
    """thresholds half-way between distinct values of ||A_IK|| ||B_KJ||, so no
    product sits on the boundary (decisions independent of rounding order)"""
    na = np.sqrt((a[2] ** 2).sum(axis=(1, 2)))
    nb = np.sqrt((b[2] ** 2).sum(axis=(1, 2)))
    prods = np.unique(np.outer(na, nb).ravel())
    mids = (prods[1:] + prods[:-1]) / 2
    return [float(mids[len(mids) // 4]), float(mids[len(mids) // 2]), float(mids[3 * len(mids) // 4])]


@pytest.mark.parametrize("bs", [4, 16])
def test_screened_product_vs_bruteforce_enumeration(bs):
    """The screened product (f4) at block sizes 4 and 16 (the paper's S^2 runs
    screen at block size 16) equals the brute-force enumeration
    of the block products that pass ||A_IK|| ||B_KJ|| >= tau."""
    rng = np.random.default_rng(41 + bs)
    nbr = 8
    a = _scaled_int_matrix(rng, nbr, bs, 0.5)
    b = _scaled_int_matrix(rng, nbr, bs, 0.5)
    na = np.sqrt((a[2] ** 2).sum(axis=(1, 2)))
    nb = np.sqrt((b[2] ** 2).sum(axis=(1, 2)))
    for tau in _separating_taus(a, b) + [0.0]:
        ref = {}
        for p in range(len(a[0])):
            for q in range(len(b[0])):
                if a[1][p] != b[0][q] or na[p] * nb[q] < tau:
                    continue
                key = (int(a[0][p]), int(b[1][q]))
                ref[key] = ref.get(key, 0) + a[2][p] @ b[2][q]
        r, c, v = oracle.spgemm(nbr, bs, a, b, tau=tau)
        assert sorted(ref) == list(zip(r.tolist(), c.tolist()))
        for t in range(len(r)):
            assert np.array_equal(v[t], ref[(r[t], c[t])])


def test_screened_zero_tau_is_exact_and_error_bound():
    rng = np.random.default_rng(42)
    nbr, bs = 10, 4
    a = _random_block_matrix(rng, nbr, bs, 0.5, "uniform")
    b = _random_block_matrix(rng, nbr, bs, 0.5, "uniform")
    full = oracle.spgemm(nbr, bs, a, b)
    zero = oracle.spgemm(nbr, bs, a, b, tau=0.0)
    assert np.array_equal(full[0], zero[0]) and np.array_equal(full[2], zero[2])
    na = np.sqrt(oracle.block_norm2(a[2]))
    nb = np.sqrt(oracle.block_norm2(b[2]))
    prev = None
    for tau in _separating_taus(a, b):
        r, c, v = oracle.spgemm(nbr, bs, a, b, tau=tau)
        F = _blocks_to_dense(nbr, bs, *full)
        S = _blocks_to_dense(nbr, bs, r, c, v)
        skipped = sum(na[p] * nb[q] for p in range(len(a[0])) for q in range(len(b[0]))
                      if a[1][p] == b[0][q] and na[p] * nb[q] < tau)
        assert np.linalg.norm(F - S) <= skipped * (1 + 1e-12)
        cur = set(zip(r.tolist(), c.tolist()))
        if prev is not None:
            assert cur <= prev          # a larger tau keeps a subset of the pattern
        prev = cur


# ------------------------------------------------- multi-rank symmetric square (reading C-26)


def _symm_needed(ur, uc, lo, hi):
    """Brute force: indices of U blocks read by some product A(I,K)·A(K,J),
    I in [lo, hi), J >= I, where A(r,c) = U(r,c) and A(c,r) = U(r,c)^T."""
    src = {}
    for t, (r, c) in enumerate(zip(ur.tolist(), uc.tolist())):
        src[(r, c)] = t
        src[(c, r)] = t
    rows = {}
    for (r, c), t in src.items():
        rows.setdefault(r, []).append((c, t))
    need = set()
    for I in range(lo, hi):
        for K, t1 in rows.get(I, []):
            for J, t2 in rows.get(K, []):
                if J >= I:
                    need.add(t1)
                    need.add(t2)
    return need


@pytest.mark.parametrize("seed,nbr,p,P", [(1, 24, 0.15, 3), (2, 30, 0.3, 4), (3, 17, 0.5, 2), (4, 40, 0.08, 5)])
def test_exchange_plan_symm_is_exactly_the_needed_blocks(seed, nbr, p, P):
    rng = np.random.default_rng(seed)
    m = np.triu(rng.random((nbr, nbr)) < p)
    ur, uc = np.nonzero(m)
    cuts = np.sort(rng.choice(np.arange(1, nbr), size=P - 1, replace=False))
    bounds = [0] + cuts.tolist() + [nbr]
    plan = oracle.exchange_plan_symm(bounds, (ur, uc), 8192)
    for g in range(P):
        lo, hi = bounds[g], bounds[g + 1]
        local = set(np.nonzero((ur >= lo) & (ur < hi))[0].tolist())
        remote_needed = _symm_needed(ur, uc, lo, hi) - local
        assert set(plan[g]["selected"].tolist()) == remote_needed
        assert plan[g]["payload_bytes"] == len(remote_needed) * 8192


@pytest.mark.parametrize("P", [2, 4, 8])
def test_exchange_plan_symm_banded_closed_form(P):
    # config 5's upper band: block band D = 32, 512 block rows per rank.  An
    # interior rank receives the D full U rows above its strip (D+1 blocks
    # each) and the parts c >= lo of the D rows below it (1..D blocks):
    # D(D+1) + D(D+1)/2 blocks, vs D(2D+1) per neighbour for the full multiply.
    nbr, D, per = 512 * P, 32, 512
    br, bc = qtgen.pattern_banded(nbr, D)
    up = br <= bc
    bounds = [g * per for g in range(P + 1)]
    plan = oracle.exchange_plan_symm(bounds, (br[up], bc[up]), 8192)
    for g in range(P):
        n = (D * (D + 1) if g < P - 1 else 0) + (D * (D + 1) // 2 if g > 0 else 0)
        assert plan[g]["blocks_received"] == n
    full = oracle.exchange_plan(bounds, (br, bc), (br, bc), 8192)
    mx, mx_full = max(q["payload_bytes"] for q in plan), max(q["payload_bytes"] for q in full)
    assert mx == (1584 if P > 2 else 1056) * 8192 and mx_full == (34078720 if P > 2 else 17039360)


def test_exchange_plan_leaf_granular_banded():
    """fetching whole leaves (the paper's chunks) instead of exact
    blocks.  Config 5 at P = 4, leaf = 64 block rows: an interior rank needs
    the 32 block rows of each neighbouring leaf row next to its strip; the
    needed blocks touch two leaves per side, which hold the full band of the
    32 needed rows (32·65 blocks) plus, for the other 32 rows of the leaf row,
    the part of their band inside those two leaf columns (Σ_{k=33}^{64} k):
    3632 blocks per side = 1.75x the exact fetch (SURVEY: "roughly doubles")."""
    P, D, per, leaf = 4, 32, 512, 64
    br, bc = qtgen.pattern_banded(512 * P, D)
    bounds = [g * per for g in range(P + 1)]
    exact = oracle.exchange_plan(bounds, (br, bc), (br, bc), 8192)
    chunks = oracle.exchange_plan_leaf_granular(bounds, (br, bc), (br, bc), 8192, leaf)
    side = D * (2 * D + 1) + sum(range(D + 1, 2 * D + 1))                           # 3632
    for g in (1, 2):
        assert exact[g]["payload_bytes"] == 2 * D * (2 * D + 1) * 8192              # 34.1 MB
        assert chunks[g] == 2 * side * 8192                                         # 59.5 MB
    assert chunks[0] == side * 8192 and exact[0]["payload_bytes"] == D * (2 * D + 1) * 8192
