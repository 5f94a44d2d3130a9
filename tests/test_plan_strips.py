"""Row-strip plan (contiguous block-row strips of C, aligned
to quadtree node rows, balanced by block products).  qt_plan_strips is host
code: these tests run without a GPU.

Pins: the per-row product counts come from oracle.row_products (enumeration
of A's blocks against B's row counts); the largest strip must equal the
optimum over ALL aligned contiguous partitions (oracle.strips_min_max, a
brute-force dynamic program), so a plan that is merely "reasonable" fails."""
import numpy as np
import pytest

import oracle
import qtgen


@pytest.fixture(scope="module")
def qt():
    from paper_1501_07800_b200 import build
    build.build()
    from paper_1501_07800_b200 import qtmm
    return qtmm


def _check(qt, nbr, bs, ar, ac, br, bc, parts, align):
    bounds, prods = qt.plan_strips(nbr * bs, bs, parts, (ar, ac), br, align_rows=align)
    assert bounds[0] == 0 and bounds[-1] == nbr and np.all(np.diff(bounds) >= 0)
    assert all(b % align == 0 for b in bounds[:-1])
    rp = oracle.row_products(nbr, (ar, ac), (br, bc))
    for g in range(parts):
        assert prods[g] == rp[bounds[g]:bounds[g + 1]].sum()
    assert prods.max() == oracle.strips_min_max(rp, parts, align)
    return bounds, prods


@pytest.mark.parametrize("seed,nbr,p,parts,align", [(1, 40, 0.1, 3, 1), (2, 64, 0.05, 4, 4), (3, 37, 0.3, 5, 2),
                                                    (4, 16, 0.5, 8, 1), (5, 12, 0.2, 20, 1)])
def test_plan_is_optimal_on_random_patterns(qt, seed, nbr, p, parts, align):
    rng = np.random.default_rng(seed)
    a = rng.random((nbr, nbr)) < p
    a[rng.integers(0, nbr, 3)] |= rng.random(nbr) < 0.8       # a few heavy rows
    b = rng.random((nbr, nbr)) < p
    ar, ac = np.nonzero(a)
    br, bc = np.nonzero(b)
    _check(qt, nbr, 32, ar, ac, br, bc, parts, align)


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_plan_eslike_small(qt, parts):
    A = qtgen.config(4, small=True)["A"]
    bounds, prods = _check(qt, A.nbr, 32, A.brow, A.bcol, A.brow, A.bcol, parts, 4)
    assert prods.max() / prods.mean() < 1.25


def test_plan_banded_cfg5_leaf_aligned(qt):
    # config 5 at P = 8, leaf-aligned strips (64 block rows per leaf): the
    # optimum is within one leaf row of the equal strips the weak-scaling run uses
    A = qtgen.config(5, P=8)["A"]
    bounds, prods = _check(qt, A.nbr, 32, A.brow, A.bcol, A.brow, A.bcol, 8, 64)
    equal = np.arange(9) * (A.nbr // 8)
    assert np.abs(bounds - equal).max() <= 64
    assert prods.sum() == 17191200                      # pin P-7: cfg5 P=8 block products


def test_plan_block_size_16_and_errors(qt):
    rng = np.random.default_rng(9)
    nbr = 24
    a = rng.random((nbr, nbr)) < 0.2
    ar, ac = np.nonzero(a)
    _check(qt, nbr, 16, ar, ac, ar, ac, 3, 2)
    with pytest.raises(qt.QtError) as e:
        qt.plan_strips(nbr * 32, 32, 2, (np.array([nbr]), np.array([0])), np.array([0]))
    assert e.value.name == "QT_ERANGE"
    with pytest.raises(qt.QtError) as e:
        qt.plan_strips(nbr * 32, 32, 0, (ar, ac), ar)
    assert e.value.name == "QT_EINVAL"
    bounds, prods = qt.plan_strips(nbr * 32, 32, 3, (np.zeros(0), np.zeros(0)), np.zeros(0))
    assert bounds[0] == 0 and bounds[-1] == nbr and prods.sum() == 0


@pytest.mark.gpu
def test_plan_multi_rank_loopback_then_multiply(qt):
    """Each rank passes the blocks it holds under an initial equal split; the
    collective plan equals the single-process one; the planned strips then
    drive a loopback multi-rank multiply whose rows match the single-rank C."""
    import threading
    import torch
    A = qtgen.config(4, small=True)["A"]
    P, align = 3, 4
    ref_bounds, _ = qt.plan_strips(A.n, 32, P, (A.brow, A.bcol), A.brow, align_rows=align)
    ctx0 = qt.Context(0)
    M = qt.Matrix.from_blocks(ctx0, A.n, A.leaf_dim, 32, A.brow, A.bcol, A.vals)
    full = (M @ M).to_blocks()
    init = [g * (A.nbr // P) for g in range(P)] + [A.nbr]
    hub = qt.LoopbackHub(P)
    out, errs = [None] * P, []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            c = qt.Context(0, stream=torch.cuda.Stream(), loopback=(hub, g, P))
            m = (A.brow >= init[g]) & (A.brow < init[g + 1])
            bounds, _ = qt.plan_strips(A.n, 32, P, (A.brow[m], A.bcol[m]), A.brow[m], align_rows=align, ctx=c)
            mine = (A.brow >= bounds[g]) & (A.brow < bounds[g + 1])       # (redistribution: the test has all blocks)
            X = qt.Matrix.from_blocks(c, A.n, A.leaf_dim, 32, A.brow[mine], A.bcol[mine], A.vals[mine],
                                      row_bounds=bounds)
            C, st = X.multiply(X)
            out[g] = (bounds, C.to_blocks(), st.block_products)
            C.close()
            X.close()
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
    rp = oracle.row_products(A.nbr, (A.brow, A.bcol), (A.brow, A.bcol))
    for g in range(P):
        bounds, (r, c, v), prods = out[g]
        assert np.array_equal(bounds, ref_bounds)
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(v, full[2][m])
        assert prods == rp[bounds[g]:bounds[g + 1]].sum()


@pytest.mark.parametrize("seed", range(6))
def test_oracle_strips_min_max_vs_enumeration(seed):
    """Pin the oracle's DP: exhaustive enumeration of every aligned boundary set."""
    import itertools
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 10))
    w = rng.integers(0, 20, n)
    parts = int(rng.integers(1, 5))
    align = int(rng.integers(1, 3))
    cuts = list(range(align, n, align))
    best = None
    for k in range(0, min(parts - 1, len(cuts)) + 1):
        for cs in itertools.combinations(cuts, k):
            b = [0, *cs, n]
            m = max(int(w[b[i]:b[i + 1]].sum()) for i in range(len(b) - 1))
            best = m if best is None else min(best, m)
    assert oracle.strips_min_max(w, parts, align) == best


def test_oracle_row_products_small_closed_form():
    """Dense nbr x nbr A and B: every row of C has nbr^2 block products."""
    nbr = 5
    r, c = np.nonzero(np.ones((nbr, nbr), bool))
    assert np.all(oracle.row_products(nbr, (r, c), (r, c)) == nbr * nbr)
    # identity A: row I of C costs nnz(B row I)
    br, bc = np.nonzero(np.tril(np.ones((nbr, nbr), bool)))
    ii = np.arange(nbr)
    assert np.array_equal(oracle.row_products(nbr, (ii, ii), (br, bc)), np.arange(1, nbr + 1))
