"""Distributed read-back (qt_gather) on the loopback transport
(the NCCL code path with rank threads on one device).  Needs a B200.

Each rank computes its block rows of C = A·A; the root gathers every rank's
blocks and must hold exactly the oracle's product (integer-valued inputs:
exact in every dtype, pin P-12) and the single-rank product (bitwise: each C
block is computed on one rank in the same k order, pin P-10)."""
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


def _rand(rng, nbr, p, bs, dtype):
    m = rng.random((nbr, nbr)) < p
    br, bc = np.nonzero(m)
    v = rng.integers(-4, 5, size=(len(br), bs, bs)).astype(dtype)
    return qtgen.BlockMatrix(nbr * bs, max(bs, 32) * 2, bs, br.astype(np.int32), bc.astype(np.int32), v)


@pytest.mark.parametrize("bs,dtype,P,root", [(32, np.float64, 3, 0), (32, np.float32, 2, 1), (64, np.float64, 2, 0),
                                             (16, np.float64, 3, 2)])
def test_gather_equals_single_rank_product(qt, bs, dtype, P, root):
    import threading
    import torch
    rng = np.random.default_rng(40 + bs + P)
    nbr = 24 if bs != 16 else 36
    M = _rand(rng, nbr, 0.2, bs, dtype)
    ctx0 = qt.Context(0)
    A0 = qt.Matrix.from_blocks(ctx0, M.n, M.leaf_dim, bs, M.brow, M.bcol, M.vals)
    full = (A0 @ A0).to_blocks()
    t = (M.brow, M.bcol, M.vals.astype(np.float64))
    ref = oracle.spgemm(nbr, bs, t, t)
    assert np.array_equal(full[0], ref[0]) and np.array_equal(full[1], ref[1])
    assert np.array_equal(full[2].astype(np.float64), ref[2])
    step = (nbr // P) // 2 * 2
    bounds = [g * step for g in range(P)] + [nbr]
    hub = qt.LoopbackHub(P)
    out, errs = [None] * P, []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            c = qt.Context(0, stream=torch.cuda.Stream(), loopback=(hub, g, P))
            m = (M.brow >= bounds[g]) & (M.brow < bounds[g + 1])
            A = qt.Matrix.from_blocks(c, M.n, M.leaf_dim, bs, M.brow[m], M.bcol[m], M.vals[m], row_bounds=bounds)
            C = A @ A
            out[g] = C.gather(root)
            C.close()
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
    for g in range(P):
        if g != root:
            assert out[g] is None
    r, c, v = out[root]
    assert np.array_equal(r, ref[0]) and np.array_equal(c, ref[1])
    assert np.array_equal(v.astype(np.float64), ref[2])                  # the oracle's product
    assert np.array_equal(v, full[2])                                    # bitwise = single rank


@pytest.mark.parametrize("P,frac", [(2, 0.0), (2, 0.5), (3, 1.0)])
def test_screened_multi_rank_loopback(qt, P, frac):
    """The norm-screened product on P loopback ranks (B_ext's norms come from
    its local and received pools) equals the single-rank screened product."""
    import threading
    import torch
    rng = np.random.default_rng(60 + P)
    nbr = 30
    M = _rand(rng, nbr, 0.25, 32, np.float64)
    M.vals *= rng.integers(1, 9, size=(M.nb, 1, 1))
    nrm = np.sqrt((M.vals.astype(np.float64) ** 2).sum(axis=(1, 2)))
    tau = frac * float(np.median(nrm)) ** 2      # (frac 1: about half of the block products are screened)
    ctx0 = qt.Context(0)
    A0 = qt.Matrix.from_blocks(ctx0, M.n, M.leaf_dim, 32, M.brow, M.bcol, M.vals)
    ref, st_ref = A0.multiply_screened(A0, tau)
    full = A0.multiply(A0)[1]
    if frac > 0:
        assert st_ref.block_products < full.block_products
    ref = ref.to_blocks()
    t = (M.brow, M.bcol, M.vals)
    orc = oracle.spgemm(nbr, 32, t, t, tau=tau)                          # integer inputs: exact
    assert np.array_equal(ref[0], orc[0]) and np.array_equal(ref[1], orc[1]) and np.array_equal(ref[2], orc[2])
    bounds = [g * (nbr // P) for g in range(P)] + [nbr]
    hub = qt.LoopbackHub(P)
    out, errs = [None] * P, []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            c = qt.Context(0, stream=torch.cuda.Stream(), loopback=(hub, g, P))
            m = (M.brow >= bounds[g]) & (M.brow < bounds[g + 1])
            A = qt.Matrix.from_blocks(c, M.n, M.leaf_dim, 32, M.brow[m], M.bcol[m], M.vals[m], row_bounds=bounds)
            C, _ = A.multiply_screened(A, tau)
            out[g] = C.to_blocks()
            C.close()
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
    for g in range(P):
        r, c, v = out[g]
        m = (ref[0] >= bounds[g]) & (ref[0] < bounds[g + 1])
        assert np.array_equal(r, ref[0][m]) and np.array_equal(c, ref[1][m]) and np.array_equal(v, ref[2][m])
