"""Multi-rank symmetric square (SURVEY f1 at P > 1; §3.3, the
paper's S^2 communication P:1179-1183; DESIGN reading C-26).  Needs a B200.

Rank g owns block rows [lo, hi) of the upper-triangular storage U and gets
its block rows of C = A^2, upper triangle.  Checked on the virtual-rank path
and on the loopback transport (the NCCL code path):
* C's rows are bitwise those of the single-rank symmetric square (itself
  pinned against the oracle in test_gpu_parity.py): every C block is computed
  on one rank from the same blocks in the same k order;
* the blocks received are exactly oracle.exchange_plan_symm's (pinned in
  test_oracle.py to the brute-force set of blocks the rank's products read):
  payload and metadata bytes;
* on the banded config the payload is ≈ 0.38x the full multiply's."""
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


def mk(qt, ctx, M):
    return qt.Matrix.from_blocks(ctx, M.n, M.leaf_dim, M.bs, M.brow, M.bcol, M.vals)


def f32(M):
    return qtgen.BlockMatrix(M.n, M.leaf_dim, M.bs, M.brow, M.bcol, M.vals.astype(np.float32))


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


def _case(name, P):
    if name == "cfg5":
        return qtgen.upper(qtgen.config(5, P=P, small=True, symmetric=True)["A"])
    if name == "cfg5int":
        return qtgen.upper(qtgen.config(5, "int", P=P, small=True, symmetric=True)["A"])
    if name == "cfg4":
        return qtgen.upper(qtgen.config(4, small=True, symmetric=True)["A"])
    return random_sym_upper(np.random.default_rng(31), 48, 0.12, "uniform", 256)


CASES = [("cfg5", 2, None), ("cfg5", 4, None), ("cfg5int", 4, None), ("cfg4", 3, None),
         ("random", 3, [0, 7, 30, 48]), ("random", 5, [0, 10, 11, 20, 35, 48])]


def _bounds(U, P, spec):
    return spec if spec is not None else [g * (U.nbr // P) for g in range(P)] + [U.nbr]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("name,P,spec", CASES)
def test_symm_virtual_bitwise_and_bytes(qt, ctx, name, P, spec, dtype):
    U = _case(name, P)
    if dtype == "f32":
        U = f32(U)
    bounds = _bounds(U, P, spec)
    A = mk(qt, ctx, U)
    full = A.symm_square()[0].to_blocks()
    plan = oracle.exchange_plan_symm(bounds, (U.brow, U.bcol), 8192 if dtype == "f64" else 4096)
    for g in range(P):
        Cg, st = A.symm_square_virtual(P, g, bounds)
        r, c, v = Cg.to_blocks()
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(c, full[1][m])
        assert np.array_equal(v, full[2][m])
        assert st.blocks_recv == plan[g]["blocks_received"]
        assert st.bytes_recv_payload == plan[g]["payload_bytes"]
        assert st.bytes_recv_meta == plan[g]["meta_bytes"]


def test_symm_virtual_banded_traffic_vs_full_multiply(qt, ctx):
    P = 4
    U = _case("cfg5", P)
    Af = qtgen.config(5, P=P, small=True, symmetric=True)["A"]
    bounds = _bounds(U, P, None)
    A, F = mk(qt, ctx, U), mk(qt, ctx, Af)
    for g in (1, 2):
        _, ss = A.symm_square_virtual(P, g, bounds)
        _, sf = F.multiply_virtual(F, P, g, bounds)
        assert 0.3 < ss.bytes_recv_payload / sf.bytes_recv_payload < 0.45
        assert ss.block_products < 0.6 * sf.block_products


def test_symm_virtual_single_rank_equals_symm_square(qt, ctx):
    U = _case("random", 1)
    A = mk(qt, ctx, U)
    ref = A.symm_square()[0].to_blocks()
    C, st = A.symm_square_virtual(1, 0, [0, U.nbr])
    got = C.to_blocks()
    assert all(np.array_equal(x, y) for x, y in zip(got, ref))
    assert st.bytes_recv_payload == 0 and st.blocks_recv == 0


def test_symm_virtual_errors(qt, ctx):
    rng = np.random.default_rng(3)
    nb = 4
    A64 = qt.Matrix.from_blocks(ctx, 256, 128, 64, np.array([0, 1], np.int32), np.array([0, 1], np.int32),
                                rng.uniform(-1, 1, size=(2, 64, 64)))
    with pytest.raises(qt.QtError) as e:
        A64.symm_square_virtual(2, 0, [0, 2, 4])
    assert e.value.name == "QT_EBS"
    L = qt.Matrix.from_blocks(ctx, nb * 32, 64, 32, np.array([1], np.int32), np.array([0], np.int32),
                              np.ones((1, 32, 32)))
    with pytest.raises(qt.QtError) as e:
        L.symm_square_virtual(2, 0, [0, 2, 4])
    assert e.value.name == "QT_EINVAL"


@pytest.mark.parametrize("dtype,P,name", [("f64", 2, "cfg5"), ("f64", 4, "cfg5"), ("f64", 3, "random"),
                                          ("f32", 2, "cfg5")])
def test_symm_loopback_nccl_path(qt, ctx, dtype, P, name):
    import threading
    import torch
    U = _case(name, P)
    if dtype == "f32":
        U = f32(U)
    bounds = _bounds(U, P, [0, 7, 30, 48] if name == "random" else None)
    full = mk(qt, ctx, U).symm_square()[0].to_blocks()
    bb = 8192 if dtype == "f64" else 4096
    plan = oracle.exchange_plan_symm(bounds, (U.brow, U.bcol), bb)
    hub = qt.LoopbackHub(P)
    out, errs = [None] * P, []

    def rank_fn(g):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            c = qt.Context(0, stream=s, loopback=(hub, g, P))
            m = (U.brow >= bounds[g]) & (U.brow < bounds[g + 1])
            A = qt.Matrix.from_blocks(c, U.n, U.leaf_dim, 32, U.brow[m], U.bcol[m], U.vals[m],
                                      row_bounds=bounds)
            C, st = A.symm_square()
            out[g] = (C.to_blocks(), st.as_dict(), C.info())
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
        (r, c, v), st, info = out[g]
        m = (full[0] >= bounds[g]) & (full[0] < bounds[g + 1])
        assert np.array_equal(r, full[0][m]) and np.array_equal(c, full[1][m])
        assert np.array_equal(v, full[2][m])
        assert st["bytes_recv_payload"] == plan[g]["payload_bytes"]
        assert st["bytes_recv_meta"] == plan[g]["meta_bytes"]
        assert (info["row_lo"], info["row_hi"]) == (bounds[g], bounds[g + 1])
    assert sum(o[1]["bytes_sent_payload"] for o in out) == sum(p["payload_bytes"] for p in plan)
