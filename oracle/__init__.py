"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU reference for the hot path of arXiv
1501.07800 (Rubensson & Rudberg): C = A*B for block-sparse matrices held as
sparse quadtrees.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1501_07800_b200/`` (neither imports
the other); the seeded inputs come from ``qtgen`` which holds none of the
method's arithmetic.

Functions and the passages they follow (P:nnn = /root/reference/PAPER.md line,
S:nnn = SPEC.md line; readings C-n are listed in DESIGN.md):

* ``spgemm``      C = A*B, block-CSR Gustavson in double, ascending k
                  (§3.2 NIL skipping; P:381-388 sum of outer
                  products; C-1 structural pattern, C-5 order).  C source in
                  ``qt_oracle.c``.
* ``dense_mm``    textbook triple loop (pin P-2).
* ``transpose`` / ``spgemm_t``  the transposed task types C = A^T B, A B^T,
                  A^T B^T by explicit block transposition.
* ``spgemm(..., tau=)`` the norm-screened product C~ (products with
                  ||A_IK|| ||B_KJ|| < tau skipped),
                  ``block_norm2`` the squared block norms it tests.
* ``symm_square`` upper block triangle of A^2 for symmetric A in upper
                  triangular storage (§3.3), by explicit expansion;
                  ``level_task_counts_sym`` its per-level tasks.
* ``pattern_product``   boolean product of block patterns (pin P-6).
* ``level_task_counts`` multiply tasks per quadtree level: the number of
                  (A-node, B-node) pairs with both non-NIL at level l
                  (§5.1; C-19).  Levels run from the root (l=0) to the
                  block level, "merging the lowest levels".
* ``tree_levels`` quadtree geometry: 2^L blocks per side, 2^L >= block rows (C-3).
* ``exchange_plan``     bytes each rank receives under block-row strips
                  (A-stationary) — the paper's "data received by each process"
                  (P:1153-1155); protocol in DESIGN.md §Multi-GPU.
* ``spsumma_volume``    2mN/sqrt(p) elements (Eq. eq:sqrtp_equation P:726-728).
* ``truncate``    drop the longest prefix of blocks, sorted ascending by
                  Frobenius norm (ties by (brow, bcol)), whose cumulative
                  squared norm stays < tau^2 (C-16).
* ``higham_bound`` 2*gamma_K*(|A||B|) elementwise (pin P-9).

Parity status: every function above is pinned by tests/test_oracle.py; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile qt_oracle.c with gcc (plain -O2, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        lib.oracle_symbolic.restype = i64
        D = ctypes.c_double
        lib.oracle_symbolic.argtypes = [i32, P, P, i32, P, P, i32, P, P, P, D]
        lib.oracle_numeric.restype = None
        lib.oracle_numeric.argtypes = [i32, i32, P, P, P, P, P, P, i32, P, P, P, i32, i32, i32, P, P, D]
        lib.oracle_block_norm2.restype = None
        lib.oracle_block_norm2.argtypes = [i64, i32, P, P]
        lib.oracle_dense.restype = None
        lib.oracle_dense.argtypes = [i32, P, P, P]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


# ----------------------------------------------------------------------------
# block-CSR


def to_bcsr(nbr: int, brow, bcol, vals):
    """Sort blocks by (brow, bcol) and build block-CSR (row_ptr int64, col int32)."""
    brow = np.asarray(brow, np.int64)
    bcol = np.asarray(bcol, np.int64)
    o = np.lexsort((bcol, brow))
    ptr = np.zeros(nbr + 1, np.int64)
    np.add.at(ptr, brow[o] + 1, 1)
    ptr = np.cumsum(ptr)
    col = np.ascontiguousarray(bcol[o], dtype=np.int32)
    val = np.ascontiguousarray(np.asarray(vals, dtype=np.float64)[o])
    return ptr, col, val


def block_norm2(vals) -> np.ndarray:
    """Squared Frobenius norm of each block (row-major, plain C loop)."""
    vals = np.ascontiguousarray(np.asarray(vals, np.float64))
    out = np.zeros(vals.shape[0], np.float64)
    if vals.shape[0]:
        _load().oracle_block_norm2(vals.shape[0], vals.shape[1], _p(vals), _p(out))
    return out


def spgemm(nbr: int, bs: int, A, B, nthreads: int | None = None, rows=None, tau: float | None = None):
    """C = A*B.  ``A``/``B`` are (brow, bcol, vals[nb,bs,bs]) tuples over an
    nbr x nbr block grid.  Returns (brow, bcol, vals) of C sorted by
    (brow, bcol); ``rows=(lo,hi)`` restricts the work to those block rows.
    ``tau``: the norm-screened product — only block products with
    ||A_IK||_F ||B_KJ||_F >= tau (squared norms: na2*nb2 >= tau^2) are taken."""
    lib = _load()
    a_ptr, a_col, a_val = to_bcsr(nbr, *A)
    b_ptr, b_col, b_val = to_bcsr(nbr, *B)
    na2 = nb2 = None
    tau2 = 0.0
    if tau is not None:
        na2, nb2, tau2 = block_norm2(a_val), block_norm2(b_val), float(tau) * float(tau)
    c_cnt = np.zeros(nbr, np.int64)
    lib.oracle_symbolic(nbr, _p(a_ptr), _p(a_col), nbr, _p(b_ptr), _p(b_col), nbr, _p(c_cnt),
                        _p(na2) if na2 is not None else None, _p(nb2) if nb2 is not None else None, tau2)
    lo, hi = rows if rows is not None else (0, nbr)
    if rows is not None:
        c_cnt[:lo] = 0
        c_cnt[hi:] = 0
    c_ptr = np.zeros(nbr + 1, np.int64)
    c_ptr[1:] = np.cumsum(c_cnt)
    nc = int(c_ptr[-1])
    c_col = np.zeros(max(nc, 1), np.int32)
    c_val = np.zeros((max(nc, 1), bs, bs), np.float64)
    nt = default_threads() if nthreads is None else nthreads
    lib.oracle_numeric(nbr, bs, _p(a_ptr), _p(a_col), _p(a_val), _p(b_ptr), _p(b_col), _p(b_val),
                       nbr, _p(c_ptr), _p(c_col), _p(c_val), lo, hi, nt,
                       _p(na2) if na2 is not None else None, _p(nb2) if nb2 is not None else None, tau2)
    c_row = np.repeat(np.arange(nbr, dtype=np.int32), c_cnt)
    return c_row, c_col[:nc], c_val[:nc]


def transpose(brow, bcol, vals):
    """X^T as a block list: block (I,J) becomes block (J,I) with its values
    transposed (the operand of the transposed task types C = A^T B, A B^T,
    A^T B^T)."""
    return (np.asarray(bcol, np.int32), np.asarray(brow, np.int32),
            np.ascontiguousarray(np.swapaxes(np.asarray(vals), 1, 2)))


def spgemm_t(nbr: int, bs: int, A, B, trans_a=False, trans_b=False, nthreads=None, rows=None):
    """C = op(A) op(B) (op = transpose when flagged), by explicit transposition."""
    a = transpose(*A) if trans_a else A
    b = transpose(*B) if trans_b else B
    return spgemm(nbr, bs, a, b, nthreads, rows)


def expand_symmetric(brow, bcol, vals):
    """The full symmetric matrix from its upper block triangle (brow <= bcol):
    every off-diagonal block (I,J) also stands for (J,I) = block^T; diagonal
    blocks are used as stored (§3.3, upper triangular storage)."""
    brow = np.asarray(brow, np.int32)
    bcol = np.asarray(bcol, np.int32)
    vals = np.asarray(vals)
    off = brow != bcol
    tr = transpose(brow[off], bcol[off], vals[off])
    return (np.concatenate([brow, tr[0]]), np.concatenate([bcol, tr[1]]),
            np.concatenate([vals, tr[2]]))


def symm_square(nbr: int, bs: int, U, nthreads=None, rows=None):
    """C = A^2 for the symmetric A given by its upper block triangle U; returns
    the upper block triangle of C (the operation of §3.3)."""
    full = expand_symmetric(*U)
    r, c, v = spgemm(nbr, bs, full, full, nthreads, rows)
    keep = r <= c
    return r[keep], c[keep], v[keep]


def level_task_counts_sym(L: int, u_rc):
    """Multiply tasks per level of the symmetric square: (I,K,J) at level l
    with A_l(I,K), A_l(K,J) non-NIL and I <= J (only C's upper triangle is
    computed), A the full symmetric pattern."""
    import scipy.sparse as sp
    r = np.asarray(u_rc[0], np.int64)
    c = np.asarray(u_rc[1], np.int64)
    fr, fc = np.concatenate([r, c]), np.concatenate([c, r])
    out = []
    for l in range(L + 1):
        s = L - l
        m = 1 << l
        ar, ac = _coarsen((fr, fc), s)
        M = sp.csr_matrix((np.ones(len(ar), np.int64), (ar, ac)), shape=(m, m))
        P = sp.triu(M @ M)
        out.append(int(P.sum()))
    return out


def dense_mm(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    lib = _load()
    n = A.shape[0]
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    C = np.zeros((n, n), np.float64)
    lib.oracle_dense(n, _p(A), _p(B), _p(C))
    return C


# ----------------------------------------------------------------------------
# patterns and quadtree levels


def pattern_product(nbr: int, a_rc, b_rc):
    """Boolean product of block patterns: sorted (brow, bcol) of S_C, via a
    library sparse product (scipy.sparse) of 0/1 matrices."""
    import scipy.sparse as sp
    one = lambda rc: sp.csr_matrix((np.ones(len(rc[0]), np.int64),
                                    (np.asarray(rc[0]), np.asarray(rc[1]))), shape=(nbr, nbr))
    C = (one(a_rc) @ one(b_rc)).tocoo()
    keep = C.data > 0
    r, c = C.row[keep].astype(np.int64), C.col[keep].astype(np.int64)
    o = np.lexsort((c, r))
    return r[o].astype(np.int32), c[o].astype(np.int32)


def tree_levels(n: int, bs: int, leaf_dim: int):
    """(L, leaf_level): the quadtree covers 2^L x 2^L blocks with 2^L the
    smallest power of two >= ceil(n/bs) — the matrix is split "as far as
    possible" into a uniform block size per level (reading C-3:
    pad to a power of two, padded children are NIL).  Level 0 is the root,
    level L the blocks, leaf level = L - log2(leaf/bs) clipped at 0.  A matrix
    of a single block has L = 0 (the root is the block)."""
    nbr = -(-n // bs)
    L = 0
    while (1 << L) < nbr:
        L += 1
    per_leaf = leaf_dim // bs
    lg = per_leaf.bit_length() - 1
    return L, max(0, L - lg)


def _coarsen(rc, s):
    r = np.asarray(rc[0], np.int64) >> s
    c = np.asarray(rc[1], np.int64) >> s
    key = np.unique(r * (1 << 31) + c)
    return key >> 31, key & ((1 << 31) - 1)


def level_task_counts(L: int, a_rc, b_rc):
    """C_l for l = 0..L: number of (I,K,J) at level l with A_l(I,K) and
    B_l(K,J) both nonzero, where X_l is the pattern coarsened to 2^l x 2^l
    nodes.  Computed as sum_K colcount(A_l)[K] * rowcount(B_l)[K]."""
    out = []
    for l in range(L + 1):
        s = L - l
        ar, ac = _coarsen(a_rc, s)
        br, bc = _coarsen(b_rc, s)
        m = 1 << l
        ca = np.bincount(ac, minlength=m).astype(np.int64)
        rb = np.bincount(br, minlength=m).astype(np.int64)
        out.append(int((ca * rb).sum()))
    return out


def level_node_counts(L: int, rc):
    """Number of non-NIL quadtree nodes per level l = 0..L."""
    return [int(_coarsen(rc, L - l)[0].shape[0]) for l in range(L + 1)]


# ----------------------------------------------------------------------------
# multi-GPU exchange plan (row strips, A-stationary)


def exchange_plan(bounds, a_rc, b_rc, block_bytes: int):
    """Per-rank received bytes when rank g owns block rows [bounds[g],
    bounds[g+1]) of A, B and C and fetches, from their owners, every B block
    row K it needs (K in cols(A[rows_g, :]) and K not owned by g).

    Returns a list of dicts: rows_requested, blocks_received, payload bytes
    (= blocks * block_bytes) and meta bytes received (protocol of DESIGN.md:
    one int32 block count per requested row and one int32 column per block)."""
    bounds = np.asarray(bounds, np.int64)
    P = len(bounds) - 1
    ar = np.asarray(a_rc[0], np.int64)
    ac = np.asarray(a_rc[1], np.int64)
    br = np.asarray(b_rc[0], np.int64)
    nbr_rows = int(bounds[-1])
    b_row_cnt = np.bincount(br, minlength=nbr_rows).astype(np.int64)
    out = []
    for g in range(P):
        lo, hi = bounds[g], bounds[g + 1]
        need = np.unique(ac[(ar >= lo) & (ar < hi)])
        need = need[(need < lo) | (need >= hi)]
        nblk = int(b_row_cnt[need].sum()) if need.size else 0
        per_src = np.zeros(P, np.int64)
        for q in range(P):
            sel = need[(need >= bounds[q]) & (need < bounds[q + 1])]
            per_src[q] = int(b_row_cnt[sel].sum()) if sel.size else 0
        out.append({
            "rows_requested": int(need.size),
            "blocks_received": nblk,
            "payload_bytes": nblk * block_bytes,
            "meta_bytes": 4 * int(need.size) + 4 * nblk,
            "blocks_from": per_src.tolist(),
        })
    return out


def exchange_plan_leaf_granular(bounds, a_rc, b_rc, block_bytes: int, leaf_blocks: int):
    """The paper's fetch granularity as a counterfactual: a
    rank fetches whole leaf matrices ("chunks") — every B leaf
    (leaf row, leaf column) holding a block it needs — instead of exactly the
    needed blocks.  Returns the bytes received per rank."""
    bounds = np.asarray(bounds, np.int64)
    P = len(bounds) - 1
    ar = np.asarray(a_rc[0], np.int64)
    ac = np.asarray(a_rc[1], np.int64)
    br = np.asarray(b_rc[0], np.int64)
    bc = np.asarray(b_rc[1], np.int64)
    out = []
    for g in range(P):
        lo, hi = bounds[g], bounds[g + 1]
        need_rows = np.unique(ac[(ar >= lo) & (ar < hi)])
        need_rows = need_rows[(need_rows < lo) | (need_rows >= hi)]
        needed = np.isin(br, need_rows)
        leaves = set(zip((br[needed] // leaf_blocks).tolist(), (bc[needed] // leaf_blocks).tolist()))
        remote = (br < lo) | (br >= hi)
        in_leaf = np.array([(r // leaf_blocks, c // leaf_blocks) in leaves for r, c in zip(br.tolist(), bc.tolist())],
                           bool) if len(br) else np.zeros(0, bool)
        out.append(int((in_leaf & remote).sum()) * block_bytes)
    return out


def exchange_plan_symm(bounds, u_rc, block_bytes: int):
    """Per-rank received bytes of the multi-rank symmetric square (DESIGN.md
    reading C-26; §3.3 P:297-311 for the operation, P:1179-1183 for the
    paper's measured communication of S^2).  Rank g owns rows [lo, hi) of the
    upper-triangular storage U and computes C rows [lo, hi), upper triangle.
    With R_g = the block columns >= hi of g's blocks, g receives every block
    (r, c) of U outside its strip with
        r >= hi and (r in R_g or c in R_g), or
        r <  lo, c >= lo and row r of U has a block in columns [lo, hi).
    This is exactly the set of other ranks' blocks read by some product
    A(I,K)·A(K,J), I in [lo, hi), J >= I (A(I,K) = U(I,K) or U(K,I)^T).
    Metadata received: one int64 key per block, one int32 count per peer, and
    the int32 lists R_q of the lower ranks q < g (sent to every higher rank)."""
    bounds = np.asarray(bounds, np.int64)
    P = len(bounds) - 1
    nbr = int(bounds[-1])
    ur = np.asarray(u_rc[0], np.int64)
    uc = np.asarray(u_rc[1], np.int64)
    R = []
    for g in range(P):
        lo, hi = bounds[g], bounds[g + 1]
        r = np.unique(uc[(ur >= lo) & (ur < hi)])
        R.append(r[r >= hi])
    out = []
    for g in range(P):
        lo, hi = bounds[g], bounds[g + 1]
        strip = (ur >= lo) & (ur < hi)
        in_r = np.zeros(nbr, bool)
        in_r[R[g]] = True
        hit = np.zeros(nbr, bool)
        hit[ur[(uc >= lo) & (uc < hi)]] = True
        sel = ~strip & (((ur >= hi) & (in_r[ur] | in_r[uc])) | ((ur < lo) & (uc >= lo) & hit[ur]))
        n = int(sel.sum())
        lists_in = int(sum(len(R[q]) for q in range(g)))
        out.append({
            "blocks_received": n,
            "payload_bytes": n * block_bytes,
            "meta_bytes": 8 * n + 4 * (P - 1) + 4 * lists_in,
            "selected": np.nonzero(sel)[0],
        })
    return out


def row_products(nbr: int, a_rc, b_rc):
    """Block products of each row of C = A·B (the work of a
    row strip), by enumeration: for every A block (I, K), the blocks of B's row K."""
    ar = np.asarray(a_rc[0], np.int64)
    ac = np.asarray(a_rc[1], np.int64)
    nnz_b = np.bincount(np.asarray(b_rc[0], np.int64), minlength=nbr)
    out = np.zeros(nbr, np.int64)
    for i, k in zip(ar.tolist(), ac.tolist()):
        out[i] += nnz_b[k]
    return out


def strips_min_max(weights, parts: int, align: int):
    """Smallest possible largest strip load over all partitions of the rows
    into `parts` contiguous strips with boundaries at multiples of `align`
    (brute-force dynamic program over the aligned chunks)."""
    w = np.asarray(weights, np.int64)
    nch = -(-len(w) // align)
    cw = [int(w[c * align:(c + 1) * align].sum()) for c in range(nch)]
    pre = [0]
    for x in cw:
        pre.append(pre[-1] + x)
    INF = float("inf")
    best = [[INF] * (nch + 1) for _ in range(parts + 1)]
    best[0][0] = 0
    for g in range(1, parts + 1):
        for j in range(nch + 1):
            for i in range(j + 1):
                v = max(best[g - 1][i], pre[j] - pre[i])
                if v < best[g][j]:
                    best[g][j] = v
    return int(min(best[g][nch] for g in range(1, parts + 1)))


def spsumma_volume(m: float, N: float, p: float) -> float:
    """Elements each process fetches under random permutation + Sparse SUMMA:
    2 m N / sqrt(p) (Eq. eq:sqrtp_equation)."""
    return 2.0 * m * N / math.sqrt(p)


# ----------------------------------------------------------------------------
# truncation and error bounds


def truncate(brow, bcol, vals, tau: float):
    """Remove the longest prefix of blocks (ascending Frobenius norm, ties by
    (brow, bcol)) whose accumulated squared norm is < tau^2.
    Returns the kept (brow, bcol, vals) sorted by (brow, bcol)."""
    brow = np.asarray(brow, np.int64)
    bcol = np.asarray(bcol, np.int64)
    vals = np.asarray(vals, np.float64)
    nb = brow.shape[0]
    nrm2 = np.array([float(np.sum(vals[t] * vals[t])) for t in range(nb)])
    order = np.lexsort((bcol, brow, nrm2))
    drop = np.zeros(nb, np.bool_)
    acc = 0.0
    t2 = tau * tau
    for t in order:
        if acc + nrm2[t] < t2:
            acc += nrm2[t]
            drop[t] = True
        else:
            break
    keep = ~drop
    o = np.lexsort((bcol[keep], brow[keep]))
    return (brow[keep][o].astype(np.int32), bcol[keep][o].astype(np.int32), vals[keep][o])


def gamma(k: int, u: float) -> float:
    return k * u / (1.0 - k * u)


def higham_bound(nbr: int, bs: int, A, B, k_terms: int, u: float = 2.0 ** -53, nthreads=None,
                 rows=None):
    """Elementwise bound 2*gamma_K*(|A||B|) on |C_computed - C_exact| valid for
    any summation order, with or without FMA (Higham, Accuracy and Stability,
    §3.5).  Returns (brow, bcol, bound_vals) aligned with spgemm's output."""
    r, c, v = spgemm(nbr, bs, (A[0], A[1], np.abs(A[2])), (B[0], B[1], np.abs(B[2])), nthreads,
                     rows=rows)
    return r, c, 2.0 * gamma(k_terms, u) * v
