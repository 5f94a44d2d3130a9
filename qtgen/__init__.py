"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is shared by the oracle side (``oracle/``, ``tests/``) and the
product side (``bench.py`` and the GPU tests).  It holds NONE of the method's
arithmetic: no multiply, no pattern product, no quadtree logic.  It only
produces block lists ``(brow, bcol, values)`` of the input matrices.

Recipe:

* Every random number is counter based: ``h(seed, i, j) = mix64((seed << 40) |
  (i << 20) | j)`` with ``mix64`` the SplitMix64 finaliser.  A value therefore
  depends only on (seed, global row, global column), never on the partition,
  the device or the leaf size, so any rank can generate any block.
* ``uniform[-1,1]``: ``u = 2 * ((h >> 11) * 2**-53) - 1`` (C-11).
* ``integers in [-4,4]``: ``v = (h mod 9) - 4`` (C-10).
* Block presence with probability p: ``h(seed_pat, I, J) < p * 2**64`` (C-14).
* Banded (C-12): half-bandwidth d, element ``a_ij`` nonzero iff ``|i-j| <= d``;
  block (I, J) is stored iff it intersects the band.  Entries of a stored
  block outside the band are exact zeros.
* ES-like (C-15): 3072 atoms on a 16x16x12 lattice, spacing 3 bohr, jitter
  uniform +-1.5 bohr, recursive divide-space ordering (median bisection of the
  longest bounding-box axis), one 32x32 block per atom pair, block kept iff
  r_IJ < 7.0 bohr, ``a_ij = u_ij * exp(-0.5 r_IJ)``.

Seeds (C-11): A values 1, B values 2, A pattern 11, B pattern 12, geometry 3.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_A_VAL = 1
SEED_B_VAL = 2
SEED_A_PAT = 11
SEED_B_PAT = 12
SEED_GEOM = 3

_U64 = np.uint64


def mix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + _U64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
    return z ^ (z >> _U64(31))


def hash3(seed: int, i, j) -> np.ndarray:
    """Counter hash of (seed, i, j); i, j < 2**20, seed < 2**24."""
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    return mix64((_U64(seed) << _U64(40)) | (i << _U64(20)) | j)


def uniform_pm1(h: np.ndarray) -> np.ndarray:
    return ((h >> _U64(11)).astype(np.float64) * 2.0 ** -53) * 2.0 - 1.0


def int_pm4(h: np.ndarray) -> np.ndarray:
    return (h % _U64(9)).astype(np.int64).astype(np.float64) - 4.0


@dataclasses.dataclass
class BlockMatrix:
    """A matrix given as a list of dense bs x bs blocks (row-major per block).

    ``brow``/``bcol`` are block coordinates, ``vals`` has shape [nb, bs, bs].
    Blocks are listed in row-major block order (brow, then bcol).
    """

    n: int
    leaf_dim: int
    bs: int
    brow: np.ndarray
    bcol: np.ndarray
    vals: np.ndarray

    @property
    def nb(self) -> int:
        return int(self.brow.shape[0])

    @property
    def nbr(self) -> int:
        return -(-self.n // self.bs)

    def dense(self) -> np.ndarray:
        """Dense n x n copy (tiny matrices only)."""
        out = np.zeros((self.nbr * self.bs, self.nbr * self.bs), dtype=self.vals.dtype)
        for t in range(self.nb):
            r, c = int(self.brow[t]) * self.bs, int(self.bcol[t]) * self.bs
            out[r:r + self.bs, c:c + self.bs] = self.vals[t]
        return out[: self.n, : self.n]


# ----------------------------------------------------------------------------
# block patterns (row-major sorted int32 arrays)


def _sorted_pattern(brow, bcol):
    brow = np.asarray(brow, dtype=np.int64)
    bcol = np.asarray(bcol, dtype=np.int64)
    o = np.lexsort((bcol, brow))
    return brow[o].astype(np.int32), bcol[o].astype(np.int32)


def pattern_dense(nbr: int, rows=None):
    lo, hi = rows if rows is not None else (0, nbr)
    I, J = np.meshgrid(np.arange(lo, hi), np.arange(nbr), indexing="ij")
    return _sorted_pattern(I.ravel(), J.ravel())


def band_blocks(d: int, bs: int) -> int:
    """Block half-bandwidth D: block (I,J) meets the element band iff |I-J| <= D."""
    return (d + bs - 1) // bs


def pattern_banded(nbr: int, D: int, rows=None):
    lo, hi = rows if rows is not None else (0, nbr)
    I = np.repeat(np.arange(lo, hi), 2 * D + 1)
    J = I + np.tile(np.arange(-D, D + 1), hi - lo)
    keep = (J >= 0) & (J < nbr)
    return _sorted_pattern(I[keep], J[keep])


def pattern_random(nbr: int, p: float, seed_pat: int, rows=None):
    lo, hi = rows if rows is not None else (0, nbr)
    thresh = _U64(min(int(p * 2.0 ** 64), 2 ** 64 - 1))
    brs, bcs = [], []
    J = np.arange(nbr)
    for I in range(lo, hi):
        h = hash3(seed_pat, np.full(nbr, I), J)
        sel = np.nonzero(h < thresh)[0]
        brs.append(np.full(sel.shape, I))
        bcs.append(sel)
    if not brs:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    return _sorted_pattern(np.concatenate(brs), np.concatenate(bcs))


# ----------------------------------------------------------------------------
# block values


def block_values(brow, bcol, bs: int, seed: int, kind: str = "uniform",
                 band_d: int | None = None, scale=None, chunk: int = 4096,
                 symmetric: bool = False) -> np.ndarray:
    """Values of the listed blocks: element (i, j) = F(h(seed, i, j)).

    ``kind``: "uniform" (uniform[-1,1]), "int" (integers -4..4), "ones".
    ``band_d``: zero the entries with |i-j| > band_d (banded configs).
    ``scale``: optional per-block multiplier (ES-like config).
    ``symmetric``: hash the unordered pair (min(i,j), max(i,j)), so that the
    matrix is symmetric (inputs of the symmetric square).
    """
    nb = len(brow)
    out = np.empty((nb, bs, bs), dtype=np.float64)
    ii = np.arange(bs, dtype=np.int64)
    for s in range(0, nb, chunk):
        e = min(nb, s + chunk)
        R = (np.asarray(brow[s:e], np.int64) * bs)[:, None, None] + ii[None, :, None]
        C = (np.asarray(bcol[s:e], np.int64) * bs)[:, None, None] + ii[None, None, :]
        if kind == "ones":
            v = np.ones((e - s, bs, bs))
        else:
            h = hash3(seed, np.minimum(R, C), np.maximum(R, C)) if symmetric else hash3(seed, R, C)
            v = uniform_pm1(h) if kind == "uniform" else int_pm4(h)
        if band_d is not None:
            v = np.where(np.abs(R - C) <= band_d, v, 0.0)
        if scale is not None:
            v = v * np.asarray(scale[s:e], dtype=np.float64)[:, None, None]
        out[s:e] = v
    return out


# ----------------------------------------------------------------------------
# ES-like geometry (config 4)


def _divide_space_order(pos: np.ndarray) -> np.ndarray:
    """Recursive divide-space ordering: bisect at the median of the longest
    bounding-box axis (paper names Ergo's default)."""
    order = []
    stack = [np.arange(pos.shape[0])]
    while stack:
        idx = stack.pop()
        if idx.shape[0] <= 1:
            order.extend(idx.tolist())
            continue
        p = pos[idx]
        ext = p.max(axis=0) - p.min(axis=0)
        ax = int(np.argmax(ext))
        o = np.lexsort((idx, p[:, ax]))
        idx = idx[o]
        half = idx.shape[0] // 2
        stack.append(idx[half:])   # processed after the left half
        stack.append(idx[:half])
    return np.asarray(order, dtype=np.int64)


def es_geometry(shape=(16, 16, 12), spacing=3.0, jitter=1.5, seed=SEED_GEOM):
    nx, ny, nz = shape
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    g = g.reshape(-1, 3).astype(np.float64) * spacing
    na = g.shape[0]
    h = hash3(seed, np.arange(na)[:, None], np.arange(3)[None, :])
    pos = g + jitter * uniform_pm1(h)
    return pos[_divide_space_order(pos)]


def pattern_es(pos: np.ndarray, rc: float, rows=None):
    na = pos.shape[0]
    lo, hi = rows if rows is not None else (0, na)
    d = np.sqrt(((pos[lo:hi, None, :] - pos[None, :, :]) ** 2).sum(-1))
    I, J = np.nonzero(d < rc)
    I = I + lo
    br, bc = _sorted_pattern(I, J)
    r = np.sqrt(((pos[br] - pos[bc]) ** 2).sum(-1))
    return br, bc, r


# ----------------------------------------------------------------------------
# the BASELINE configs


def upper(M: "BlockMatrix") -> "BlockMatrix":
    """The upper block triangle (brow <= bcol) of a block list."""
    k = M.brow <= M.bcol
    return BlockMatrix(M.n, M.leaf_dim, M.bs, M.brow[k], M.bcol[k], M.vals[k])


def config(idx: int, kind: str = "uniform", P: int = 1, rank: int | None = None,
           rows=None, small: bool = False, symmetric: bool = False) -> dict:
    """Inputs of BASELINE.json configs[idx-1] (idx in 1..5).

    Returns ``{"name", "A", "B", "same"}``; ``B is A`` when the config computes
    C = A*A.  ``rank`` (with ``P``) restricts the generated blocks to the block
    rows the rank owns under equal row strips (configs 5 and 2); ``rows`` gives
    an explicit block-row range instead.  ``small`` gives a reduced-size
    variant of the same recipe for fast tests.
    """
    bs = 32
    if idx == 1:
        n, leaf = 512, 128
        nbr = n // bs
        rng = rows
        ar, ac = pattern_dense(nbr, rng)
        br, bc = pattern_dense(nbr, rng)
        A = BlockMatrix(n, leaf, bs, ar, ac, block_values(ar, ac, bs, SEED_A_VAL, kind))
        B = BlockMatrix(n, leaf, bs, br, bc, block_values(br, bc, bs, SEED_B_VAL, kind))
        return {"name": "cfg1-dense-N512", "A": A, "B": B, "same": False}
    if idx in (2, 5):
        d = 1024
        if idx == 2:
            n, leaf = (2048 if small else 16384), 1024
            if small:
                d = 128
        else:
            n, leaf = (2048 if small else 16384) * P, 2048
            if small:
                d, leaf = 128, 256
        nbr = n // bs
        D = band_blocks(d, bs)
        if rank is not None and rows is None:
            per = nbr // P
            rows = (rank * per, (rank + 1) * per)
        ar, ac = pattern_banded(nbr, D, rows)
        A = BlockMatrix(n, leaf, bs, ar, ac,
                        block_values(ar, ac, bs, SEED_A_VAL, kind, band_d=d, symmetric=symmetric))
        name = f"cfg{idx}-banded-N{n}-d{d}"
        return {"name": name, "A": A, "B": A, "same": True, "d": d}
    if idx == 3:
        n, leaf, p = (8192, 2048, 0.04) if small else (32768, 2048, 0.01)
        nbr = n // bs
        ar, ac = pattern_random(nbr, p, SEED_A_PAT, rows)
        br, bc = pattern_random(nbr, p, SEED_B_PAT, rows)
        A = BlockMatrix(n, leaf, bs, ar, ac, block_values(ar, ac, bs, SEED_A_VAL, kind))
        B = BlockMatrix(n, leaf, bs, br, bc, block_values(br, bc, bs, SEED_B_VAL, kind))
        return {"name": f"cfg3-random-N{n}-p{p}", "A": A, "B": B, "same": False}
    if idx == 4:
        shape = (8, 8, 6) if small else (16, 16, 12)
        pos = es_geometry(shape)
        na = pos.shape[0]
        n, leaf = na * bs, 4096
        if small:
            leaf = 1024
        ar, ac, r = pattern_es(pos, 7.0, rows)
        scale = np.exp(-0.5 * r) if kind == "uniform" else None
        A = BlockMatrix(n, leaf, bs, ar, ac,
                        block_values(ar, ac, bs, SEED_A_VAL, kind, scale=scale, symmetric=symmetric))
        return {"name": f"cfg4-eslike-N{n}", "A": A, "B": A, "same": True}
    raise ValueError(f"unknown config {idx}")

