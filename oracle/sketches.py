"""Sketch operators, restated on the CPU (test infrastructure only).

Reference kinds (restating `pkg/src/sketch_krylov/sketching.py`):
  * srht       -- signs/sample drawn from numpy's Philox exactly as
                  `SketchOperator.__post_init__` does (sketching.py:62-70);
                  applied as zero-pad -> sign -> unnormalised FWHT with the
                  ascending-h butterfly (a+b, a-b) (sketching.py:115-126)
                  -> gather -> * (1/sqrt(k)) (sketching.py:129-137).
  * rademacher -- k x n int8 signs from the same Philox stream
                  (sketching.py:71-73); applied by the fixed-order fp64
                  gemm, l ascending, then * (1/sqrt(k)) (sketching.py:151-155,
                  kernels.py:200-208).
  * identity   -- copy (sketching.py:146-147).

North-star kinds (absent from the reference; definitions are
ours and are documented in DESIGN.md section 3; the CUDA path implements the
same functions in `csrc/philox.cuh`):
  * gaussian    -- Theta[r, i] = q(r, i) / (2048 sqrt(k)), q an int16: the
                   Box-Muller normal of Philox4x32-10 quad
                   (counter = (i lo, i hi, r // 4, 'GAUS'), key = seed),
                   rounded to the 2^-11 grid.
  * sparse_sign -- column i holds s = min(nnz, k) entries +-1/sqrt(s) at
                   distinct rows drawn from the Philox word stream
                   (counter = (i lo, i hi, t, 'SPRS')), duplicates skipped.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse

from .philox import philox4x32_10

TAG_GAUSS = 0x47415553   # 'GAUS'
TAG_SPARSE = 0x53505253  # 'SPRS'
GAUSS_GRID = 2048.0      # int16 grid of the gaussian kind: 11 fractional bits
TWO_PI = 6.283185307179586


def next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p <<= 1
    return p


class OracleSketch:
    """Plain-data operator: (kind, k, n, seed) plus its realised tables."""

    def __init__(self, kind, k, n, seed, nnz=8, bits=16):
        self.kind, self.k, self.n, self.seed = kind, int(k), int(n), int(seed)
        self.nnz = int(nnz)
        self.bits = int(bits)  # gaussian kind: 16 (grid 2^-11) or 8 (grid 2^-5, |q| <= 127)
        if kind in ("srht", "rademacher"):
            gen = np.random.Generator(np.random.Philox(self.seed))
            if kind == "srht":
                self.n_pad = next_pow2(self.n)
                bits = gen.integers(0, 2, size=self.n_pad, dtype=np.int64)
                self.sign_diagonal = (bits * 2 - 1).astype(np.float64)
                self.sample_indices = gen.permutation(self.n_pad)[: self.k]
            else:
                self.signs = gen.integers(0, 2, size=(self.k, self.n),
                                          dtype=np.int8) * 2 - 1
        elif kind not in ("identity", "gaussian", "sparse_sign"):
            raise ValueError(kind)


# ---------------------------------------------------------------------------
# gaussian kind
# ---------------------------------------------------------------------------

def gaussian_int16(seed: int, k: int, rows: np.ndarray, bits: int = 16) -> np.ndarray:
    """int16 table q[r, t] for global W-rows `rows` (shape k x len(rows))."""
    rows = np.asarray(rows, dtype=np.uint64)
    nq = (k + 3) // 4
    quad = np.arange(nq, dtype=np.uint64)[:, None]
    lo = (rows & np.uint64(0xFFFFFFFF))[None, :]
    hi = (rows >> np.uint64(32))[None, :]
    a, b, c, d = philox4x32_10(lo, hi, quad, TAG_GAUSS, seed & 0xFFFFFFFF,
                               (seed >> 32) & 0xFFFFFFFF)
    scale = 2.0 ** -32

    def unif(w):
        return (w.astype(np.float64) + 0.5) * scale

    r1 = np.sqrt(-2.0 * np.log(unif(a)))
    t1 = TWO_PI * unif(b)
    r2 = np.sqrt(-2.0 * np.log(unif(c)))
    t2 = TWO_PI * unif(d)
    g = np.empty((4 * nq, rows.size), dtype=np.float64)
    g[0::4] = r1 * np.cos(t1)
    g[1::4] = r1 * np.sin(t1)
    g[2::4] = r2 * np.cos(t2)
    g[3::4] = r2 * np.sin(t2)
    if bits == 8:  # the same normals on the int8 grid 2^-5 (the one-plane tensor sketch)
        return np.clip(np.rint(GAUSS_GRID8 * g[:k]), -127, 127).astype(np.int16)
    q = np.clip(np.rint(GAUSS_GRID * g[:k]), -32767, 32767)
    return q.astype(np.int16)


GAUSS_GRID8 = 32.0


def gaussian_scale(k: int, bits: int = 16) -> float:
    return 1.0 / ((GAUSS_GRID8 if bits == 8 else GAUSS_GRID) * math.sqrt(k))


def gaussian_apply(seed, k, X, row0=0, chunk=8192, bits=16):
    """Theta[:, row0:row0+n] @ X in fp64, Theta regenerated chunk by chunk."""
    X = np.asarray(X, dtype=np.float64)
    out = np.zeros((k, X.shape[1]))
    for s in range(0, X.shape[0], chunk):
        e = min(X.shape[0], s + chunk)
        q = gaussian_int16(seed, k, np.arange(row0 + s, row0 + e), bits)
        out += q.astype(np.float64) @ X[s:e]
    return out * gaussian_scale(k, bits)


# ---------------------------------------------------------------------------
# sparse-sign kind
# ---------------------------------------------------------------------------

def sparse_sign_rows(seed: int, k: int, nnz: int, rows: np.ndarray):
    """(row index [s, len], sign [s, len]) of the nonzeros of Theta columns."""
    rows = np.asarray(rows, dtype=np.uint64)
    s = min(nnz, k)
    m = rows.size
    pick = np.full((s, m), -1, dtype=np.int64)
    sign = np.zeros((s, m), dtype=np.int8)
    have = np.zeros(m, dtype=np.int64)
    lo = rows & np.uint64(0xFFFFFFFF)
    hi = rows >> np.uint64(32)
    t = 0
    while np.any(have < s):
        words = philox4x32_10(lo, hi, np.uint64(t), TAG_SPARSE,
                              seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
        for w in words:
            w = w.astype(np.uint64)
            cand = ((w >> np.uint64(1)) * np.uint64(k)) >> np.uint64(31)
            cand = cand.astype(np.int64)
            sg = np.where((w & np.uint64(1)) == 0, 1, -1).astype(np.int8)
            dup = np.any(pick == cand[None, :], axis=0)
            take = (have < s) & ~dup
            idx = np.nonzero(take)[0]
            pick[have[idx], idx] = cand[idx]
            sign[have[idx], idx] = sg[idx]
            have[idx] += 1
        t += 1
    return pick, sign


def sparse_sign_matrix(seed, k, nnz, n, row0=0):
    pick, sign = sparse_sign_rows(seed, k, nnz, np.arange(row0, row0 + n))
    s = pick.shape[0]
    vals = sign.T.reshape(-1).astype(np.float64) / math.sqrt(s)
    indptr = np.arange(0, s * n + 1, s)
    return scipy.sparse.csc_matrix((vals, pick.T.reshape(-1), indptr), shape=(k, n))


# ---------------------------------------------------------------------------
# reference kinds
# ---------------------------------------------------------------------------

def fwht_ascending(Z: np.ndarray) -> np.ndarray:
    """In-place unnormalised Walsh-Hadamard along axis 0, stages h = 1, 2, 4,
    ... with (lo, hi) -> (lo + hi, lo - hi) (sketching.py:115-126)."""
    n = Z.shape[0]
    h = 1
    while h < n:
        V = Z.reshape(n // (2 * h), 2, h, *Z.shape[1:])
        lo = V[:, 0].copy()
        hi = V[:, 1].copy()
        V[:, 0] = lo + hi
        V[:, 1] = lo - hi
        h <<= 1
    return Z


def srht_apply(op: OracleSketch, X: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    Z = np.zeros((op.n_pad, X.shape[1]))
    Z[: X.shape[0]] = op.sign_diagonal[: X.shape[0], None] * X
    fwht_ascending(Z)
    return Z[op.sample_indices] * (1.0 / math.sqrt(op.k))


def rademacher_apply(op: OracleSketch, X: np.ndarray) -> np.ndarray:
    """Fixed-order fp64 accumulation over l ascending (kernels.py:200-208)."""
    X = np.asarray(X, dtype=np.float64)
    S = op.signs.astype(np.float64)
    acc = np.zeros((op.k, X.shape[1]))
    for l in range(X.shape[0]):
        acc += S[:, l:l + 1] * X[l:l + 1, :]
    return acc * (1.0 / math.sqrt(op.k))


def apply(op: OracleSketch, X) -> np.ndarray:
    """Theta @ X in fine precision (sketching.py:140-155), returned in the
    Fortran layout of the reference's `Matrix` wrapper."""
    return np.asfortranarray(_apply(op, X))


def materialize(op: OracleSketch) -> OracleSketch:
    """Cache the dense fp64 matrix of a gaussian operator (operator
    construction, as the reference does for its SRHT tables), so apply is
    one BLAS product.  For timing the CPU baseline on row samples."""
    if op.kind == "gaussian":
        op.dense = (gaussian_int16(op.seed, op.k, np.arange(op.n), op.bits).astype(np.float64)
                    * gaussian_scale(op.k, op.bits))
    return op


def _apply(op: OracleSketch, X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    if X.shape[0] != op.n:
        raise ValueError(f"sketch expects {op.n} rows, got {X.shape[0]}")
    if op.kind == "identity":
        return X.copy()
    if op.kind == "srht":
        return srht_apply(op, X)
    if op.kind == "rademacher":
        return rademacher_apply(op, X)
    if op.kind == "gaussian":
        if getattr(op, "dense", None) is not None:
            return op.dense @ X
        return gaussian_apply(op.seed, op.k, X, bits=op.bits)
    M = sparse_sign_matrix(op.seed, op.k, op.nnz, op.n)
    return np.asarray(M @ X)
