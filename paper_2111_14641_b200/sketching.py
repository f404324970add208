"""Oblivious sketching operators (reference `pkg/src/sketch_krylov/sketching.py`).

`SketchOperator(kind, k, n, seed)` accepts exactly the reference kinds
(`KINDS`, sketching.py:33) and draws its tables with the reference's own
recipe -- numpy `Generator(Philox(seed))`, `integers(0, 2, n_pad)` signs then
`permutation(n_pad)[:k]` for srht, `integers(0, 2, (k, n), int8)` for
rademacher (sketching.py:62-73) -- so an operator built here and one built by
the reference are the same matrix.  The two north-star kinds (`gaussian`,
`sparse_sign`; SPEC.md:212 lists them as reference non-goals) are built with
`gaussian_operator` / `sparse_sign_operator`, which keeps
`SketchOperator("gaussian", ...)` rejected as the reference's tests pin
(tests/test_sketching.py:108-110).

`apply(theta, X)` runs on the GPU.  Device tables are realised lazily per
(device, row range): srht sign bits + sample indices, rademacher sign bits,
the gaussian int16 table of the local rows.  The
sparse_sign kind needs no table; its rows are hashed in-kernel.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from .errors import ShapeError
from .kernels import Matrix, as_array

__all__ = ["KINDS", "EXTENDED_KINDS", "SketchOperator", "make_operator", "apply", "sketch_into",
           "gaussian_operator", "sparse_sign_operator", "to_line", "from_line", "srht_apply", "materialize",
           "gauss_mode"]

KINDS = ("rademacher", "srht", "identity")
EXTENDED_KINDS = ("gaussian", "sparse_sign")
GAUSS_GRID = 2048.0
# gaussian sketch engine: "auto" (tensor pipe for binary32 inputs, fp64 CUDA
# cores for binary64), "fp64" or "tensor"; overridable for tests/benchmarks.
GAUSS_MODE = os.environ.get("RB_GAUSS_MODE", "auto")


def _next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p <<= 1
    return p


def _pack_bits(neg: np.ndarray, words: int) -> np.ndarray:
    """bool array (last axis) -> little-endian uint32 words (bit set = -1)."""
    neg = np.asarray(neg, dtype=bool)
    lead = neg.shape[:-1]
    pad = words * 32 - neg.shape[-1]
    if pad:
        neg = np.concatenate([neg, np.zeros(lead + (pad,), dtype=bool)], axis=-1)
    b = np.packbits(neg.reshape(lead + (words, 32)), axis=-1, bitorder="little")
    return b.view(np.uint32).reshape(lead + (words,))


@dataclass(frozen=True, eq=False)
class SketchOperator:
    """Seeded k x n sketching operator, immutable after construction."""

    kind: str
    k: int
    n: int
    seed: int

    _allowed = KINDS

    def __post_init__(self):
        if self.kind not in self._allowed:
            raise ValueError(f"unknown sketch kind {self.kind!r}")
        if self.k < 1 or self.n < 1:
            raise ShapeError(f"sketch dims must be positive, got k={self.k}, n={self.n}")
        if self.kind == "identity":
            if self.k != self.n:
                raise ShapeError("identity sketch requires k == n")
        elif self.k > self.n:
            raise ShapeError(f"sketch rows k={self.k} exceed columns n={self.n}")
        object.__setattr__(self, "_dev", {})
        if self.kind == "sparse_sign":
            object.__setattr__(self, "nnz", 8)
        if self.kind in ("srht", "rademacher"):
            gen = np.random.Generator(np.random.Philox(self.seed))
            if self.kind == "srht":
                n_pad = _next_pow2(self.n)
                signs = (gen.integers(0, 2, size=n_pad, dtype=np.int64) * 2 - 1).astype(np.float64)
                object.__setattr__(self, "n_pad", n_pad)
                object.__setattr__(self, "sign_diagonal", signs)
                object.__setattr__(self, "sample_indices", gen.permutation(n_pad)[: self.k])
            else:
                object.__setattr__(self, "_signs",
                                   gen.integers(0, 2, size=(self.k, self.n), dtype=np.int8) * 2 - 1)

    # -- device realisation ------------------------------------------------
    def device_tables(self, device, row0=0, nrows=None):
        """Device tables for rows row0 .. row0+nrows-1 (cached)."""
        dev = D.cuda_device(device)
        nrows = self.n - row0 if nrows is None else nrows
        key = (dev.index, row0, nrows)
        cache = self._dev
        if key in cache:
            return cache[key]
        if self.kind == "srht":
            words = -(-self.n_pad // 2048) * 64
            bits = _pack_bits(self.sign_diagonal < 0, words)
            tab = dict(bits=torch.from_numpy(bits.view(np.int32)).to(dev),
                       sample=torch.from_numpy(np.asarray(self.sample_indices, dtype=np.int64)).to(dev))
        elif self.kind == "rademacher":
            if row0 % 32:
                raise ValueError("rademacher shards must start at a multiple of 32 rows")
            sl = self._signs[:, row0:row0 + nrows]
            words = max(1, -(-nrows // 32))
            bits = _pack_bits(sl < 0, words)
            tab = dict(bits=torch.from_numpy(np.ascontiguousarray(bits).view(np.int32)).to(dev), ldb=words)
        elif self.kind == "gaussian":
            ldt = max(-(-nrows // 128) * 128, 128)
            theta = torch.empty((2 * (-(-self.k // 128)) * 128, ldt), dtype=torch.uint8, device=dev)
            with torch.cuda.device(dev):
                D.gaussian_fill(self.seed, self.k, row0, nrows, theta, ldt, getattr(self, "theta_bits", 16))
            tab = dict(theta=theta, ldt=ldt)
        elif self.kind == "sparse_sign":
            with torch.cuda.device(dev):
                tab = dict(table=D.sparse_sign_table(self.seed, self.k, self.nnz, row0, nrows, dev))
        else:
            tab = {}
        cache[key] = tab
        return tab

    def release_device_tables(self):
        self._dev.clear()


class _ExtendedSketchOperator(SketchOperator):
    _allowed = KINDS + EXTENDED_KINDS


def gaussian_operator(k: int, n: int, seed: int, digits: int = 6, theta_bits: int = 16) -> SketchOperator:
    """Dense gaussian sketch, entries q / (2048 sqrt(k)) with q the int16
    Box-Muller normal of Philox4x32-10.

    digits  byte digits of each binary32 X entry the tensor-pipe sketch
            keeps: 6 (default; fixed point at 2^-47 of each 16384-row chunk's
            max -- binary64-grade sketches), 4 (2^-31) or 3 (2^-23); the
            tensor work is proportional to it.  The operator (Theta) is the
            same; only the rounding of X inside Theta X changes.
    theta_bits  16 (default): the normals on the int16 grid 2^-11.  8: the
            SAME normals on the int8 grid 2^-5 (255 levels, clamped at
            +-127/32) -- a different, coarser-grained operator (still iid,
            symmetric, unit variance to 1e-4: a valid embedding), whose
            table needs one byte plane: half the table stream and half the
            tensor work.  Opt-in; the oracle builds the same operator
            (OracleSketch(..., bits=8))."""
    if digits not in (6, 4, 3):
        raise ValueError("digits must be 6, 4 or 3")
    if theta_bits not in (16, 8):
        raise ValueError("theta_bits must be 16 or 8")
    op = _ExtendedSketchOperator("gaussian", int(k), int(n), int(seed))
    object.__setattr__(op, "digits", int(digits))
    object.__setattr__(op, "theta_bits", int(theta_bits))
    return op


def gauss_scale(theta) -> float:
    """1 / (grid sqrt(k)) of a gaussian operator's table (q units)."""
    grid = 8192.0 if getattr(theta, "theta_bits", 16) == 8 else GAUSS_GRID
    return 1.0 / (grid * math.sqrt(theta.k))


def gauss_mode(theta, digits=None) -> str:
    """rb_sketch_gaussian mode of an operator (RB_GAUSS_MODE overrides)."""
    if GAUSS_MODE != "auto":
        return GAUSS_MODE
    d = digits or getattr(theta, "digits", 6)
    return {6: "auto", 4: "tensor4", 3: "tensor3"}[d] + ("+q8" if getattr(theta, "theta_bits", 16) == 8 else "")


def sparse_sign_operator(k: int, n: int, seed: int, nnz: int = 8) -> SketchOperator:
    """Sparse sign embedding: min(nnz, k) entries +-1/sqrt(s) per column."""
    op = _ExtendedSketchOperator("sparse_sign", int(k), int(n), int(seed))
    if not 1 <= nnz <= 16:
        raise ValueError("nnz must be in [1, 16]")
    object.__setattr__(op, "nnz", int(nnz))
    return op


def make_operator(kind: str, k: int, n: int, seed: int) -> SketchOperator:
    return SketchOperator(kind, int(k), int(n), int(seed))


def sketch_into(theta: SketchOperator, X: torch.Tensor, out: torch.Tensor, row0: int = 0,
                accumulate: bool = False, gauss: str = None) -> None:
    """out (k x cols, fp64, device) = Theta[:, row0:row0+rows] @ X (device,
    column-major).  The building block of every sketch in the sweep."""
    n, cols = X.shape
    k = theta.k
    if cols > 64 and theta.kind != "identity":
        # the kernels take at most 64 columns per call (a block is never
        # wider); wider inputs (e.g. the reference's materialize(): Theta @ I)
        # go through in column slabs
        for j in range(0, cols, 64):
            sketch_into(theta, X[:, j:j + 64], out[:, j:j + 64], row0, accumulate, gauss)
        return
    if theta.kind == "identity":
        if row0 != 0 or n != theta.n:
            raise ShapeError("identity sketch cannot be row-sharded")
        if accumulate:
            out.add_(X.to(torch.float64))
        else:
            out.copy_(X)
        return
    tab = theta.device_tables(X.device, row0, n) if theta.kind != "srht" else theta.device_tables(X.device)
    if theta.kind == "srht":
        D.sketch_srht(X, row0, theta.n_pad, tab["bits"], tab["sample"], k, 1.0 / math.sqrt(k), out,
                      accumulate)
    elif theta.kind == "rademacher":
        D.sketch_signs(X, tab["bits"], tab["ldb"], k, 1.0 / math.sqrt(k), out, accumulate)
    elif theta.kind == "gaussian":
        D.sketch_gaussian(X, tab["theta"], tab["ldt"], k, gauss_scale(theta), out,
                          accumulate, gauss or gauss_mode(theta))
    else:
        # the pre-bucketed table of exactly this row range (cached on the
        # operator; shards and whole-matrix calls each get their own)
        D.sketch_sparse_sign(X, row0, theta.seed, k, theta.nnz, out, accumulate, table=tab["table"])


def apply(theta: SketchOperator, X, device=None) -> Matrix:
    """Theta @ X in fine precision (sketching.py:140-155), on the GPU.

    X may be a numpy array / Matrix (uploaded; the result is a host-readable
    Matrix) or a CUDA tensor (the result stays on that device)."""
    if isinstance(X, torch.Tensor) and X.is_cuda:
        Xd = D.to_cm(X.reshape(X.shape[0], -1) if X.dim() == 1 else X)
    else:
        A = as_array(X)
        Xd = D.to_cm(torch.from_numpy(np.asfortranarray(A)), torch.float64, device)
    if Xd.shape[0] != theta.n:
        raise ShapeError(f"sketch expects {theta.n} rows, got {Xd.shape[0]}")
    out = D.empty_cm(theta.k, Xd.shape[1], torch.float64, Xd.device)
    with torch.cuda.device(Xd.device):
        sketch_into(theta, Xd, out)
    return Matrix(out)


def srht_apply(X, sign_diagonal, sample_indices, k: int, device=None):
    """Core SRHT path (sketching.py:129-137): zero-pad to len(sign_diagonal),
    sign-flip, Walsh-Hadamard transform (the pruned warp FWHT, same stage
    order as `_fwht_rows`), subsample, scale 1 / sqrt(k).  Returns the
    k x cols numpy array like the reference (the device result downloaded)."""
    A = as_array(X)
    signs = np.asarray(sign_diagonal, dtype=np.float64)
    n_pad = len(signs)
    if n_pad & (n_pad - 1) or n_pad < A.shape[0]:
        raise ShapeError(f"sign diagonal of length {n_pad} must be a power of two >= rows {A.shape[0]}")
    sample = np.asarray(sample_indices, dtype=np.int64)
    Xd = D.to_cm(torch.from_numpy(np.asfortranarray(A)), torch.float64, device)
    dev = Xd.device
    words = -(-n_pad // 2048) * 64
    bits = torch.from_numpy(_pack_bits(signs < 0, words).view(np.int32)).to(dev)
    out = D.empty_cm(len(sample), Xd.shape[1], torch.float64, dev)
    with torch.cuda.device(dev):
        for j in range(0, Xd.shape[1], 64):
            D.sketch_srht(Xd[:, j:j + 64], 0, n_pad, bits, torch.from_numpy(sample).to(dev), len(sample),
                          1.0 / math.sqrt(k), out[:, j:j + 64], False)
    return out.cpu().numpy()


def materialize(theta: SketchOperator, device=None) -> np.ndarray:
    """Dense k x n realization (sketching.py:158-160); test-scale diagnostics only."""
    return apply(theta, np.eye(theta.n), device).data


def to_line(theta: SketchOperator) -> str:
    return f"{theta.kind} {theta.k} {theta.n} {theta.seed}"


def from_line(line: str) -> SketchOperator:
    parts = line.split()
    if len(parts) != 4:
        raise ValueError(f"operator line must be 'kind k n seed', got {line!r}")
    kind, k, n, seed = parts
    if kind == "gaussian":
        return gaussian_operator(int(k), int(n), int(seed))
    if kind == "sparse_sign":
        return sparse_sign_operator(int(k), int(n), int(seed))
    return make_operator(kind, int(k), int(n), int(seed))
