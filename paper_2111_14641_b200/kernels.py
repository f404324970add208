"""Domain types of the drop-in (reference `pkg/src/sketch_krylov/kernels.py:44-164`).

`PrecisionSpec` / `COARSE` / `FINE` and `BlockPartition` keep the reference
semantics exactly.  `Matrix` keeps the reference's contract (2-D, binary64
values, finite entries, `.data` is a Fortran-ordered numpy array) but may be
backed by a device tensor: `.tensor` is the device array the kernels
produced, `.data` downloads it lazily (once) for host-side consumers.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import NotPositiveDefiniteError, ShapeError, SingularTriangularError

__all__ = ["PrecisionSpec", "COARSE", "FINE", "Matrix", "BlockPartition", "as_array", "cond_estimate",
           "gemm", "householder_qr", "cholesky", "triangular_solve"]


@dataclass(frozen=True)
class PrecisionSpec:
    """'coarse' = binary32, 'fine' = binary64 (kernels.py:44-61)."""

    format: str

    def __post_init__(self):
        if self.format not in ("coarse", "fine"):
            raise ValueError(f"unknown precision format {self.format!r}")

    @property
    def u(self) -> float:
        return 2.0 ** -24 if self.format == "coarse" else 2.0 ** -53

    @property
    def dtype(self):
        return np.float32 if self.format == "coarse" else np.float64

    @property
    def torch_dtype(self):
        return torch.float32 if self.format == "coarse" else torch.float64


COARSE = PrecisionSpec("coarse")
FINE = PrecisionSpec("fine")


class Matrix:
    """2-D binary64 matrix, host (numpy) or device (torch) backed."""

    def __init__(self, data, precision: PrecisionSpec = FINE):
        self.precision = precision
        self._host = None
        self._dev = None
        if isinstance(data, Matrix):
            self._host, self._dev = data._host, data._dev
            return
        if type(data).__name__ == "DevArray":
            data = data.tensor
        if isinstance(data, torch.Tensor):
            t = data
            if t.ndim == 1:
                t = t.reshape(-1, 1)
            if t.ndim != 2:
                raise ShapeError(f"Matrix requires 2-D data, got ndim={t.ndim}")
            self._dev = t
            return
        A = np.asarray(data, dtype=np.float64)
        if A.ndim == 1:
            A = A.reshape(-1, 1)
        if A.ndim != 2:
            raise ShapeError(f"Matrix requires 2-D data, got ndim={A.ndim}")
        if not np.all(np.isfinite(A)):
            raise ValueError("Matrix entries must be finite")
        self._host = np.asfortranarray(A)

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            A = self._dev.detach().to("cpu", torch.float64).numpy()
            if not np.all(np.isfinite(A)):
                raise ValueError("Matrix entries must be finite")
            self._host = np.asfortranarray(A)
        return self._host

    @property
    def tensor(self) -> torch.Tensor:
        return self._dev if self._dev is not None else torch.from_numpy(self._host)

    @property
    def shape(self):
        return tuple(self._dev.shape) if self._dev is not None else self._host.shape

    @property
    def rows(self) -> int:
        return self.shape[0]

    @property
    def cols(self) -> int:
        return self.shape[1]

    def __array__(self, dtype=None, copy=None):
        if dtype is None and not copy:
            return self.data
        return np.array(self.data, dtype=dtype)

    def __repr__(self):
        where = "device" if self._dev is not None else "host"
        return f"Matrix({self.shape[0]}x{self.shape[1]}, {where})"


class DevArray:
    """What `RbgsSweep.Q / S / P / R` hand to a caller: the reference keeps
    these as numpy arrays that consumers slice and feed to numpy / scipy
    (rbgs.py:343-347; krylov.py:229-262 does `sweep.R[:c, mp:c]`,
    `sweep.Q[:, :j] @ Z`).  Here the data live on the device, so the public
    attribute is this lazy view: slicing stays on the device (`.tensor` is
    the CUDA tensor, used by this package's own drivers), and anything numpy
    asks of it -- `np.asarray`, `@`, arithmetic, `.copy()`, `.T`,
    `np.linalg.*` -- downloads the viewed block once as binary64."""

    __slots__ = ("tensor",)
    __array_priority__ = 100.0

    def __init__(self, t):
        self.tensor = t

    def __getitem__(self, idx):
        return DevArray(self.tensor[idx])

    def __setitem__(self, idx, value):
        v = value.tensor if isinstance(value, DevArray) else value
        if not isinstance(v, torch.Tensor):
            v = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64)))
        self.tensor[idx] = v.to(self.tensor.device, self.tensor.dtype)

    def __array__(self, dtype=None, copy=None):
        A = self.tensor.detach().to("cpu", torch.float64).numpy()
        return A if dtype is None else A.astype(dtype, copy=False)

    @property
    def shape(self):
        return tuple(self.tensor.shape)

    @property
    def ndim(self):
        return self.tensor.dim()

    @property
    def dtype(self):
        return np.dtype(np.float64)

    def __len__(self):
        return self.tensor.shape[0]

    def __getattr__(self, name):  # .copy(), .T, .sum(), ... : numpy semantics on the downloaded block
        if name.startswith("__"):
            raise AttributeError(name)
        return getattr(np.asarray(self), name)

    def __repr__(self):
        return f"DevArray({tuple(self.tensor.shape)}, {self.tensor.dtype}, {self.tensor.device})"


def _devarray_op(name):
    def op(self, *others):
        return getattr(np.asarray(self), name)(*[np.asarray(o) if isinstance(o, DevArray) else o for o in others])
    op.__name__ = name
    return op


for _n in ("__matmul__", "__rmatmul__", "__add__", "__radd__", "__sub__", "__rsub__", "__mul__", "__rmul__",
           "__truediv__", "__rtruediv__", "__neg__", "__abs__", "__eq__", "__ne__", "__lt__", "__le__", "__gt__",
           "__ge__", "__iter__"):
    setattr(DevArray, _n, _devarray_op(_n))
DevArray.__hash__ = None


def as_array(X) -> np.ndarray:
    """Host fp64 2-D view (kernels.py:68-77)."""
    if isinstance(X, Matrix):
        return X.data
    if isinstance(X, DevArray):
        X = X.tensor
    if isinstance(X, torch.Tensor):
        X = X.detach().cpu().numpy()
    A = np.asarray(X, dtype=np.float64)
    if A.ndim == 1:
        A = A.reshape(-1, 1)
    if A.ndim != 2:
        raise ShapeError(f"expected a 2-D array, got ndim={A.ndim}")
    return A


@dataclass(frozen=True)
class BlockPartition:
    """Column blocks: `num_blocks` of width `block_width` with a ragged tail,
    or explicit `widths` (kernels.py:119-164)."""

    block_width: int
    num_blocks: int
    total_cols: int
    widths: tuple = field(default=None)

    def __post_init__(self):
        mp, nb, m = self.block_width, self.num_blocks, self.total_cols
        if mp < 1 or nb < 1 or m < 1:
            raise ValueError("partition counts must be positive")
        if self.widths is not None:
            w = tuple(int(x) for x in self.widths)
            object.__setattr__(self, "widths", w)
            if len(w) != nb or sum(w) != m or min(w) < 1:
                raise ValueError(f"explicit widths {w} inconsistent with p={nb}, m={m}")
        else:
            tail = m - mp * (nb - 1)
            if not 1 <= tail <= mp:
                raise ValueError(f"partition m={m}, m_p={mp}, p={nb} has invalid tail width {tail}")

    @classmethod
    def uniform(cls, total_cols: int, block_width: int) -> "BlockPartition":
        return cls(block_width, -(-total_cols // block_width), total_cols)

    def block_widths(self) -> tuple:
        if self.widths is not None:
            return self.widths
        mp, nb, m = self.block_width, self.num_blocks, self.total_cols
        return tuple([mp] * (nb - 1) + [m - mp * (nb - 1)])

    def offsets(self) -> tuple:
        out = [0]
        for w in self.block_widths():
            out.append(out[-1] + w)
        return tuple(out)


def cond_estimate(A, device=None) -> float:
    """sigma_max / sigma_min of a tall matrix on the GPU (kernels.py:552-566);
    see post.cond_estimate."""
    from .post import cond_estimate as _ce

    return _ce(A, device)


# ---------------------------------------------------------------------------
# The reference's kernel-level entry points (kernels.py:171-270) on the device.
# The sweep calls the device kernels directly; these wrappers keep the module
# API for callers that use them standalone.


def _dev_cm(X, dtype, device=None):
    from . import _device as D

    if isinstance(X, Matrix):
        X = X._dev if X._dev is not None else X.data
    if isinstance(X, DevArray):
        X = X.tensor
    if isinstance(X, torch.Tensor):
        t = X if X.dim() == 2 else X.reshape(-1, 1)
        return D.to_cm(t, dtype, device if device is not None else (t.device if t.is_cuda else None))
    return D.to_cm(torch.from_numpy(np.asfortranarray(as_array(X))), dtype, device)


def gemm(alpha: float, A, B, beta: float = 0.0, C=None, prec: PrecisionSpec = FINE, device=None) -> Matrix:
    """fl(alpha A B + beta C) with every elementary multiply / add rounded per
    `prec`, l ascending (kernels.py:171-209) -- bit-identical to the
    reference.  alpha = +-1 (every call of the RBGS path) runs on rb_project's
    separately-rounded multiply-add kernels in 64-column slabs; any other
    alpha keeps the reference's extra rounding fl(alpha fl(a b)) with one
    elementwise device pass per l."""
    from . import _device as D
    from ._lib import F32, F64, ORDER_REFERENCE, require_cuda

    require_cuda()
    Ad = _dev_cm(A, prec.torch_dtype, device)
    dev = Ad.device
    Bd = _dev_cm(B, torch.float64, dev)
    if Ad.shape[1] != Bd.shape[0]:
        raise ShapeError(f"gemm inner dimensions disagree: {tuple(Ad.shape)} x {tuple(Bd.shape)}")
    n, m = Ad.shape[0], Bd.shape[1]
    dt = prec.torch_dtype
    if C is not None:
        Cd = _dev_cm(C, torch.float64, dev)
        if tuple(Cd.shape) != (n, m):
            raise ShapeError(f"gemm C has shape {tuple(Cd.shape)}, expected {(n, m)}")
    elif beta != 0.0:
        raise ShapeError("gemm beta != 0 requires C")
    with torch.cuda.device(dev):
        acc = D.zeros_cm(n, m, dt, dev)
        if C is not None and beta != 0.0:
            acc.copy_(Cd)  # rounds to prec.dtype like C.astype(dt)
            if beta != 1.0:
                acc.mul_(torch.tensor(beta, dtype=dt, device=dev))
        K = Ad.shape[1]
        if K and alpha in (1.0, -1.0):
            compute = F32 if prec.format == "coarse" else F64
            X = Bd if alpha == -1.0 else D.to_cm(-Bd)  # acc - A (-B): negation is exact
            for j in range(0, m, 64):
                D.project(Ad, X[:, j:j + 64], acc[:, j:j + 64], acc[:, j:j + 64], compute, ORDER_REFERENCE)
        elif K:
            a = torch.tensor(alpha, dtype=dt, device=dev)
            Bt = Bd.to(dt)
            for l in range(K):
                term = Ad[:, l:l + 1] * Bt[l:l + 1, :]
                acc += a * term
        return Matrix(D.to_cm(acc, torch.float64), precision=prec)


def householder_qr(A, device=None) -> tuple:
    """Economic Householder QR with diag(R) >= 0 (kernels.py:216-231) on the
    device (single-CTA Householder kernel: meant for the k-dimensional
    problems of the path; a tall n runs, slowly)."""
    from . import _device as D
    from ._lib import require_cuda

    require_cuda()
    Ad = _dev_cm(A, torch.float64, device)
    n, m = Ad.shape
    if n < m:
        raise ShapeError(f"householder_qr requires rows >= cols, got {(n, m)}")
    with torch.cuda.device(Ad.device):
        Q = D.empty_cm(n, m, torch.float64, Ad.device)
        Q.copy_(Ad)
        R = D.zeros_cm(m, m, torch.float64, Ad.device)
        D.geqrf(Q, R)
    return Matrix(Q), Matrix(R)


def cholesky(G, device=None) -> Matrix:
    """Upper-triangular R with R^T R = G (kernels.py:234-247), dpotrf
    semantics: NotPositiveDefiniteError(column) at the first bad pivot."""
    from . import _device as D
    from ._lib import require_cuda

    require_cuda()
    Gd = _dev_cm(G, torch.float64, device)
    n, m = Gd.shape
    if n != m:
        raise ShapeError(f"cholesky requires a square matrix, got {(n, m)}")
    if n > 128:
        raise ShapeError(f"cholesky on the device handles n <= 128 (block-sized Gram matrices), got {n}")
    with torch.cuda.device(Gd.device):
        tol = 1e-10 * max(1.0, float(Gd.abs().max()))
        if float((Gd - Gd.t()).abs().max()) > tol:
            raise ShapeError("cholesky input is not symmetric")
        R = D.zeros_cm(n, n, torch.float64, Gd.device)
        info = torch.zeros(1, dtype=torch.int32, device=Gd.device)
        D.potrf(Gd, R, info)
        bad = int(info.item())
    if bad > 0:
        raise NotPositiveDefiniteError(bad)
    return Matrix(R)


def triangular_solve(R, B, side: str = "left", device=None) -> Matrix:
    """Solve R X = B ('left') or X R = B ('right') for upper-triangular R
    (kernels.py:250-270)."""
    from . import _device as D
    from ._lib import require_cuda

    require_cuda()
    Rd = _dev_cm(R, torch.float64, device)
    n = Rd.shape[0]
    if Rd.shape[1] != n:
        raise ShapeError(f"triangular_solve requires square R, got {tuple(Rd.shape)}")
    Bd = _dev_cm(B, torch.float64, Rd.device)
    d = Rd.diagonal().abs()
    if bool((d == 0.0).any()):
        raise SingularTriangularError(int(torch.argmax((d == 0.0).to(torch.int32)).item()))
    with torch.cuda.device(Rd.device):
        if side == "left":
            if Bd.shape[0] != n:
                raise ShapeError(f"RX=B shape mismatch: {tuple(Rd.shape)} vs {tuple(Bd.shape)}")
            X = D.empty_cm(Bd.shape[0], Bd.shape[1], torch.float64, Rd.device)
            X.copy_(Bd)
            info = torch.zeros(1, dtype=torch.int32, device=Rd.device)
            D.trsm_left_upper(Rd, X, info)
        elif side == "right":
            if Bd.shape[1] != n:
                raise ShapeError(f"XR=B shape mismatch: {tuple(Bd.shape)} vs {tuple(Rd.shape)}")
            if n > 64:
                raise ShapeError(f"right solves on the device handle n <= 64 (one block), got {n}")
            X = D.empty_cm(Bd.shape[0], n, torch.float64, Rd.device)
            D.trsm_right(Bd, Rd, X)
        else:
            raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    return Matrix(X)
