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

from .errors import ShapeError

__all__ = ["PrecisionSpec", "COARSE", "FINE", "Matrix", "BlockPartition", "as_array", "cond_estimate"]


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
