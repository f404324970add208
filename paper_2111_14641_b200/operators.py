"""Linear operators for the Krylov drivers (reference
`pkg/src/sketch_krylov/operators.py`), applied on the GPU.

`LinearOperator.apply(X)` keeps the reference protocol (2-D block in, same
shape out, 1-D squeezed) and accepts numpy arrays or CUDA tensors; device
subclasses implement `_apply_dev(Xd, out_dtype)` on column-major device
blocks.  `Poisson3D` is the C4 operator (7-point Dirichlet Laplacian, the
3-D analogue of `gen_laplacian`, bench.py:214-233) with z-slab sharding and
a halo exchange of one plane per neighbour.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse
import torch

from . import _device as D
from ._lib import require_cuda
from .errors import ShapeError

__all__ = ["LinearOperator", "DenseOperator", "CsrOperator", "ShiftedOperator", "ComposedOperator",
           "Poisson3D"]


class LinearOperator:
    """Abstract n x n operator (operators.py:24-42)."""

    def __init__(self, n: int, description: str = ""):
        self.n = int(n)
        self.description = description

    @property
    def n_local(self) -> int:
        return self.n

    def apply(self, X, out_dtype=torch.float64):
        """A X.  numpy in -> numpy out; CUDA tensor in -> CUDA tensor out."""
        require_cuda()
        host = not (isinstance(X, torch.Tensor) and X.is_cuda)
        if host:
            A = np.asarray(X, dtype=np.float64)
            squeeze = A.ndim == 1
            if squeeze:
                A = A.reshape(-1, 1)
            Xd = D.to_cm(torch.from_numpy(np.asfortranarray(A)), torch.float64, getattr(self, "device", None))
        else:
            squeeze = X.dim() == 1
            Xd = D.to_cm(X.reshape(-1, 1) if squeeze else X)
        if Xd.shape[0] != self.n_local:
            raise ShapeError(f"operator dim {self.n_local} vs block rows {Xd.shape[0]}")
        with torch.cuda.device(Xd.device):
            Y = self._apply_dev(Xd, out_dtype)
        if host:
            Yh = Y.cpu().numpy()
            return Yh[:, 0] if squeeze else np.asfortranarray(Yh)
        return Y[:, 0] if squeeze else Y

    def _apply_dev(self, Xd, out_dtype):
        raise NotImplementedError


class DenseOperator(LinearOperator):
    def __init__(self, A, description: str = "dense", device=None):
        A = np.asarray(A, dtype=np.float64)
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ShapeError(f"dense operator must be square, got {A.shape}")
        super().__init__(A.shape[0], description)
        self.A = A
        self.device = D.cuda_device(device) if torch.cuda.is_available() else None
        self._Ad = None

    def _apply_dev(self, Xd, out_dtype):
        if self._Ad is None or self._Ad.device != Xd.device:
            self._Ad = D.to_cm(torch.from_numpy(np.asfortranarray(self.A)), torch.float64, Xd.device)
        X64 = D.to_cm(Xd, torch.float64)
        Y = D.empty_cm(self.n, Xd.shape[1], torch.float64, Xd.device)
        D.gemm(0, 0, 1.0, self._Ad, X64, 0.0, Y)
        return Y if out_dtype == torch.float64 else Y.to(out_dtype)


class CsrOperator(LinearOperator):
    def __init__(self, matrix, description: str = "csr", device=None):
        matrix = scipy.sparse.csr_matrix(matrix)
        if matrix.shape[0] != matrix.shape[1]:
            raise ShapeError(f"csr operator must be square, got {matrix.shape}")
        super().__init__(matrix.shape[0], description)
        self.matrix = matrix
        self.device = D.cuda_device(device) if torch.cuda.is_available() else None
        self._dev = None

    @classmethod
    def from_coo(cls, n, m, rows, cols, vals, description: str = "csr"):
        if n != m:
            raise ShapeError(f"operator must be square, got {n}x{m}")
        return cls(scipy.sparse.coo_matrix((vals, (rows, cols)), shape=(n, m)).tocsr(), description)

    def _apply_dev(self, Xd, out_dtype):
        if self._dev is None or self._dev[0].device != Xd.device:
            M = self.matrix
            self._dev = (torch.from_numpy(M.indptr.astype(np.int64)).to(Xd.device),
                         torch.from_numpy(M.indices.astype(np.int64)).to(Xd.device),
                         torch.from_numpy(M.data.astype(np.float64)).to(Xd.device))
        Y = D.empty_cm(self.n, Xd.shape[1], out_dtype, Xd.device)
        D.csr_spmm(*self._dev, Xd, Y)
        return Y


class ShiftedOperator(LinearOperator):
    """alpha I + sign A (operators.py:76-88)."""

    def __init__(self, base: LinearOperator, alpha: float, sign: int = 1):
        if sign not in (1, -1):
            raise ValueError(f"sign must be +-1, got {sign}")
        super().__init__(base.n, f"{alpha}*I{'+' if sign > 0 else '-'}({base.description})")
        self.base, self.alpha, self.sign = base, float(alpha), sign
        self.device = getattr(base, "device", None)

    def _apply_dev(self, Xd, out_dtype):
        Y = self.base._apply_dev(Xd, torch.float64)
        return (self.alpha * Xd.to(torch.float64) + self.sign * Y).to(out_dtype)


class ComposedOperator(LinearOperator):
    """x -> A(M(x)) (operators.py:91-102)."""

    def __init__(self, A: LinearOperator, M: LinearOperator):
        if A.n != M.n:
            raise ShapeError(f"composition dims disagree: {A.n} vs {M.n}")
        super().__init__(A.n, f"({A.description})o({M.description})")
        self.outer, self.inner = A, M
        self.device = getattr(A, "device", None)

    def _apply_dev(self, Xd, out_dtype):
        return self.outer._apply_dev(self.inner._apply_dev(Xd, torch.float64), out_dtype)


class Poisson3D(LinearOperator):
    """7-point Dirichlet Laplacian on nx*ny*nz (x fastest), stencil 6 / -1.

    With `comm` (a comm.Comm over world ranks) the grid is cut into z-slabs:
    rank r owns planes [z0, z0 + nz_local); `apply` exchanges the boundary
    planes with the neighbouring ranks (one plane x ncols each way) before
    the stencil kernel.  The stencil accumulates in the reference CSR order,
    so results equal `CsrOperator(kron-sum matrix).apply` bit for bit."""

    def __init__(self, nx, ny, nz, comm=None, device=None):
        super().__init__(nx * ny * nz, f"poisson{nx}x{ny}x{nz}")
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.comm = comm
        world = comm.world if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        base, extra = divmod(self.nz, world)
        self.z0 = rank * base + min(rank, extra)
        self.nz_local = base + (1 if rank < extra else 0)
        self.device = D.cuda_device(device) if torch.cuda.is_available() else None

    @property
    def n_local(self):
        return self.nx * self.ny * self.nz_local

    @property
    def row0(self):
        return self.nx * self.ny * self.z0

    def _halos(self, Xd):
        comm = self.comm
        if comm is None or not comm.active:
            return None, None
        import torch.distributed as dist
        plane = self.nx * self.ny
        cols = Xd.shape[1]
        lo = hi = None
        ops = []
        rank, world = comm.rank, comm.world
        first = Xd[:plane].contiguous()
        last = Xd[-plane:].contiguous()
        g = comm.group
        # gloo has no device-memory point-to-point: stage the planes on the host
        staged = Xd.is_cuda and dist.get_backend(g) != "nccl"
        if staged:
            first, last = first.cpu(), last.cpu()
        if rank > 0:
            lo = torch.empty_like(first)
            ops += [dist.P2POp(dist.isend, first, dist.get_global_rank(g, rank - 1) if g else rank - 1, g),
                    dist.P2POp(dist.irecv, lo, dist.get_global_rank(g, rank - 1) if g else rank - 1, g)]
        if rank < world - 1:
            hi = torch.empty_like(last)
            ops += [dist.P2POp(dist.isend, last, dist.get_global_rank(g, rank + 1) if g else rank + 1, g),
                    dist.P2POp(dist.irecv, hi, dist.get_global_rank(g, rank + 1) if g else rank + 1, g)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if staged:
            lo = lo.to(Xd.device) if lo is not None else None
            hi = hi.to(Xd.device) if hi is not None else None
        # contiguous (plane, cols) row-major -> column-major views
        to = lambda t: D.to_cm(t) if t is not None else None
        return to(lo), to(hi)

    def _apply_dev(self, Xd, out_dtype):
        lo, hi = self._halos(Xd)
        Y = D.empty_cm(self.n_local, Xd.shape[1], out_dtype, Xd.device)
        D.stencil7(self.nx, self.ny, self.nz_local, Xd, Y, lo, hi)
        return Y
