"""Randomized block Gram-Schmidt on the GPU -- drop-in for
`sketch_krylov.rbgs` (reference `pkg/src/sketch_krylov/rbgs.py`).

Public names and signatures follow the reference: `RbgsConfig`, `CertReport`,
`BlockQR`, `RbgsSweep(n, theta, cfg).push_block(W_i) / finish()`,
`rbgs(W, theta, cfg)`, `certify(S, P, R)`, the Step-2 solvers `ls_*` and the
Step-4/5 routines `interblock_*`.  Device-only knobs live in a separate
`DeviceConfig` ("Config / flags"), so reference configs
round-trip unchanged.

Per block i (paper Alg. 2; rbgs.py:352-399), on one rank
holding rows [row0, row0 + n_local):

  Step 1   P_i = Theta W_i                  sketch kernel  (+ allreduce)
  Step 2   X = argmin ||S X - P_i||          small fp64 kernels (replicated)
  Step 3   Q' = W_i - Q_(1:i-1) X            rb_project, reference order,
                                             fused sum-of-squares of W_i, Q'
  Step 4-5 inter-block QR of Q'             sketch of Q' (+ allreduce),
                                             fp64 Cholesky / TRSM, tall TRSM
                                             writing Q_i into its slot
  checks   one device->host read of the status words per block: the
           dependence test (rbgs.py:373-376, GLOBAL n and norms), the
           Cholesky info (-> InterblockError) and a finiteness flag
           (the reference's Matrix() check, kernels.py:97-98).

Storage: Q is n_local x m in the coarse format (binary32) when
`cfg.coarse` is COARSE -- bit-identical to what the reference's coarse gemm
reads (`Q.astype(float32)`, kernels.py:192) -- and binary64 otherwise;
S, P (k x m) and R (m x m) are binary64 and replicated.
"""

from __future__ import annotations

import math
import os
import re
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from . import sketching
from ._lib import F32, F64, ORDER_FMA, ORDER_REFERENCE, ORDER_TC, require_cuda
from .comm import Comm, RowShard
from .errors import (
    CertificationError,
    DependentBlockError,
    InterblockError,
    NotPositiveDefiniteError,
    RankDeficiencyError,
    ShapeError,
)
from .kernels import COARSE, FINE, BlockPartition, DevArray, Matrix, PrecisionSpec, as_array

__all__ = ["RbgsConfig", "DeviceConfig", "BlockQR", "CertReport", "rbgs", "RbgsSweep", "RbgsPlan", "certify",
           "ls_richardson", "ls_bmgs_reorth", "ls_cg_normal", "ls_householder_direct",
           "interblock_rgs", "interblock_sketched_cholqr", "interblock_l2_cholqr", "parse_method",
           "cholesky_qr_postprocess", "certify_embedding", "save_blockqr", "load_blockqr",
           "save_blockqr_binary", "load_blockqr_binary"]

U_FINE = 2.0 ** -53
U_COARSE = 2.0 ** -24

_METHOD = re.compile(r"^([a-z0-9_]+)(?:[(:]\s*(\d+)\s*\)?)?$")
_DEFAULTS = {"richardson": 5, "bmgs_reorth": 1, "cg_normal": 20, "sketched_cholqr": 1}


def parse_method(spec: str):
    """'name', 'name(3)' or 'name:3' -> (name, param) (rbgs.py:64-82)."""
    m = _METHOD.match(spec.strip().lower())
    if not m:
        raise ValueError(f"cannot parse method spec {spec!r}")
    name, param = m.group(1), m.group(2)
    if param is None:
        return name, _DEFAULTS.get(name)
    param = int(param)
    if param < 1:
        raise ValueError(f"method parameter must be >= 1 in {spec!r}")
    return name, param


@dataclass
class RbgsConfig:
    """Reference knobs, same fields and validation (rbgs.py:85-107)."""

    partition: BlockPartition = None
    ls_solver: str = "richardson(5)"
    interblock: str = "l2_plus_cholqr"
    coarse: PrecisionSpec = COARSE
    fine: PrecisionSpec = FINE
    certify_blocks: bool = False
    resketch: bool = False

    def __post_init__(self):
        if self.fine.u > self.coarse.u:
            raise ValueError("fine precision must not be coarser than coarse")
        name, param = parse_method(self.ls_solver)
        if name not in ("richardson", "bmgs_reorth", "cg_normal", "householder_direct"):
            raise ValueError(f"unknown ls solver {self.ls_solver!r}")
        if name != "householder_direct" and (param is None or param < 1):
            raise ValueError(f"solver {name} needs a positive iteration count")
        if parse_method(self.interblock)[0] not in ("rgs_single", "sketched_cholqr", "l2_plus_cholqr"):
            raise ValueError(f"unknown interblock method {self.interblock!r}")


@dataclass
class DeviceConfig:
    """Device-side knobs (no reference counterpart).

    device            CUDA device (default: current).
    q_dtype           storage of Q (default binary32 when cfg.coarse is
                      COARSE, else binary64); binary64 keeps the reference's
                      fp64 Q (e.g. for Arnoldi, whose operator reads fp64 Q).
    projection_order  "reference" (bit-identical Step 3), "fma" (fused
                      multiply-subtract on the CUDA cores) or "tc" (tensor
                      pipe, 3xTF32: HBM-bound); the last two are faster and
                      not bit-identical -- for inputs whose R is insensitive
                      to the Step-3 rounding order (bench.py gates them on
                      the measured oracle drift).
    sketch_digits     gaussian kind on the tensor pipe: byte digits kept of
                      each binary32 entry inside Theta X (6, 4 or 3; default:
                      the operator's own, 6 = binary64-grade).  Fewer digits
                      cost proportionally less tensor work; like the fast
                      projection orders, for inputs whose R tolerates it.
    comm / shard      row sharding: this rank's rows and the group that owns
                      the other shards (comm.py).  Default: all rows here.
    overwrite_w       one-shot rbgs() only: Q is written over W's own device
                      storage (W must be a column-major CUDA tensor of Q's
                      dtype), block by block as each W_i is consumed -- the
                      n x m buffer that lets the C5 shard (2^24 x 1024 fp32
                      plus its 2^24 x 2048 gaussian table) fit one GPU.  W
                      is destroyed; failures raise at the failing block.
    coarse_shadow     binary64 Q with binary32 Step 3: keep a binary32 copy
                      of Q for the projection (same bits, half the bytes).
    """

    device: object = None
    q_dtype: torch.dtype = None
    projection_order: str = "reference"
    sketch_digits: int = None
    comm: Comm = None
    shard: RowShard = None
    overwrite_w: bool = False
    coarse_shadow: bool = True


@dataclass(frozen=True)
class CertReport:
    delta: float
    delta_tilde: float
    per_block_ortho: tuple = ()
    per_block_resid: tuple = ()

    def __post_init__(self):
        vals = (self.delta, self.delta_tilde, *self.per_block_ortho, *self.per_block_resid)
        if not all(np.isfinite(v) and v >= 0.0 for v in vals):
            raise ValueError("certification quantities must be finite and nonnegative")


@dataclass(eq=False)
class BlockQR:
    Q: Matrix
    R: Matrix
    S: Matrix
    P: Matrix
    partition: BlockPartition
    cert: CertReport = None


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def _dev_f64(A, device):
    """fp64 column-major device copy of a host or device matrix."""
    if isinstance(A, Matrix):
        A = A._dev if A._dev is not None else A.data
    if isinstance(A, torch.Tensor):
        return D.to_cm(A if A.dim() == 2 else A.reshape(-1, 1), torch.float64, device)
    return D.to_cm(torch.from_numpy(np.asfortranarray(as_array(A))), torch.float64, device)


class _Scratch:
    """Per-sweep device scratch, allocated once at the largest block width."""

    def __init__(self, k, m, w, device):
        f64 = torch.float64
        self.Pi = D.empty_cm(k, w, f64, device)
        self.Pn = [D.empty_cm(k, w, f64, device), D.empty_cm(k, w, f64, device)]  # fused next-block sketches
        self.pn_flip = 0
        self.Sp = D.empty_cm(k, w, f64, device)
        self.Ss = D.empty_cm(k, w, f64, device)
        self.Si = D.empty_cm(k, w, f64, device)
        self.T = D.empty_cm(k, w, f64, device)
        self.X = D.empty_cm(max(m, 1), w, f64, device)
        self.G = D.empty_cm(w, w, f64, device)
        self.R1 = D.empty_cm(w, w, f64, device)
        self.R2 = D.empty_cm(w, w, f64, device)
        self.Rt = D.empty_cm(w, w, f64, device)
        self.Pr = D.empty_cm(k, w, f64, device)  # binary32-rounded P_i (fine = COARSE)
        self.P32 = D.empty_cm(k, w, torch.float32, device)
        self.Rb = D.empty_cm(w, w, f64, device)  # l2 stage, fallback path
        self.Sb = D.empty_cm(k, w, f64, device)
        self.norms = torch.zeros(8, dtype=f64, device=device)  # [w2, q2, fin, ...]
        # status words: [0..3] checked per block (Cholesky infos), [6..7]
        # solver / RGS, [8..10] the l2 stage's two paths (selector, A, B)
        self.info = torch.zeros(16, dtype=torch.int32, device=device)
        self.status_host = torch.zeros(8, dtype=f64).pin_memory()
        self.info_host = torch.zeros(16, dtype=torch.int32).pin_memory()


# ---------------------------------------------------------------------------
# Step 2 solvers (rbgs.py:144-225) -- device, fp64
# ---------------------------------------------------------------------------

def _richardson_dev(S, P, l, X, T):
    D.richardson(S, P, l, X, T)


def _bmgs_dev(S, offsets, P, l, X, T):
    c = S.shape[1]
    T.copy_(P)
    X.zero_()
    blocks = [(offsets[j], min(offsets[j + 1], c)) for j in range(len(offsets) - 1) if offsets[j] < c]
    for _ in range(l):
        for a, b in blocks:
            Sj = S[:, a:b]
            inc = D.empty_cm(b - a, P.shape[1], torch.float64, S.device)
            D.gemm(1, 0, 1.0, Sj, T, 0.0, inc)
            X[a:b].add_(inc)
            D.gemm(0, 0, -1.0, Sj, inc, 1.0, T)


def _cg_dev(S, P, iters, X):
    k, c = S.shape
    p = P.shape[1]
    dev = S.device
    b = D.empty_cm(c, p, torch.float64, dev)
    D.gemm(1, 0, 1.0, S, P, 0.0, b)
    X.zero_()
    r = b.clone()
    d = r.clone()
    rs = (r * r).sum(0)
    SD = D.empty_cm(k, p, torch.float64, dev)
    Ad = D.empty_cm(c, p, torch.float64, dev)
    for _ in range(iters):
        D.gemm(0, 0, 1.0, S, d, 0.0, SD)
        D.gemm(1, 0, 1.0, S, SD, 0.0, Ad)
        dAd = (d * Ad).sum(0)
        alpha = torch.where(dAd > 0, rs / torch.where(dAd > 0, dAd, torch.ones_like(dAd)), torch.zeros_like(dAd))
        X.add_(alpha * d)
        r.sub_(alpha * Ad)
        rs2 = (r * r).sum(0)
        beta = torch.where(rs > 0, rs2 / torch.where(rs > 0, rs, torch.ones_like(rs)), torch.zeros_like(rs))
        rs = rs2
        d = r + beta * d


def _householder_direct_dev(S, P, X, scr, sync=True, u=None):
    k, c = S.shape
    dev = S.device
    A = D.empty_cm(k, c, torch.float64, dev)
    A.copy_(S)
    Rs = D.empty_cm(c, c, torch.float64, dev)
    D.geqrf(A, Rs)
    d = Rs.diagonal().abs()
    if sync:
        dmin, dmax = float(d.min()), float(d.max())
        if dmin <= k * (U_FINE if u is None else u) * max(dmax, 1e-300):
            raise RankDeficiencyError(f"least-squares matrix numerically rank deficient (min diag {dmin:.3e})")
    D.gemm(1, 0, 1.0, A, P, 0.0, X)
    D.trsm_left_upper(Rs, X, scr.info[6:7])


def _solve_ls_f32(name, param, S, offsets, P, X, scr):
    """Step 2 in binary32 (fine = COARSE): the reference casts S and P_i to
    float32 and runs the solver in float32 BLAS (rbgs.py:144-212); here
    the library's own binary32 GEMM (binary32 accumulation, no TF32).  X comes back as binary64 values
    of the binary32 solution (`X.astype(np.float64)`)."""
    k, c = S.shape
    p = P.shape[1]
    dev = S.device
    f32 = torch.float32
    S32 = D.empty_cm(k, c, f32, dev)
    D.convert(S, S32)
    P32 = D.empty_cm(k, p, f32, dev)
    D.convert(P, P32)
    X32 = D.zeros_cm(c, p, f32, dev)
    if name == "richardson":
        T = D.empty_cm(k, p, f32, dev)
        for _ in range(param):
            T.copy_(P32)
            D.gemm32(0, 0, -1.0, S32, X32, 1.0, T)     # Pd - Sd X
            D.gemm32(1, 0, 1.0, S32, T, 1.0, X32)      # X + Sd^T (...)
    elif name == "bmgs_reorth":
        T = P32.clone()
        blocks = [(offsets[j], min(offsets[j + 1], c)) for j in range(len(offsets) - 1) if offsets[j] < c]
        for _ in range(param):
            for a, b in blocks:
                inc = D.empty_cm(b - a, p, f32, dev)
                D.gemm32(1, 0, 1.0, S32[:, a:b], T, 0.0, inc)
                X32[a:b].add_(inc)
                D.gemm32(0, 0, -1.0, S32[:, a:b], inc, 1.0, T)
    elif name == "cg_normal":
        b = D.empty_cm(c, p, f32, dev)
        D.gemm32(1, 0, 1.0, S32, P32, 0.0, b)
        r = b.clone()
        d = r.clone()
        rs = (r * r).sum(0)
        SD = D.empty_cm(k, p, f32, dev)
        Ad = D.empty_cm(c, p, f32, dev)
        for _ in range(param):
            D.gemm32(0, 0, 1.0, S32, d, 0.0, SD)
            D.gemm32(1, 0, 1.0, S32, SD, 0.0, Ad)
            dAd = (d * Ad).sum(0)
            alpha = torch.where(dAd > 0, rs / torch.where(dAd > 0, dAd, torch.ones_like(dAd)),
                                torch.zeros_like(dAd))
            X32.add_(alpha * d)
            r.sub_(alpha * Ad)
            rs2 = (r * r).sum(0)
            beta = torch.where(rs > 0, rs2 / torch.where(rs > 0, rs, torch.ones_like(rs)), torch.zeros_like(rs))
            rs = rs2
            d = r + beta * d
    else:
        # Householder on the binary32-rounded data, factorised in binary64,
        # rank test at u = 2^-24 (rbgs.py:208 with prec = COARSE)
        Sr = D.empty_cm(k, c, torch.float64, dev)
        D.convert(S32, Sr)
        Pr = D.empty_cm(k, p, torch.float64, dev)
        D.convert(P32, Pr)
        Xd = D.empty_cm(c, p, torch.float64, dev)
        _householder_direct_dev(Sr, Pr, Xd, scr, u=U_COARSE)
        D.convert(Xd, X32)
    D.convert(X32, X)


# ---------------------------------------------------------------------------
# the sweep
# ---------------------------------------------------------------------------

class RbgsSweep:
    """Incremental RBGS on the GPU (rbgs.py:318-407).

    Feed blocks left to right with `push_block`; `Q`, `S`, `P`, `R` are the
    device buffers (torch, column-major; Q holds this rank's rows only)."""

    def __init__(self, n: int, theta, cfg: RbgsConfig, device_cfg: DeviceConfig = None, *, _q_storage=None):
        require_cuda()
        if cfg.partition is None:
            raise ShapeError("config needs a partition")
        m = cfg.partition.total_cols
        if theta.n != n:
            raise ShapeError(f"sketch built for n={theta.n}, input has n={n}")
        if not (m <= theta.k <= n):
            raise ShapeError(f"need total cols m={m} <= sketch k={theta.k} <= n={n}")
        # unique coarse precision (fine = COARSE): P_i is rounded to binary32
        # values (rbgs.py:363 _round_to) and the Step-2 solvers run in
        # binary32 (prec.dtype, rbgs.py:144-212); inter-block stays binary64
        self.fine32 = cfg.fine.format != "fine"
        dc = device_cfg or DeviceConfig()
        self.device = D.cuda_device(dc.device)
        self.comm = dc.comm or Comm(None)
        self.shard = dc.shard or RowShard.whole(n)
        if self.shard.n != n:
            raise ShapeError("shard built for a different n")
        self.n = n
        self.n_local = self.shard.n_local
        self.row0 = self.shard.row0
        self.theta = theta
        self.cfg = cfg
        self.solver = parse_method(cfg.ls_solver)
        self.inter = parse_method(cfg.interblock)
        self.offsets = cfg.partition.offsets()
        self.compute = F32 if cfg.coarse.format == "coarse" else F64
        self.q_dtype = dc.q_dtype or (torch.float32 if self.compute == F32 else torch.float64)
        if dc.projection_order not in ("reference", "fma", "tc"):
            raise ValueError("projection_order must be 'reference', 'fma' or 'tc'")
        self.order = {"fma": ORDER_FMA, "tc": ORDER_TC}.get(dc.projection_order, ORDER_REFERENCE)
        if dc.sketch_digits not in (None, 6, 4, 3):
            raise ValueError("sketch_digits must be 6, 4 or 3")
        self._gmode = sketching.gauss_mode(theta, dc.sketch_digits) if theta.kind == "gaussian" else "auto"
        dev = self.device
        k = theta.k
        if _q_storage is not None:  # Q over W's storage (DeviceConfig.overwrite_w)
            if (_q_storage.shape != (self.n_local, m) or _q_storage.dtype != self.q_dtype
                    or not D.is_cm(_q_storage) or _q_storage.device != dev):
                raise ShapeError("overwrite_w needs W as a column-major CUDA tensor of Q's dtype")
            self.Qd = _q_storage
        else:
            self.Qd = D.zeros_cm(self.n_local, m, self.q_dtype, dev)
        # binary64 Q with binary32 projections (Arnoldi: the operator reads
        # the binary64 basis): keep a binary32 shadow -- exactly the
        # Q.astype(float32) the reference's coarse gemm reads (kernels.py:192)
        # -- so Step 3 streams half the bytes through the staged kernel
        self.Q32 = None
        if self.q_dtype == torch.float64 and self.compute == F32 and dc.coarse_shadow:
            self.Q32 = D.zeros_cm(self.n_local, m, torch.float32, dev)
        self.Sd = D.zeros_cm(k, m, torch.float64, dev)
        self.Pd = D.zeros_cm(k, m, torch.float64, dev)
        self.Rd = D.zeros_cm(m, m, torch.float64, dev)
        wmax = max(cfg.partition.block_widths())
        self._scr = _Scratch(k, m, wmax, dev)
        self._tmp64 = None
        self.blocks_done = 0
        self.cols_done = 0
        self.per_block_ortho = []
        self.per_block_resid = []
        self.pending_P = None
        self._next_P = None  # (key of the next block, its sketch) from a fused pass
        self._deferred = None  # (status, info) per block when checks are deferred
        # one-shot sweeps: the Step-5 scaling of the previous block, deferred
        # into the next projection (rb_project_trsm): (slot, R_S) or None
        self._fuse_scaling = False
        self._prepass_bufs = None
        self._prepass_flip = 0
        self._pending_scale = None
        self._lookahead_event = None  # upload event of the lookahead block (pinned host W)
        self._pending = []  # this block's partials (norms, l2 Gram) not yet allreduced
        self._g_given = None  # l2 stage: Q'^T Q' reduced with the block's sketches

    # -- small utilities ---------------------------------------------------
    # the reference's public state (rbgs.py:343-347) as numpy-compatible
    # views of the device tensors Qd / Sd / Pd / Rd (kernels.DevArray)
    @property
    def Q(self):
        return DevArray(self.Qd)

    @property
    def S(self):
        return DevArray(self.Sd)

    @property
    def P(self):
        return DevArray(self.Pd)

    @property
    def R(self):
        return DevArray(self.Rd)

    def _sketch(self, X, out):
        sketching.sketch_into(self.theta, X, out, self.row0, gauss=self._gmode if self.theta.kind == "gaussian" else None)

    def _sketch_reduce(self, X, out):
        self._sketch(X, out)
        self._reduce(out)

    def _reduce(self, *tensors):
        """Allreduce of this block's sketch partials, with the block's other
        pending partials -- the norms (rbgs.py:373-374, projection epilogue),
        the l2 stage's tall Gram -- riding along: one collective per block
        (PAPER.md:200)."""
        pend = self._pending
        self._pending = []
        self.comm.allreduce_(*tensors, *pend)

    def _flush_norms(self):
        if self._pending:
            self._reduce()

    def _as_block(self, W_i, w):
        """Device view of this rank's rows of block W_i (dtype kept: binary32
        blocks are read as binary32, binary64 as binary64)."""
        if isinstance(W_i, Matrix):
            W_i = W_i._dev if W_i._dev is not None else W_i.data
        if isinstance(W_i, torch.Tensor):
            t = W_i if W_i.dim() == 2 else W_i.reshape(-1, 1)
            if t.dtype not in (torch.float32, torch.float64):
                t = t.to(torch.float64)
            t = D.to_cm(t, t.dtype, self.device)
        else:
            A = np.asarray(W_i)
            if A.dtype not in (np.float32, np.float64):
                A = A.astype(np.float64)
            if A.ndim == 1:
                A = A.reshape(-1, 1)
            t = D.to_cm(torch.from_numpy(np.asfortranarray(A)), None, self.device)
        if t.shape != (self.n_local, w):
            raise ShapeError(f"block {self.blocks_done + 1} has shape {tuple(t.shape)}, "
                             f"expected {(self.n_local, w)}")
        return t

    def _tmp(self, w):
        if self._tmp64 is None or self._tmp64.shape[1] < w:
            self._tmp64 = D.empty_cm(self.n_local, w, torch.float64, self.device)
        return self._tmp64[:, :w]

    # -- Step 2 ------------------------------------------------------------
    def _solve_ls(self, S, Pi, X):
        name, param = self.solver
        scr = self._scr
        if self.fine32:
            _solve_ls_f32(name, param, S, self.offsets, Pi, X, scr)
            return
        if name == "richardson":
            _richardson_dev(S, Pi, param, X, scr.T[:, :Pi.shape[1]])
        elif name == "bmgs_reorth":
            _bmgs_dev(S, self.offsets, Pi, param, X, scr.T[:, :Pi.shape[1]])
        elif name == "cg_normal":
            _cg_dev(S, Pi, param, X)
        else:
            _householder_direct_dev(S, Pi, X, scr)

    # -- Steps 4-5 -----------------------------------------------------------
    def _interblock(self, Qp, Pi, slot, block1, sp_given=None):
        """Writes Q_i into `slot`; returns (R_ii, S_i, Sp_of_Qp or None).
        `sp_given`: Theta Q' already computed (fused pass) -- used for the
        first sketch instead of recomputing it."""
        name, param = self.inter
        scr = self._scr
        w = Qp.shape[1]
        k = self.theta.k
        Sp = scr.Sp[:, :w]
        reuse = block1  # sketch(W_1) is P_1 bit for bit (same kernel, same data)
        if name == "rgs_single":
            return self._interblock_rgs(Qp, slot)
        if name == "sketched_cholqr":
            l = param or 1
            Rt = scr.Rt[:w, :w]
            Qcur = Qp
            RS = scr.R1[:w, :w]
            for it in range(l):
                if it == 0 and reuse:
                    Sp.copy_(Pi)
                elif it == 0 and sp_given is not None:
                    Sp = sp_given
                else:
                    self._sketch_reduce(Qcur, Sp)
                if it == 0:
                    sp_qp = Sp.clone() if self.cfg.certify_blocks else None
                # G = Sp^T Sp, R_S = chol(G), Ss = Sp R_S^{-1}: one launch
                D.sketched_cholqr_small(Sp, RS, scr.Ss[:, :w], scr.info[it % 4:it % 4 + 1])
                last = it == l - 1
                # resketch sketches the binary64 Q_i before it is rounded to
                # the slot's format (rbgs.py:286-287 sketches fp64 Q)
                out = slot if (last and not self.cfg.resketch) else self._tmp(w)
                if not last and Qcur.data_ptr() == out.data_ptr():
                    out = D.empty_cm(self.n_local, w, torch.float64, self.device)
                if (last and l == 1 and self._fuse_scaling and out.data_ptr() == Qcur.data_ptr()
                        and self.cols_done + w < self.Qd.shape[1]):
                    # in-place scaling of this block: done by the next block's
                    # projection (rb_project_trsm), which alone reads it next
                    self._pending_scale = (out, RS)
                else:
                    D.trsm_right(Qcur, RS, out)
                if it == 0:  # R_total = R_S I
                    Rt.copy_(RS)
                else:
                    Rn = scr.R2[:w, :w]
                    D.gemm(0, 0, 1.0, RS, Rt, 0.0, Rn)
                    Rt.copy_(Rn)
                Qcur = out
            if self.cfg.resketch:
                Si = scr.Si[:, :w]
                self._sketch_reduce(Qcur, Si)
                D.convert(Qcur, slot)
            else:
                Si = scr.Ss[:, :w]  # the last pass's Sp R_S^{-1}
            return Rt, Si, sp_qp
        # l2_plus_cholqr -- Gram realisation of the l2 stage:
        # R' = chol(Q'^T Q'), S* = (Theta Q') R'^{-1} = Theta Q*, then the
        # sketched CholQR of Q*: R'' = chol(S*^T S*), R_ii = R'' R',
        # Q_i = Q' R_ii^{-1}, S_i = S* R''^{-1}.
        G = scr.G[:w, :w]
        if self._g_given is not None:  # reduced with the block's sketches
            Sp.copy_(Pi if reuse else sp_given)
        else:
            D.cross(Qp, Qp, G)
            if reuse or sp_given is not None:
                Sp.copy_(Pi if reuse else sp_given)
                self._reduce(G)
            else:
                self._sketch(Qp, Sp)
                self._reduce(G, Sp)
        sp_qp = Sp.clone() if self.cfg.certify_blocks else None
        # No host branch (deferrable, graph-capturable): both outcomes of the
        # Gram stage run on the device and rb_l2_select keeps one.
        #  (A) R' = chol(Q'^T Q'), S* = Sp R'^{-1}, R'' = chol(S*^T S*),
        #      R_ii = R'' R', S_i = S* R''^{-1}
        #      If the Gram Cholesky broke down (cond(Q') > ~1e8) R' is replaced
        #      by the Householder R of Q' (rb_tsqr_r: binary64 TSQR, the
        #      reference's own l2 stage, kernels.py:216-231) -- launched
        #      unconditionally, a no-op unless the status word is set.
        #      (Row-sharded runs keep (B): the tall QR would need its own
        #      collective.)
        #  (B) last resort (A still failed / sharded): the one-pass sketched
        #      CholQR of Q' -- the same R_ii in exact arithmetic.
        info = scr.info
        R1 = scr.R1[:w, :w]
        D.potrf(G, R1, info[8:9])
        if not self.comm.active and TSQR_FALLBACK:
            D.tsqr_r(Qp, R1, info[8:9], cond=info[8:9])
        Ss = scr.Ss[:, :w]
        D.trsm_right(Sp, R1, Ss)
        R2 = scr.R2[:w, :w]
        Sa = scr.T[:, :w]
        D.sketched_cholqr_small(Ss, R2, Sa, info[9:10])
        Ra = scr.G[:w, :w]  # (G is consumed)
        D.gemm(0, 0, 1.0, R2, R1, 0.0, Ra)
        Rb = scr.Rb[:w, :w]
        Sb = scr.Sb[:, :w]
        D.sketched_cholqr_small(Sp, Rb, Sb, info[10:11])
        Rt = scr.Rt[:w, :w]
        Si = scr.Si[:, :w]
        D.l2_select(info[8:9], info[9:10], info[10:11], Ra, Sa, Rb, Sb, Rt, Si, info[1:2])
        if self.cfg.resketch:
            q64 = self._tmp(w)
            D.trsm_right(Qp, Rt, q64)
            self._sketch_reduce(q64, Si)
            D.convert(q64, slot)
        else:
            D.trsm_right(Qp, Rt, slot)
        return Rt, Si, sp_qp

    def _interblock_rgs(self, Qp, slot):
        """Column-wise randomized Gram-Schmidt (rbgs.py:232-264), fp64 block."""
        scr = self._scr
        dev = self.device
        w = Qp.shape[1]
        k = self.theta.k
        Qi = self._tmp(w)
        D.convert(Qp, Qi)
        Rb = scr.Rt[:w, :w]
        Rb.zero_()
        Sb = scr.Si[:, :w]
        pv = D.empty_cm(k, 1, torch.float64, dev)
        s2 = D.empty_cm(k, 1, torch.float64, dev)
        nrm = torch.zeros(w + 1, dtype=torch.float64, device=dev)
        D.sumsq(Qp, nrm[w:w + 1])
        self._reduce(nrm[w:w + 1])
        sp_qp = None
        if self.cfg.certify_blocks:
            sp_qp = D.empty_cm(k, w, torch.float64, dev)
            self._sketch_reduce(Qp, sp_qp)
        for t in range(w):
            v = Qi[:, t:t + 1]
            self._sketch_reduce(v, pv)
            if t:
                A = D.empty_cm(k, t, torch.float64, dev)
                A.copy_(Sb[:, :t])
                rf = D.empty_cm(t, t, torch.float64, dev)
                D.geqrf(A, rf)
                y = D.empty_cm(t, 1, torch.float64, dev)
                D.gemm(1, 0, 1.0, A, pv, 0.0, y)
                D.trsm_left_upper(rf, y, scr.info[7:8])
                Rb[:t, t:t + 1].copy_(y)
                D.project(Qi[:, :t], y, v, v, F64, ORDER_REFERENCE)
            self._sketch_reduce(v, s2)
            rtt = nrm[t:t + 1]
            D.sumsq(s2, rtt)
            rtt.sqrt_()
            Rb[t, t:t + 1].copy_(rtt)
            rr = rtt.reshape(1, 1)
            D.trsm_right(v, rr, v)
            D.trsm_right(s2, rr, Sb[:, t:t + 1])
        D.convert(Qi, slot)
        self._rgs_norms = nrm
        return Rb, Sb, sp_qp

    # -- one block -------------------------------------------------------------
    def push_block(self, W_i, lookahead=None) -> tuple:
        """One RBGS iteration on block W_i (rbgs.py:352-399); returns (j0, j1).

        `lookahead` (optional, device-path extension): the NEXT block, when
        the caller already has it (one-shot `rbgs`).  Its Step-1 sketch is
        then computed in the same pass over the gaussian table as this
        block's Step-4 sketch of Q' (one table read and, when sharded, one
        allreduce per block instead of two); the next push_block of that
        same tensor reuses it."""
        self.pending_P = None
        i = self.blocks_done + 1
        if self.blocks_done >= len(self.offsets) - 1:
            raise ShapeError(f"all {len(self.offsets) - 1} blocks already pushed")
        j0, j1 = self.offsets[self.blocks_done], self.offsets[self.blocks_done + 1]
        w = j1 - j0
        with torch.cuda.device(self.device):
            Wn = None
            if lookahead is not None and self.blocks_done + 2 < len(self.offsets):
                wn = self.offsets[self.blocks_done + 2] - j1
                Wn = self._as_block(lookahead, wn)
            return self._push(i, j0, j1, w, self._as_block(W_i, w), Wn)

    @staticmethod
    def _key(t):
        return (t.data_ptr(), tuple(t.shape), t.stride(), t.dtype)

    def _fusable(self, A, B):
        """Two sketches can share one table pass (gaussian kind, tensor pipe)."""
        return (self.theta.kind == "gaussian" and self.inter[0] in ("sketched_cholqr", "l2_plus_cholqr")
                and not self.cfg.certify_blocks and A.dtype == torch.float32 and B.dtype == torch.float32
                and A.shape[1] <= 64 and B.shape[1] <= 64 and sketching.GAUSS_MODE != "fp64")

    def _sketch_pair(self, A, B, outA, outB, pre=None):
        tab = self.theta.device_tables(A.device, self.row0, A.shape[0])
        pre2 = None
        if pre is not None:  # B's pre-pass ran on the side stream (_fork_prepass)
            pre2, ev = pre
            torch.cuda.current_stream(self.device).wait_event(ev)
        D.sketch_gaussian2(A, B, tab["theta"], tab["ldt"], self.theta.k,
                           sketching.gauss_scale(self.theta), outA, outB,
                           False, self._gmode, pre2=pre2)
        self._reduce(outA, outB)

    def _fork_prepass(self, slot, Wn):
        """The digit pre-pass of W_(i+1) (chunk exponents + planes: two small
        streaming kernels that depend on nothing block i computes) on the
        side stream while this stream runs block i's projection, for the
        paired sketch [Q'_i | W_(i+1)] that follows it.  Returns (buffer,
        event) or None when the paired tensor form will not be taken."""
        if not (PREPASS_OVERLAP and self._fusable(slot, Wn) and slot.shape[1] + Wn.shape[1] > 64
                and self._gmode.split("+")[0] in ("auto", "tensor", "tensor4", "tensor3") and Wn.shape[0] >= 1):
            return None
        dev = self.device
        nb = D.gauss_prepass_bytes(Wn.shape[0], Wn.shape[1], slot.shape[1], self._gmode)
        bufs = self._prepass_bufs
        if bufs is None or bufs[0].numel() < nb:
            bufs = self._prepass_bufs = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
            self._prepass_flip = 0
        buf = bufs[self._prepass_flip]
        self._prepass_flip ^= 1
        cur = torch.cuda.current_stream(dev)
        side = _SIDE_STREAMS.get(dev.index)
        if side is None:
            side = _SIDE_STREAMS[dev.index] = torch.cuda.Stream(dev, priority=-1)
        side.wait_stream(cur)
        ev = self._lookahead_event
        self._lookahead_event = None
        with torch.cuda.stream(side):
            if ev is not None:
                side.wait_event(ev)  # W_(i+1)'s upload (pinned / staged host W)
            D.gauss_prepass(Wn, slot.shape[1], self._gmode, buf)
            done = torch.cuda.Event()
            done.record(side)
        return buf, done

    # -- sketch / projection overlap -------------------------------------------
    def _overlap_ok(self, Wn):
        """The next block's W sketch can run beside this block's projection:
        gaussian kind on the tensor pipe, <= 40 columns (the lean sketch CTA
        and one staged-projection CTA share an SM), binary32 Q."""
        return (OVERLAP and self._fusable(Wn, Wn) and Wn.shape[1] <= 40 and self.q_dtype == torch.float32
                and self.compute == F32 and self.order == ORDER_REFERENCE)

    def _fork_next_sketch(self, Wn, Pn):
        """Sketch W_(i+1) into Pn on a high-priority side stream (lean CTAs,
        tensor pipe) while the current stream runs this block's projection
        (FP32 pipe); returns the event the consumer waits for."""
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        side = _SIDE_STREAMS.get(dev.index)
        if side is None:  # one per device, shared by every sweep (and its workspace)
            side = _SIDE_STREAMS[dev.index] = torch.cuda.Stream(dev, priority=-1)
        side.wait_stream(cur)
        ev = self._lookahead_event
        self._lookahead_event = None
        tab = self.theta.device_tables(dev, self.row0, Wn.shape[0])
        with torch.cuda.stream(side):
            if ev is not None:
                side.wait_event(ev)
            D.sketch_gaussian(Wn, tab["theta"], tab["ldt"], self.theta.k,
                              sketching.gauss_scale(self.theta), Pn, False, "lean")
            done = torch.cuda.Event()
            done.record(side)
        return done

    def _push(self, i, j0, j1, w, W, Wn=None):
        scr = self._scr
        cfg = self.cfg
        c = self.cols_done
        norms = scr.norms
        norms.zero_()
        scr.info.zero_()
        sharded = self.comm.active
        if not c:
            # Q' = W_1 itself (rbgs.py:371-372): ||W_1|| = ||Q'_1||, read in its
            # own format; sharded, the partial rides Step 1's allreduce
            D.sumsq(W, norms[0:1])
            norms[1:2].copy_(norms[0:1])
            if sharded:
                self._pending.append(norms[0:2])
                if self.inter[0] == "l2_plus_cholqr" and not cfg.certify_blocks:
                    # the l2 stage's W_1^T W_1 rides Step 1's allreduce too
                    self._g_given = scr.G[:w, :w]
                    D.cross(W, W, self._g_given)
                    self._pending.append(self._g_given)
        # Step 1 (possibly already done by the previous block's fused pass)
        nxt = self._next_P
        self._next_P = None
        if nxt is not None and nxt[0] == self._key(W):
            Pi = nxt[1]
        else:
            Pi = scr.Pi[:, :w]
            if Wn is not None and c == 0 and self._fusable(W, Wn):
                Pn = scr.Pn[scr.pn_flip][:, :Wn.shape[1]]
                scr.pn_flip ^= 1
                self._wait_lookahead()
                self._sketch_pair(W, Wn, Pi, Pn)
                self._next_P = (self._key(Wn), Pn)
                Wn = None
            elif Wn is not None and c == 0 and sharded and not cfg.certify_blocks:
                # row-sharded, any kind: Step 1 of blocks 1 and 2 (and the
                # norms of W_1) in one allreduce
                Pn = scr.Pn[scr.pn_flip][:, :Wn.shape[1]]
                scr.pn_flip ^= 1
                self._wait_lookahead()
                self._sketch(W, Pi)
                self._sketch(Wn, Pn)
                self._reduce(Pi, Pn)
                self._next_P = (self._key(Wn), Pn)
                Wn = None
            else:
                self._sketch_reduce(W, Pi)
        Pu = Pi  # as sketched (the inter-block step re-sketches Q' unrounded)
        if self.fine32:
            D.convert(Pi, scr.P32[:, :w])
            Pi = scr.Pr[:, :w]
            D.convert(scr.P32[:, :w], Pi)
        slot = self.Qd[:, j0:j1]
        sp_given = None
        if c:
            self._g_given = None
        fork = None
        pre = None
        if c and Wn is not None and self._next_P is None and not self._overlap_ok(Wn):
            pre = self._fork_prepass(slot, Wn)
        if c and Wn is not None and self._next_P is None and self._overlap_ok(Wn):
            # the next block's Step 1 does not depend on this block: issue it
            # first, on the side stream, so it overlaps the projection
            Pn = scr.Pn[scr.pn_flip][:, :Wn.shape[1]]
            scr.pn_flip ^= 1
            fork = (self._fork_next_sketch(Wn, Pn), Pn)
        if c:
            X = scr.X[:c, :w]
            self._solve_ls(self.Sd[:, :c], Pi, X)
            self.Rd[:c, j0:j1].copy_(X)
            if self.Q32 is not None:
                # Q' in binary32 into the (not yet committed) shadow slot,
                # then widened exactly into the binary64 slot
                D.project(self.Q32[:, :c], X, W, self.Q32[:, j0:j1], self.compute, self.order, norms[0:2])
                D.convert(self.Q32[:, j0:j1], slot)
            elif self._pending_scale is not None:
                Qf, RSf = self._pending_scale
                self._pending_scale = None
                D.project_trsm(self.Qd[:, :c], X, W, slot, self.compute, self.order, norms[0:2], Qf, RSf)
            else:
                D.project(self.Qd[:, :c], X, W, slot, self.compute, self.order, norms[0:2])
            if sharded:
                # the norm partials join the block's next allreduce
                self._pending.append(norms[0:2])
            if fork is not None:
                # Step 4's sketch of Q' on this stream, then join the side
                # stream's Step 1 of the next block; one allreduce for both
                sp_given = scr.Sp[:, :w]
                self._sketch(slot, sp_given)
                torch.cuda.current_stream(self.device).wait_event(fork[0])
                self._reduce(sp_given, fork[1])
                self._next_P = (self._key(Wn), fork[1])
            elif Wn is not None and self._next_P is None and self._fusable(slot, Wn):
                sp_given = scr.Sp[:, :w]
                Pn = scr.Pn[scr.pn_flip][:, :Wn.shape[1]]
                scr.pn_flip ^= 1
                self._wait_lookahead()
                self._sketch_pair(slot, Wn, sp_given, Pn, pre=pre)
                self._next_P = (self._key(Wn), Pn)
            elif (Wn is not None and self._next_P is None and sharded and not cfg.certify_blocks
                  and self.inter[0] in ("sketched_cholqr", "l2_plus_cholqr")):
                # row-sharded, any sketch kind: Step 4's sketch of Q'_i, Step 1
                # of block i+1, the norms (and the l2 stage's tall Gram) in
                # ONE allreduce (one synchronization per block)
                sp_given = scr.Sp[:, :w]
                Pn = scr.Pn[scr.pn_flip][:, :Wn.shape[1]]
                scr.pn_flip ^= 1
                self._wait_lookahead()
                self._sketch(slot, sp_given)
                self._sketch(Wn, Pn)
                if self.inter[0] == "l2_plus_cholqr":
                    self._g_given = scr.G[:w, :w]
                    D.cross(slot, slot, self._g_given)
                self._reduce(sp_given, Pn, self._g_given)
                self._next_P = (self._key(Wn), Pn)
            Qp = slot
        else:
            Qp = W
        Rii, Si, sp_qp = self._interblock(Qp, Pu, slot, block1=(c == 0), sp_given=sp_given)
        self._flush_norms()
        # finiteness of everything the block produced (Matrix() checks)
        if Pi.dtype == torch.float64 and Si.dtype == torch.float64 and Rii.dtype == torch.float64:
            D.sumsq3(Pi, Si, Rii, norms[2:5])
        else:
            D.sumsq(Pi, norms[2:3])
            D.sumsq(Si, norms[3:4])
            D.sumsq(Rii, norms[4:5])
        if self._deferred is not None:
            # one-shot rbgs(): record this block's status words on the device
            # and carry on without a host round trip; rbgs() checks every
            # block once at the end (and replays eagerly on a failure)
            self._deferred[0][i - 1].copy_(norms)
            self._deferred[1][i - 1].copy_(scr.info)
            self._commit_block(j0, j1, Pi, Si, Rii)
            return j0, j1
        scr.status_host.copy_(norms, non_blocking=True)
        scr.info_host.copy_(scr.info, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        self._check_status(i, scr.status_host.numpy(), scr.info_host.numpy(), Pi, slot, c, w)
        if cfg.certify_blocks:
            if sp_qp is None:
                sp_qp = D.empty_cm(self.theta.k, w, torch.float64, self.device)
                self._sketch_reduce(Qp, sp_qp)
        self._commit_block(j0, j1, Pi, Si, Rii)
        if cfg.certify_blocks:
            self._certify_block(Si, Rii, sp_qp)
        return j0, j1

    def _wait_lookahead(self):
        """The stream waits for the upload of the lookahead block (pinned
        host W in one-shot rbgs()) only where that block is first read."""
        ev = self._lookahead_event
        self._lookahead_event = None
        if ev is not None:
            torch.cuda.current_stream(self.device).wait_event(ev)

    def _flush_scaling(self):
        if self._pending_scale is not None:
            Qf, RSf = self._pending_scale
            self._pending_scale = None
            D.trsm_right(Qf, RSf, Qf)

    def _commit_block(self, j0, j1, Pi, Si, Rii):
        if self.Q32 is not None:
            D.convert(self.Qd[:, j0:j1], self.Q32[:, j0:j1])
        self.Sd[:, j0:j1].copy_(Si)
        self.Pd[:, j0:j1].copy_(Pi)
        self.Rd[j0:j1, j0:j1].copy_(Rii)
        self.blocks_done += 1
        self.cols_done = j1

    def _check_status(self, i, st, info, Pi, slot, c, w):
        """The reference's per-block failure tests (rbgs.py:373-399 and the
        Matrix() finiteness checks) on the block's status words."""
        w_norm = math.sqrt(st[0]) if st[0] >= 0 else float("nan")
        q_norm = math.sqrt(st[1]) if st[1] >= 0 else float("nan")
        if not (np.isfinite(st[0]) and np.isfinite(st[1]) and np.isfinite(st[2])):
            raise ValueError("Matrix entries must be finite")
        if q_norm <= self.n * U_FINE * w_norm:
            self.pending_P = Matrix(Pi.clone())
            if c:
                slot.zero_()
            raise DependentBlockError(i, "projected block vanished")
        if self.inter[0] == "rgs_single":
            self._check_rgs(i, q_norm, w)
        for col in info[:4]:
            if col:
                if c:
                    slot.zero_()
                raise InterblockError(i, str(NotPositiveDefiniteError(int(col)))) from \
                    NotPositiveDefiniteError(int(col))
        if not (np.isfinite(st[3]) and np.isfinite(st[4])):
            raise ValueError("Matrix entries must be finite")

    def _defer_status(self):
        """Switch to deferred status checks (one-shot rbgs() only, variants
        without data-dependent host branches)."""
        B = len(self.offsets) - 1
        self._deferred = (torch.zeros(B, 8, dtype=torch.float64, device=self.device),
                          torch.zeros(B, 16, dtype=torch.int32, device=self.device))

    def _deferred_ok(self) -> bool:
        """One host read of every block's status words; True when no block
        would have raised in the eager sweep."""
        st_all = self._deferred[0].cpu().numpy()
        info_all = self._deferred[1].cpu().numpy()
        for b in range(self.blocks_done):
            st, info = st_all[b], info_all[b]
            if not np.all(np.isfinite(st[:5])) or np.any(info[:4]):
                return False
            if math.sqrt(st[1]) <= self.n * U_FINE * math.sqrt(st[0]):
                return False
        return True

    def _check_rgs(self, i, q_norm, w):
        r = self._rgs_norms[:w].cpu().numpy()
        thr = self.n * U_FINE * q_norm
        for t in range(w):
            if not r[t] > thr:
                # rbgs.py:258-260 raised inside interblock_rgs, re-raised by the sweep (rbgs.py:381)
                inner = DependentBlockError(t + 1, f"sketched norm {r[t]:.3e} below dependence threshold")
                raise DependentBlockError(i, f"dependent column: {inner}") from inner

    def _certify_block(self, Si, Rii, Sp):
        w = Si.shape[1]
        dev = self.device
        G = D.empty_cm(w, w, torch.float64, dev)
        D.gemm(1, 0, 1.0, Si, Si, 0.0, G)
        T = D.empty_cm(Sp.shape[0], w, torch.float64, dev)
        T.copy_(Sp)
        D.gemm(0, 0, -1.0, Si, Rii, 1.0, T)
        out = torch.zeros(3, dtype=torch.float64, device=dev)
        D.sumsq(G, out[0:1], minus_identity=True)
        D.sumsq(T, out[1:2])
        D.sumsq(Sp, out[2:3])
        o = out.cpu().numpy()
        self.per_block_ortho.append(float(math.sqrt(o[0])))
        self.per_block_resid.append(float(math.sqrt(o[1]) / math.sqrt(o[2])))

    def finish(self) -> BlockQR:
        c = self.cols_done
        with torch.cuda.device(self.device):
            cert0 = certify(self.Sd[:, :c], self.Pd[:, :c], self.Rd[:c, :c])
        cert = CertReport(cert0.delta, cert0.delta_tilde, tuple(self.per_block_ortho),
                          tuple(self.per_block_resid))
        return BlockQR(Matrix(self.Qd, precision=self.cfg.coarse), Matrix(self.Rd), Matrix(self.Sd),
                       Matrix(self.Pd), self.cfg.partition, cert)


REPLAYS = 0  # one-shot factorizations replayed eagerly after a deferred-status failure
# next-block sketch overlapped with the projection on a side stream
# (RB_OVERLAP=1).  Off by default: measured on B200 (tools/overlap_probe.py,
# profiles/r02_overlap_probe.json) the two kernels do co-reside, but the
# projection's LDS traffic and the sketch's UMMA operand reads share each
# SM's shared-memory bandwidth, and the pair takes as long as the two in
# series (2.89 vs 2.77 ms at C2's last block); the default is the fused
# two-input sketch after the projection (one table pass).
OVERLAP = os.environ.get("RB_OVERLAP", "0") == "1"
# W_(i+1)'s digit pre-pass on a side stream beside the projection: built, bitwise neutral, measured without
# gain at C2 (54.3 / 54.8 ms off, 54.4 / 54.1 ms on: the staged projection fills every SM's shared memory, so
# the side kernels run in its tail) -- off by default
PREPASS_OVERLAP = os.environ.get("RB_PREPASS_OVERLAP", "0") == "1"
TSQR_FALLBACK = os.environ.get("RB_L2_TSQR", "1") == "1"  # Householder R when the l2 Gram breaks down
_SIDE_STREAMS = {}


def _deferrable(cfg) -> bool:
    """Inter-block variants whose block step has no data-dependent host
    branch (RGS reads its column norms; the l2 stage selects its fallback on
    the device), and no per-block certificate read."""
    return parse_method(cfg.interblock)[0] in ("sketched_cholqr", "l2_plus_cholqr") and not cfg.certify_blocks


_STAGE_POOL = {}  # (device index, rows, cols, dtype) -> pinned staging slots, reused across calls
_STAGE_SLOTS = 3
# host copy threads (measured on the 16-core GPU box, C2: 2 -> 12.7, 4 -> 23.3, 8 -> 31.1, 12 -> 23.7 GB/s e2e)
_STAGE_THREADS = int(os.environ.get("RB_STAGE_THREADS", str(max(1, min(8, len(os.sched_getaffinity(0)) // 2)))))
_STAGE_MAX_BLOCK_BYTES = 1 << 30


class _StagedUpload:
    """Block-by-block upload of a PAGEABLE host W (a numpy array, the
    reference-style input): a background thread copies block b into a pinned
    staging slot with a few host threads (numpy releases the GIL in its copy
    loops), enqueues the H2D copy on the copy stream and records its event,
    while the main thread is already factoring earlier blocks -- so the host
    copy, the PCIe transfer and the factorization overlap like the pinned
    path.  Indexing [b] blocks until block b's transfer has been enqueued and
    returns its CUDA event (what _sweep_blocks waits on)."""

    def __init__(self, Wh, Wd, off, dev, copy_stream):
        import threading
        from concurrent.futures import ThreadPoolExecutor

        self.Wh, self.Wd, self.off, self.dev, self.copy_stream = Wh, Wd, off, dev, copy_stream
        self.nb = len(off) - 1
        rows = Wd.shape[0]
        wmax = max(off[b + 1] - off[b] for b in range(self.nb))
        key = (dev.index, rows, wmax, Wd.dtype)
        slots = _STAGE_POOL.get(key)
        if slots is None:
            slots = [torch.empty((wmax, rows), dtype=Wd.dtype).pin_memory().t() for _ in range(_STAGE_SLOTS)]
            _STAGE_POOL.clear()  # one shape at a time: pinned memory is not free
            _STAGE_POOL[key] = slots
        self.slots = slots
        self.events = [torch.cuda.Event() for _ in range(self.nb)]
        self.ready = [threading.Event() for _ in range(self.nb)]
        self.error = None
        self.pool = ThreadPoolExecutor(max_workers=max(1, _STAGE_THREADS))
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        try:
            torch.cuda.set_device(self.dev)
            rows = self.Wd.shape[0]
            nt = max(1, _STAGE_THREADS)
            step = -(-rows // nt)
            for b in range(self.nb):
                j0, j1 = self.off[b], self.off[b + 1]
                slot = self.slots[b % _STAGE_SLOTS]
                if b >= _STAGE_SLOTS:
                    self.events[b - _STAGE_SLOTS].synchronize()  # the slot's previous transfer has left it
                dst = slot.numpy()

                def chunk(r0, r1, j0=j0, j1=j1, dst=dst):
                    dst[r0:r1, :j1 - j0] = self.Wh[r0:r1, j0:j1]

                futs = [self.pool.submit(chunk, r0, min(rows, r0 + step)) for r0 in range(0, rows, step)]
                for f in futs:
                    f.result()
                with torch.cuda.stream(self.copy_stream):
                    self.Wd[:, j0:j1].copy_(slot[:, :j1 - j0], non_blocking=True)
                    self.events[b].record(self.copy_stream)
                self.ready[b].set()
        except BaseException as exc:  # noqa: BLE001 -- re-raised in the consumer
            self.error = exc
        finally:
            for r in self.ready:
                r.set()
            self.pool.shutdown(wait=False)

    def __len__(self):
        return self.nb

    def __getitem__(self, b):
        self.ready[b].wait()
        if self.error is not None:
            raise self.error
        return self.events[b]

    def __iter__(self):
        return (self[b] for b in range(self.nb))


def _stageable(W, cfg):
    """A pageable 2-D host array big enough for the staged upload to pay."""
    if isinstance(W, torch.Tensor):
        if W.is_cuda or W.is_pinned() or W.dim() != 2 or W.dtype not in (torch.float32, torch.float64):
            return None
        A = W.numpy()
    else:
        A = np.asarray(W)
        if A.ndim != 2 or A.dtype not in (np.float32, np.float64):
            return None
    if os.environ.get("RB_STAGED_UPLOAD", "1") != "1" or A.nbytes < (64 << 20):
        return None
    if cfg.partition.total_cols != A.shape[1]:
        return None
    wmax = max(cfg.partition.block_widths())
    if A.shape[0] * wmax * A.itemsize > _STAGE_MAX_BLOCK_BYTES:
        return None
    return A


def _sweep_blocks(Wd, n, theta, cfg, dc, q_storage, deferred, events=None):
    """The block loop of rbgs() (rbgs.py:417-421) on a device W."""
    dev = Wd.device
    sweep = RbgsSweep(n, theta, cfg, dc, _q_storage=q_storage)
    if deferred:
        sweep._defer_status()
        # nothing observes a block's Q_i before the next projection: fuse
        # the scaling into it (binary32 Q only; rb_project_trsm checks the
        # rest and falls back to the separate kernels)
        sweep._fuse_scaling = (sweep.q_dtype == torch.float32 and sweep.compute == F32
                               and os.environ.get("RB_FUSE_SCALING", "1") != "0")
    off = cfg.partition.offsets()
    for b in range(cfg.partition.num_blocks):
        nxt = Wd[:, off[b + 1]:off[b + 2]] if b + 2 < len(off) else None
        if events is not None:
            # block b needs W_b now; W_(b+1) only for the fused sketch at the
            # end of block b (waited for there), so the projection of block b
            # overlaps the upload of W_(b+1)
            torch.cuda.current_stream(dev).wait_event(events[b])
            sweep._lookahead_event = events[b + 1] if nxt is not None else None
        sweep.push_block(Wd[:, off[b]:off[b + 1]], lookahead=nxt)
    sweep._flush_scaling()
    return sweep


class RbgsPlan:
    """One-shot factorization of a FIXED device W, captured once as a CUDA
    graph and replayed (device-path extension, no reference counterpart --
    SURVEY.md 8(e): with the per-block stream time down to ~0.5 ms at 8
    GPUs, launch latency and the host's launch rate bound the sweep).

    W must be a column-major CUDA tensor; its CONTENTS may change between
    replays, its storage may not.  The capture runs after one eager
    factorization (tables, workspaces and library handles are created
    outside the capture).  Each replay is the complete factorization --
    every kernel of every block -- followed by the one host read of the
    deferred block statuses and the final certification; if a block
    failed, the factorization is re-run eagerly so the exception is the
    reference's.  The returned BlockQR ALIASES the plan's buffers: the next
    replay overwrites it (copy what must survive)."""

    def __init__(self, W, theta, cfg: RbgsConfig, device_cfg: DeviceConfig = None):
        require_cuda()
        dc = device_cfg or DeviceConfig()
        if not (isinstance(W, torch.Tensor) and W.is_cuda and W.dim() == 2 and D.is_cm(W)
                and W.dtype in (torch.float32, torch.float64)):
            raise ShapeError("RbgsPlan needs W as a column-major binary32/binary64 CUDA tensor")
        if not _deferrable(cfg):
            raise ValueError("RbgsPlan needs a sketched_cholqr / l2_plus_cholqr inter-block variant without "
                             "certify_blocks")
        if dc.overwrite_w:
            raise ValueError("RbgsPlan cannot overwrite its own input")
        if cfg.partition.total_cols != W.shape[1]:
            raise ShapeError(f"partition covers {cfg.partition.total_cols} cols, W has {W.shape[1]}")
        self.W, self.theta, self.cfg, self.dc = W, theta, cfg, dc
        self.n = theta.n if dc.shard is not None else W.shape[0]
        dev = W.device
        with torch.cuda.device(dev):
            rbgs(W, theta, cfg, dc)  # warm-up outside the capture
            torch.cuda.synchronize(dev)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self._sweep = _sweep_blocks(W, self.n, theta, cfg, dc, None, True)
            torch.cuda.synchronize(dev)

    def replay(self) -> BlockQR:
        """Run the captured factorization on the current contents of W."""
        self.graph.replay()
        if not self._sweep._deferred_ok():
            global REPLAYS
            REPLAYS += 1
            return rbgs(self.W, self.theta, self.cfg, self.dc, _eager=True)
        return self._sweep.finish()


def rbgs(W, theta, cfg: RbgsConfig, device_cfg: DeviceConfig = None, *, _eager: bool = False) -> BlockQR:
    """Factor W = QR with Q orthonormal in the sketched inner product
    (rbgs.py:410-421).  W: numpy / Matrix (uploaded once; binary32 arrays
    stay binary32) or a CUDA tensor (used in place); with a sharded
    DeviceConfig, W holds this rank's rows."""
    require_cuda()
    W_in = W
    dc = device_cfg or DeviceConfig()
    dev = D.cuda_device(dc.device)
    if isinstance(W, Matrix):
        W = W._dev if W._dev is not None else W.data
    events = None
    if isinstance(W, torch.Tensor) and not W.is_cuda and W.is_pinned() and W.dim() == 2 and D.is_cm(W) \
            and W.dtype in (torch.float32, torch.float64):
        # pinned column-major host W: upload block by block on a side stream,
        # so block b's transfer overlaps the factorization of earlier blocks
        Wd = D.empty_cm(W.shape[0], W.shape[1], W.dtype, dev)
        off = cfg.partition.offsets()
        copy_stream = torch.cuda.Stream(dev)
        copy_stream.wait_stream(torch.cuda.current_stream(dev))
        # the uploads write Wd on copy_stream: the caching allocator must not
        # hand its memory to the current stream while they may be in flight
        # (e.g. after a block raises before the later uploads completed)
        Wd.record_stream(copy_stream)
        events = []
        with torch.cuda.stream(copy_stream):
            for b in range(cfg.partition.num_blocks):
                Wd[:, off[b]:off[b + 1]].copy_(W[:, off[b]:off[b + 1]], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                events.append(ev)
    elif _stageable(W, cfg) is not None:
        # pageable host W (numpy): staged block-by-block upload (see _StagedUpload)
        A = _stageable(W, cfg)
        Wd = D.empty_cm(A.shape[0], A.shape[1], torch.float32 if A.dtype == np.float32 else torch.float64, dev)
        copy_stream = torch.cuda.Stream(dev)
        copy_stream.wait_stream(torch.cuda.current_stream(dev))
        Wd.record_stream(copy_stream)
        events = _StagedUpload(A, Wd, cfg.partition.offsets(), dev, copy_stream)
    elif isinstance(W, torch.Tensor):
        Wd = D.to_cm(W, W.dtype if W.dtype in (torch.float32, torch.float64) else torch.float64, dev)
    else:
        A = np.asarray(W)
        if A.dtype not in (np.float32, np.float64):
            A = A.astype(np.float64)
        if A.ndim != 2:
            raise ShapeError(f"expected a 2-D array, got ndim={A.ndim}")
        Wd = D.to_cm(torch.from_numpy(np.asfortranarray(A)), None, dev)
    n_rows, m = Wd.shape
    if cfg.partition.total_cols != m:
        raise ShapeError(f"partition covers {cfg.partition.total_cols} cols, W has {m}")
    n = theta.n if dc.shard is not None else n_rows
    # Q over W's storage: always for the private upload of a pinned host W
    # (the slot of block i is written only after W_i has been consumed),
    # on request (overwrite_w) for a caller's device W
    q_storage = None
    qd = dc.q_dtype or (torch.float32 if cfg.coarse.format == "coarse" else torch.float64)
    if dc.overwrite_w or events is not None:
        if Wd.dtype == qd and Wd.is_cuda and D.is_cm(Wd):
            q_storage = Wd
        elif dc.overwrite_w:
            raise ShapeError("overwrite_w needs W as a column-major CUDA tensor of Q's dtype")
    destroys_input = (q_storage is not None and isinstance(W_in, torch.Tensor) and W_in.is_cuda
                      and Wd.data_ptr() == W_in.data_ptr())
    # Per-block host round trips are only needed to raise at the failing
    # block; the one-shot driver defers them to one read at the end and, if
    # any block failed, replays the factorization eagerly so the exception
    # (type, message, block index) is exactly the reference's.
    deferred = (not _eager and not destroys_input and _deferrable(cfg)
                and os.environ.get("RB_EAGER_STATUS", "0") != "1")
    try:
        sweep = _sweep_blocks(Wd, n, theta, cfg, dc, q_storage, deferred, events)
    except BaseException:
        if events is not None:
            # a block raised: no stream reads the remaining uploads, so
            # order them before anything that may reuse Wd's memory
            cur = torch.cuda.current_stream(dev)
            for ev in events:
                cur.wait_event(ev)
        raise
    if deferred and not sweep._deferred_ok():
        global REPLAYS
        REPLAYS += 1
        del sweep
        return rbgs(W_in, theta, cfg, device_cfg, _eager=True)
    return sweep.finish()


def certify(S, P, R, device=None) -> CertReport:
    """Delta = ||I - S^T S||_F, Delta~ = ||P - S R||_F / ||P||_F on the GPU
    (rbgs.py:428-443); k-dimensional data only."""
    require_cuda()
    dev = D.cuda_device(device if device is not None else
                        (S.device if isinstance(S, torch.Tensor) and S.is_cuda else None))
    with torch.cuda.device(dev):
        Sd, Pd, Rd = _dev_f64(S, dev), _dev_f64(P, dev), _dev_f64(R, dev)
        k, m = Sd.shape
        out = torch.zeros(3, dtype=torch.float64, device=dev)
        if m:
            D.certify_sums(Sd, Pd, Rd, out)
        else:
            D.sumsq(Pd, out[2:3])
        o = out.cpu().numpy()
    if not np.all(np.isfinite(o)):
        raise ValueError("Matrix entries must be finite")
    if o[2] == 0.0:
        raise CertificationError("certification undefined for a zero sketch P")
    return CertReport(float(math.sqrt(o[0])), float(math.sqrt(o[1]) / math.sqrt(o[2])))


# ---------------------------------------------------------------------------
# standalone Step-2 / Step-4-5 entry points (reference signatures)
# ---------------------------------------------------------------------------

def _ls_entry(fn, S, Pi, param, prec, device=None, name=None, offsets=None):
    dev = D.cuda_device(device)
    with torch.cuda.device(dev):
        Sd, Pd = _dev_f64(S, dev), _dev_f64(Pi, dev)
        X = D.empty_cm(Sd.shape[1], Pd.shape[1], torch.float64, dev)
        if prec.format != "fine":  # binary32 solve (prec.dtype = float32)
            class _S:
                info = torch.zeros(8, dtype=torch.int32, device=dev)
            _solve_ls_f32(name, param, Sd, offsets, Pd, X, _S())
        else:
            fn(Sd, Pd, param, X)
        return Matrix(X)


def ls_richardson(S, Pi, l: int, prec: PrecisionSpec = FINE) -> Matrix:
    def f(Sd, Pd, l, X):
        T = D.empty_cm(Sd.shape[0], Pd.shape[1], torch.float64, Sd.device)
        _richardson_dev(Sd, Pd, l, X, T)
    return _ls_entry(f, S, Pi, l, prec, name="richardson")


def ls_bmgs_reorth(S_blocks, Pi, l: int, prec: PrecisionSpec = FINE) -> Matrix:
    blocks = [as_array(B) if not isinstance(B, torch.Tensor) else B for B in S_blocks]
    widths = [B.shape[1] for B in blocks]
    off = [0]
    for w in widths:
        off.append(off[-1] + w)
    S = np.hstack([as_array(B) for B in blocks]) if blocks else np.zeros((as_array(Pi).shape[0], 0))

    def f(Sd, Pd, l, X):
        T = D.empty_cm(Sd.shape[0], Pd.shape[1], torch.float64, Sd.device)
        _bmgs_dev(Sd, off, Pd, l, X, T)
    return _ls_entry(f, S, Pi, l, prec, name="bmgs_reorth", offsets=off)


def ls_cg_normal(S, Pi, iters: int, prec: PrecisionSpec = FINE) -> Matrix:
    return _ls_entry(lambda Sd, Pd, it, X: _cg_dev(Sd, Pd, it, X), S, Pi, iters, prec, name="cg_normal")


def ls_householder_direct(S, Pi, prec: PrecisionSpec = FINE) -> Matrix:
    class _S:
        info = None

    def f(Sd, Pd, _, X):
        scr = _S()
        scr.info = torch.zeros(8, dtype=torch.int32, device=Sd.device)
        _householder_direct_dev(Sd, Pd, X, scr)
    return _ls_entry(f, S, Pi, None, prec, name="householder_direct")


def _standalone_interblock(Qprime, theta, cfg):
    W = Qprime
    if isinstance(W, Matrix):
        W = W._dev if W._dev is not None else W.data
    A = W if isinstance(W, torch.Tensor) else torch.from_numpy(np.asfortranarray(as_array(W)))
    n, w = A.shape
    if w > theta.k:
        raise ShapeError(f"block width {w} exceeds sketch size {theta.k}")
    sw = RbgsSweep(n, theta, RbgsConfig(partition=BlockPartition(w, 1, w), coarse=FINE, **cfg))
    try:
        sw.push_block(A.to(torch.float64) if isinstance(A, torch.Tensor) else A)
    except InterblockError as e:
        cause = e.__cause__
        raise (cause if cause is not None else e)
    except DependentBlockError as e:
        cause = e.__cause__
        raise (cause if cause is not None else e)
    return Matrix(sw.Qd), Matrix(sw.Rd), Matrix(sw.Sd)


def interblock_sketched_cholqr(Qprime, theta, l: int = 1, resketch: bool = False):
    """Sketched Cholesky QR of one block, l passes (rbgs.py:267-290)."""
    return _standalone_interblock(Qprime, theta, dict(interblock=f"sketched_cholqr({l})", resketch=resketch))


def interblock_l2_cholqr(Qprime, theta, resketch: bool = False):
    """l2 stage then one sketched CholQR pass (rbgs.py:293-302)."""
    return _standalone_interblock(Qprime, theta, dict(interblock="l2_plus_cholqr", resketch=resketch))


def interblock_rgs(Qprime, theta):
    """Column-wise randomized Gram-Schmidt (rbgs.py:232-264)."""
    return _standalone_interblock(Qprime, theta, dict(interblock="rgs_single"))


# ---------------------------------------------------------------------------
# post-processing, embedding certificate, serialization (rbgs.py:446-552;
# device implementations in post.py)
# ---------------------------------------------------------------------------

from .post import (  # noqa: E402
    certify_embedding,
    cholesky_qr_postprocess,
    load_blockqr,
    load_blockqr_binary,
    save_blockqr,
    save_blockqr_binary,
)
