"""Block randomized Arnoldi and GMRES on the GPU sweep -- drop-in for
`sketch_krylov.krylov.rbgs_arnoldi` / `block_gmres`
(reference `pkg/src/sketch_krylov/krylov.py:49-281`).

The operator products, the RBGS block steps, the n-dimensional basis
combinations U_j = Q Z and the true-residual / basis-conditioning
diagnostics all run on the device; the Hessenberg least-squares problems
(at most (p mp) x ((p-1) mp)) use the single-CTA Householder kernel.
Only the spectrum of the (rows x rows) basis Gram matrix used for the
`basis_cond_history` diagnostic is taken on the host (a <= 244 x 244
symmetric eigenproblem; the n-dimensional Gram itself is a device kernel).
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import require_cuda
from .comm import Comm, RowShard
from .errors import DependentBlockError, ShapeError
from .kernels import FINE, BlockPartition, Matrix, PrecisionSpec, as_array
from .operators import LinearOperator
from .rbgs import DeviceConfig, RbgsConfig, RbgsSweep, certify

__all__ = ["ArnoldiDecomposition", "KrylovSolveReport", "rbgs_arnoldi", "block_gmres"]


@dataclass(eq=False)
class ArnoldiDecomposition:
    """Basis Q, Hessenberg data H = R[:, mp:], R_first = R[:, :mp]
    (krylov.py:49-64)."""

    Q: Matrix
    H: Matrix
    R_first: Matrix
    S: Matrix
    P: Matrix
    cert: object
    partition: BlockPartition


@dataclass(eq=False)
class KrylovSolveReport:
    """Solution plus per-inner-iteration histories (krylov.py:67-95)."""

    solution: Matrix
    residual_history: list
    basis_cond_history: list
    restarts: int
    breakdown: int = 0
    cert_history: list = None

    def __post_init__(self):
        if not self.residual_history:
            raise ValueError("residual history must be non-empty")
        if len(self.residual_history) != len(self.basis_cond_history):
            raise ValueError("history lengths must agree")
        if self.cert_history is None:
            self.cert_history = [(np.nan, np.nan)] * len(self.residual_history)
        elif len(self.cert_history) != len(self.residual_history):
            raise ValueError("history lengths must agree")


def _partition(mp, p):
    return BlockPartition(mp, p, p * mp)


def _device_cfg(device_cfg, A):
    dc = device_cfg or DeviceConfig(q_dtype=torch.float64)
    if dc.q_dtype is None:
        dc = dataclasses.replace(dc, q_dtype=torch.float64)
    if dc.device is None and getattr(A, "device", None) is not None:
        dc = dataclasses.replace(dc, device=A.device)
    return dc


def _to_dev(B, device):
    if isinstance(B, Matrix):
        B = B._dev if B._dev is not None else B.data
    if isinstance(B, torch.Tensor):
        return D.to_cm(B if B.dim() == 2 else B.reshape(-1, 1), torch.float64, device)
    return D.to_cm(torch.from_numpy(np.asfortranarray(as_array(B))), torch.float64, device)


def _matvec(A, X, prec):
    Y = A._apply_dev(X, torch.float64)
    if prec.format == "coarse":  # _round_to (rbgs.py:134-137)
        Y = D.to_cm(Y, torch.float32)
    return Y


def rbgs_arnoldi(A: LinearOperator, B, theta, p: int, cfg: RbgsConfig = None,
                 matvec_precision: PrecisionSpec = FINE, device_cfg: DeviceConfig = None) -> ArnoldiDecomposition:
    """Block Arnoldi: W_1 = B, W_i = A Q_(i-1), orthogonalized by RBGS
    (krylov.py:110-135).  Q is kept in binary64 by default because the
    reference applies A to its binary64 Q."""
    require_cuda()
    dc = _device_cfg(device_cfg, A)
    dev = D.cuda_device(dc.device)
    with torch.cuda.device(dev):
        Bd = _to_dev(B, dev)
        n_local, mp = Bd.shape
        if p < 2:
            raise ShapeError("Arnoldi needs p >= 2 blocks")
        n = A.n
        cfg = dataclasses.replace(cfg or RbgsConfig(), partition=_partition(mp, p))
        sweep = RbgsSweep(n, theta, cfg, dc)
        sweep.push_block(Bd)
        off = sweep.offsets
        for i in range(2, p + 1):
            sweep.push_block(_matvec(A, sweep.Qd[:, off[i - 2]:off[i - 1]], matvec_precision))
        f = sweep.finish()
        R = sweep.Rd
        return ArnoldiDecomposition(f.Q, Matrix(R[:, mp:]), Matrix(R[:, :mp]), f.S, f.P, f.cert,
                                    cfg.partition)


def _ls_qr_dev(M, T):
    """min ||M Z - T||_F via Householder QR (krylov.py:164-167), device."""
    rows, q = M.shape
    A = D.empty_cm(rows, q, torch.float64, M.device)
    A.copy_(M)
    Rm = D.empty_cm(q, q, torch.float64, M.device)
    D.geqrf(A, Rm)
    Z = D.empty_cm(q, T.shape[1], torch.float64, M.device)
    D.gemm(1, 0, 1.0, A, T, 0.0, Z)
    info = torch.zeros(1, dtype=torch.int32, device=M.device)
    D.trsm_left_upper(Rm, Z, info)
    return Z


def _ls_nested_dev(Hf, Rf, q, mp):
    """Z_j = argmin ||H[:(j+1)mp, :j mp] Z - R_first[:(j+1)mp]|| for every
    j = 1 .. q-1 from ONE Householder QR of the widest block Hessenberg
    matrix (krylov.py:229-233 solves each j separately): column l of H is
    zero below row (l // mp + 2) mp, so the reflectors of the first j mp
    columns -- hence the thin Q and R of the truncated problem -- are the
    leading parts of the full factorization; Z_j = R[:j mp, :j mp]^{-1}
    (Q^T R_first)[:j mp]."""
    if q < 2:
        return []
    rows, w = q * mp, (q - 1) * mp
    A = D.empty_cm(rows, w, torch.float64, Hf.device)
    A.copy_(Hf[:rows, :w])
    Rm = D.empty_cm(w, w, torch.float64, Hf.device)
    D.geqrf(A, Rm)
    QtT = D.empty_cm(w, mp, torch.float64, Hf.device)
    D.gemm(1, 0, 1.0, A, Rf[:rows, :], 0.0, QtT)
    info = torch.zeros(1, dtype=torch.int32, device=Hf.device)
    out = []
    for j in range(1, q):
        Z = D.empty_cm(j * mp, mp, torch.float64, Hf.device)
        Z.copy_(QtT[:j * mp])
        D.trsm_left_upper(Rm[:j * mp, :j * mp], Z, info)
        out.append(Z)
    return out


def _cond2_dev(Q, comm):
    """2-norm condition of the (row-sharded) basis from its Gram matrix."""
    q = Q.shape[1]
    G = D.empty_cm(q, q, torch.float64, Q.device)
    D.cross(Q, Q, G)
    comm.allreduce_(G)
    ev = np.linalg.eigvalsh(G.cpu().numpy())
    if ev.size == 0 or ev[0] <= 0.0:
        return float("inf")
    return float(math.sqrt(ev[-1] / ev[0]))


def _sketched_history(A, X, Bd, bn, sweep, cands, Hf, Rf, mp, c, bk, comm, history, conds, certs, pair, it,
                      colsq):
    """diagnostics="sketched": histories from k-dimensional data; one
    n-dimensional correction and one true residual per cycle (the last
    candidate: the sketched residual is non-increasing in j)."""
    dev = Bd.device
    k = sweep.Sd.shape[0]
    # sketched residuals of the nested problems: ||R_first - H Z_j|| per column
    est = []
    for t, (w, Z, rows) in enumerate(cands):
        if bk and t == len(cands) - 1:
            # breakdown candidate (krylov.py:258-268): || P_1 - [P_2.. | pending] Z ||
            PA = D.empty_cm(k, c, torch.float64, dev)
            PA[:, :c - mp].copy_(sweep.Pd[:, mp:c])
            PA[:, c - mp:].copy_(sweep.pending_P.tensor)
            Rk = D.empty_cm(k, mp, torch.float64, dev)
            Rk.copy_(sweep.Pd[:, :mp])
            D.gemm(0, 0, -1.0, PA, Z, 1.0, Rk)
        else:
            Rk = D.empty_cm(rows, mp, torch.float64, dev)
            Rk.copy_(Rf[:rows])
            Hj = D.empty_cm(rows, w, torch.float64, dev)
            Hj.copy_(Hf[:rows, :w])
            D.gemm(0, 0, -1.0, Hj, Z, 1.0, Rk)
        est.append((Rk * Rk).sum(0).sqrt())
    rels = (torch.stack(est) / bn).amax(1).cpu().tolist()
    # cond(S[:, :rows]) brackets cond(Q[:, :rows]) (epsilon-embedding); one
    # k-dimensional Gram, leading principal blocks on the host
    rmax = max(r for _, _, r in cands)
    G = D.empty_cm(rmax, rmax, torch.float64, dev)
    Sc = D.empty_cm(k, rmax, torch.float64, dev)
    Sc.copy_(sweep.Sd[:, :rmax])
    D.gemm(1, 0, 1.0, Sc, Sc, 0.0, G)
    Gh = G.cpu().numpy()
    Gh = np.triu(Gh) + np.triu(Gh, 1).T
    # the last candidate in n dimensions, with its true residual
    w, Z, _ = cands[-1]
    U = D.empty_cm(Bd.shape[0], mp, torch.float64, dev)
    Zc = D.empty_cm(w, mp, torch.float64, dev)
    Zc.copy_(Z)
    D.gemm(0, 0, 1.0, sweep.Qd[:, :w], Zc, 0.0, U)
    Rr = Bd - A._apply_dev(D.to_cm(X + U), torch.float64)
    rels[-1] = float((colsq(Rr).sqrt() / bn).max())
    for t, (_, _, r) in enumerate(cands):
        it += 1
        history.append((it, rels[t]))
        ev = np.linalg.eigvalsh(Gh[:r, :r])
        conds.append(float("inf") if ev.size == 0 or ev[0] <= 0.0 else float(math.sqrt(ev[-1] / ev[0])))
        certs.append(pair)
    return U, rels[-1], it


def block_gmres(A: LinearOperator, B, theta, p: int, restarts: int = 1, cfg=None, tol: float = 0.0,
                matvec_precision: PrecisionSpec = FINE, device_cfg: DeviceConfig = None,
                diagnostics: str = "full") -> KrylovSolveReport:
    """Restarted block GMRES over a sketch-orthonormal basis (krylov.py:170-281).

    RBGS backend only (the reference's classical backend is a baseline,
    out of scope).  With a sharded DeviceConfig, B, the solution and every
    operator block hold this rank's rows; residual norms are global.

    diagnostics  "full" (default, the reference's histories, krylov.py:247-257:
                 per inner iterate one n-dimensional correction, one operator
                 apply for the true residual and the basis condition number);
                 "sketched": the inner-iterate histories come from k-dimensional
                 data only -- the residual of iterate j is the sketched one,
                 ||R_first - H Z_j|| column-wise (= ||Theta r_j|| up to the
                 certified orthonormality of S; eq. 4.4), the basis
                 condition that of S[:, :rows] (the epsilon-embedding bracket
                 of cond(Q)) -- and only the LAST iterate of a cycle is formed
                 in n dimensions, with ONE true residual; its history entry
                 is the true value."""
    if diagnostics not in ("full", "sketched"):
        raise ValueError(f"unknown diagnostics mode {diagnostics!r}")
    require_cuda()
    dc = _device_cfg(device_cfg, A)
    dev = D.cuda_device(dc.device)
    comm = dc.comm or Comm(None)
    with torch.cuda.device(dev):
        Bd = _to_dev(B, dev)
        n_local, mp = Bd.shape
        if p < 2:
            raise ShapeError("GMRES needs p >= 2 blocks")
        n = A.n
        part = _partition(mp, p)

        def colsq(M):
            s = (M * M).sum(0)
            comm.allreduce_(s)
            return s

        bn = colsq(Bd).sqrt()
        bn = torch.where(bn == 0.0, torch.ones_like(bn), bn)
        X = D.zeros_cm(n_local, mp, torch.float64, dev)
        history, conds, certs = [], [], []
        it = 0
        breakdown = 0
        cycles = 0

        def rel_residual(Xc):
            Rr = Bd - A._apply_dev(Xc, torch.float64)
            return float((colsq(Rr).sqrt() / bn).max())

        for cycle in range(max(restarts, 1)):
            cycles += 1
            Bres = D.to_cm(Bd - A._apply_dev(X, torch.float64)) if cycle else Bd.clone()
            sweep = RbgsSweep(n, theta, dataclasses.replace(cfg or RbgsConfig(), partition=part), dc)
            bk = 0
            try:
                sweep.push_block(Bres)
                off = sweep.offsets
                for i in range(2, p + 1):
                    sweep.push_block(_matvec(A, sweep.Qd[:, off[i - 2]:off[i - 1]], matvec_precision))
            except DependentBlockError as e:
                bk = e.block
            q, c = sweep.blocks_done, sweep.cols_done
            if q == 0:
                it += 1
                history.append((it, rel_residual(X)))
                conds.append(1.0)
                certs.append((np.nan, np.nan))
                breakdown = bk
                break
            rep = certify(sweep.Sd[:, :c], sweep.Pd[:, :c], sweep.Rd[:c, :c])
            pair = (rep.delta, rep.delta_tilde)
            Hf = sweep.Rd[:c, mp:c]
            Rf = sweep.Rd[:c, :mp]
            # Every inner iterate j = 1 .. q-1 (plus the breakdown candidate)
            # of krylov.py:229-262, evaluated in batches: the small LS
            # solves first, then ONE pass over the basis for all corrections
            # U_j = Q[:, :j mp] Z_j (a block upper-triangular right factor),
            # one operator apply per candidate for the true residual, and one
            # basis Gram for the cond(Q[:, :rows]) history -- one host read
            # for all of them.
            cands = []  # (width of Q used, Z, rows of the cond basis)
            for j, Z in enumerate(_ls_nested_dev(Hf, Rf, q, mp), start=1):
                cands.append((j * mp, Z, (j + 1) * mp))
            if bk:
                PA = D.empty_cm(theta.k, c - mp + mp, torch.float64, dev)
                PA[:, :c - mp].copy_(sweep.Pd[:, mp:c])
                PA[:, c - mp:].copy_(sweep.pending_P.tensor)
                cands.append((c, _ls_qr_dev(PA, sweep.Pd[:, :mp]), c))
            U_best, rel_best = None, None
            if cands and diagnostics == "sketched":
                U_best, rel_best, it = _sketched_history(A, X, Bd, bn, sweep, cands, Hf, Rf, mp, c, bk, comm,
                                                         history, conds, certs, pair, it, colsq)
            elif cands:
                wmax = max(w for w, _, _ in cands)
                Zb = D.zeros_cm(wmax, mp * len(cands), torch.float64, dev)
                for t, (w, Z, _) in enumerate(cands):
                    Zb[:w, t * mp:(t + 1) * mp].copy_(Z)
                U = D.empty_cm(n_local, mp * len(cands), torch.float64, dev)
                D.gemm(0, 0, 1.0, sweep.Qd[:, :wmax], Zb, 0.0, U)
                res2 = torch.empty(len(cands), mp, dtype=torch.float64, device=dev)
                for t in range(len(cands)):
                    Rr = Bd - A._apply_dev(D.to_cm(X + U[:, t * mp:(t + 1) * mp]), torch.float64)
                    res2[t] = (Rr * Rr).sum(0)
                comm.allreduce_(res2)
                rels = (res2.sqrt() / bn).amax(1).cpu().tolist()
                # ONE Gram of the widest basis (a single pass over Q): every
                # cond(Q[:, :rows]) is that of a leading principal block
                rmax = max(r for _, _, r in cands)
                G = D.empty_cm(rmax, rmax, torch.float64, dev)
                G.zero_()
                D.syrk(sweep.Qd[:, :rmax], G)  # upper triangle (tiles below the diagonal are skipped)
                comm.allreduce_(G)
                Gh = G.cpu().numpy()
                Gh = np.triu(Gh) + np.triu(Gh, 1).T
                for t, (w, Z, r) in enumerate(cands):
                    it += 1
                    history.append((it, rels[t]))
                    ev = np.linalg.eigvalsh(Gh[:r, :r])
                    conds.append(float("inf") if ev.size == 0 or ev[0] <= 0.0
                                 else float(math.sqrt(ev[-1] / ev[0])))
                    certs.append(pair)
                    if rel_best is None or rels[t] <= rel_best:
                        U_best, rel_best = U[:, t * mp:(t + 1) * mp], rels[t]
            if U_best is not None:
                X = D.to_cm(X + U_best)
            if bk:
                breakdown = bk
                break
            if tol > 0.0 and rel_best is not None and rel_best <= tol:
                break
        if not history:
            history.append((1, rel_residual(X)))
            conds.append(1.0)
            certs.append((np.nan, np.nan))
        return KrylovSolveReport(Matrix(X), history, conds, cycles, breakdown, certs)
