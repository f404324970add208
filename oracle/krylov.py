"""Block Arnoldi / GMRES on the RBGS sweep, restated (test infrastructure only).

Restates `pkg/src/sketch_krylov/krylov.py:98-281`.  The operator is any
callable X -> A X on 2-D fp64 blocks.
"""

from __future__ import annotations

import numpy as np

from . import sweep as sw


def arnoldi(apply_A, B, op, p, cfg_kw=None, matvec_fmt="fine"):
    """rbgs_arnoldi (krylov.py:110-135): returns (sweep, H, R_first, cert)."""
    B = np.asarray(B, dtype=np.float64)
    n, mp = B.shape
    cfg = sw.OracleConfig((mp,) * p, **(cfg_kw or {}))
    s = sw.OracleSweep(n, op, cfg)
    s.push_block(B)
    off = s.offsets
    for i in range(2, p + 1):
        s.push_block(sw.round_to(apply_A(s.Q[:, off[i - 2]:off[i - 1]]), matvec_fmt))
    cert = s.finish()
    return s, s.R[:, mp:], s.R[:, :mp], cert


def _cond2(A):
    sv = np.linalg.svd(A, compute_uv=False)
    if sv.size == 0 or sv[-1] == 0.0:
        return float("inf")
    return float(sv[0] / sv[-1])


def _ls_qr(M, T):
    Qm, Rm = sw.householder_qr(M)
    return sw.trsm(Rm, Qm.T @ T, "left")


def gmres(apply_A, B, op, p, restarts=1, cfg_kw=None, tol=0.0, matvec_fmt="fine"):
    """block_gmres (krylov.py:170-281), RBGS backend only.

    Returns dict(solution, residual_history, basis_cond_history, restarts,
    breakdown, cert_history)."""
    B = np.asarray(B, dtype=np.float64)
    n, mp = B.shape
    bn = np.linalg.norm(B, axis=0)
    bn[bn == 0.0] = 1.0
    X = np.zeros_like(B)
    hist, conds, certs = [], [], []
    it = 0
    breakdown = 0
    cycles = 0

    def rel(Xc):
        Rr = B - apply_A(Xc)
        return float(np.max(np.linalg.norm(Rr, axis=0) / bn))

    for cycle in range(max(restarts, 1)):
        cycles += 1
        Bres = B - apply_A(X) if cycle else B.copy()
        s = sw.OracleSweep(n, op, sw.OracleConfig((mp,) * p, **(cfg_kw or {})))
        bk = 0
        try:
            s.push_block(Bres)
            off = s.offsets
            for i in range(2, p + 1):
                s.push_block(sw.round_to(apply_A(s.Q[:, off[i - 2]:off[i - 1]]),
                                         matvec_fmt))
        except sw.DependentBlock as e:
            bk = e.block
        q, c = s.blocks_done, s.cols_done
        if q == 0:
            it += 1
            hist.append((it, rel(X)))
            conds.append(1.0)
            certs.append((np.nan, np.nan))
            breakdown = bk
            break
        cert = sw.certify(s.S[:, :c], s.P[:, :c], s.R[:c, :c])
        Hf = s.R[:c, mp:c]
        Rf = s.R[:c, :mp]
        best, rbest = None, None
        for j in range(1, q):
            rows = (j + 1) * mp
            Z = _ls_qr(Hf[:rows, :j * mp], Rf[:rows, :])
            U = s.Q[:, :j * mp] @ Z
            r = rel(X + U)
            it += 1
            hist.append((it, r))
            conds.append(_cond2(s.Q[:, :rows]))
            certs.append(cert)
            if rbest is None or r <= rbest:
                best, rbest = U, r
        if bk:
            PA = np.hstack([s.P[:, mp:c], s.pending_P])
            Z = _ls_qr(PA, s.P[:, :mp])
            U = s.Q[:, :c] @ Z
            r = rel(X + U)
            it += 1
            hist.append((it, r))
            conds.append(_cond2(s.Q[:, :c]))
            certs.append(cert)
            if rbest is None or r <= rbest:
                best, rbest = U, r
        if best is not None:
            X = X + best
        if bk:
            breakdown = bk
            break
        if tol > 0.0 and rbest is not None and rbest <= tol:
            break
    if not hist:
        hist.append((1, rel(X)))
        conds.append(1.0)
        certs.append((np.nan, np.nan))
    return dict(solution=X, residual_history=hist, basis_cond_history=conds,
                restarts=cycles, breakdown=breakdown, cert_history=certs)


def poisson3d_apply(nx, ny, nz):
    """7-point Dirichlet Laplacian on an nx*ny*nz grid, x fastest: the 3-D
    Kronecker sum of tridiag(-1, 2, -1) that `gen_laplacian` builds in 1-D/2-D
    (bench.py:214-233).  Returns X -> A X on (n, cols) fp64 blocks."""
    def f(X):
        X = np.asarray(X, dtype=np.float64)
        squeeze = X.ndim == 1
        if squeeze:
            X = X.reshape(-1, 1)
        c = X.shape[1]
        V = X.reshape(nz, ny, nx, c)
        Y = 6.0 * V
        Y[:, :, 1:] -= V[:, :, :-1]
        Y[:, :, :-1] -= V[:, :, 1:]
        Y[:, 1:] -= V[:, :-1]
        Y[:, :-1] -= V[:, 1:]
        Y[1:] -= V[:-1]
        Y[:-1] -= V[1:]
        Y = Y.reshape(-1, c)
        return Y[:, 0] if squeeze else Y
    return f
