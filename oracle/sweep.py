"""RBGS sweep restated on the CPU (test infrastructure only).

Follows `pkg/src/sketch_krylov/rbgs.py` (Algorithm 2 of the paper,
PAPER.md:184-192) step by step; every function names the reference lines it
restates.  Exceptions are raised as `OracleError` subclasses that carry the
same attributes as the reference ones (`block`, `column`, `index`).
"""

from __future__ import annotations

import re

import numpy as np
import scipy.linalg
from scipy.linalg import lapack

from . import sketches

U_COARSE = 2.0 ** -24
U_FINE = 2.0 ** -53
DTYPE = {"coarse": np.float32, "fine": np.float64}
UNIT = {"coarse": U_COARSE, "fine": U_FINE}


class OracleError(Exception):
    pass


class DependentBlock(OracleError):
    def __init__(self, block, detail=""):
        self.block = block
        super().__init__(f"block {block} numerically dependent: {detail}")


class Interblock(OracleError):
    def __init__(self, block, detail):
        self.block = block
        super().__init__(f"inter-block QR failed at block {block}: {detail}")


class NotPD(OracleError):
    def __init__(self, column):
        self.column = column
        super().__init__(f"not positive definite at column {column}")


class SingularTri(OracleError):
    def __init__(self, index):
        self.index = index
        super().__init__(f"zero diagonal entry at index {index}")


class RankDeficient(OracleError):
    pass


def parse_spec(spec: str):
    """'name', 'name(3)', 'name:3' -> (name, param)  (rbgs.py:64-82)."""
    defaults = {"richardson": 5, "bmgs_reorth": 1, "cg_normal": 20,
                "sketched_cholqr": 1}
    m = re.match(r"^([a-z0-9_]+)(?:[(:]\s*(\d+)\s*\)?)?$", spec.strip().lower())
    if not m:
        raise ValueError(spec)
    p = m.group(2)
    return m.group(1), int(p) if p is not None else defaults.get(m.group(1))


def _finite(A):
    """Emulates the `Matrix(...)` wrapper every reference routine returns
    through (kernels.py:91-99): finiteness check and Fortran layout (the
    layout matters for bit-identity, BLAS picks its kernel by it)."""
    if not np.all(np.isfinite(A)):
        raise ValueError("Matrix entries must be finite")
    return np.asfortranarray(A, dtype=np.float64)


# ---------------------------------------------------------------------------
# L1 primitives (kernels.py)
# ---------------------------------------------------------------------------

def gemm_ordered(alpha, A, B, beta=0.0, C=None, fmt="fine"):
    """fl(alpha A B + beta C), each elementary op rounded in `fmt`, inner index
    ascending, accumulator seeded with fl(beta C) (kernels.py:171-209)."""
    dt = DTYPE[fmt]
    A = np.asarray(A, dtype=np.float64).astype(dt)
    B = np.asarray(B, dtype=np.float64).astype(dt)
    n, m = A.shape[0], B.shape[1]
    if C is None or beta == 0.0:
        acc = np.zeros((n, m), dtype=dt, order="F")
    elif beta == 1.0:
        acc = np.array(np.asarray(C, dtype=np.float64).astype(dt), order="F")
    else:
        acc = np.array(dt(beta) * np.asarray(C, dtype=np.float64).astype(dt), order="F")
    a = dt(alpha)
    for l in range(A.shape[1]):
        t = A[:, l:l + 1] * B[l:l + 1, :]
        if alpha == -1.0:
            acc -= t
        elif alpha == 1.0:
            acc += t
        else:
            acc += a * t
    return _finite(acc.astype(np.float64))


# tests may route the binary32 Step 3 through the plain-C restatement of the
# same order (oracle/cproj, pinned bit-identical to gemm_ordered by
# tests/test_oracle_golden.py); the bench's CPU arms keep the numpy loop,
# which has the reference's own cost profile (a Python loop over l).
FAST_PROJECT = False


def project(Q, X, W, fmt="coarse"):
    """Step 3: Q' = W - Q X in reference order (rbgs.py:369-370)."""
    if FAST_PROJECT and fmt == "coarse" and np.asarray(W).shape[1] <= 64 and np.asarray(Q).shape[1] > 0:
        from . import cproj
        Q32 = np.asarray(Q, dtype=np.float64).astype(np.float32)
        W32 = np.asarray(W, dtype=np.float64).astype(np.float32)
        X32 = np.asarray(X, dtype=np.float64).astype(np.float32).astype(np.float64)
        return _finite(cproj.project_f32(Q32, X32, W32).astype(np.float64))
    return gemm_ordered(-1.0, Q, X, 1.0, W, fmt)


def householder_qr(A):
    """Economic QR with diag(R) >= 0 (kernels.py:216-231)."""
    A = np.asarray(A, dtype=np.float64)
    Q, R = scipy.linalg.qr(A, mode="economic")
    d = np.sign(np.diag(R))
    d[d == 0.0] = 1.0
    return _finite(Q * d), _finite(d[:, None] * R)


def cholesky_upper(G):
    """Upper R with R^T R = G via dpotrf (kernels.py:234-247)."""
    G = np.asarray(G, dtype=np.float64)
    if not np.allclose(G, G.T, rtol=0.0, atol=1e-10 * max(1.0, np.abs(G).max())):
        raise ValueError("cholesky input is not symmetric")
    R, info = lapack.dpotrf(G, lower=0, clean=1)
    if info > 0:
        raise NotPD(info)
    return _finite(R)


def trsm(R, B, side):
    """RX = B (left) or XR = B (right), R upper (kernels.py:250-270)."""
    R = np.asarray(R, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    if B.ndim == 1:
        B = B.reshape(-1, 1)
    d = np.abs(np.diag(R))
    if np.any(d == 0.0):
        raise SingularTri(int(np.argmin(d != 0.0)))
    if side == "left":
        return _finite(scipy.linalg.solve_triangular(R, B, lower=False))
    return _finite(scipy.linalg.solve_triangular(R, B.T, trans="T", lower=False).T)


def round_to(A, fmt):
    """_round_to (rbgs.py:134-137)."""
    return A.astype(np.float32).astype(np.float64) if fmt == "coarse" else A


# ---------------------------------------------------------------------------
# Step 2 solvers (rbgs.py:144-225)
# ---------------------------------------------------------------------------

def ls_richardson(S, P, l, fmt="fine"):
    dt = DTYPE[fmt]
    S = np.asarray(S, dtype=np.float64).astype(dt)
    P = np.asarray(P, dtype=np.float64).astype(dt)
    X = np.zeros((S.shape[1], P.shape[1]), dtype=dt)
    for _ in range(l):
        X = X + S.T @ (P - S @ X)
    return _finite(X.astype(np.float64))


def ls_bmgs_reorth(blocks, P, l, fmt="fine"):
    dt = DTYPE[fmt]
    Sb = [np.asarray(B, dtype=np.float64).astype(dt) for B in blocks]
    R = np.asarray(P, dtype=np.float64).astype(dt).copy()
    Xs = [np.zeros((B.shape[1], R.shape[1]), dtype=dt) for B in Sb]
    for _ in range(l):
        for j, B in enumerate(Sb):
            inc = B.T @ R
            Xs[j] += inc
            R -= B @ inc
    return _finite(np.vstack(Xs).astype(np.float64))


def ls_cg_normal(S, P, iters, fmt="fine"):
    dt = DTYPE[fmt]
    S = np.asarray(S, dtype=np.float64).astype(dt)
    P = np.asarray(P, dtype=np.float64).astype(dt)
    b = S.T @ P
    X = np.zeros_like(b)
    r = b.copy()
    d = r.copy()
    rs = np.sum(r * r, axis=0)
    for _ in range(iters):
        Ad = S.T @ (S @ d)
        dAd = np.sum(d * Ad, axis=0)
        alpha = np.where(dAd > 0, rs / np.where(dAd > 0, dAd, 1.0), 0.0).astype(dt)
        X += alpha * d
        r -= alpha * Ad
        rs2 = np.sum(r * r, axis=0)
        beta = np.where(rs > 0, rs2 / np.where(rs > 0, rs, 1.0), 0.0).astype(dt)
        rs = rs2
        d = r + beta * d
    return _finite(X.astype(np.float64))


def ls_householder_direct(S, P, fmt="fine"):
    dt = DTYPE[fmt]
    S = np.asarray(S, dtype=np.float64).astype(dt)
    P = np.asarray(P, dtype=np.float64).astype(dt)
    Qs, Rs = scipy.linalg.qr(S, mode="economic")
    d = np.abs(np.diag(Rs))
    if d.size and d.min() <= S.shape[0] * UNIT[fmt] * max(d.max(), 1e-300):
        raise RankDeficient("least-squares matrix numerically rank deficient")
    X = scipy.linalg.solve_triangular(Rs, Qs.T @ P, lower=False)
    return _finite(X.astype(np.float64))


def solve_ls(name, param, S, offsets, P, fmt):
    if name == "richardson":
        return ls_richardson(S, P, param, fmt)
    if name == "bmgs_reorth":
        blocks = [S[:, offsets[j]:offsets[j + 1]]
                  for j in range(len(offsets) - 1) if offsets[j] < S.shape[1]]
        return ls_bmgs_reorth(blocks, P, param, fmt)
    if name == "cg_normal":
        return ls_cg_normal(S, P, param, fmt)
    return ls_householder_direct(S, P, fmt)


# ---------------------------------------------------------------------------
# Steps 4-5: inter-block QR, always fp64 (rbgs.py:232-311)
# ---------------------------------------------------------------------------

def interblock_rgs(Qp, op):
    Qp = np.asarray(Qp, dtype=np.float64)
    n, w = Qp.shape
    Q = np.empty((n, w), order="F")
    S = np.empty((op.k, w), order="F")
    R = np.zeros((w, w), order="F")
    thr = n * U_FINE * np.linalg.norm(Qp, "fro")
    for t in range(w):
        v = Qp[:, t].copy()
        pv = sketches.apply(op, v.reshape(-1, 1))
        if t:
            qf, rf = scipy.linalg.qr(S[:, :t], mode="economic")
            y = scipy.linalg.solve_triangular(rf, qf.T @ pv, lower=False)
            R[:t, t] = y[:, 0]
            v -= Q[:, :t] @ y[:, 0]
        s2 = sketches.apply(op, v.reshape(-1, 1))[:, 0]
        rtt = float(np.linalg.norm(s2))
        if rtt <= thr:
            raise DependentBlock(t + 1, "sketched norm below dependence threshold")
        R[t, t] = rtt
        Q[:, t] = v / rtt
        S[:, t] = s2 / rtt
    return _finite(Q), _finite(R), _finite(S)


def interblock_sketched_cholqr(Qp, op, l=1, resketch=False):
    Q = np.array(Qp, dtype=np.float64)
    Rt = np.eye(Q.shape[1])
    for _ in range(max(l, 1)):
        Sp = sketches.apply(op, Q)
        RS = cholesky_upper(Sp.T @ Sp)
        Q = trsm(RS, Q, "right")
        Rt = RS @ Rt
    S = sketches.apply(op, Q) if resketch else trsm(RS, Sp, "right")
    return Q, _finite(Rt), S


def interblock_l2_cholqr(Qp, op, resketch=False):
    Qs, Rp = householder_qr(Qp)
    Q, R2, S = interblock_sketched_cholqr(Qs, op, 1, resketch)
    return Q, _finite(R2 @ Rp), S


def interblock(name, param, Qp, op, resketch):
    if name == "rgs_single":
        return interblock_rgs(Qp, op)
    if name == "sketched_cholqr":
        return interblock_sketched_cholqr(Qp, op, param or 1, resketch)
    return interblock_l2_cholqr(Qp, op, resketch)


# ---------------------------------------------------------------------------
# the sweep (rbgs.py:318-421)
# ---------------------------------------------------------------------------

def widths_offsets(widths):
    off = [0]
    for w in widths:
        off.append(off[-1] + int(w))
    return tuple(off)


class OracleConfig:
    def __init__(self, widths, ls_solver="richardson(5)", interblock="l2_plus_cholqr",
                 coarse="coarse", fine="fine", certify_blocks=False, resketch=False):
        self.widths = tuple(int(w) for w in widths)
        self.ls_solver, self.interblock = ls_solver, interblock
        self.coarse, self.fine = coarse, fine
        self.certify_blocks, self.resketch = certify_blocks, resketch


def uniform_widths(m, mp):
    nb = -(-m // mp)
    return tuple([mp] * (nb - 1) + [m - mp * (nb - 1)])


class OracleSweep:
    def __init__(self, n, op, cfg: OracleConfig):
        m = sum(cfg.widths)
        if not (m <= op.k <= n):
            raise ValueError("need m <= k <= n")
        self.n, self.op, self.cfg = n, op, cfg
        self.solver = parse_spec(cfg.ls_solver)
        self.inter = parse_spec(cfg.interblock)
        self.offsets = widths_offsets(cfg.widths)
        self.Q = np.zeros((n, m), order="F")
        self.S = np.zeros((op.k, m), order="F")
        self.P = np.zeros((op.k, m), order="F")
        self.R = np.zeros((m, m), order="F")
        self.blocks_done = 0
        self.cols_done = 0
        self.per_block_ortho = []
        self.per_block_resid = []
        self.pending_P = None

    def push_block(self, Wi):
        Wi = np.asarray(Wi, dtype=np.float64)
        if Wi.ndim == 1:
            Wi = Wi.reshape(-1, 1)
        self.pending_P = None
        i = self.blocks_done + 1
        j0, j1 = self.offsets[self.blocks_done], self.offsets[self.blocks_done + 1]
        if Wi.shape != (self.n, j1 - j0):
            raise ValueError("block shape")
        cfg = self.cfg
        Pi = round_to(sketches.apply(self.op, Wi), cfg.fine)
        if self.cols_done:
            c = self.cols_done
            X = solve_ls(self.solver[0], self.solver[1], self.S[:, :c],
                         self.offsets, Pi, cfg.fine)
            self.R[:c, j0:j1] = X
            Qp = project(self.Q[:, :c], X, Wi, cfg.coarse)
        else:
            Qp = Wi.copy()
        if np.linalg.norm(Qp, "fro") <= self.n * U_FINE * np.linalg.norm(Wi, "fro"):
            self.pending_P = Pi
            raise DependentBlock(i, "projected block vanished")
        try:
            Qi, Rii, Si = interblock(self.inter[0], self.inter[1], Qp, self.op,
                                     cfg.resketch)
        except DependentBlock as e:
            raise DependentBlock(i, f"dependent column: {e}") from e
        except (RankDeficient, NotPD, SingularTri) as e:
            raise Interblock(i, str(e)) from e
        self.Q[:, j0:j1] = Qi
        self.S[:, j0:j1] = Si
        self.P[:, j0:j1] = Pi
        self.R[j0:j1, j0:j1] = Rii
        if cfg.certify_blocks:
            Sp = sketches.apply(self.op, Qp)
            w = j1 - j0
            self.per_block_ortho.append(float(np.linalg.norm(np.eye(w) - Si.T @ Si, "fro")))
            self.per_block_resid.append(float(np.linalg.norm(Sp - Si @ Rii, "fro")
                                              / np.linalg.norm(Sp, "fro")))
        self.blocks_done += 1
        self.cols_done = j1
        return j0, j1

    def finish(self):
        c = self.cols_done
        return certify(self.S[:, :c], self.P[:, :c], self.R[:c, :c])


def certify(S, P, R):
    """Delta = ||I - S^T S||_F, Delta~ = ||P - S R||_F / ||P||_F (rbgs.py:428-443)."""
    pn = np.linalg.norm(P, "fro")
    if pn == 0.0:
        raise OracleError("certification undefined for a zero sketch P")
    m = S.shape[1]
    return (float(np.linalg.norm(np.eye(m) - S.T @ S, "fro")),
            float(np.linalg.norm(P - S @ R, "fro") / pn))


def rbgs(W, op, cfg: OracleConfig):
    """One-shot sweep (rbgs.py:410-421); returns (sweep, (delta, delta_tilde))."""
    W = np.asarray(W, dtype=np.float64)
    sw = OracleSweep(W.shape[0], op, cfg)
    off = sw.offsets
    for b in range(len(cfg.widths)):
        sw.push_block(W[:, off[b]:off[b + 1]])
    return sw, sw.finish()
