"""Typed wrappers of the C ABI over column-major torch tensors.

A device matrix is a 2-D torch tensor with stride (1, ld) -- column-major,
exactly the layout the kernels take.  `empty_cm` allocates one; slicing
columns keeps the layout.  Every wrapper enqueues on the current stream and
never synchronises.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import F32, F64, call, dtype_code, ptr, stream_handle


def empty_cm(rows, cols, dtype, device):
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def zeros_cm(rows, cols, dtype, device):
    return torch.zeros((cols, rows), dtype=dtype, device=device).t()


def to_cm(t, dtype=None, device=None):
    """Column-major device copy (or view when already suitable)."""
    dtype = dtype or t.dtype
    if t.dim() == 1:
        t = t.reshape(-1, 1)
    dev = cuda_device(device if device is not None else (t.device if t.is_cuda else None))
    if t.device == dev and t.dtype == dtype and is_cm(t):
        return t
    out = empty_cm(t.shape[0], t.shape[1], dtype, dev)
    out.copy_(t)
    return out


def cuda_device(device=None):
    """Normalise to torch.device('cuda', index)."""
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device) if not isinstance(device, torch.device) else device
    if isinstance(device, int):
        d = torch.device("cuda", device)
    if d.type != "cuda":
        raise ValueError(f"device {d} is not a CUDA device (no CPU fallback)")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


def is_cm(t):
    return t.dim() == 2 and (t.stride(0) == 1 or t.shape[0] <= 1) and \
        (t.shape[1] <= 1 or t.stride(1) >= max(t.shape[0], 1))


def ld(t):
    if not is_cm(t):
        raise ValueError(f"tensor of shape {tuple(t.shape)} strides {t.stride()} is not column-major")
    return max(t.stride(1) if t.shape[1] > 1 else t.shape[0], t.shape[0], 1)


def _ws(n, ncols, k, device):
    return _lib.ws_for(n, ncols, k, device)


# ---------------------------------------------------------------------------
# optional per-kernel timing (bench.py's roofline): CUDA events recorded on
# the launching stream around the hot entry points, with the algorithmic
# bytes / flops of each call.

class KernelTimer:
    def __init__(self):
        self.records = []  # (name, ev0, ev1, bytes, flops)

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for name, e0, e1, nb, nf in self.records:
            d = out.setdefault(name, dict(calls=0, ms=0.0, bytes=0.0, flops=0.0))
            d["calls"] += 1
            d["ms"] += e0.elapsed_time(e1)
            d["bytes"] += nb
            d["flops"] += nf
        return out


_TIMER = None


class timed_kernels:
    """Context manager enabling the KernelTimer."""

    def __enter__(self):
        global _TIMER
        _TIMER = KernelTimer()
        return _TIMER

    def __exit__(self, *a):
        global _TIMER
        _TIMER = None


def _t0():
    if _TIMER is None:
        return None
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def _t1(e0, name, nbytes, nflops=0.0):
    if e0 is None or _TIMER is None:
        return
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    _TIMER.records.append((name, e0, e1, float(nbytes), float(nflops)))


def st(device=None):
    return stream_handle(device)


# ---------------------------------------------------------------------------

def project(Q, X, W, Qp, compute, order, norms2=None):
    """Qp = W - Q X in reference order (K3); Q may have zero columns."""
    n, p = W.shape
    c = 0 if Q is None else Q.shape[1]
    ws, wsb = _ws(n, p, 64, W.device)
    e0 = _t0()
    call("rb_project", dtype_code(Qp), dtype_code(W), compute, order, n, c, p,
         ptr(Q) if c else None, ld(Q) if c else 1, ptr(X) if c else None, ld(X) if c else 1,
         ptr(W), ld(W), ptr(Qp), ld(Qp), ptr(norms2), ws, wsb, st(W.device))
    if e0 is not None:
        qs = Q.element_size() if c else 0
        _t1(e0, "project", n * (c * qs + p * W.element_size() + p * Qp.element_size()), 2.0 * n * c * p)


def project_trsm(Q, X, W, Qp, compute, order, norms2, Qf, Rf):
    """Qf <- Qf Rf^{-1} (the previous block's Step-5 scaling, in place; Qf
    must be the last columns of Q) fused in front of Qp = W - Q X."""
    n, p = W.shape
    c, pf = Q.shape[1], Qf.shape[1]
    ws, wsb = _ws(n, p, 64, W.device)
    e0 = _t0()
    call("rb_project_trsm", dtype_code(Qp), dtype_code(W), compute, order, n, c, p, ptr(Q), ld(Q), ptr(X), ld(X),
         ptr(W), ld(W), ptr(Qp), ld(Qp), ptr(norms2), ptr(Qf), ld(Qf), ptr(Rf), ld(Rf), pf, ws, wsb, st(W.device))
    if e0 is not None:
        qs = Q.element_size()
        _t1(e0, "project", n * (c * qs + p * W.element_size() + p * Qp.element_size() + 2 * pf * qs),
            2.0 * n * c * p)


GAUSS_MODE = {"auto": 0, "fp64": 1, "tensor": 2, "lean": 3, "tensor4": 4, "tensor3": 5}
# "+q8": the table of an 8-bit operator (lo plane zero): mode + 16
GAUSS_MODE.update({m + "+q8": c + 16 for m, c in list(GAUSS_MODE.items()) if m != "lean"})


def sketch_gaussian(X, theta, ldt, k, scale, out, accumulate=False, mode="auto"):
    n, cols = X.shape
    ws, wsb = _ws(n, cols, k, X.device)
    e0 = _t0()
    call("rb_sketch_gaussian", dtype_code(X), n, cols, ptr(X), ld(X), ptr(theta), ldt, k, scale,
         ptr(out), ld(out), int(accumulate), GAUSS_MODE[mode], ws, wsb, st(X.device))
    _t1(e0, "sketch_gaussian", n * (cols * X.element_size() + 2 * k), 2.0 * k * n * cols)


GAUSS_DIGITS = {"auto": 6, "tensor": 6, "tensor4": 4, "tensor3": 3}
GAUSS_DIGITS.update({m + "+q8": d for m, d in list(GAUSS_DIGITS.items())})


def gauss_prepass_bytes(n, c, c_partner, mode):
    from ._lib import require_cuda
    return int(require_cuda().rb_gauss_prepass_bytes(int(n), int(c), int(c_partner), GAUSS_DIGITS[mode]))


def gauss_prepass(X, c_partner, mode, buf):
    """Digit planes + chunk exponents of X (the second input of a later
    paired sketch_gaussian2 with a c_partner-column first input) into buf."""
    n, c = X.shape
    call("rb_gauss_prepass", dtype_code(X), ptr(X), ld(X), c, int(c_partner), n, GAUSS_DIGITS[mode], ptr(buf),
         buf.numel() * buf.element_size(), st(X.device))


def sketch_gaussian2(X1, X2, theta, ldt, k, scale, out1, out2, accumulate=False, mode="auto", pre2=None):
    """[out1 | out2] = Theta [X1 | X2] in one pass over the gaussian table;
    pre2: X2's pre-pass already done (gauss_prepass)."""
    n, c1 = X1.shape
    c2 = X2.shape[1]
    ws, wsb = _ws(n, c1 + c2, k, X1.device)
    e0 = _t0()
    if pre2 is not None:
        call("rb_sketch_gaussian2_pre", dtype_code(X1), ptr(X1), ld(X1), c1, dtype_code(X2), ptr(X2), ld(X2), c2, n,
             ptr(theta), ldt, k, scale, ptr(out1), ld(out1), ptr(out2), ld(out2), int(accumulate), GAUSS_MODE[mode],
             ptr(pre2), ws, wsb, st(X1.device))
    else:
        call("rb_sketch_gaussian2", dtype_code(X1), ptr(X1), ld(X1), c1, dtype_code(X2), ptr(X2), ld(X2), c2, n,
             ptr(theta), ldt, k, scale, ptr(out1), ld(out1), ptr(out2), ld(out2), int(accumulate), GAUSS_MODE[mode],
             ws, wsb, st(X1.device))
    _t1(e0, "sketch_gaussian", n * ((c1 + c2) * X1.element_size() + 2 * k), 2.0 * k * n * (c1 + c2))


def gaussian_fill(seed, k, row0, nrows, theta, ldt, bits=16):
    call("rb_gaussian_fill_bits", ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), k, row0, nrows, ptr(theta), ldt,
         int(bits), st(theta.device))


def sketch_srht(X, row0, n_pad, bits, sample, k, scale, out, accumulate=False):
    n, cols = X.shape
    ws, wsb = _ws(n, cols, k, X.device)
    e0 = _t0()
    call("rb_sketch_srht", dtype_code(X), n, cols, ptr(X), ld(X), row0, n_pad, ptr(bits), ptr(sample), k,
         scale, ptr(out), ld(out), int(accumulate), ws, wsb, st(X.device))
    _t1(e0, "sketch_srht", n * cols * X.element_size())


def sketch_sparse_sign(X, row0, seed, k, nnz, out, accumulate=False, table=None):
    """table: (offs, lists) from sparse_sign_table for THIS row range (the
    per-call path then streams X and the table; else rows are hashed)."""
    n, cols = X.shape
    ws, wsb = _ws(n, cols, k, X.device)
    e0 = _t0()
    if table is not None:
        offs, lists = table
        call("rb_sketch_sparse_sign_tab", dtype_code(X), n, cols, ptr(X), ld(X), ptr(offs), ptr(lists), k, nnz,
             ptr(out), ld(out), int(accumulate), ws, wsb, st(X.device))
    else:
        call("rb_sketch_sparse_sign", dtype_code(X), n, cols, ptr(X), ld(X), row0,
             ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), k, nnz, ptr(out), ld(out), int(accumulate), ws, wsb,
             st(X.device))
    _t1(e0, "sketch_sparse_sign", n * cols * X.element_size())


def sparse_sign_table(seed, k, nnz, row0, nrows, device):
    """Pre-bucketed sparse-sign table of rows row0 .. row0 + nrows - 1."""
    s = min(nnz, k)
    ntiles = -(-nrows // 1024)
    offs = torch.empty(max(ntiles, 1) * (k + 1), dtype=torch.int32, device=device)
    lists = torch.empty(max(ntiles, 1) * 1024 * s, dtype=torch.int16, device=device)
    call("rb_sparse_sign_table", ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), k, nnz, row0, nrows, ptr(offs),
         ptr(lists), st(device))
    return offs, lists


def sketch_signs(X, bits, ldb, k, scale, out, accumulate=False):
    n, cols = X.shape
    ws, wsb = _ws(n, cols, k, X.device)
    call("rb_sketch_signs", dtype_code(X), n, cols, ptr(X), ld(X), ptr(bits), ldb, k, scale, ptr(out),
         ld(out), int(accumulate), ws, wsb, st(X.device))


def trsm_right(B, R, out):
    """out = B R^{-1} (rows solved in fp64, rounded to out's dtype)."""
    n, p = B.shape
    e0 = _t0()
    call("rb_trsm_right", dtype_code(B), dtype_code(out), n, p, ptr(B), ld(B), ptr(R), ld(R), ptr(out),
         ld(out), st(B.device))
    _t1(e0, "trsm_right", n * p * (B.element_size() + out.element_size()), 1.0 * n * p * p)


def gemm(tA, tB, alpha, A, B, beta, C):
    m, n = C.shape
    k = A.shape[0] if tA else A.shape[1]
    ws, wsb = _ws(1, 1, 1, C.device)  # split-K partials: <= 2 x SMs x 128 x 64 doubles
    call("rb_gemm_f64", int(tA), int(tB), m, n, k, alpha, ptr(A), ld(A), ptr(B), ld(B), beta, ptr(C), ld(C),
         ws, wsb, st(C.device))


def gemm32(tA, tB, alpha, A, B, beta, C):
    """binary32 C = alpha op(A) B + beta C (own kernel, binary32 accumulation)."""
    m, n = C.shape
    k = A.shape[0] if tA else A.shape[1]
    ws, wsb = _ws(1, 1, 1, C.device)
    call("rb_gemm_f32", int(tA), int(tB), m, n, k, alpha, ptr(A), ld(A), ptr(B), ld(B), beta, ptr(C), ld(C),
         ws, wsb, st(C.device))


def syrk(A, C):
    """Upper triangle of C = A^T A (binary64; the full product is formed)."""
    k, n = A.shape
    ws, wsb = _ws(1, 1, 1, C.device)
    call("rb_syrk_f64", n, k, 1.0, ptr(A), ld(A), 0.0, ptr(C), ld(C), ws, wsb, st(C.device))


def cross(A, B, out, accumulate=False):
    """out = A^T B for tall A (n x p), B (n x q)."""
    n, p = A.shape
    q = B.shape[1]
    ws, wsb = _ws(n, max(p, q), max(p, q), A.device)
    call("rb_cross", dtype_code(A), dtype_code(B), n, p, q, ptr(A), ld(A), ptr(B), ld(B), ptr(out), ld(out),
         int(accumulate), ws, wsb, st(A.device))


def potrf(G, R, info):
    p = G.shape[0]
    call("rb_potrf_upper", p, ptr(G), ld(G), ptr(R), ld(R), ptr(info), st(G.device))


def tsqr_r(A, R, info, cond=None):
    """R <- the Householder-QR R factor of the tall A (TSQR, binary64); with
    `cond` (a device int) the call is a no-op unless cond != 0."""
    n, p = A.shape
    ws, wsb = _ws(n, p, 64, A.device)
    call("rb_tsqr_r", dtype_code(A), n, p, ptr(A), ld(A), ptr(R), ld(R), ptr(cond), ptr(info), ws, wsb, st(A.device))


def trsm_left_upper(R, B, info):
    m = R.shape[0]
    call("rb_trsm_left_upper", m, B.shape[1], ptr(R), ld(R), ptr(B), ld(B), ptr(info), st(R.device))


def geqrf(A, R):
    m, q = A.shape
    ws, wsb = _ws(m, q, m, A.device)
    call("rb_geqrf_small", m, q, ptr(A), ld(A), ptr(R), ld(R), ws, wsb, st(A.device))


def sumsq(A, out, minus_identity=False):
    m, n = A.shape
    ws, wsb = _ws(m, n, 64, A.device)
    call("rb_sumsq", dtype_code(A), m, n, ptr(A), ld(A), int(minus_identity), ptr(out), ws, wsb, st(A.device))


def sumsq3(A1, A2, A3, out):
    """out[0:3] = sums of squares of three binary64 matrices (one launch)."""
    args = []
    for A in (A1, A2, A3):
        args += [A.shape[0], A.shape[1], ptr(A), ld(A)]
    ws, wsb = _ws(1, 1, 1, out.device)
    call("rb_sumsq3", *args, ptr(out), ws, wsb, st(out.device))


def richardson(S, P, l, X, T):
    k, c = S.shape
    p = P.shape[1]
    ws, wsb = _ws(max(k, c), max(p, 64), max(k, c, 64), S.device)
    call("rb_ls_richardson", k, c, p, ptr(S), ld(S), ptr(P), ld(P), l, ptr(X), ld(X), ptr(T), ld(T), ws, wsb,
         st(S.device))


def certify_sums(S, P, R, out):
    """out[0:3] = ||I - S^T S||^2, ||P - S R||^2, ||P||^2 (one launch)."""
    k, m = S.shape
    ws, wsb = _ws(max(k, 64), m, k, S.device)
    call("rb_certify", k, m, ptr(S), ld(S), ptr(P), ld(P), ptr(R), ld(R), ptr(out), ws, wsb, st(S.device))


def l2_select(info_sel, info_a, info_b, Ra, Sa, Rb, Sb, R, S, info_out):
    k, p = S.shape
    call("rb_l2_select", k, p, ptr(info_sel), ptr(info_a), ptr(info_b), ptr(Ra), ld(Ra), ptr(Sa), ld(Sa), ptr(Rb),
         ld(Rb), ptr(Sb), ld(Sb), ptr(R), ld(R), ptr(S), ld(S), ptr(info_out), st(S.device))


def sketched_cholqr_small(Sp, R, Sout, info):
    k, p = Sp.shape
    ws, wsb = _ws(k, p, k, Sp.device)
    call("rb_sketched_cholqr_small", k, p, ptr(Sp), ld(Sp), ptr(R), ld(R), ptr(Sout), ld(Sout), ptr(info), ws,
         wsb, st(Sp.device))


def stencil7(nx, ny, nzl, X, Y, halo_lo=None, halo_hi=None):
    ldh = ld(halo_lo) if halo_lo is not None else (ld(halo_hi) if halo_hi is not None else 0)
    call("rb_stencil7", dtype_code(X), dtype_code(Y), nx, ny, nzl, X.shape[1], ptr(X), ld(X), ptr(halo_lo),
         ptr(halo_hi), ldh, ptr(Y), ld(Y), st(X.device))


def csr_spmm(indptr, indices, values, X, Y):
    call("rb_csr_spmm", dtype_code(X), dtype_code(Y), X.shape[0], X.shape[1], ptr(indptr), ptr(indices),
         ptr(values), ptr(X), ld(X), ptr(Y), ld(Y), st(X.device))


def convert(X, Y):
    call("rb_convert", dtype_code(X), dtype_code(Y), X.shape[0], X.shape[1], ptr(X), ld(X), ptr(Y), ld(Y),
         st(X.device))


__all__ = ["F32", "F64", "empty_cm", "zeros_cm", "to_cm", "ld"]
