"""SURVEY.md 8(f) rows on the device: factor post-processing, the embedding
certificate, factorization diagnostics and BlockQR serialization.

  cholesky_qr_postprocess  rbgs.py:446-463   Gram (rb_cross) + Cholesky +
                                             blocked tall TRSM (rb_trsm_right
                                             panels, rb_gemm_f64 updates)
  certify_embedding        rbgs.py:466-486   both sketches on the device,
                                             Householder R of Phi M, SVD of
                                             (Theta M) R_phi^{-1}
  cond_estimate            kernels.py:552-566  sigma_max / sigma_min
  rel_fact_error           bench.py:327-328  ||W - Q R||_F / ||W||_F, fp64,
                                             streamed in row chunks
  sketched_cond            (new)             cond(Q) bracket from S = Theta Q
  save_blockqr/load_blockqr rbgs.py:493-552  the reference's Matrix Market
                                             directory, bit-compatible
  save_blockqr_binary/...  (new)             raw little-endian, sharded Q

The m x m factorizations (Cholesky of the m x m Gram, QR / SVD of k x m
sketches) are small dense library calls (cuSOLVER through torch.linalg) on
the device; every n-dimensional pass goes through the C ABI.
"""

from __future__ import annotations

import json
import math
import os

import numpy as np
import torch

from . import _device as D
from . import sketching
from ._lib import require_cuda
from .errors import CertificationError, NotPositiveDefiniteError, RankDeficiencyError, ShapeError
from .kernels import FINE, BlockPartition, Matrix

PANEL = 64  # widest panel of the hand-written tall kernels (rb_trsm_right)


def _dev(A, device=None, dtype=None):
    """Column-major device tensor of a Matrix / tensor / array (dtype kept
    unless given; host arrays upload as binary64)."""
    if isinstance(A, Matrix):
        A = A._dev if A._dev is not None else A.data
    if isinstance(A, torch.Tensor):
        t = A if A.dim() == 2 else A.reshape(-1, 1)
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        return D.to_cm(t, dtype or t.dtype, device if not t.is_cuda else t.device)
    a = np.asarray(A, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return D.to_cm(torch.from_numpy(np.asfortranarray(a)), dtype or torch.float64, device)


def gram(Q) -> torch.Tensor:
    """G = Q^T Q in binary64 (rb_cross: split-K fp64 accumulation, binary32
    Q read as is)."""
    n, m = Q.shape
    G = D.empty_cm(m, m, torch.float64, Q.device)
    D.cross(Q, Q, G)
    return G


def trsm_right_tall(B, R):
    """In place B <- B R^{-1} for tall binary64 B (n x m) and upper R (m x m):
    right-looking over 64-column panels -- the trailing update is one DGEMM,
    each diagonal panel the hand-written row-substitution kernel."""
    m = R.shape[0]
    d = torch.diagonal(R)
    if bool((d == 0).any()):
        from .errors import SingularTriangularError
        raise SingularTriangularError(int(torch.nonzero(d == 0)[0, 0]))
    for j0 in range(0, m, PANEL):
        j1 = min(m, j0 + PANEL)
        if j0:
            D.gemm(0, 0, -1.0, B[:, :j0], R[:j0, j0:j1], 1.0, B[:, j0:j1])
        D.trsm_right(B[:, j0:j1], R[j0:j1, j0:j1], B[:, j0:j1])
    return B


def _cond_from_gram(G) -> float:
    ev = torch.linalg.eigvalsh(G)
    lo, hi = float(ev[0]), float(ev[-1])
    if not hi > 0.0:
        return float("inf")
    if not lo > 0.0:
        return float("inf")
    return math.sqrt(hi / lo)


def cond_estimate(A, device=None) -> float:
    """sigma_max / sigma_min of a tall matrix (kernels.py:552-566), +inf when
    sigma_min underflows.  The Gram route (one rb_cross pass + an m x m
    eigensolve) is accurate to ~cond^2 u64 relative; above 1e5 the estimate
    is recomputed from the singular values of the Householder R of A, which
    is accurate at any condition number (the reference's Jacobi SVD)."""
    require_cuda()
    Ad = _dev(A, D.cuda_device(device))
    n, m = Ad.shape
    if n < m:
        raise ShapeError(f"cond_estimate requires rows >= cols, got {tuple(Ad.shape)}")
    with torch.cuda.device(Ad.device):
        c = _cond_from_gram(gram(Ad))
        if c > 1e5:
            A64 = Ad if Ad.dtype == torch.float64 else Ad.to(torch.float64)
            sv = torch.linalg.svdvals(torch.linalg.qr(A64, mode="r")[1])
            smin = float(sv[-1])
            c = float("inf") if smin == 0.0 else float(sv[0]) / smin
    return c


def cholesky_qr_postprocess(f, device=None):
    """One Cholesky-QR pass turning a sketch-orthonormal Q into an
    l2-orthonormal one (rbgs.py:446-463): R' = chol(Q^T Q), Q <- Q R'^{-1},
    R <- R' R, S <- S R'^{-1}, re-certified.  Q comes back in binary64."""
    from .rbgs import BlockQR, certify

    require_cuda()
    Qd = _dev(f.Q, D.cuda_device(device))
    dev = Qd.device
    with torch.cuda.device(dev):
        G = gram(Qd)
        c = _cond_from_gram(G)
        if not (c <= 100.0):
            raise RankDeficiencyError(
                f"cond(Q) = {c:.3e} exceeds 100; refusing Cholesky post-processing")
        # G is symmetric to rounding (kernels.py:240-241 tolerance); the
        # factorization reads the upper triangle, like dpotrf(lower=0)
        if not torch.allclose(G, G.t(), rtol=0.0, atol=1e-10 * max(1.0, float(G.abs().max()))):
            raise ShapeError("cholesky input is not symmetric")
        Rp, info = torch.linalg.cholesky_ex(torch.triu(G) + torch.triu(G, 1).t(), upper=True)
        if int(info) > 0:
            raise NotPositiveDefiniteError(int(info))
        Rp = D.to_cm(Rp, torch.float64)
        Qn = D.empty_cm(Qd.shape[0], Qd.shape[1], torch.float64, dev)
        D.convert(Qd, Qn)
        trsm_right_tall(Qn, Rp)
        Rd = _dev(f.R, dev, torch.float64)
        Rn = D.empty_cm(Rd.shape[0], Rd.shape[1], torch.float64, dev)
        D.gemm(0, 0, 1.0, Rp, Rd, 0.0, Rn)
        Sn = _dev(f.S, dev, torch.float64).clone()
        Sn = D.to_cm(Sn, torch.float64)
        trsm_right_tall(Sn, Rp)
        cert = certify(Sn, f.P, Rn, device=dev)
    return BlockQR(Matrix(Qn), Matrix(Rn), Matrix(Sn), f.P, f.partition, cert)


def _sketch_cols(theta, M):
    out = D.empty_cm(theta.k, M.shape[1], torch.float64, M.device)
    for j0 in range(0, M.shape[1], PANEL):
        j1 = min(M.shape[1], j0 + PANEL)
        sketching.sketch_into(theta, M[:, j0:j1], out[:, j0:j1])
    return out


def _householder_r(A):
    """R of the economic Householder QR with diag(R) >= 0 (kernels.py:216-231)."""
    R = torch.linalg.qr(A, mode="r")[1]
    d = torch.sign(torch.diagonal(R))
    d[d == 0] = 1.0
    return d[:, None] * R


def certify_embedding(Q, W, theta, phi, device=None) -> tuple:
    """Embedding distortion of theta on range(Q) and range(W), estimated with
    an independent second sketch phi (rbgs.py:466-486)."""
    require_cuda()
    dev = D.cuda_device(device)
    out = []
    for M in (Q, W):
        Md = _dev(M, dev)
        if Md.shape[0] != theta.n or Md.shape[0] != phi.n:
            raise ShapeError(f"sketch expects {theta.n} rows, got {Md.shape[0]}")
        with torch.cuda.device(Md.device):
            Rphi = _householder_r(_sketch_cols(phi, Md))
            d = torch.abs(torch.diagonal(Rphi))
            dmin, dmax = float(d.min()), float(d.max())
            if d.numel() and dmin <= phi.k * FINE.u * max(dmax, 1e-300):
                raise RankDeficiencyError(
                    f"second sketch of the factor is rank deficient (min diag {dmin:.3e})")
            G = torch.linalg.solve_triangular(Rphi, _sketch_cols(theta, Md), upper=True, left=False)
            sv = torch.linalg.svdvals(G)
            out.append(float(max(float(sv[0]) ** 2 - 1.0, 1.0 - float(sv[-1]) ** 2)))
    return out[0], out[1]


def rel_fact_error(W, Q, R, device=None, rows_per_chunk: int = 1 << 16) -> float:
    """||W - Q R||_F / ||W||_F in binary64 (bench.py:327-328's diagnostic),
    streamed over row chunks so no n x m binary64 copy is formed."""
    require_cuda()
    Qd = _dev(Q, D.cuda_device(device))
    dev = Qd.device
    Wd = _dev(W, dev)
    Rd = _dev(R, dev, torch.float64)
    n, m = Qd.shape
    if Wd.shape != (n, Rd.shape[1]) or Rd.shape[0] != m:
        raise ShapeError("rel_fact_error: shape mismatch")
    num = torch.zeros(1, dtype=torch.float64, device=dev)
    den = torch.zeros(1, dtype=torch.float64, device=dev)
    part = torch.zeros(1, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        T = D.empty_cm(min(n, rows_per_chunk), Wd.shape[1], torch.float64, dev)
        Qc = D.empty_cm(min(n, rows_per_chunk), m, torch.float64, dev)
        for r0 in range(0, n, rows_per_chunk):
            r1 = min(n, r0 + rows_per_chunk)
            t, q = T[:r1 - r0], Qc[:r1 - r0]
            D.convert(Wd[r0:r1], t)
            D.sumsq(t, part)
            den.add_(part)
            D.convert(Qd[r0:r1], q)
            D.gemm(0, 0, -1.0, q, Rd, 1.0, t)
            D.sumsq(t, part)
            num.add_(part)
    wn = float(den)
    if wn == 0.0:
        raise CertificationError("relative factorization error undefined for W = 0")
    return math.sqrt(float(num) / wn)


def sketched_cond(S, eps: float) -> tuple:
    """Bracket of cond(Q) from its sketch S = Theta Q alone: for an
    eps-embedding, sigma_i(Q) lies in [sigma_i(S) / sqrt(1 + eps),
    sigma_i(S) / sqrt(1 - eps)] (section 2), so cond(Q) lies in
    cond(S) * [sqrt((1 - eps) / (1 + eps)), sqrt((1 + eps) / (1 - eps))].
    k x m work only -- the device replacement of the per-block full SVD of
    bench._qr_driver (bench.py:326)."""
    if not 0.0 <= eps < 1.0:
        raise ValueError("eps must lie in [0, 1)")
    Sd = S if isinstance(S, torch.Tensor) else _dev(S)
    sv = torch.linalg.svdvals(Sd.to(torch.float64))
    smin = float(sv[-1])
    cs = float("inf") if smin == 0.0 else float(sv[0]) / smin
    f = math.sqrt((1.0 - eps) / (1.0 + eps))
    return cs * f, cs / f


# ---------------------------------------------------------------------------
# serialization
# ---------------------------------------------------------------------------

def _write_mm_array(path, A):
    """'array real general', column-major values, shortest round-trip
    decimals (mmio.py:27-40): a write-then-read cycle is bit-exact."""
    A = np.asarray(A, dtype=np.float64)
    n, m = A.shape
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix array real general\n")
        fh.write(f"{n} {m}\n")
        for j in range(m):
            col = A[:, j].tolist()
            if col:
                fh.write("\n".join(map(repr, col)))
                fh.write("\n")


def _read_mm_array(path):
    """Reads the 'array real general' files the reference writes
    (mmio.py:72-113 semantics: comments, blank lines, count checks)."""
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise ValueError(f"{path}: empty file")
    parts = lines[0].strip().lower().split()
    if len(parts) != 5 or parts[0] != "%%matrixmarket" or parts[1] != "matrix" or parts[2] != "array":
        raise ValueError(f"{os.path.basename(path)} must be an array file")
    body = [s for s in (ln.strip() for ln in lines[1:]) if s and not s.startswith("%")]
    if not body:
        raise ValueError(f"{path}: missing size line")
    n, m = (int(x) for x in body[0].split())
    vals = np.array([float(s) for s in body[1:]], dtype=np.float64)
    if vals.size != n * m:
        raise ValueError(f"{path}: expected {n * m} values, got {vals.size}")
    return vals.reshape((m, n)).T.copy(order="F")


def save_blockqr(f, directory: str) -> None:
    """Q/R/S/P as Matrix Market array files plus cert.txt and meta.txt, the
    reference's directory layout (rbgs.py:493-517); binary32-stored Q is
    written as its exact binary64 values.  Text is slow for a large Q: see
    save_blockqr_binary."""
    os.makedirs(directory, exist_ok=True)
    for name, M in (("Q", f.Q), ("R", f.R), ("S", f.S), ("P", f.P)):
        if M is not None:
            _write_mm_array(os.path.join(directory, name + ".mtx"), M.data)
    if f.cert is not None:
        with open(os.path.join(directory, "cert.txt"), "w") as fh:
            fh.write(f"delta={f.cert.delta!r}\n")
            fh.write(f"delta_tilde={f.cert.delta_tilde!r}\n")
            fh.write("per_block_ortho=" + ",".join(repr(v) for v in f.cert.per_block_ortho) + "\n")
            fh.write("per_block_resid=" + ",".join(repr(v) for v in f.cert.per_block_resid) + "\n")
    part = f.partition
    with open(os.path.join(directory, "meta.txt"), "w") as fh:
        fh.write(f"block_width={part.block_width}\n")
        fh.write(f"num_blocks={part.num_blocks}\n")
        fh.write(f"total_cols={part.total_cols}\n")
        if part.widths is not None:
            fh.write("widths=" + ",".join(str(w) for w in part.widths) + "\n")


def _read_kv(path):
    kv = {}
    with open(path) as fh:
        for line in fh:
            if "=" in line:
                key, val = line.strip().split("=", 1)
                kv[key] = val
    return kv


def _floats(s):
    return tuple(float(x) for x in s.split(",")) if s else ()


def load_blockqr(directory: str):
    """Inverse of save_blockqr; also reads directories the reference wrote
    (rbgs.py:520-552).  S.mtx / P.mtx may be absent."""
    from .rbgs import BlockQR, CertReport

    mats = {}
    for name in ("Q", "R", "S", "P"):
        path = os.path.join(directory, name + ".mtx")
        if not os.path.exists(path) and name in ("S", "P"):
            mats[name] = None
            continue
        mats[name] = Matrix(_read_mm_array(path))
    meta = _read_kv(os.path.join(directory, "meta.txt"))
    widths = tuple(int(x) for x in meta["widths"].split(",")) if meta.get("widths") else None
    part = BlockPartition(int(meta["block_width"]), int(meta["num_blocks"]), int(meta["total_cols"]),
                          widths=widths)
    cert = None
    cp = os.path.join(directory, "cert.txt")
    if os.path.exists(cp):
        kv = _read_kv(cp)
        cert = CertReport(float(kv["delta"]), float(kv["delta_tilde"]), _floats(kv.get("per_block_ortho", "")),
                          _floats(kv.get("per_block_resid", "")))
    return BlockQR(mats["Q"], mats["R"], mats["S"], mats["P"], part, cert)


_BIN_VERSION = 1


def save_blockqr_binary(f, directory: str, shard=None, rank: int = 0) -> None:
    """Binary BlockQR: raw little-endian column-major arrays, Q in its
    storage dtype (binary32 for two-precision factors), S, P, R in binary64,
    and meta.json.  Row-sharded factors write one Q file per rank
    (`Q.rank{r}.bin`, rows [row0, row0 + n_local)); rank 0 also writes the
    replicated S, P, R and the metadata, so `certify` (k-dimensional data
    only) needs nothing but rank 0's files."""
    os.makedirs(directory, exist_ok=True)
    Qt = f.Q._dev if f.Q._dev is not None else torch.from_numpy(f.Q.data)
    row0 = shard.row0 if shard is not None else 0
    n_local = Qt.shape[0]
    qname = f"Q.rank{rank}.bin"
    Qt.detach().t().contiguous().cpu().numpy().tofile(os.path.join(directory, qname))
    if rank != 0:
        return
    arrays = {}
    for name, M in (("R", f.R), ("S", f.S), ("P", f.P)):
        if M is not None:
            np.asfortranarray(M.data).T.astype("<f8").tofile(os.path.join(directory, name + ".bin"))
            arrays[name] = list(M.shape)
    part = f.partition
    meta = {"version": _BIN_VERSION, "n": shard.n if shard is not None else n_local, "m": Qt.shape[1],
            "q_dtype": str(Qt.dtype).replace("torch.", ""), "arrays": arrays,
            "partition": {"block_width": part.block_width, "num_blocks": part.num_blocks,
                          "total_cols": part.total_cols,
                          "widths": list(part.widths) if part.widths is not None else None},
            "cert": None if f.cert is None else {
                "delta": f.cert.delta, "delta_tilde": f.cert.delta_tilde,
                "per_block_ortho": list(f.cert.per_block_ortho),
                "per_block_resid": list(f.cert.per_block_resid)},
            "shards": [] if shard is None else None}
    if shard is None:
        meta["shards"] = [{"rank": 0, "row0": row0, "n_local": n_local}]
    with open(os.path.join(directory, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def register_shard(directory: str, rank: int, row0: int, n_local: int) -> None:
    """Rank 0 records every shard's rows (call after the ranks' saves)."""
    path = os.path.join(directory, "meta.json")
    with open(path) as fh:
        meta = json.load(fh)
    shards = [s for s in (meta.get("shards") or []) if s["rank"] != rank]
    shards.append({"rank": rank, "row0": row0, "n_local": n_local})
    meta["shards"] = sorted(shards, key=lambda s: s["row0"])
    with open(path, "w") as fh:
        json.dump(meta, fh, indent=1)


def load_blockqr_binary(directory: str, rank=None, device=None):
    """Inverse of save_blockqr_binary.  rank=None stitches every shard's Q
    rows (host); an int loads that rank's rows only.  With `device`, Q, S,
    P, R are placed on that CUDA device."""
    from .rbgs import BlockQR, CertReport

    with open(os.path.join(directory, "meta.json")) as fh:
        meta = json.load(fh)
    if meta.get("version") != _BIN_VERSION:
        raise ValueError(f"unsupported binary BlockQR version {meta.get('version')}")
    m = meta["m"]
    qdt = np.float32 if meta["q_dtype"] == "float32" else np.float64

    def read_q(s):
        a = np.fromfile(os.path.join(directory, f"Q.rank{s['rank']}.bin"), dtype="<f4" if qdt == np.float32
                        else "<f8")
        if a.size != s["n_local"] * m:
            raise ValueError(f"Q.rank{s['rank']}.bin: expected {s['n_local'] * m} values, got {a.size}")
        return a.reshape(m, s["n_local"]).T

    shards = meta["shards"]
    if rank is None:
        if sum(s["n_local"] for s in shards) != meta["n"]:
            raise ValueError("binary BlockQR: shards do not cover all rows")
        Q = np.vstack([read_q(s) for s in sorted(shards, key=lambda s: s["row0"])])
    else:
        Q = read_q(next(s for s in shards if s["rank"] == rank))
    mats = {}
    for name in ("R", "S", "P"):
        shp = meta["arrays"].get(name)
        if shp is None:
            mats[name] = None
            continue
        a = np.fromfile(os.path.join(directory, name + ".bin"), dtype="<f8").reshape(shp[1], shp[0]).T
        mats[name] = a

    def wrap(a, prec=FINE):
        if a is None:
            return None
        if device is not None:
            return Matrix(D.to_cm(torch.from_numpy(np.ascontiguousarray(a)), None, D.cuda_device(device)),
                          precision=prec)
        return Matrix(a.astype(np.float64), precision=prec)

    p = meta["partition"]
    part = BlockPartition(p["block_width"], p["num_blocks"], p["total_cols"],
                          widths=tuple(p["widths"]) if p["widths"] else None)
    c = meta["cert"]
    cert = None if c is None else CertReport(c["delta"], c["delta_tilde"], tuple(c["per_block_ortho"]),
                                             tuple(c["per_block_resid"]))
    from .kernels import COARSE
    return BlockQR(wrap(Q, COARSE if qdt == np.float32 else FINE), wrap(mats["R"]), wrap(mats["S"]),
                   wrap(mats["P"]), part, cert)
