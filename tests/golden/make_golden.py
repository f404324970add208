"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports `sketch_krylov` from /root/reference/pkg/src, runs the reference's
own public entry points (`kernels.gemm`, `sketching.apply`, `rbgs.rbgs`,
`rbgs.RbgsSweep`, `krylov.rbgs_arnoldi`, `krylov.block_gmres`) on seeded
inputs, and writes small .npz files.  The GPU parity tests and the oracle
pinning tests read only these files, never /root/reference.

The gaussian / sparse_sign kinds do not exist in the reference; their
golden sweeps run the reference's own RbgsSweep on an operator whose
`sketching.apply` path (the fixed-order dense gemm, sketching.py:151-155)
is fed the dense matrix that `oracle.sketches` materialises.
"""

from __future__ import annotations

import dataclasses
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from sketch_krylov import kernels, krylov, rbgs as R, sketching  # noqa: E402
from sketch_krylov.bench import gen_oscillatory  # noqa: E402
from sketch_krylov.errors import DependentBlockError, InterblockError  # noqa: E402
from sketch_krylov.operators import CsrOperator, DenseOperator  # noqa: E402

from oracle import sketches as osk  # noqa: E402


def rng(seed):
    return np.random.Generator(np.random.Philox(seed))


def conditioned(g, n, m, cond):
    U, _ = np.linalg.qr(g.standard_normal((n, m)))
    V, _ = np.linalg.qr(g.standard_normal((m, m)))
    return (U * np.geomspace(1.0, 1.0 / cond, m)) @ V.T


def trig_family(n, m, seed):
    """BASELINE.json configs[0]/[1] generator: W_ij = sin(10 mu_j (x_i+1)) /
    (cos(100 mu_j (x_i+1)) + 1.1), x_i = i/(n-1), mu_j ~ U[1, pi]."""
    mu = 1.0 + (math.pi - 1.0) * rng(seed).random(m)
    x = np.arange(n, dtype=np.float64) / (n - 1)
    a = np.outer(x + 1.0, mu)
    return np.sin(10.0 * a) / (np.cos(100.0 * a) + 1.1)


def dense_kind_operator(kind, k, n, seed, nnz=8):
    """Reference SketchOperator whose dense-gemm apply path carries the
    oracle's materialised gaussian / sparse_sign matrix times sqrt(k)."""
    th = sketching.SketchOperator("rademacher", k, n, 0)
    if kind == "gaussian":
        M = osk.gaussian_int16(seed, k, np.arange(n)).astype(np.float64) \
            * osk.gaussian_scale(k)
    else:
        M = osk.sparse_sign_matrix(seed, k, nnz, n).toarray()
    object.__setattr__(th, "_signs", M * math.sqrt(k))
    return th


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1e3:.1f} kB")


# ---------------------------------------------------------------------------

def gen_gemm():
    g = rng(101)
    out = {}
    for t, (n, c, p) in enumerate([(7, 5, 3), (64, 17, 8), (257, 40, 12), (1000, 33, 10)]):
        Q = g.standard_normal((n, c))
        X = g.standard_normal((c, p))
        W = g.standard_normal((n, p))
        out[f"Q{t}"], out[f"X{t}"], out[f"W{t}"] = Q, X, W
        out[f"coarse{t}"] = kernels.gemm(-1.0, Q, X, 1.0, W, prec=kernels.COARSE).data
        out[f"fine{t}"] = kernels.gemm(-1.0, Q, X, 1.0, W, prec=kernels.FINE).data
    save("gemm", **out)


def gen_sketch():
    g = rng(102)
    out = {}
    specs = [("srht", 64, 300, 11), ("srht", 24, 64, 3), ("srht", 1, 2, 5),
             ("srht", 333, 5000, 17), ("srht", 1024, 4096, 5),
             ("rademacher", 24, 64, 3), ("rademacher", 64, 256, 5),
             ("identity", 16, 16, 0)]
    for t, (kind, k, n, seed) in enumerate(specs):
        th = sketching.SketchOperator(kind, k, n, seed)
        X = g.standard_normal((n, 5))
        out[f"spec{t}"] = np.array([kind.encode(), str(k).encode(), str(n).encode(),
                                    str(seed).encode()])
        out[f"X{t}"] = X
        out[f"Y{t}"] = sketching.apply(th, X).data
        if kind == "srht":
            out[f"signs{t}"] = th.sign_diagonal.astype(np.int8)
            out[f"sample{t}"] = np.asarray(th.sample_indices)
        if kind == "rademacher":
            out[f"signs{t}"] = th._signs
    save("sketch", **out)


def run_rbgs(W, th, **cfg_kw):
    cfg = R.RbgsConfig(**cfg_kw)
    f = R.rbgs(W, th, cfg)
    return dict(Q=f.Q.data, R=f.R.data, S=f.S.data, P=f.P.data,
                cert=np.array([f.cert.delta, f.cert.delta_tilde]),
                pbo=np.array(f.cert.per_block_ortho), pbr=np.array(f.cert.per_block_resid))


def gen_rbgs():
    cases = {}
    P = kernels.BlockPartition
    g = rng(103)
    W = conditioned(g, 512, 24, 1e3)
    th = ("srht", 320, 512, 12)
    base = dict(partition=P.uniform(24, 6))
    for name, kw in [
        ("default", {}),
        ("fp64", dict(coarse=kernels.FINE)),
        ("sk1", dict(interblock="sketched_cholqr(1)")),
        ("sk2", dict(interblock="sketched_cholqr(2)")),
        ("rgs", dict(interblock="rgs_single")),
        ("bmgs", dict(ls_solver="bmgs_reorth(2)")),
        ("cg", dict(ls_solver="cg_normal(20)")),
        ("hh", dict(ls_solver="householder_direct")),
        ("resketch", dict(interblock="sketched_cholqr(1)", resketch=True)),
        ("coarse_all", dict(fine=kernels.COARSE)),
        ("certblocks", dict(certify_blocks=True)),
    ]:
        cases[name] = (W, th, {**base, **kw})
    g = rng(104)
    cases["rad_ragged"] = (g.standard_normal((256, 11)), ("rademacher", 64, 256, 5),
                           dict(partition=P.uniform(11, 4), certify_blocks=True))
    g = rng(105)
    cases["identity_hh"] = (conditioned(g, 400, 30, 50.0), ("identity", 400, 400, 0),
                            dict(partition=P.uniform(30, 5), ls_solver="householder_direct",
                                 coarse=kernels.FINE))
    cases["osc"] = (np.asarray(gen_oscillatory(2048, 120)), ("srht", 1200, 2048, 13),
                    dict(partition=P.uniform(120, 10)))
    Wt = trig_family(3000, 40, 7)
    cases["trig2p"] = (Wt, ("srht", 80, 3000, 3), dict(partition=P.uniform(40, 10),
                                                       interblock="sketched_cholqr(1)"))
    cases["trig64"] = (Wt, ("srht", 80, 3000, 3), dict(partition=P.uniform(40, 10),
                                                       interblock="sketched_cholqr(1)",
                                                       coarse=kernels.FINE))
    Wg = trig_family(1000, 20, 9)
    cases["gauss2p"] = (Wg.astype(np.float32).astype(np.float64), ("gaussian", 80, 1000, 7),
                        dict(partition=P.uniform(20, 5), interblock="sketched_cholqr(1)"))
    cases["gauss64"] = (Wg, ("gaussian", 80, 1000, 7),
                        dict(partition=P.uniform(20, 5), interblock="sketched_cholqr(1)",
                             coarse=kernels.FINE))
    g = rng(106)
    cases["sparse2p"] = (g.standard_normal((1200, 12)), ("sparse_sign", 48, 1200, 9),
                         dict(partition=P.uniform(12, 4), interblock="sketched_cholqr(1)"))
    out = {}
    shared = {}
    regen = {"osc": "osc", "trig2p": "trig:3000:40:7", "trig64": "trig:3000:40:7",
             "gauss64": "trig:1000:20:9"}
    for name, (W, spec, kw) in cases.items():
        kind, k, n, seed = spec
        if kind in ("gaussian", "sparse_sign"):
            th_obj = dense_kind_operator(kind, k, n, seed)
        else:
            th_obj = sketching.SketchOperator(kind, k, n, seed)
        res = run_rbgs(W, th_obj, **kw)
        if name in regen:
            out[f"{name}/Wgen"] = np.array(regen[name])
        else:
            key = next((kk for kk, vv in shared.items() if vv is W), None)
            if key is None:
                shared[name] = W
                out[f"{name}/W"] = W
            else:
                out[f"{name}/Wref"] = np.array(key)
        out[f"{name}/spec"] = np.array([kind, str(k), str(n), str(seed)])
        cfg = R.RbgsConfig(**kw)
        out[f"{name}/cfg"] = np.array([
            ",".join(str(w) for w in cfg.partition.block_widths()), cfg.ls_solver,
            cfg.interblock, cfg.coarse.format, cfg.fine.format,
            str(int(cfg.certify_blocks)), str(int(cfg.resketch))])
        for key, v in res.items():
            out[f"{name}/{key}"] = v
        print(name, res["cert"])
    save("rbgs", **out)


def gen_errors():
    out = {}
    g = rng(27)
    W = np.hstack([g.standard_normal((300, 10)), np.zeros((300, 5))])
    try:
        R.rbgs(W, sketching.SketchOperator("srht", 60, 300, 7),
               R.RbgsConfig(partition=kernels.BlockPartition(5, 3, 15)))
    except DependentBlockError as e:
        out["vanished/W"], out["vanished/block"] = W, np.array(e.block)
    g = rng(28)
    dup = g.standard_normal((300, 1))
    W = np.hstack([g.standard_normal((300, 10)), dup, dup, g.standard_normal((300, 3))])
    try:
        R.rbgs(W, sketching.SketchOperator("srht", 60, 300, 7),
               R.RbgsConfig(partition=kernels.BlockPartition(5, 3, 15),
                            interblock="sketched_cholqr(1)"))
    except InterblockError as e:
        out["interblock/W"], out["interblock/block"] = W, np.array(e.block)
        out["interblock/msg"] = np.array(str(e))
    save("errors", **out)


def gen_krylov():
    out = {}
    n = 200
    import scipy.sparse
    T = scipy.sparse.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)],
                           [-1, 0, 1]).tocsr()
    g = rng(107)
    B = g.standard_normal((n, 2))
    dec = krylov.rbgs_arnoldi(CsrOperator(T), B, sketching.SketchOperator("srht", 64, n, 1), 5)
    out.update({"arn/B": B, "arn/Q": dec.Q.data, "arn/H": dec.H.data,
                "arn/Rf": dec.R_first.data, "arn/S": dec.S.data, "arn/P": dec.P.data,
                "arn/cert": np.array([dec.cert.delta, dec.cert.delta_tilde])})
    g = rng(121)
    d = np.arange(1.0, 101.0)
    b = g.standard_normal((100, 1))
    rep = krylov.block_gmres(DenseOperator(np.diag(d)), b,
                             sketching.SketchOperator("srht", 48, 100, 21), 12)
    out.update({"gm/b": b, "gm/x": rep.solution.data,
                "gm/hist": np.array(rep.residual_history),
                "gm/conds": np.array(rep.basis_cond_history),
                "gm/certs": np.array(rep.cert_history)})
    g = rng(120)
    B = g.standard_normal((50, 2))
    rep = krylov.block_gmres(DenseOperator(np.eye(50)), B,
                             sketching.SketchOperator("identity", 50, 50, 0), 4)
    out.update({"gmid/B": B, "gmid/x": rep.solution.data,
                "gmid/hist": np.array(rep.residual_history),
                "gmid/breakdown": np.array(rep.breakdown)})
    # 3-D Poisson, small grid, restarted, the C4 shape in miniature
    nx = 12
    from oracle.krylov import poisson3d_apply
    A3 = poisson3d_apply(nx, nx, nx)
    I = np.eye(nx)
    T1 = scipy.sparse.diags([-np.ones(nx - 1), 2 * np.ones(nx), -np.ones(nx - 1)], [-1, 0, 1])
    K = (scipy.sparse.kron(scipy.sparse.kron(I, I), T1)
         + scipy.sparse.kron(scipy.sparse.kron(I, T1), I)
         + scipy.sparse.kron(scipy.sparse.kron(T1, I), I)).tocsr()
    g = rng(122)
    B = g.standard_normal((nx ** 3, 4))
    assert np.allclose(K @ B, A3(B))
    th = dense_kind_operator("sparse_sign", 2 * 4 * 9, nx ** 3, 11)
    rep = krylov.block_gmres(CsrOperator(K), B, th, 8, restarts=2,
                             cfg=R.RbgsConfig(interblock="sketched_cholqr(1)"))
    out.update({"p3/B": B, "p3/x": rep.solution.data, "p3/hist": np.array(rep.residual_history),
                "p3/conds": np.array(rep.basis_cond_history),
                "p3/certs": np.array(rep.cert_history), "p3/nx": np.array(nx)})
    save("krylov", **out)


def gen_operators():
    """Pins of the two north-star kinds (checked by the oracle tests too)."""
    out = {}
    out["gauss_q"] = osk.gaussian_int16(20240917, 37, np.arange(0, 50))
    out["gauss_q_far"] = osk.gaussian_int16(7, 9, np.arange(2 ** 33, 2 ** 33 + 5))
    pick, sign = osk.sparse_sign_rows(11, 72, 8, np.arange(0, 64))
    out["sparse_pick"], out["sparse_sign"] = pick, sign
    save("operators", **out)


def gen_post():
    """Post-processing / embedding certificate / serialization:
    cholesky_qr_postprocess, certify_embedding and save_blockqr on the
    reference's own test shapes (test_rbgs.py:570-651)."""
    out = {}
    W = gen_oscillatory(2048, 100)
    th = sketching.SketchOperator("srht", 1000, 2048, 3)
    f = R.rbgs(W, th, R.RbgsConfig(partition=kernels.BlockPartition.uniform(100, 10)))
    o = R.cholesky_qr_postprocess(f)
    out.update({"p1/R_in": f.R.data, "p1/R": o.R.data, "p1/S": o.S.data,
                "p1/cert": np.array([o.cert.delta, o.cert.delta_tilde])})
    # fp64 hand-made factor: Q orthonormal times a column scaling
    g = rng(131)
    Q0, _ = np.linalg.qr(g.standard_normal((400, 6)))
    Qs = Q0 * np.array([1.0, 2.0, 0.5, 3.0, 1.5, 0.25])
    ident = sketching.SketchOperator("identity", 400, 400, 0)
    S = sketching.apply(ident, Qs).data
    f2 = R.BlockQR(kernels.Matrix(Qs), kernels.Matrix(np.eye(6)), kernels.Matrix(S), kernels.Matrix(S),
                   kernels.BlockPartition.uniform(6, 3), None)
    o2 = R.cholesky_qr_postprocess(f2)
    out.update({"p2/Q_in": Qs, "p2/Q": o2.Q.data, "p2/R": o2.R.data, "p2/S": o2.S.data,
                "p2/cert": np.array([o2.cert.delta, o2.cert.delta_tilde])})
    # certify_embedding
    n = 300
    M = g.standard_normal((n, 6)) @ np.diag(np.logspace(0, -3, 6))
    Wm = g.standard_normal((n, 6))
    th7 = sketching.SketchOperator("srht", 60, n, 7)
    phi = sketching.SketchOperator("rademacher", 80, n, 99)
    eq, ew = R.certify_embedding(M, Wm, th7, phi)
    out.update({"e1/M": M, "e1/W": Wm, "e1/eps": np.array([eq, ew])})
    _, _, Vt = np.linalg.svd(sketching.materialize(th7) if hasattr(sketching, "materialize")
                             else sketching.apply(th7, np.eye(n)).data)
    Mb = Vt[60:].T[:, :6] + 1e-9 * g.standard_normal((n, 6))
    eq2, ew2 = R.certify_embedding(Mb, Wm, th7, phi)
    out.update({"e2/M": Mb, "e2/eps": np.array([eq2, ew2])})
    save("post", **out)
    # a reference-written BlockQR directory (Matrix Market text) for the
    # load_blockqr interoperability test
    Wc = conditioned(rng(30), 300, 12, 50.0)
    th72 = sketching.SketchOperator("srht", 72, 300, 19)
    fc = R.rbgs(Wc, th72, R.RbgsConfig(partition=kernels.BlockPartition.uniform(12, 4),
                                       certify_blocks=True))
    d = os.path.join(HERE, "blockqr_ref")
    R.save_blockqr(fc, d)
    print("blockqr_ref:", sorted(os.listdir(d)))


if __name__ == "__main__":
    gen_gemm()
    gen_sketch()
    gen_operators()
    gen_errors()
    gen_rbgs()
    gen_krylov()
    gen_post()
