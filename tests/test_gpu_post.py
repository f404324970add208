"""GPU parity of the SURVEY 8(f) rows: cholesky_qr_postprocess and
certify_embedding (rbgs.py:446-486) against golden vectors the unmodified
reference wrote (tests/golden/post.npz), plus the reference's own property
tests for them (test_rbgs.py:583-651), cond_estimate, rel_fact_error and the
sketched cond bracket."""

import math

import numpy as np
import pytest
import torch

import goldens

pytestmark = pytest.mark.gpu

U32, U64 = 2.0 ** -24, 2.0 ** -53


@pytest.fixture(scope="module")
def mods():
    from paper_2111_14641_b200 import kernels, post, rbgs, sketching

    return rbgs, sketching, post, kernels


def _conditioned(g, n, m, cond):
    U, _ = np.linalg.qr(g.standard_normal((n, m)))
    V, _ = np.linalg.qr(g.standard_normal((m, m)))
    return (U * np.geomspace(1.0, 1.0 / cond, m)) @ V.T


def test_postprocess_after_two_precision_sweep_vs_golden(mods):
    rbgs, sk, post, K = mods
    z = goldens.load("post")
    W = goldens.oscillatory(2048, 100)
    th = sk.SketchOperator("srht", 1000, 2048, 3)
    f = rbgs.rbgs(W, th, rbgs.RbgsConfig(partition=K.BlockPartition.uniform(100, 10)))
    dR = np.linalg.norm(f.R.data - z["p1/R_in"]) / np.linalg.norm(z["p1/R_in"])
    assert dR <= 1e-5
    o = rbgs.cholesky_qr_postprocess(f)
    R = o.R.data
    assert np.linalg.norm(R - z["p1/R"]) / np.linalg.norm(z["p1/R"]) <= 1e-5
    Q = o.Q.data
    m = 100
    # the reference's own bounds (test_rbgs.py:603-612)
    assert np.linalg.norm(np.eye(m) - Q.T @ Q) <= 1e-13 * m
    assert np.linalg.norm(W - Q @ R) <= 4 * U32 * m ** 1.5 * np.linalg.norm(W)
    assert np.linalg.norm(o.S.data - z["p1/S"]) / np.linalg.norm(z["p1/S"]) <= 1e-5
    # certificates: same order as the reference's
    assert o.cert.delta <= 10 * max(z["p1/cert"][0], 1e-12)


def test_postprocess_fp64_factor_vs_golden(mods):
    rbgs, sk, post, K = mods
    z = goldens.load("post")
    Qs = z["p2/Q_in"]
    ident = sk.SketchOperator("identity", 400, 400, 0)
    S = sk.apply(ident, Qs).data
    f = rbgs.BlockQR(K.Matrix(Qs), K.Matrix(np.eye(6)), K.Matrix(S), K.Matrix(S),
                     K.BlockPartition.uniform(6, 3), None)
    o = rbgs.cholesky_qr_postprocess(f)
    assert np.allclose(o.R.data, z["p2/R"], rtol=0, atol=1e-13)
    assert np.allclose(o.Q.data, z["p2/Q"], rtol=0, atol=1e-13)
    assert np.allclose(o.S.data, z["p2/S"], rtol=0, atol=1e-13)
    assert np.allclose(o.R.data, np.diag([1.0, 2.0, 0.5, 3.0, 1.5, 0.25]), atol=1e-13)
    assert abs(o.cert.delta - z["p2/cert"][0]) <= 1e-13


def test_postprocess_rejects_ill_conditioned_q(mods):
    rbgs, sk, post, K = mods
    from paper_2111_14641_b200.errors import RankDeficiencyError

    Q = _conditioned(np.random.Generator(np.random.Philox(32)), 100, 6, 1e3)
    f = rbgs.BlockQR(K.Matrix(Q), K.Matrix(np.eye(6)), K.Matrix(Q[:20]), K.Matrix(Q[:20]),
                     K.BlockPartition.uniform(6, 3), None)
    with pytest.raises(RankDeficiencyError, match="exceeds 100"):
        rbgs.cholesky_qr_postprocess(f)


def test_postprocess_wide_factor_blocked_trsm(mods):
    """m = 200 > 64: the blocked tall TRSM (panels + DGEMM updates)."""
    rbgs, sk, post, K = mods
    g = np.random.Generator(np.random.Philox(41))
    n, m = 5000, 200
    Q = _conditioned(g, n, m, 20.0)
    th = sk.SketchOperator("identity", n, n, 0)
    f = rbgs.BlockQR(K.Matrix(Q), K.Matrix(np.eye(m)), K.Matrix(Q), K.Matrix(Q),
                     K.BlockPartition.uniform(m, 20), None)
    o = rbgs.cholesky_qr_postprocess(f)
    Qn = o.Q.data
    assert np.linalg.norm(np.eye(m) - Qn.T @ Qn) <= 1e-13 * m
    assert np.linalg.norm(Q - Qn @ o.R.data) <= 1e-13 * np.linalg.norm(Q)


def test_certify_embedding_vs_golden(mods):
    rbgs, sk, post, K = mods
    z = goldens.load("post")
    th7 = sk.SketchOperator("srht", 60, 300, 7)
    phi = sk.SketchOperator("rademacher", 80, 300, 99)
    eq, ew = rbgs.certify_embedding(z["e1/M"], z["e1/W"], th7, phi)
    assert math.isclose(eq, z["e1/eps"][0], rel_tol=1e-8)
    assert math.isclose(ew, z["e1/eps"][1], rel_tol=1e-8)
    eq2, _ = rbgs.certify_embedding(z["e2/M"], z["e1/W"], th7, phi)
    assert eq2 >= 0.5 and abs(eq2 - z["e2/eps"][0]) <= 1e-6


def test_certify_embedding_identity_and_rank_deficiency(mods):
    rbgs, sk, post, K = mods
    from paper_2111_14641_b200.errors import RankDeficiencyError

    g = np.random.Generator(np.random.Philox(33))
    M = g.standard_normal((150, 8))
    th = sk.SketchOperator("identity", 150, 150, 0)
    eq, ew = rbgs.certify_embedding(M, M, th, th)
    assert eq <= 1e-10 and ew <= 1e-10
    Md = np.hstack([M[:, :4], M[:, :4]])
    with pytest.raises(RankDeficiencyError):
        rbgs.certify_embedding(Md, M, th, th)


def test_cond_estimate_and_diagnostics(mods):
    rbgs, sk, post, K = mods
    g = np.random.Generator(np.random.Philox(51))
    for cond in (1e3, 1e9):
        A = _conditioned(g, 3000, 40, cond)
        c = K.cond_estimate(A)
        assert math.isclose(c, np.linalg.cond(A), rel_tol=1e-6 if cond > 1e5 else 1e-9), (cond, c)
        c32 = K.cond_estimate(torch.from_numpy(A.astype(np.float32)).cuda())
        assert math.isclose(c32, np.linalg.cond(A.astype(np.float32).astype(np.float64)), rel_tol=1e-3)
    # ||W - QR|| / ||W|| and the sketched bracket on a real sweep
    W = goldens.trig_family(20_000, 60, 5).astype(np.float32)
    th = sk.gaussian_operator(400, 20_000, 3)
    f = rbgs.rbgs(W, th, rbgs.RbgsConfig(partition=K.BlockPartition.uniform(60, 12),
                                         interblock="sketched_cholqr(1)"))
    Q, R = f.Q.data, f.R.data
    W64 = W.astype(np.float64)
    want = np.linalg.norm(W64 - Q @ R) / np.linalg.norm(W64)
    got = post.rel_fact_error(W, f.Q, f.R, rows_per_chunk=4096)
    assert math.isclose(got, want, rel_tol=1e-6), (got, want)
    eps_q, _ = rbgs.certify_embedding(f.Q, W, th, sk.SketchOperator("rademacher", 300, 20_000, 9))
    lo, hi = post.sketched_cond(f.S, min(0.95, 2 * eps_q + 0.1))
    cq = np.linalg.cond(Q)
    assert lo <= cq * (1 + 1e-6) and cq <= hi * (1 + 1e-6), (lo, cq, hi)
