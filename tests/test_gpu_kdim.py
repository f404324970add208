"""The hand-written k-dimensional kernels (csrc/kdim.cu) against numpy /
the oracle: Richardson (rbgs.py:144-156), one sketched-CholQR pass
(rbgs.py:282-289), certification (rbgs.py:428-443) and the generic
binary64 / binary32 GEMMs.  Tolerances: binary64 reassociation level
(the kernels and OpenBLAS sum in different fixed orders); the results are
also checked to be bit-reproducible run to run."""

import numpy as np
import pytest
import torch

from oracle import sweep as osw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2111_14641_b200 import _device

    return _device


def _dev(A, dtype=torch.float64):
    from paper_2111_14641_b200 import _device as Dm

    return Dm.to_cm(torch.from_numpy(np.asfortranarray(A)), dtype, "cuda")


def _orth(g, k, c):
    return np.linalg.qr(g.standard_normal((k, c)))[0] + 1e-3 * g.standard_normal((k, c))


@pytest.mark.parametrize("k,c,p,l", [(1600, 760, 40, 5), (2048, 960, 64, 5), (400, 190, 10, 5), (100, 7, 3, 1),
                                     (488, 240, 4, 2), (1024, 480, 32, 3)])
def test_richardson_vs_oracle(D, k, c, p, l):
    g = np.random.Generator(np.random.Philox(k + c))
    S = _orth(g, k, c)
    P = g.standard_normal((k, p))
    X = D.empty_cm(c, p, torch.float64, "cuda")
    T = D.empty_cm(k, p, torch.float64, "cuda")
    Sd, Pd = _dev(S), _dev(P)
    D.richardson(Sd, Pd, l, X, T)
    got = X.cpu().numpy()
    want = osw.ls_richardson(S, P, l)
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    X2 = torch.zeros_like(X)
    D.richardson(Sd, Pd, l, X2, T)
    assert torch.equal(X, X2)


@pytest.mark.parametrize("k,p", [(1600, 40), (2048, 64), (400, 10), (1024, 32), (488, 4), (70, 37)])
def test_sketched_cholqr_small_vs_numpy(D, k, p):
    import scipy.linalg

    g = np.random.Generator(np.random.Philox(p))
    Sp = g.standard_normal((k, p)) @ np.diag(np.logspace(0, -4, p))
    R = D.empty_cm(p, p, torch.float64, "cuda")
    So = D.empty_cm(k, p, torch.float64, "cuda")
    info = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    D.sketched_cholqr_small(_dev(Sp), R, So, info)
    assert int(info.item()) == 0
    Rw = osw.cholesky_upper(Sp.T @ Sp)
    assert np.linalg.norm(R.cpu().numpy() - Rw) <= 1e-12 * np.linalg.norm(Rw)
    Sw = scipy.linalg.solve_triangular(Rw, Sp.T, trans="T").T
    assert np.linalg.norm(So.cpu().numpy() - Sw) <= 1e-10 * np.linalg.norm(Sw)
    # not positive definite: dpotrf's 1-based column
    Sb = Sp.copy()
    Sb[:, 5 % p] = 0.0  # an exactly zero pivot
    D.sketched_cholqr_small(_dev(Sb), R, So, info)
    want = 1 + (5 % p)
    assert int(info.item()) == want


@pytest.mark.parametrize("k,m", [(1600, 800), (400, 200), (2048, 1024), (96, 5)])
def test_certify_sums_vs_numpy(D, k, m):
    g = np.random.Generator(np.random.Philox(m))
    S = _orth(g, k, m)
    R = np.triu(g.standard_normal((m, m)))
    P = S @ R + 1e-6 * g.standard_normal((k, m))
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    D.certify_sums(_dev(S), _dev(P), _dev(R), out)
    o = out.cpu().numpy()
    want = [np.linalg.norm(np.eye(m) - S.T @ S) ** 2, np.linalg.norm(P - S @ R) ** 2, np.linalg.norm(P) ** 2]
    assert np.allclose(o[[0, 2]], np.array(want)[[0, 2]], rtol=1e-11)
    # ||P - S R|| is a cancellation (~1e-6 of ||P||): absolute binary64 level
    assert abs(o[1] - want[1]) <= 1e-12 * want[2] + 1e-9 * want[1]


@pytest.mark.parametrize("tA,m,n,k", [(1, 760, 40, 1600), (0, 1600, 40, 760), (1, 240, 240, 300_000),
                                      (0, 300_000, 60, 240), (1, 3, 2, 5), (0, 1, 1, 1)])
@pytest.mark.parametrize("dt", [torch.float64, torch.float32])
def test_gemm_vs_numpy(D, tA, m, n, k, dt):
    g = np.random.Generator(np.random.Philox(m + n))
    A = g.standard_normal((k, m) if tA else (m, k))
    B = g.standard_normal((k, n))
    C0 = g.standard_normal((m, n))
    Ad, Bd = _dev(A, dt), _dev(B, dt)
    for alpha, beta in ((1.0, 0.0), (-1.0, 1.0), (0.5, 2.0)):
        C = _dev(C0, dt)
        (D.gemm if dt == torch.float64 else D.gemm32)(tA, 0, alpha, Ad, Bd, beta, C)
        Aw = A.astype(np.float32).astype(np.float64) if dt == torch.float32 else A
        Bw = B.astype(np.float32).astype(np.float64) if dt == torch.float32 else B
        Cw = C0.astype(np.float32).astype(np.float64) if dt == torch.float32 else C0
        want = alpha * ((Aw.T if tA else Aw) @ Bw) + beta * Cw
        scale = np.abs(Aw.T if tA else Aw) @ np.abs(Bw) + np.abs(Cw)
        u = 2.0 ** -24 if dt == torch.float32 else 2.0 ** -53
        assert np.all(np.abs(C.double().cpu().numpy() - want) <= 4 * k * u * scale + 1e-300)


@pytest.mark.parametrize("n,k", [(244, 200_000), (64, 5000), (130, 777), (8, 64)])
def test_syrk_upper_vs_numpy(D, n, k):
    """rb_syrk_f64 (the GMRES basis Gram, krylov.py:98-103): the upper
    triangle of A^T A; 128 x 64 tiles wholly below the diagonal are not formed
    and stay as they were."""
    g = np.random.Generator(np.random.Philox(n))
    A = g.standard_normal((k, n))
    C = _dev(np.full((n, n), 7.0), torch.float64)
    D.syrk(_dev(A, torch.float64), C)
    got = C.cpu().numpy()
    want = A.T @ A
    iu = np.triu_indices(n)
    assert np.all(np.abs(got[iu] - want[iu]) <= 4 * k * 2.0 ** -53 * (np.abs(A).T @ np.abs(A))[iu])
    if n == 244:  # the block (rows 128.., cols 0..63) lies below the diagonal: untouched
        assert np.all(got[128:, :64] == 7.0)


@pytest.mark.parametrize("n,p,q,sym", [(100_003, 40, 40, True), (65536, 64, 64, True), (5000, 16, 16, True),
                                       (33_000, 33, 20, False), (70_000, 64, 9, False), (64, 48, 48, True)])
@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_cross_dmma_vs_numpy(D, n, p, q, sym, dt):
    """rb_cross for 8 < max(p, q) <= 64 (the l2 stage's tall Gram Q'^T Q',
    rbgs.py:293-302) on the FP64 tensor pipe, Gram (mirrored upper tiles) and
    general A^T B, accumulate flag included."""
    g = np.random.Generator(np.random.Philox(n + p))
    A = g.standard_normal((n, p))
    B = A if sym else g.standard_normal((n, q))
    Ad = _dev(A, dt)
    Bd = Ad if sym else _dev(B, dt)
    Aw = Ad.double().cpu().numpy()
    Bw = Aw if sym else Bd.double().cpu().numpy()
    want = Aw.T @ Bw
    bound = 4 * n * 2.0 ** -53 * (np.abs(Aw).T @ np.abs(Bw))
    out = _dev(np.ones((p, q)), torch.float64)
    D.cross(Ad, Bd, out)
    assert np.all(np.abs(out.cpu().numpy() - want) <= bound)
    D.cross(Ad, Bd, out, accumulate=True)
    assert np.all(np.abs(out.cpu().numpy() - 2 * want) <= 2 * bound)


@pytest.mark.parametrize("n,p,cond", [(100_003, 40, 1e3), (65536, 64, 1e12), (300, 7, 1e6), (50_000, 33, 1e14),
                                      (64, 64, 10.0)])
@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_tsqr_r_vs_lapack(D, n, p, cond, dt):
    """rb_tsqr_r: the Householder R factor of a tall matrix (kernels.py:216-231),
    binary64 TSQR, against LAPACK's QR of the same (rounded) input -- normwise
    1e-13 even at cond 1e14 where the Gram route has long broken down; the
    conditional form is a no-op when the status word is zero."""
    g = np.random.Generator(np.random.Philox(n + p))
    U, _ = np.linalg.qr(g.standard_normal((n, p)))
    V, _ = np.linalg.qr(g.standard_normal((p, p)))
    A = (U * np.geomspace(1.0, 1.0 / cond, p)) @ V.T
    Ad = _dev(A, dt)
    Aw = Ad.double().cpu().numpy()
    Rw = np.linalg.qr(Aw, mode="r")
    Rw = np.sign(np.diag(Rw))[:, None] * Rw
    R = _dev(np.full((p, p), 3.0), torch.float64)
    info = torch.full((1,), 5, dtype=torch.int32, device="cuda")
    D.tsqr_r(Ad, R, info, cond=info)
    got = R.cpu().numpy()
    assert int(info.item()) == 0
    assert np.array_equal(got, np.triu(got)) and np.all(np.diag(got) >= 0)
    assert np.linalg.norm(got - Rw) <= 1e-13 * np.linalg.norm(Rw) * max(1.0, np.sqrt(n) / 30)
    # R^T R reproduces the Gram to working accuracy
    assert np.linalg.norm(got.T @ got - Aw.T @ Aw) <= 1e-13 * np.linalg.norm(Aw) ** 2
    R2 = _dev(np.full((p, p), 3.0), torch.float64)
    zero = torch.zeros(1, dtype=torch.int32, device="cuda")
    D.tsqr_r(Ad, R2, zero, cond=zero)
    assert np.all(R2.cpu().numpy() == 3.0)
