"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the CPU oracle.

Tolerances (north star): R within 1e-10 relative in all-fp64 mode and 1e-5
in fp32-coarse mode; Step 3 bit-exact; the SRHT / rademacher / identity
sketches to fp64 reassociation level (1e-13 relative)."""

import math

import numpy as np
import pytest
import torch

import goldens
from oracle import sketches as osk
from oracle import sweep as osw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_2111_14641_b200 import _device, rbgs, sketching

    return rbgs, sketching, _device


def _dev(A, dtype=torch.float64):
    from paper_2111_14641_b200 import _device as D

    return D.to_cm(torch.from_numpy(np.asfortranarray(A)), dtype, "cuda")


# ---------------------------------------------------------------------------
# K3 projection

@pytest.mark.parametrize("t", range(4))
def test_project_bitexact_vs_reference(pkg, t):
    rbgs, sketching, D = pkg
    z = goldens.load("gemm")
    Q, X, W = z[f"Q{t}"], z[f"X{t}"], z[f"W{t}"]
    for compute, want in ((0, z[f"coarse{t}"]), (1, z[f"fine{t}"])):
        Qd = _dev(Q, torch.float32 if compute == 0 else torch.float64)
        out = D.empty_cm(W.shape[0], W.shape[1], Qd.dtype, "cuda")
        norms = torch.zeros(2, dtype=torch.float64, device="cuda")
        D.project(Qd, _dev(X), _dev(W), out, compute, 0, norms)
        got = out.double().cpu().numpy()
        assert np.array_equal(got, want), f"compute={compute}: {np.sum(got != want)} mismatches"
        nw, nq = norms.cpu().numpy()
        assert math.isclose(nw, np.sum(W * W), rel_tol=1e-13)
        assert math.isclose(nq, np.sum(want * want), rel_tol=1e-13)


def test_project_fp32_inputs_bitexact_large(pkg):
    """Large random instance, binary32 storage, vs the oracle loop (kernels.py:171-209)."""
    rbgs, sketching, D = pkg
    g = np.random.Generator(np.random.Philox(9))
    for n, c, p in [(100_003, 96, 40), (4099, 200, 64), (7, 3, 1), (1000, 0, 13)]:
        Q = g.standard_normal((n, c)).astype(np.float32)
        X = g.standard_normal((c, p))
        W = g.standard_normal((n, p)).astype(np.float32)
        want = osw.project(Q, X, W, "coarse")
        out = D.empty_cm(n, p, torch.float32, "cuda")
        D.project(_dev(Q, torch.float32) if c else None, _dev(X) if c else None, _dev(W, torch.float32), out, 0, 0)
        got = out.double().cpu().numpy()
        assert np.array_equal(got, want), (n, c, p, int(np.sum(got != want)))


def test_project_fma_mode_close(pkg):
    rbgs, sketching, D = pkg
    g = np.random.Generator(np.random.Philox(10))
    n, c, p = 20000, 64, 32
    Q = g.standard_normal((n, c)).astype(np.float32)
    X = g.standard_normal((c, p))
    W = g.standard_normal((n, p)).astype(np.float32)
    want = osw.project(Q, X, W, "coarse")
    out = D.empty_cm(n, p, torch.float32, "cuda")
    D.project(_dev(Q, torch.float32), _dev(X), _dev(W, torch.float32), out, 0, 1)
    got = out.double().cpu().numpy()
    scale = np.abs(Q).astype(np.float64) @ np.abs(X) + np.abs(W)
    assert np.all(np.abs(got - want) <= 2 * c * 2.0 ** -24 * scale)


# ---------------------------------------------------------------------------
# K1/K2 sketches

def test_reference_kind_sketches_vs_golden(pkg):
    rbgs, sketching, D = pkg
    z = goldens.load("sketch")
    t = 0
    while f"spec{t}" in z.files:
        kind, k, n, seed = [x.decode() for x in z[f"spec{t}"]]
        op = sketching.SketchOperator(kind, int(k), int(n), int(seed))
        Y = sketching.apply(op, z[f"X{t}"]).data
        want = z[f"Y{t}"]
        tol = 0.0 if kind == "identity" else 1e-13
        assert np.linalg.norm(Y - want) <= tol * np.linalg.norm(want), (kind, k, n)
        # column-wise linearity (test_sketching.py:149-156): bitwise
        Y1 = sketching.apply(op, z[f"X{t}"][:, 1:2]).data
        assert np.array_equal(Y[:, 1:2], Y1)
        t += 1


def test_gaussian_table_matches_oracle(pkg):
    rbgs, sketching, D = pkg
    for k, n, seed, row0 in [(37, 50, 20240917, 0), (1600, 3000, 7, 0), (9, 5, 7, 2 ** 33), (81, 4096, 3, 1000)]:
        op = sketching.gaussian_operator(k, row0 + n, seed)
        tab = op.device_tables("cuda", row0, n)
        flat = tab["theta"].cpu().numpy().reshape(-1)
        ldt = tab["ldt"]
        r = np.arange(k)[:, None]
        i = np.arange(n)[None, :]
        KT = ldt // 128
        base = (((r // 128) * KT + i // 128) * 2) * 16384 + ((i % 128) // 16) * 2048 + (r % 128) * 16 + i % 16
        hi = flat[base].view(np.int8).astype(np.int32)
        lo = flat[base + 16384].astype(np.int32)
        got = (hi * 256 + lo).astype(np.int16)
        want = osk.gaussian_int16(seed, k, np.arange(row0, row0 + n))
        bad = np.sum(got != want)
        # CUDA and glibc log/sincos may differ by an ulp; a flip of the
        # rounded grid value needs g within 1e-13 of a half-step: ~never
        assert bad == 0 or (bad <= 1 and np.max(np.abs(got.astype(int) - want)) <= 1), bad


@pytest.mark.parametrize("kind", ["gaussian", "sparse_sign", "srht", "rademacher"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_sketch_vs_oracle(pkg, kind, dtype):
    rbgs, sketching, D = pkg
    g = np.random.Generator(np.random.Philox(12))
    n, k, cols = 5000, 240, 7
    X = g.standard_normal((n, cols))
    if dtype == torch.float32:
        X = X.astype(np.float32).astype(np.float64)
    if kind == "gaussian":
        op, oop = sketching.gaussian_operator(k, n, 5), osk.OracleSketch("gaussian", k, n, 5)
    elif kind == "sparse_sign":
        op, oop = sketching.sparse_sign_operator(k, n, 5), osk.OracleSketch("sparse_sign", k, n, 5)
    else:
        op, oop = sketching.SketchOperator(kind, k, n, 5), osk.OracleSketch(kind, k, n, 5)
    Xd = _dev(X, dtype)
    out = D.empty_cm(k, cols, torch.float64, "cuda")
    sketching.sketch_into(op, Xd, out)
    got = out.cpu().numpy()
    want = osk.apply(oop, X)
    # binary32 gaussian sketches run on the tensor pipe (exact byte-split
    # products, inputs fixed-point at 2^-46 of each 16384-row chunk max)
    tol = 1e-11 if (kind == "gaussian" and dtype == torch.float32) else 1e-13
    assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want), kind


@pytest.mark.parametrize("n,k,cols", [(100, 37, 1), (8192, 128, 16), (20_001, 300, 40), (70_000, 1600, 64),
                                      (9000, 129, 5)])
def test_gaussian_tensor_pipe_vs_fp64(pkg, n, k, cols):
    """tcgen05 kind::i8 gaussian sketch vs the fp64 CUDA-core kernel and the
    oracle, on columns with 10 decades of dynamic range."""
    rbgs, sketching, D = pkg
    g = np.random.Generator(np.random.Philox(n + k))
    X = g.standard_normal((n, cols)) * np.logspace(0, -10, cols)
    X[::7] *= 1e-3  # rows far below their chunk max
    X = X.astype(np.float32).astype(np.float64)
    op = sketching.gaussian_operator(k, n, 99)
    tab = op.device_tables("cuda", 0, n)
    Xd = _dev(X, torch.float32)
    res = {}
    for mode in ("tensor", "fp64"):
        out = D.empty_cm(k, cols, torch.float64, "cuda")
        D.sketch_gaussian(Xd, tab["theta"], tab["ldt"], k, 1.0 / (2048 * math.sqrt(k)), out, False, mode)
        res[mode] = out.cpu().numpy()
    want = osk.apply(osk.OracleSketch("gaussian", k, n, 99), X)
    for j in range(cols):
        wn = np.linalg.norm(want[:, j])
        assert np.linalg.norm(res["fp64"][:, j] - want[:, j]) <= 1e-13 * wn
        assert np.linalg.norm(res["tensor"][:, j] - want[:, j]) <= 1e-11 * wn, (j, np.linalg.norm(
            res["tensor"][:, j] - want[:, j]) / wn)
    # accumulate flag adds
    out = D.empty_cm(k, cols, torch.float64, "cuda")
    out.copy_(torch.from_numpy(res["tensor"]))
    D.sketch_gaussian(Xd, tab["theta"], tab["ldt"], k, 1.0 / (2048 * math.sqrt(k)), out, True, "tensor")
    assert np.allclose(out.cpu().numpy(), 2 * res["tensor"], rtol=1e-15, atol=0)


@pytest.mark.parametrize("c1,c2", [(64, 64), (64, 50), (49, 64)])
def test_gaussian_tensor_pair_matches_separate_calls(pkg, c1, c2):
    """More than 96 columns: one launch of CTA pairs sharing the table stream
    gives, per input, the bits of that input's own launch."""
    rbgs, sketching, D = pkg
    n, k = 70_001, 300
    g = np.random.Generator(np.random.Philox(c1 + c2))
    X = (g.standard_normal((n, c1 + c2)) * np.logspace(0, -6, c1 + c2)).astype(np.float32)
    op = sketching.gaussian_operator(k, n, 5)
    tab = op.device_tables("cuda", 0, n)
    Xd = _dev(X.astype(np.float64), torch.float32)
    A, B = Xd[:, :c1], Xd[:, c1:]
    sc = 1.0 / (2048 * math.sqrt(k))
    oa, ob = D.empty_cm(k, c1, torch.float64, "cuda"), D.empty_cm(k, c2, torch.float64, "cuda")
    D.sketch_gaussian2(A, B, tab["theta"], tab["ldt"], k, sc, oa, ob, False, "tensor")
    sa, sb = D.empty_cm(k, c1, torch.float64, "cuda"), D.empty_cm(k, c2, torch.float64, "cuda")
    D.sketch_gaussian(A, tab["theta"], tab["ldt"], k, sc, sa, False, "tensor")
    D.sketch_gaussian(B, tab["theta"], tab["ldt"], k, sc, sb, False, "tensor")
    assert torch.equal(oa, sa) and torch.equal(ob, sb)
    want = osk.apply(osk.OracleSketch("gaussian", k, n, 5), X.astype(np.float64))
    got = np.concatenate([oa.cpu().numpy(), ob.cpu().numpy()], axis=1)
    for j in range(c1 + c2):
        wn = np.linalg.norm(want[:, j])
        assert np.linalg.norm(got[:, j] - want[:, j]) <= 1e-11 * wn, j


@pytest.mark.parametrize("scale", [1e-30, 1e-40, 1e30, 1.0])
def test_gaussian_tensor_extreme_magnitudes(pkg, scale):
    """Chunk exponents at both ends of binary32: 2^(46-E) leaves the normal
    binary32 range below ~1e-25 (the pre-pass then scales in binary64),
    subnormal entries, exact zeros and an all-zero column."""
    rbgs, sketching, D = pkg
    n, k, cols = 40_000, 200, 6
    g = np.random.Generator(np.random.Philox(int(-math.log10(scale)) + 50))
    X = g.standard_normal((n, cols)) * scale
    X[::5, 1] *= 1e-6
    X[::3, 2] = 0.0
    X[:, 3] = 0.0
    X[:100, 4] = 1e-45  # binary32 subnormals (2^-149)
    X = X.astype(np.float32).astype(np.float64)
    op = sketching.gaussian_operator(k, n, 17)
    tab = op.device_tables("cuda", 0, n)
    Xd = _dev(X, torch.float32)
    sc = 1.0 / (2048 * math.sqrt(k))
    res = {}
    for mode in ("tensor", "fp64"):
        out = D.empty_cm(k, cols, torch.float64, "cuda")
        D.sketch_gaussian(Xd, tab["theta"], tab["ldt"], k, sc, out, False, mode)
        res[mode] = out.cpu().numpy()
    assert np.all(np.isfinite(res["tensor"]))
    assert np.all(res["tensor"][:, 3] == 0.0)
    for j in range(cols):
        wn = np.linalg.norm(res["fp64"][:, j])
        assert np.linalg.norm(res["tensor"][:, j] - res["fp64"][:, j]) <= 1e-11 * wn, j


def test_gaussian_prepass_variants_same_bits(pkg):
    """The streaming pre-pass (chunk_max + encode_planes), the single-kernel
    split_planes (RB_SPLIT_MODE=1) and its binary64 conversion path
    (RB_SPLIT_SLOW=1) write the same planes: the sketch bits agree."""
    import os
    import subprocess
    import sys
    code = r"""
import hashlib, math, sys, torch
sys.path.insert(0, %r)
from paper_2111_14641_b200 import _device as D, sketching
g = torch.Generator().manual_seed(4)
n, k = 50_001, 300
X = (torch.randn(n, 70, generator=g, dtype=torch.float64) * torch.logspace(0, -9, 70, dtype=torch.float64))
X[::4] *= 1e-20
Xd = X.to(torch.float32).cuda().t().contiguous().t()
tab = sketching.gaussian_operator(k, n, 3).device_tables("cuda", 0, n)
o1 = D.empty_cm(k, 30, torch.float64, "cuda"); o2 = D.empty_cm(k, 40, torch.float64, "cuda")
D.sketch_gaussian2(Xd[:, :30], Xd[:, 30:], tab["theta"], tab["ldt"], k, 1.0, o1, o2, False, "tensor")
o3 = D.empty_cm(k, 60, torch.float64, "cuda")
D.sketch_gaussian(Xd[:, 10:], tab["theta"], tab["ldt"], k, 1.0, o3, False, "tensor")
print(hashlib.sha256(o1.cpu().numpy().tobytes() + o2.cpu().numpy().tobytes() + o3.cpu().numpy().tobytes()).hexdigest())
""" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),)
    shas = set()
    for env in ({}, {"RB_SPLIT_MODE": "1"}, {"RB_SPLIT_SLOW": "1"}):
        e = dict(os.environ)
        e.pop("RB_SPLIT_MODE", None)
        e.pop("RB_SPLIT_SLOW", None)
        e.update(env)
        out = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        shas.add(out.stdout.strip().splitlines()[-1])
    assert len(shas) == 1, shas


def test_fused_lookahead_pair_sketch_is_bitwise_neutral(pkg):
    """p = 64: [Q'_i | W_(i+1)] (128 columns) runs as one paired launch."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.kernels import BlockPartition
    import goldens as G

    n, m, p, k = 20_000, 192, 64, 400
    W = G.trig_family(n, m, 9).astype(np.float32)
    th = sketching.gaussian_operator(k, n, 4)
    cfg = rbgs.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
    f = rbgs.rbgs(W, th, cfg)
    sw = rbgs.RbgsSweep(n, th, cfg)
    Wd = _dev(W.astype(np.float64), torch.float32)
    for b in range(m // p):
        sw.push_block(Wd[:, b * p:(b + 1) * p])
    g = sw.finish()
    assert np.array_equal(f.R.data, g.R.data)
    assert np.array_equal(f.Q.data, g.Q.data)


@pytest.mark.parametrize("kind", ["gaussian", "sparse_sign", "srht"])
def test_sharded_sketch_sums_to_whole(pkg, kind):
    """Virtual shards on one GPU: per-shard partial sketches (global row
    keys) summed on the host equal the unsharded sketch."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.comm import RowShard

    g = np.random.Generator(np.random.Philox(13))
    n, k, cols = 3 * 4096 + 100, 128, 5
    X = g.standard_normal((n, cols))
    op = {"gaussian": lambda: sketching.gaussian_operator(k, n, 3),
          "sparse_sign": lambda: sketching.sparse_sign_operator(k, n, 3),
          "srht": lambda: sketching.SketchOperator("srht", k, n, 3)}[kind]()
    whole = D.empty_cm(k, cols, torch.float64, "cuda")
    sketching.sketch_into(op, _dev(X), whole)
    acc = np.zeros((k, cols))
    for r in range(4):
        sh = RowShard.split(n, 4, r, align=2048)
        part = D.empty_cm(k, cols, torch.float64, "cuda")
        sketching.sketch_into(op, _dev(X[sh.row0:sh.row0 + sh.n_local]), part, row0=sh.row0)
        acc += part.cpu().numpy()
    w = whole.cpu().numpy()
    assert np.linalg.norm(acc - w) <= 1e-13 * np.linalg.norm(w)


def test_srht_large_pruned_fwht(pkg):
    """n_pad = 2^16 with 16 tiles and k = 2048 samples vs the full FWHT."""
    rbgs, sketching, D = pkg
    g = np.random.Generator(np.random.Philox(14))
    n, k = 50_000, 2048
    X = g.standard_normal((n, 3))
    op = sketching.SketchOperator("srht", k, n, 21)
    got = sketching.apply(op, X).data
    want = osk.apply(osk.OracleSketch("srht", k, n, 21), X)
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


# ---------------------------------------------------------------------------
# full sweep vs golden

CASES = goldens.rbgs_cases()
SKIP = {}


def _make_op(sketching, c):
    if c["kind"] == "gaussian":
        return sketching.gaussian_operator(c["k"], c["n"], c["seed"])
    if c["kind"] == "sparse_sign":
        return sketching.sparse_sign_operator(c["k"], c["n"], c["seed"])
    return sketching.SketchOperator(c["kind"], c["k"], c["n"], c["seed"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_rbgs_vs_reference_golden(pkg, name):
    rbgs, sketching, D = pkg
    if name in SKIP:
        pytest.skip(SKIP[name])
    c = CASES[name]
    from paper_2111_14641_b200.kernels import BlockPartition, COARSE, FINE

    part = BlockPartition(max(c["widths"]), len(c["widths"]), sum(c["widths"]), widths=c["widths"])
    cfg = rbgs.RbgsConfig(partition=part, ls_solver=c["ls_solver"], interblock=c["interblock"],
                          coarse=COARSE if c["coarse"] == "coarse" else FINE,
                          fine=COARSE if c["fine"] == "coarse" else FINE,
                          certify_blocks=c["certify_blocks"], resketch=c["resketch"])
    f = rbgs.rbgs(c["W"], _make_op(sketching, c), cfg)
    R = f.R.data
    dR = goldens.rel(R, c["R"])
    tol = 1e-10 if c["coarse"] == "fine" else 1e-5
    assert dR <= tol, f"{name}: ||dR||/||R|| = {dR:.3e} > {tol}"
    assert np.array_equal(R, np.triu(R))
    assert np.all(np.diag(R) >= 0)
    qtol = 1e-9 if c["coarse"] == "fine" else 5e-5
    assert goldens.rel(f.Q.data, c["Q"]) <= qtol
    assert goldens.rel(f.P.data, c["P"]) <= 1e-12
    d, dt = c["cert"]
    if c["coarse"] == "fine":
        assert abs(f.cert.delta - d) <= 1e-2 * d + 1e-12, (f.cert.delta, d)
        assert abs(f.cert.delta_tilde - dt) <= 1e-2 * dt + 1e-14, (f.cert.delta_tilde, dt)
    else:
        # two-precision certificates sit at the binary32 rounding level:
        # "same order" (north star), i.e. within a factor 1.5
        assert d / 1.5 <= f.cert.delta <= 1.5 * d + 1e-12, (f.cert.delta, d)
        assert dt / 1.5 <= f.cert.delta_tilde <= 1.5 * dt + 1e-14, (f.cert.delta_tilde, dt)
    if c["certify_blocks"]:
        assert np.allclose(f.cert.per_block_ortho, c["pbo"], rtol=1e-2, atol=1e-12)
        assert np.allclose(f.cert.per_block_resid, c["pbr"], rtol=1e-2, atol=1e-14)


def test_rbgs_errors_vs_golden(pkg):
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.errors import DependentBlockError, InterblockError
    from paper_2111_14641_b200.kernels import BlockPartition

    z = goldens.load("errors")
    th = sketching.SketchOperator("srht", 60, 300, 7)
    with pytest.raises(DependentBlockError) as e:
        rbgs.rbgs(z["vanished/W"], th, rbgs.RbgsConfig(partition=BlockPartition(5, 3, 15)))
    assert e.value.block == int(z["vanished/block"])
    with pytest.raises(InterblockError) as e:
        rbgs.rbgs(z["interblock/W"], th, rbgs.RbgsConfig(partition=BlockPartition(5, 3, 15),
                                                         interblock="sketched_cholqr(1)"))
    assert e.value.block == int(z["interblock/block"])
    assert "sketch size k" in str(e.value)


def test_sweep_state_semantics(pkg):
    """blocks_done / cols_done / pending_P semantics on failure (rbgs.py:352-399)."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.errors import DependentBlockError
    from paper_2111_14641_b200.kernels import BlockPartition

    g = np.random.Generator(np.random.Philox(27))
    W = np.hstack([g.standard_normal((300, 10)), np.zeros((300, 5))])
    th = sketching.SketchOperator("srht", 60, 300, 7)
    sw = rbgs.RbgsSweep(300, th, rbgs.RbgsConfig(partition=BlockPartition(5, 3, 15)))
    sw.push_block(W[:, :5])
    sw.push_block(W[:, 5:10])
    with pytest.raises(DependentBlockError):
        sw.push_block(W[:, 10:])
    assert sw.blocks_done == 2 and sw.cols_done == 10
    assert sw.pending_P is not None and sw.pending_P.shape == (60, 5)
    assert np.allclose(sw.pending_P.data, 0.0)


def test_fused_lookahead_sketch_is_bitwise_neutral(pkg):
    """rbgs() fuses the next block's Step-1 sketch into this block's Step-4
    pass; pushing blocks one by one (no lookahead) must give the same bits."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.kernels import BlockPartition
    import goldens as G

    n, m, p, k = 20_000, 60, 12, 200
    W = G.trig_family(n, m, 5).astype(np.float32)
    th = sketching.gaussian_operator(k, n, 3)
    cfg = rbgs.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
    f = rbgs.rbgs(W, th, cfg)
    sw = rbgs.RbgsSweep(n, th, cfg)
    Wd = _dev(W.astype(np.float64), torch.float32)
    for b in range(m // p):
        sw.push_block(Wd[:, b * p:(b + 1) * p])
    g = sw.finish()
    assert np.array_equal(f.R.data, g.R.data)
    assert np.array_equal(f.Q.data, g.Q.data)
    assert np.array_equal(f.S.data, g.S.data)


def test_overwrite_w_and_pinned_upload_are_bitwise_neutral(pkg):
    """Q written over W's storage (DeviceConfig.overwrite_w; always for the
    private upload of a pinned host W) gives the same bits as a separate Q,
    and the deferred-status one-shot path matches the eager per-block one."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.kernels import BlockPartition
    import goldens as G

    n, m, p, k = 20_000, 60, 12, 200
    W = G.trig_family(n, m, 5).astype(np.float32)
    th = sketching.gaussian_operator(k, n, 3)
    cfg = rbgs.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
    f = rbgs.rbgs(W, th, cfg)
    Wd = _dev(W.astype(np.float64), torch.float32)
    g = rbgs.rbgs(Wd, th, cfg, rbgs.DeviceConfig(overwrite_w=True))
    assert g.Q._dev.data_ptr() == Wd.data_ptr()
    Wh = torch.empty((m, n), dtype=torch.float32).pin_memory().t()
    Wh.copy_(torch.from_numpy(W))
    h = rbgs.rbgs(Wh, th, cfg)
    for other in (g, h):
        assert np.array_equal(f.R.data, other.R.data)
        assert np.array_equal(f.Q.data, other.Q.data)
        assert np.array_equal(f.S.data, other.S.data)
    import os
    os.environ["RB_EAGER_STATUS"] = "1"
    try:
        e = rbgs.rbgs(W, th, cfg)
    finally:
        del os.environ["RB_EAGER_STATUS"]
    assert np.array_equal(f.R.data, e.R.data) and np.array_equal(f.Q.data, e.Q.data)


def test_deferred_status_replays_to_the_reference_exception(pkg):
    """A failing block in the one-shot (deferred-status) path raises the same
    exception, at the same block, as the eager sweep (rbgs.py:373-399)."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.errors import DependentBlockError
    from paper_2111_14641_b200.kernels import BlockPartition

    g = np.random.Generator(np.random.Philox(27))
    W = np.hstack([g.standard_normal((3000, 10)), np.zeros((3000, 5)), g.standard_normal((3000, 5))])
    th = sketching.gaussian_operator(200, 3000, 7)
    cfg = rbgs.RbgsConfig(partition=BlockPartition.uniform(20, 5), interblock="sketched_cholqr(1)")
    before = rbgs.REPLAYS
    with pytest.raises(DependentBlockError) as ei:
        rbgs.rbgs(W.astype(np.float32), th, cfg)
    assert ei.value.block == 3
    assert rbgs.REPLAYS == before + 1


@pytest.mark.parametrize("solver", ["richardson", "bmgs_reorth", "cg_normal", "householder_direct"])
def test_ls_solvers_coarse_precision_vs_oracle(pkg, solver):
    """Step-2 solvers with prec = COARSE run in binary32 (rbgs.py:144-212,
    prec.dtype); compared with the oracle's float32 numpy restatement."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.kernels import COARSE, FINE

    g = np.random.Generator(np.random.Philox(31))
    k, c, p = 300, 40, 8
    S, _ = np.linalg.qr(g.standard_normal((k, c)))
    S = S @ np.diag(1 + 0.01 * g.standard_normal(c))
    P = g.standard_normal((k, p))
    if solver == "richardson":
        got = rbgs.ls_richardson(S, P, 5, COARSE).data
        want = osw.ls_richardson(S, P, 5, "coarse")
        ref64 = rbgs.ls_richardson(S, P, 5, FINE).data
    elif solver == "bmgs_reorth":
        blocks = [S[:, :20], S[:, 20:]]
        got = rbgs.ls_bmgs_reorth(blocks, P, 2, COARSE).data
        want = osw.ls_bmgs_reorth(blocks, P, 2, "coarse")
        ref64 = rbgs.ls_bmgs_reorth(blocks, P, 2, FINE).data
    elif solver == "cg_normal":
        got = rbgs.ls_cg_normal(S, P, 10, COARSE).data
        want = osw.ls_cg_normal(S, P, 10, "coarse")
        ref64 = rbgs.ls_cg_normal(S, P, 10, FINE).data
    else:
        got = rbgs.ls_householder_direct(S, P, COARSE).data
        want = osw.ls_householder_direct(S, P, "coarse")
        ref64 = rbgs.ls_householder_direct(S, P, FINE).data
    # binary32 values, same answer as the float32 restatement to binary32
    # rounding, and visibly different from the binary64 solve
    assert np.array_equal(got, got.astype(np.float32).astype(np.float64))
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want)
    assert np.linalg.norm(got - ref64) > 0


# ---------------------------------------------------------------------------
# Krylov drivers (krylov.py:110-281) vs the reference golden vectors

def _lap1d(n):
    import scipy.sparse as sp
    return sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")


def test_arnoldi_vs_reference_golden(pkg):
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200 import krylov, operators

    z = goldens.load("krylov")
    n = 200
    A = operators.CsrOperator(_lap1d(n))
    arn = krylov.rbgs_arnoldi(A, z["arn/B"], sketching.SketchOperator("srht", 64, n, 1), 5)
    # two-precision (reference default coarse = COARSE): binary32 rounding level
    assert goldens.rel(arn.H.data, z["arn/H"]) <= 1e-5
    assert goldens.rel(arn.Q.data, z["arn/Q"]) <= 5e-5
    assert goldens.rel(arn.R_first.data, z["arn/Rf"]) <= 1e-5
    assert goldens.rel(arn.P.data, z["arn/P"]) <= 1e-5


def test_block_gmres_vs_reference_golden(pkg):
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200 import krylov, operators

    z = goldens.load("krylov")
    d = np.arange(1.0, 101.0)
    A = operators.DenseOperator(np.diag(d))
    rep = krylov.block_gmres(A, z["gm/b"], sketching.SketchOperator("srht", 48, 100, 21), 12)
    assert goldens.rel(rep.solution.data, z["gm/x"]) <= 1e-5
    hist = np.array(rep.residual_history)
    assert hist.shape == z["gm/hist"].shape
    assert np.array_equal(hist[:, 0], z["gm/hist"][:, 0])
    assert np.allclose(hist[:, 1], z["gm/hist"][:, 1], rtol=1e-3, atol=1e-7)
    # happy breakdown: identity operator, block 2 vanishes
    rep = krylov.block_gmres(operators.DenseOperator(np.eye(50)), z["gmid/B"],
                             sketching.SketchOperator("identity", 50, 50, 0), 4)
    assert rep.breakdown == int(z["gmid/breakdown"]) == 2
    assert goldens.rel(rep.solution.data, z["gmid/x"]) <= 1e-6


def test_block_gmres_poisson3d_vs_reference_golden(pkg):
    """C4 shape family at a reduced grid: 7-point 3-D Poisson, sparse-sign
    sketch, 2 restarts, sketched CholQR."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200 import krylov, operators

    z = goldens.load("krylov")
    nx = int(z["p3/nx"])
    A = operators.Poisson3D(nx, nx, nx)
    op = sketching.sparse_sign_operator(72, nx ** 3, 11)
    cfg = rbgs.RbgsConfig(interblock="sketched_cholqr(1)")
    rep = krylov.block_gmres(A, z["p3/B"], op, 8, restarts=2, cfg=cfg)
    assert goldens.rel(rep.solution.data, z["p3/x"]) <= 1e-4
    hist = np.array(rep.residual_history)
    assert hist.shape == z["p3/hist"].shape
    assert np.allclose(hist[:, 1], z["p3/hist"][:, 1], rtol=1e-2)
    assert np.allclose(np.array(rep.basis_cond_history), z["p3/conds"], rtol=1e-2)


def test_block_gmres_sketched_diagnostics(pkg):
    """diagnostics="sketched" (the reference's per-iterate
    diagnostics, krylov.py:247-257, made optional): same solution and final
    true residual as the full mode; the k-dimensional residual estimates sit
    inside the epsilon-embedding bracket of the true ones."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200 import krylov, operators

    z = goldens.load("krylov")
    nx = int(z["p3/nx"])
    A = operators.Poisson3D(nx, nx, nx)
    op = sketching.sparse_sign_operator(72, nx ** 3, 11)
    cfg = rbgs.RbgsConfig(interblock="sketched_cholqr(1)")
    full = krylov.block_gmres(A, z["p3/B"], op, 8, restarts=2, cfg=cfg)
    sk = krylov.block_gmres(A, z["p3/B"], op, 8, restarts=2, cfg=cfg, diagnostics="sketched")
    assert goldens.rel(sk.solution.data, full.solution.data) <= 1e-12
    hf, hs = np.array(full.residual_history), np.array(sk.residual_history)
    assert hf.shape == hs.shape
    last = [7 * c - 1 for c in (1, 2)]  # the cycle's last iterate carries the true residual
    assert np.allclose(hs[last, 1], hf[last, 1], rtol=1e-10)
    assert np.all(hs[:, 1] <= 2.0 * hf[:, 1]) and np.all(hs[:, 1] >= 0.5 * hf[:, 1])
    cf, cs = np.array(full.basis_cond_history), np.array(sk.basis_cond_history)
    # cond(S) brackets cond(Q) through the embedding's epsilon; with k = 72 for
    # up to 32 columns epsilon is large (cond(Q) reaches 4.5 while S is
    # sketch-orthonormal, cond 1): the bracket holds with a wide factor only
    assert np.all(cs <= 6.0 * cf) and np.all(cs >= cf / 6.0)
    with pytest.raises(ValueError):
        krylov.block_gmres(A, z["p3/B"], op, 8, diagnostics="none")


def test_sparse_sign_table_path_matches_hashed_path(pkg):
    """The pre-bucketed table (fixed summation order) and the per-row hashing
    path sketch with the same operator; ragged tiles and shards included."""
    rbgs, sketching, D = pkg
    g = np.random.Generator(np.random.Philox(77))
    for n, k, nnz, row0, cols in [(5000, 120, 8, 0, 5), (1024, 64, 3, 0, 4), (3001, 488, 8, 7, 9),
                                  (2500, 40, 16, 2048, 1)]:
        X = _dev(g.standard_normal((n, cols)))
        a = torch.zeros(k, cols, dtype=torch.float64, device="cuda").t().contiguous().t()
        b = a.clone()
        D.sketch_sparse_sign(X, row0, 11, k, nnz, a)
        tab = D.sparse_sign_table(11, k, nnz, row0, n, X.device)
        D.sketch_sparse_sign(X, row0, 11, k, nnz, b, table=tab)
        D.sketch_sparse_sign(X, row0, 11, k, nnz, b, accumulate=True, table=tab)
        ref = a.cpu().numpy()
        got = b.cpu().numpy() / 2
        assert np.allclose(got, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max()), (n, k, nnz)
        # deterministic: a second table-path call gives the same bits
        c = torch.zeros_like(a)
        D.sketch_sparse_sign(X, row0, 11, k, nnz, c, table=tab)
        assert torch.equal(c * 2, b)


def test_rbgs_plan_graph_replay_matches_eager(pkg):
    """RbgsPlan (captured CUDA graph) == eager rbgs() bit for bit, follows
    new contents of W, and raises the reference exception on a failing
    block (eager re-run)."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.errors import DependentBlockError
    from paper_2111_14641_b200.kernels import BlockPartition
    import goldens as G

    n, m, p, k = 20_000, 60, 12, 200
    th = sketching.gaussian_operator(k, n, 3)
    cfg = rbgs.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
    W1 = G.trig_family(n, m, 5).astype(np.float32)
    W2 = (np.random.Generator(np.random.Philox(8)).standard_normal((n, m)) @ np.diag(np.logspace(0, -5, m)))
    Wd = _dev(W1.astype(np.float64), torch.float32)
    plan = rbgs.RbgsPlan(Wd, th, cfg)
    for Wh in (W1, W2.astype(np.float32), W1):
        Wd.copy_(torch.from_numpy(Wh.astype(np.float32)))
        got = plan.replay()
        want = rbgs.rbgs(Wh.astype(np.float32), th, cfg)
        assert np.array_equal(got.R.data, want.R.data)
        assert np.array_equal(got.Q.data, want.Q.data)
        assert got.cert == want.cert
    Wbad = W1.copy()
    Wbad[:, 24:36] = 0.0
    Wd.copy_(torch.from_numpy(Wbad))
    with pytest.raises(DependentBlockError) as ei:
        plan.replay()
    assert ei.value.block == 3


def test_fused_scaling_is_bitwise_neutral(pkg):
    """One-shot sweeps fold block i-1's Step-5 scaling into block i's
    projection (rb_project_trsm); bits equal the separate kernels, for a
    ragged partition too (widths 40, 40, 24, 40 -> fallback where pf > p)."""
    import os
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.kernels import BlockPartition
    import goldens as G

    n, k = 30_000, 300
    W = G.trig_family(n, 144, 6).astype(np.float32)
    th = sketching.gaussian_operator(k, n, 4)
    for part in (BlockPartition.uniform(144, 36), BlockPartition(40, 4, 144, widths=(40, 40, 24, 40))):
        cfg = rbgs.RbgsConfig(partition=part, interblock="sketched_cholqr(1)")
        a = rbgs.rbgs(W, th, cfg)
        os.environ["RB_FUSE_SCALING"] = "0"
        try:
            b = rbgs.rbgs(W, th, cfg)
        finally:
            del os.environ["RB_FUSE_SCALING"]
        assert np.array_equal(a.Q.data, b.Q.data)
        assert np.array_equal(a.R.data, b.R.data)
        assert np.array_equal(a.S.data, b.S.data)


@pytest.mark.parametrize("config", ["c2", "c1"])
def test_bench_workload_sample_vs_oracle(pkg, config):
    """The bench workload's own shape (same m, p, k, sketch kind and input
    family) on an 8192-row sample: R against the CPU oracle within the
    north-star tolerance, certificates of the same order (bench.py reports
    the same numbers in cpu_baseline.parity)."""
    import bench

    cfgd = bench.CONFIGS[config]
    _, par = bench._oracle_sample(cfgd, 8192, parity=True)
    tol = 1e-5 if cfgd["coarse"] == "coarse" else 1e-10
    assert par["rel_R_diff"] <= tol, par
    d, do = par["delta"]
    assert abs(d - do) <= 0.05 * do + 1e-12, par


def test_repeat_and_two_stream_determinism(pkg):
    """Race evidence in place of compute-sanitizer (closed on this pool,
    profiles/r02_sanitizer_record.txt): the warp-specialised kernels
    (gauss_tc_partial, project_staged, project_tc2), the last-CTA combine of
    sumsq3 and the cooperative k-dimensional kernels give bitwise identical
    factors (a) run after run and (b) when two factorizations are in flight
    on two streams of the same device at once (the C ABI's per-stream
    workspaces; formerly one constant bank / counter per device)."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.kernels import BlockPartition
    import goldens as G

    n, m, p, k = 65536, 120, 40, 256
    W = G.trig_family(n, m, 5).astype(np.float32)
    Wd = _dev(W.astype(np.float64), torch.float32)
    th = sketching.gaussian_operator(k, n, 3)
    cfg = rbgs.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
    for order in ("reference", "tc"):
        dc = rbgs.DeviceConfig(projection_order=order)
        base = rbgs.rbgs(Wd, th, cfg, dc)
        torch.cuda.synchronize()
        Rb, Qb = base.R.data.copy(), base.Q.data.copy()
        for _ in range(3):
            f = rbgs.rbgs(Wd, th, cfg, dc)
            torch.cuda.synchronize()
            assert np.array_equal(f.R.data, Rb) and np.array_equal(f.Q.data, Qb), order
        import threading

        outs, errs = [], []

        def worker():
            try:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    for _ in range(3):  # (each call ends with one status read of its own stream)
                        outs.append(rbgs.rbgs(Wd, th, cfg, dc))
                s.synchronize()
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        ts = [threading.Thread(target=worker) for _ in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        torch.cuda.synchronize()
        assert not errs, errs
        assert len(outs) == 6
        for f in outs:
            assert np.array_equal(f.R.data, Rb) and np.array_equal(f.Q.data, Qb), order


@pytest.mark.parametrize("fmt", ["coarse", "fine"])
def test_kernels_gemm_bit_identical_to_reference_order(pkg, fmt):
    """kernels.gemm (kernels.py:171-209) on the device: every alpha / beta
    branch of the reference loop, bit for bit against the oracle's
    restatement (itself pinned bit-exact to the reference's golden vectors)."""
    from paper_2111_14641_b200 import kernels as K
    from paper_2111_14641_b200.errors import ShapeError

    prec = K.COARSE if fmt == "coarse" else K.FINE
    g = np.random.Generator(np.random.Philox(31))
    for n, kk, m in [(257, 33, 5), (1024, 96, 70), (64, 1, 3)]:
        A, B, C = g.standard_normal((n, kk)), g.standard_normal((kk, m)), g.standard_normal((n, m))
        for alpha, beta, Cin in [(-1.0, 1.0, C), (1.0, 0.0, None), (1.0, 1.0, C), (-1.0, 2.5, C), (0.5, 1.0, C),
                                 (-2.0, 0.0, None)]:
            got = K.gemm(alpha, A, B, beta, Cin, prec).data
            want = osw.gemm_ordered(alpha, A, B, beta, Cin, fmt)
            assert np.array_equal(got, want), (fmt, n, kk, m, alpha, beta)
    with pytest.raises(ShapeError):
        K.gemm(1.0, np.ones((3, 2)), np.ones((3, 2)))
    with pytest.raises(ShapeError):
        K.gemm(1.0, np.ones((3, 2)), np.ones((2, 2)), beta=1.0)


def test_kernels_factorizations_vs_oracle(pkg):
    """kernels.householder_qr / cholesky / triangular_solve (kernels.py:216-270)
    on the device: values against the oracle's LAPACK restatement, errors with
    the reference's classes and attributes."""
    from paper_2111_14641_b200 import kernels as K
    from paper_2111_14641_b200.errors import NotPositiveDefiniteError, ShapeError, SingularTriangularError

    g = np.random.Generator(np.random.Philox(32))
    A = g.standard_normal((300, 12))
    Q, R = K.householder_qr(A)
    Qo, Ro = osw.householder_qr(A)
    assert np.all(np.diag(R.data) >= 0) and np.allclose(R.data, Ro, rtol=0, atol=1e-12 * np.abs(Ro).max())
    assert np.allclose(Q.data, Qo, rtol=0, atol=1e-12) and np.allclose(Q.data @ R.data, A, atol=1e-12)
    with pytest.raises(ShapeError):
        K.householder_qr(np.ones((2, 3)))
    G = A.T @ A
    Rc = K.cholesky(G).data
    assert np.allclose(Rc, osw.cholesky_upper(G), rtol=1e-12, atol=1e-12) and np.array_equal(Rc, np.triu(Rc))
    Gb = G.copy()
    Gb[4, 4] = -1.0
    with pytest.raises(NotPositiveDefiniteError) as e:
        K.cholesky(Gb)
    assert e.value.column == 5
    with pytest.raises(ShapeError):
        K.cholesky(np.triu(G) + 1.0)
    Bl, Br = g.standard_normal((12, 4)), g.standard_normal((500, 12))
    assert np.allclose(K.triangular_solve(Ro, Bl).data, osw.trsm(Ro, Bl, "left"), rtol=1e-10, atol=1e-12)
    assert np.allclose(K.triangular_solve(Ro, Br, side="right").data, osw.trsm(Ro, Br, "right"), rtol=1e-10,
                       atol=1e-12)
    Rs = Ro.copy()
    Rs[3, 3] = 0.0
    with pytest.raises(SingularTriangularError) as e:
        K.triangular_solve(Rs, Bl)
    assert e.value.index == 3
    with pytest.raises(ValueError):
        K.triangular_solve(Ro, Bl, side="up")


def test_srht_apply_and_materialize_vs_reference_recipe(pkg):
    """sketching.srht_apply / materialize (sketching.py:129-160) on the device
    against the reference recipe restated in numpy (zero-pad, signs, FWHT in
    ascending-h stage order, subsample, 1 / sqrt(k))."""
    rbgs, sketching, D = pkg

    def fwht(Z):
        n = Z.shape[0]
        h = 1
        while h < n:
            Y = Z.reshape(n // (2 * h), 2, -1)
            a = Y[:, 0, :].copy()
            Y[:, 0, :] += Y[:, 1, :]
            Y[:, 1, :] = a - Y[:, 1, :]
            h *= 2
        return Z

    g = np.random.Generator(np.random.Philox(41))
    for n, n_pad, k, cols in [(1, 4, 4, 1), (300, 512, 64, 5), (5000, 8192, 700, 3), (2048, 2048, 1500, 70)]:
        X = g.standard_normal((n, cols))
        signs = g.integers(0, 2, n_pad) * 2.0 - 1.0
        sample = g.permutation(n_pad)[:k]
        Z = np.zeros((n_pad, cols))
        Z[:n] = signs[:n, None] * X
        want = fwht(Z.copy())[sample] / math.sqrt(k)
        got = sketching.srht_apply(X, signs, sample, k)
        assert got.shape == want.shape
        assert np.linalg.norm(got - want) <= 1e-13 * max(np.linalg.norm(want), 1e-300)
    th = sketching.SketchOperator("srht", 24, 100, 3)
    M = sketching.materialize(th)
    Xr = g.standard_normal((100, 4))
    assert M.shape == (24, 100)
    assert np.allclose(M @ Xr, sketching.apply(th, Xr).data, rtol=0, atol=1e-12)


def test_l2_plus_cholqr_survives_gram_breakdown(pkg):
    """The reference default inter-block QR on a block whose l2 condition
    number (1e10) breaks the Gram Cholesky of the l2 stage: the device falls
    through to the Householder R (rb_tsqr_r) like the reference's own
    householder_qr stage (rbgs.py:293-302), without a host branch -- same R as
    the oracle, Q sketch-orthonormal; with the tall QR disabled the last
    resort (one-pass sketched CholQR) is visibly worse or fails."""
    rbgs, sketching, D = pkg

    g = np.random.Generator(np.random.Philox(51))
    n, w, k = 20_000, 12, 160
    U, _ = np.linalg.qr(g.standard_normal((n, w)))
    V, _ = np.linalg.qr(g.standard_normal((w, w)))
    Qp = (U * np.geomspace(1.0, 1e-10, w)) @ V.T
    th = sketching.SketchOperator("srht", k, n, 9)
    Q, R, S = rbgs.interblock_l2_cholqr(Qp, th)
    Qo, Ro, So = osw.interblock_l2_cholqr(Qp, osk.OracleSketch("srht", k, n, 9))
    assert np.linalg.norm(R.data - Ro) <= 1e-6 * np.linalg.norm(Ro)
    G = S.data.T @ S.data
    assert np.linalg.norm(G - np.eye(w)) <= 1e-8
    assert np.linalg.norm(Qp - Q.data @ R.data) <= 1e-12 * np.linalg.norm(Qp)


def test_staged_pageable_upload_is_bitwise_neutral(pkg):
    """rbgs() on a pageable numpy W (the reference-style input) above 64 MB
    takes the staged block-by-block upload (pinned staging ring, host copy
    threads, copy stream): same bits as the factorization of the same W
    already on the device, for Fortran- and C-ordered inputs, and a failing
    block still raises the reference's exception with its block index."""
    rbgs, sketching, D = pkg
    from paper_2111_14641_b200.errors import DependentBlockError
    from paper_2111_14641_b200.kernels import BlockPartition
    import goldens as G

    n, m, p, k = 200_000, 120, 40, 256
    W = G.trig_family(n, m, 5).astype(np.float32)
    assert W.nbytes >= 64 << 20
    th = sketching.gaussian_operator(k, n, 3)
    cfg = rbgs.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
    base = rbgs.rbgs(_dev(W.astype(np.float64), torch.float32), th, cfg)
    torch.cuda.synchronize()
    for Wh in (np.asfortranarray(W), np.ascontiguousarray(W)):
        assert rbgs._stageable(Wh, cfg) is not None
        for _ in range(2):
            f = rbgs.rbgs(Wh, th, cfg)
            assert np.array_equal(f.R.data, base.R.data) and np.array_equal(f.Q.data, base.Q.data)
    Wz = np.asfortranarray(W.copy())
    Wz[:, 80:] = 0.0
    with pytest.raises(DependentBlockError) as e:
        rbgs.rbgs(Wz, th, cfg)
    assert e.value.block == 3
