"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
the host-side logic mirrors the reference (configs, partitions, operator
tables, errors), the sharding / allreduce plumbing works across 2 gloo
ranks, and the integer / tiling algebra the CUDA kernels rely on is exact
(emulated in numpy against the oracle)."""

import math
import os
import socket

import numpy as np
import pytest
import torch

import goldens
from oracle import sketches as osk
from oracle import sweep as osw

from paper_2111_14641_b200 import _lib
from paper_2111_14641_b200.comm import Comm, RowShard
from paper_2111_14641_b200.errors import DependentBlockError, InterblockError, NotPositiveDefiniteError
from paper_2111_14641_b200.kernels import COARSE, FINE, BlockPartition, Matrix, PrecisionSpec


# ---------------------------------------------------------------------------
# the C ABI

def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), set(declared) ^ set(_lib.SIGNATURES)
    assert lib.rb_version().decode().startswith("rbgs_b200")
    assert int(lib.rb_workspace_bytes(10 ** 6, 40, 1600)) > 0
    assert _lib.launch_count() >= 0


def test_library_is_sm100a_native():
    """The shared library carries sm_100a SASS with tcgen05 / TMA instructions."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UTCIMMA" in out        # tcgen05.mma kind::i8
    assert "LDTM" in out           # tcgen05.ld
    assert "UBLKCP" in out or "UTMALDG" in out  # bulk async copies (TMA engine)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    from paper_2111_14641_b200 import rbgs, sketching
    with pytest.raises(_lib.DeviceUnavailable):
        rbgs.rbgs(np.ones((64, 4)), sketching.SketchOperator("srht", 8, 64, 1),
                  rbgs.RbgsConfig(partition=BlockPartition.uniform(4, 2)))


# ---------------------------------------------------------------------------
# host logic mirrors the reference (tests/test_rbgs.py:67-95, test_kernels.py:35-73)

def test_parse_method_and_config_validation():
    from paper_2111_14641_b200.rbgs import CertReport, RbgsConfig, parse_method
    assert parse_method("richardson(5)") == ("richardson", 5)
    assert parse_method("richardson:3") == ("richardson", 3)
    assert parse_method("householder_direct") == ("householder_direct", None)
    assert parse_method("cg_normal") == ("cg_normal", 20)
    with pytest.raises(ValueError):
        parse_method("richardson(0)")
    with pytest.raises(ValueError):
        parse_method("not a method!")
    part = BlockPartition.uniform(4, 2)
    with pytest.raises(ValueError):
        RbgsConfig(partition=part, coarse=FINE, fine=COARSE)
    with pytest.raises(ValueError):
        RbgsConfig(partition=part, ls_solver="gauss_seidel(3)")
    with pytest.raises(ValueError):
        RbgsConfig(partition=part, interblock="gram_schmidt")
    with pytest.raises(ValueError):
        CertReport(-1e-3, 0.0)
    with pytest.raises(ValueError):
        CertReport(0.0, float("nan"))


def test_domain_types():
    assert COARSE.u == 2.0 ** -24 and FINE.u == 2.0 ** -53
    with pytest.raises(ValueError):
        PrecisionSpec("half")
    with pytest.raises(ValueError):
        Matrix(np.array([[1.0, np.nan]]))
    M = Matrix(np.arange(6, dtype=np.float32).reshape(2, 3))
    assert M.data.dtype == np.float64 and M.data.flags.f_contiguous and M.shape == (2, 3)
    part = BlockPartition.uniform(10, 3)
    assert part.block_widths() == (3, 3, 3, 1) and part.offsets() == (0, 3, 6, 9, 10)
    with pytest.raises(ValueError):
        BlockPartition(3, 4, 14)
    assert BlockPartition(3, 4, 10, widths=(1, 3, 3, 3)).offsets() == (0, 1, 4, 7, 10)


def test_error_messages_match_reference():
    e = InterblockError(3, str(NotPositiveDefiniteError(2)))
    assert e.block == 3 and "sketch size k" in str(e) and "not positive definite at column 2" in str(e)
    d = DependentBlockError(4, "projected block vanished")
    assert d.block == 4 and str(d) == "block 4 numerically dependent: projected block vanished"


def test_sketch_operator_tables_match_reference():
    from paper_2111_14641_b200 import sketching
    z = goldens.load("sketch")
    t = 0
    while f"spec{t}" in z.files:
        kind, k, n, seed = [x.decode() for x in z[f"spec{t}"]]
        op = sketching.SketchOperator(kind, int(k), int(n), int(seed))
        if kind == "srht":
            assert np.array_equal(op.sign_diagonal.astype(np.int8), z[f"signs{t}"])
            assert np.array_equal(op.sample_indices, z[f"sample{t}"])
            words = -(-op.n_pad // 2048) * 64
            bits = sketching._pack_bits(op.sign_diagonal < 0, words)
            unpacked = np.unpackbits(bits.view(np.uint8), bitorder="little")[: op.n_pad]
            assert np.array_equal(unpacked.astype(bool), op.sign_diagonal < 0)
        if kind == "rademacher":
            assert np.array_equal(op._signs, z[f"signs{t}"])
        t += 1
    with pytest.raises(ValueError):  # the reference pins this rejection (test_sketching.py:108-110)
        sketching.SketchOperator("gaussian", 4, 5, 0)
    g = sketching.gaussian_operator(80, 1000, 7)
    assert g.kind == "gaussian" and isinstance(g, sketching.SketchOperator)
    s = sketching.sparse_sign_operator(48, 1200, 9, nnz=8)
    assert s.nnz == 8
    assert sketching.to_line(g) == "gaussian 80 1000 7"
    assert sketching.from_line("sparse_sign 48 1200 9").kind == "sparse_sign"


def test_workload_generators_match_golden_family():
    from paper_2111_14641_b200 import workloads
    assert np.array_equal(workloads.trig_host(3000, 40, 7), goldens.trig_family(3000, 40, 7))


# ---------------------------------------------------------------------------
# sharding

@pytest.mark.parametrize("n,world,align", [(10 ** 6, 8, 2048), (2 ** 24, 4, 2048), (1000, 3, 32), (5, 8, 1)])
def test_row_shards_tile_the_rows(n, world, align):
    shards = [RowShard.split(n, world, r, align) for r in range(world)]
    assert shards[0].row0 == 0
    for a, b in zip(shards, shards[1:]):
        assert a.row0 + a.n_local == b.row0
    assert shards[-1].row0 + shards[-1].n_local == n
    for s in shards:
        assert s.row0 % align == 0 or s.n_local == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        comm = Comm(dist.group.WORLD)
        # column-major k x p views as the sweep uses them (slices of a wider buffer)
        buf = torch.zeros((6, 5), dtype=torch.float64).t()  # 5 x 6 column-major
        a = buf[:, 1:4]
        a.copy_(torch.full((5, 3), float(rank + 1)))
        b = torch.arange(4, dtype=torch.float64) * (rank + 1)
        c = torch.tensor([2.0 ** -30 * (rank + 1)], dtype=torch.float64)
        comm.allreduce_(a, b, c)
        tot = world * (world + 1) / 2
        ok = (torch.all(a == tot).item() and torch.equal(b, torch.arange(4, dtype=torch.float64) * tot)
              and c.item() == 2.0 ** -30 * tot and torch.all(buf[:, 0] == 0).item())
        m = comm.max_scalar(float(rank))
        q.put((rank, bool(ok), m))
    finally:
        dist.destroy_process_group()


def test_allreduce_packing_two_gloo_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(m == 1.0 for _, _, m in res)


# ---------------------------------------------------------------------------
# the algebra the kernels rely on, emulated exactly in numpy

def test_sharded_srht_kronecker_split_matches_fwht():
    """rb_sketch_srht: per 2048-row tile g, a local FWHT evaluated at the
    sampled local index, times (-1)^popc(g_s & g), summed over tiles (and
    over row shards) equals the reference's full FWHT (sketching.py:115-137)."""
    n, k = 3 * 2048 + 77, 300
    op = osk.OracleSketch("srht", k, n, 5)
    X = np.random.Generator(np.random.Philox(1)).standard_normal((n, 3))
    want = osk.apply(op, X)
    T = 2048
    Z = np.zeros((op.n_pad, 3))
    Z[:n] = op.sign_diagonal[:n, None] * X
    out = np.zeros((k, 3))
    gs, ls = op.sample_indices // T, op.sample_indices % T
    for g in range(op.n_pad // T):
        z = osk.fwht_ascending(Z[g * T:(g + 1) * T].copy())
        sign = np.array([(-1.0) ** bin(int(a) & g).count("1") for a in gs])
        out += sign[:, None] * z[ls]
    out /= math.sqrt(k)
    assert np.linalg.norm(out - want) <= 1e-13 * np.linalg.norm(want)


def _digits6(xi):
    """The six balanced signed byte digits of sketch_tc.cu::planes4:
    y = xi + 0x80_8080_8080 has the unsigned bytes b_q + 128 (q < 5) and
    y >> 40 = b5; returns (b5, b4, b3, b2, b1, b0)."""
    y = xi + 0x8080808080
    b = [((y >> (8 * q)) & 255) - 128 for q in range(5)]
    b5 = y >> 40
    return (b5, b[4], b[3], b[2], b[1], b[0])


def test_int8_ozaki_split_is_exact():
    """The tensor-core gaussian sketch as shipped (csrc/sketch_tc.cu): per
    (column, 16384-row chunk) x = xi 2^(E-46), |xi| <= 2^46, six balanced
    signed byte digits; q = 256 qh + ql.  One MMA multiplies qh by the six
    digit planes, a second ql shifted by one block, so the seven int32 TMEM
    blocks hold the weights 2^48 .. 2^0.  Checks: digits in s8 range, exact
    recombination of q . xi over the chunk, every block and every prefix
    sum < 2^31 (no int32 overflow; < 2^16 per row, < 2^30 per chunk), and
    the two-half int64 recombination of the epilogue."""
    g = np.random.Generator(np.random.Philox(2))
    rows = 16384
    q = osk.gaussian_int16(3, 1, np.arange(rows))[0].astype(np.int64)
    q[:4] = [32767, -32767, 32639, -32768]  # extreme int16 table values
    for case in range(3):
        x = g.standard_normal(rows).astype(np.float32)
        if case == 1:
            x[:8] = [np.float32(3.4e38), np.float32(-3.4e38), 1e-30, -1e-30, 0.0, -0.0, 1e-45, 2.0 ** -126]
        if case == 2:  # columns spanning many binades (the chunk max rules the scale)
            x *= np.float32(2.0) ** g.integers(-40, 1, rows).astype(np.float32)
        m = float(np.max(np.abs(x.astype(np.float64))))
        E = math.frexp(m)[1]
        xi = np.rint(x.astype(np.float64) * 2.0 ** (46 - E)).astype(np.int64)
        assert np.max(np.abs(xi)) <= 2 ** 46
        b5, b4, b3, b2, b1, b0 = _digits6(xi)
        for b in (b4, b3, b2, b1, b0):
            assert b.min() >= -128 and b.max() <= 127
        assert np.abs(b5).max() <= 65
        digits = (b5, b4, b3, b2, b1, b0)  # weights 2^40 .. 2^0
        assert np.array_equal(sum(d << (8 * (5 - i)) for i, d in enumerate(digits)), xi)
        qh, ql = q >> 8, q & 255
        assert qh.min() >= -128 and qh.max() <= 127 and ql.min() >= 0 and ql.max() <= 255
        # block w (w = 0..6) carries weight 2^(48 - 8w): qh x digit w, ql x digit w - 1
        blocks = []
        for w in range(7):
            blk = np.zeros(rows, dtype=np.int64)
            if w < 6:
                blk += qh * digits[w]
            if w >= 1:
                blk += ql * digits[w - 1]
            blocks.append(blk)
        for blk in blocks:
            assert np.abs(blk).max() < 2 ** 16
            assert np.abs(np.cumsum(blk)).max() < 2 ** 30
        sums = [int(blk.sum()) for blk in blocks]
        total = sum(s_ << (48 - 8 * w) for w, s_ in enumerate(sums))
        assert total == int(np.dot(q, xi))
        # the epilogue's two exact int64 halves: hi = weights 2^48..2^32 (/2^32), lo = 2^24..2^0
        hi = (sums[0] << 16) + (sums[1] << 8) + sums[2]
        lo = (sums[3] << 24) + (sums[4] << 16) + (sums[5] << 8) + sums[6]
        assert abs(hi) < 2 ** 47 and abs(lo) < 2 ** 55
        assert (hi << 32) + lo == total
        # fixed point: binary32 entries within 22 binades of the chunk max are
        # exact; the rest round at 2^(E-47) absolute
        err = np.abs(xi * 2.0 ** (E - 46) - x.astype(np.float64))
        assert err.max() <= 2.0 ** (E - 47)
        near = np.abs(x.astype(np.float64)) >= 2.0 ** (E - 23)
        assert np.all(err[near] == 0.0)


def test_reference_order_projection_is_sequential_fp32():
    """Step 3's arithmetic (kernels.py:200-208): acc - fl32(q x) per l, which
    the CUDA kernel computes as acc + fl32(q (-x)) -- the same bits."""
    g = np.random.Generator(np.random.Philox(3))
    Q = g.standard_normal((50, 9)).astype(np.float32)
    X = g.standard_normal((9, 4)).astype(np.float32)
    W = g.standard_normal((50, 4)).astype(np.float32)
    acc = W.copy()
    for l in range(9):
        acc = (acc + (Q[:, l:l + 1] * (-X[l:l + 1, :])).astype(np.float32)).astype(np.float32)
    assert np.array_equal(acc.astype(np.float64), osw.project(Q, X.astype(np.float64), W, "coarse"))


def test_reference_arm_runs_on_cpu():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--sample-rows", "2048", "--config", "c1"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    import json
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "port"


def test_devarray_is_numpy_compatible():
    """kernels.DevArray (what RbgsSweep.Q/S/P/R return): slicing stays a view
    of the tensor, numpy consumers (asarray, @, .copy(), .T, linalg) see the
    binary64 block -- the reference's consumers (krylov.py:229-262) do
    `sweep.R[:c, mp:c].copy()` and `sweep.Q[:, :j] @ Z`."""
    import torch

    from paper_2111_14641_b200.kernels import DevArray, Matrix, as_array

    A = np.arange(12.0).reshape(3, 4)
    t = torch.from_numpy(A.copy())
    d = DevArray(t)
    assert d.shape == (3, 4) and len(d) == 3 and d.ndim == 2
    v = d[:, 1:3]
    assert isinstance(v, DevArray) and v.tensor.data_ptr() == t[:, 1:3].data_ptr()
    assert np.array_equal(np.asarray(v), A[:, 1:3])
    assert np.array_equal(v.copy(), A[:, 1:3]) and isinstance(v.copy(), np.ndarray)
    assert np.array_equal(d.T, A.T)
    Z = np.ones((4, 2))
    assert np.array_equal(d @ Z, A @ Z) and np.array_equal(Z.T @ d.T, Z.T @ A.T)
    assert np.array_equal(d - A, np.zeros_like(A)) and np.array_equal(2.0 * d, 2.0 * A)
    assert np.allclose(np.linalg.svd(d, compute_uv=False), np.linalg.svd(A, compute_uv=False))
    assert np.array_equal(np.hstack([d[:, :1], d[:, 1:]]), A)
    assert np.array_equal(Matrix(d).data, A) and np.array_equal(as_array(d), A)
    d[0:1, 0:2] = np.array([[7.0, 8.0]])
    assert t[0, 0].item() == 7.0 and t[0, 1].item() == 8.0


def test_device_knobs_validate_without_a_gpu():
    """Round-2 device-only knobs: operator digits and the rb_sketch_gaussian
    mode they select; block_gmres diagnostics modes are validated before any
    device work."""
    from paper_2111_14641_b200 import krylov, sketching
    from paper_2111_14641_b200._device import GAUSS_MODE

    op = sketching.gaussian_operator(8, 64, 1)
    assert op.digits == 6 and sketching.gauss_mode(op) in ("auto", sketching.GAUSS_MODE)
    if sketching.GAUSS_MODE == "auto":
        assert sketching.gauss_mode(sketching.gaussian_operator(8, 64, 1, digits=4)) == "tensor4"
        assert sketching.gauss_mode(op, 3) == "tensor3"
    assert GAUSS_MODE["tensor4"] == 4 and GAUSS_MODE["tensor3"] == 5
    with pytest.raises(ValueError):
        sketching.gaussian_operator(8, 64, 1, digits=5)
    with pytest.raises(ValueError):
        krylov.block_gmres(None, None, None, 4, diagnostics="none")
