"""SURVEY 8(f) serialization on the host: the reference's Matrix Market
BlockQR directory (rbgs.py:493-552) read and re-written byte for byte, and
the binary (sharded) format round trip.  No GPU needed."""

import os

import numpy as np

import goldens
from paper_2111_14641_b200 import post, rbgs
from paper_2111_14641_b200.comm import RowShard
from paper_2111_14641_b200.kernels import BlockPartition, Matrix

REF_DIR = os.path.join(goldens.GOLDEN, "blockqr_ref")


def test_load_reference_directory_and_rewrite_byte_identical(tmp_path):
    f = rbgs.load_blockqr(REF_DIR)
    assert f.Q.shape == (300, 12) and f.R.shape == (12, 12) and f.S.shape == (72, 12)
    assert f.partition.block_width == 4 and f.partition.num_blocks == 3
    assert len(f.cert.per_block_ortho) == 3
    rbgs.save_blockqr(f, str(tmp_path))
    for name in ("Q.mtx", "R.mtx", "S.mtx", "P.mtx", "cert.txt", "meta.txt"):
        with open(os.path.join(REF_DIR, name), "rb") as a, open(os.path.join(tmp_path, name), "rb") as b:
            assert a.read() == b.read(), name


def test_load_without_sketches(tmp_path):
    f = rbgs.load_blockqr(REF_DIR)
    g = rbgs.BlockQR(f.Q, f.R, None, None, f.partition, None)
    rbgs.save_blockqr(g, str(tmp_path))
    h = rbgs.load_blockqr(str(tmp_path))
    assert h.S is None and h.P is None and h.cert is None
    assert np.array_equal(h.Q.data, f.Q.data)


def test_binary_round_trip_and_shards(tmp_path):
    f = rbgs.load_blockqr(REF_DIR)
    d1 = str(tmp_path / "whole")
    rbgs.save_blockqr_binary(f, d1)
    g = rbgs.load_blockqr_binary(d1)
    for a, b in ((f.Q, g.Q), (f.R, g.R), (f.S, g.S), (f.P, g.P)):
        assert np.array_equal(a.data, b.data)
    assert g.cert == f.cert and g.partition == f.partition
    # two row shards (ranks write their own Q rows; rank 0 the rest)
    d2 = str(tmp_path / "sharded")
    Q = f.Q.data
    cut = 128
    for rank, (r0, r1) in enumerate(((0, cut), (cut, 300))):
        part = rbgs.BlockQR(Matrix(Q[r0:r1]), f.R, f.S, f.P, f.partition, f.cert)
        rbgs.save_blockqr_binary(part, d2, shard=RowShard(300, r0, r1 - r0), rank=rank)
    post.register_shard(d2, 0, 0, cut)
    post.register_shard(d2, 1, cut, 300 - cut)
    h = rbgs.load_blockqr_binary(d2)
    assert np.array_equal(h.Q.data, Q)
    assert np.array_equal(rbgs.load_blockqr_binary(d2, rank=1).Q.data, Q[cut:])


def test_binary32_q_is_kept_binary32(tmp_path):
    import torch

    g = np.random.Generator(np.random.Philox(4))
    Q32 = g.standard_normal((50, 4)).astype(np.float32)
    f = rbgs.BlockQR(Matrix(torch.from_numpy(Q32)), Matrix(np.eye(4)), Matrix(np.eye(8, 4)),
                     Matrix(np.eye(8, 4)), BlockPartition.uniform(4, 2), None)
    rbgs.save_blockqr_binary(f, str(tmp_path))
    assert os.path.getsize(tmp_path / "Q.rank0.bin") == 50 * 4 * 4
    h = rbgs.load_blockqr_binary(str(tmp_path))
    assert np.array_equal(h.Q.data, Q32.astype(np.float64))
