"""Row-sharded execution with two ranks.

Two processes on cuda:0 with the gloo backend (host-staged collectives: the
ranks' kernels never wait on one another on the device -- a functional
check of the sharded algorithm on a one-GPU box, never a timing).  Each rank
owns a contiguous row shard; the sharded factorization must equal the
unsharded one (the sketches are sums over rows, reduced in fp64, so only
the summation order of the shard partials differs), and the sweep must
issue exactly ONE collective per block."""

import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent(r'''
    import os, sys, json
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.environ["RB_ROOT"])
    from paper_2111_14641_b200 import rbgs as R, sketching, workloads, krylov, operators
    from paper_2111_14641_b200.comm import Comm, RowShard
    from paper_2111_14641_b200.kernels import BlockPartition, COARSE, FINE

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["RB_PORT"], rank=rank,
                            world_size=world)
    case = os.environ["RB_CASE"]
    out = {}
    comm = Comm(dist.group.WORLD)
    if case in ("gauss", "srht_l2", "sparse"):
        n, m, p = 16384, 96, 16
        if case == "gauss":
            W = workloads.colscaled_host(n, m, 7).astype(np.float32)
            theta = sketching.gaussian_operator(256, n, 11)
            cfg = R.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
        elif case == "srht_l2":
            W = workloads.trig_host(n, m, 7)
            theta = sketching.SketchOperator("srht", 256, n, 11)
            cfg = R.RbgsConfig(partition=BlockPartition.uniform(m, p), coarse=FINE)
        else:
            W = workloads.colscaled_host(n, m, 7).astype(np.float32)
            theta = sketching.sparse_sign_operator(256, n, 11)
            cfg = R.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
        sh = RowShard.split(n, world, rank, align=2048)
        dc = R.DeviceConfig(comm=comm, shard=sh)
        f = R.rbgs(np.ascontiguousarray(W[sh.row0:sh.row0 + sh.n_local]), theta, cfg, dc)
        out["R"] = f.R.data.tolist()
        out["delta"] = f.cert.delta
        out["collectives"] = comm.collectives
        out["blocks"] = cfg.partition.num_blocks
    else:  # block GMRES, z-slab halo
        nx = 24
        B = np.random.Generator(np.random.Philox(3)).standard_normal((nx ** 3, 4))
        A = operators.Poisson3D(nx, nx, nx, comm=comm)
        theta = sketching.sparse_sign_operator(2 * 4 * 8, nx ** 3, 11)
        dc = R.DeviceConfig(comm=comm, shard=RowShard(A.n, A.row0, A.n_local))
        rep = krylov.block_gmres(A, B[A.row0:A.row0 + A.n_local], theta, 8, cfg=R.RbgsConfig(), device_cfg=dc)
        out["hist"] = [list(map(float, h)) for h in rep.residual_history]
    if rank == 0:
        with open(os.environ["RB_OUT"], "w") as fh:
            json.dump(out, fh)
    dist.destroy_process_group()
''')


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(case, tmp_path, world=2):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    outp = tmp_path / f"{case}.json"
    port = str(_free_port())
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), RB_PORT=port, RB_CASE=case, RB_OUT=str(outp),
                   RB_ROOT=ROOT, MASTER_ADDR="127.0.0.1")
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    logs = []
    for pr in procs:
        o, _ = pr.communicate(timeout=600)
        logs.append(o.decode()[-3000:])
        assert pr.returncode == 0, "\n".join(logs)
    import json
    return json.loads(outp.read_text())


@pytest.mark.parametrize("case", ["gauss", "srht_l2", "sparse"])
def test_sharded_rbgs_equals_unsharded_one_collective_per_block(case, tmp_path):
    import torch

    from paper_2111_14641_b200 import rbgs as R, sketching, workloads
    from paper_2111_14641_b200.kernels import FINE, BlockPartition

    got = _run(case, tmp_path)
    n, m, p = 16384, 96, 16
    if case == "gauss":
        W = workloads.colscaled_host(n, m, 7).astype(np.float32)
        theta = sketching.gaussian_operator(256, n, 11)
        cfg = R.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
        tol = 1e-12
    elif case == "srht_l2":
        W = workloads.trig_host(n, m, 7)
        theta = sketching.SketchOperator("srht", 256, n, 11)
        cfg = R.RbgsConfig(partition=BlockPartition.uniform(m, p), coarse=FINE)
        tol = 1e-12
    else:
        W = workloads.colscaled_host(n, m, 7).astype(np.float32)
        theta = sketching.sparse_sign_operator(256, n, 11)
        cfg = R.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
        tol = 1e-12
    f = R.rbgs(W, theta, cfg)
    torch.cuda.synchronize()
    Rs = np.array(got["R"])
    d = np.linalg.norm(Rs - f.R.data) / np.linalg.norm(f.R.data)
    assert d <= tol, (case, d)
    assert abs(got["delta"] - f.cert.delta) <= 1e-6 * max(f.cert.delta, 1e-12) + 1e-13
    # one collective per block (the norms and, for l2, the tall Gram ride along)
    assert got["collectives"] == got["blocks"], got["collectives"]


def test_sharded_block_gmres_zslab_halo_equals_unsharded(tmp_path):
    import torch

    from paper_2111_14641_b200 import krylov, operators, rbgs as R, sketching

    got = _run("gmres", tmp_path)
    nx = 24
    B = np.random.Generator(np.random.Philox(3)).standard_normal((nx ** 3, 4))
    rep = krylov.block_gmres(operators.Poisson3D(nx, nx, nx), B, sketching.sparse_sign_operator(64, nx ** 3, 11), 8,
                             cfg=R.RbgsConfig())
    torch.cuda.synchronize()
    h, hs = np.array(rep.residual_history), np.array(got["hist"])
    assert h.shape == hs.shape
    assert np.allclose(h[:, 1], hs[:, 1], rtol=1e-9), (h[:, 1], hs[:, 1])
