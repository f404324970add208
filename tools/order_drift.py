"""R drift between projection orders on the full-size bench workloads.

    python tools/order_drift.py [c2|c3 ...]

Factorizes the bench's synthetic W (bench.CONFIGS) once per projection
order and prints ||R_order - R_reference||_F / ||R_reference||_F and the max
relative drift of diag(R), plus each run's certificate -- the evidence that
a non-reference order stays within the north star's 1e-5 R tolerance.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2111_14641_b200 import sketching, workloads  # noqa: E402
from paper_2111_14641_b200.kernels import COARSE, BlockPartition  # noqa: E402
from paper_2111_14641_b200.rbgs import DeviceConfig, RbgsConfig, rbgs  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    orders = [o for o in ("fma", "tc") if o in DeviceConfig.ORDERS] if hasattr(DeviceConfig, "ORDERS") else ["fma"]
    out = {}
    for name in sys.argv[1:] or ["c2"]:
        c = bench.CONFIGS[name]
        n, m, p, k = c["n"], c["m"], c["p"], c["k"]
        if c["gen"] == "trig":
            W = workloads.trig_device(n, m, bench.SEED_W, 0, n, torch.float32, dev)
        elif c["gen"] == "lowrank":
            W = workloads.lowrank_device(n, m, bench.SEED_W, dtype=torch.float32, device=dev, rank=0)
        else:
            W = workloads.colscaled_gaussian_device(n, m, bench.SEED_W, dtype=torch.float32, device=dev, rank=0)
        if c["kind"] == "gaussian":
            theta = sketching.gaussian_operator(k, n, bench.SEED_THETA)
            theta.device_tables(dev, 0, n)
        else:
            theta = sketching.SketchOperator(c["kind"], k, n, bench.SEED_THETA)
            theta.device_tables(dev)
        cfg = RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)", coarse=COARSE)
        res = {}
        Rref = None
        for order in ["reference"] + orders:
            f = rbgs(W, theta, cfg, DeviceConfig(device=dev, projection_order=order))
            R = torch.as_tensor(f.R.data, dtype=torch.float64)
            d = {"delta": f.cert.delta, "delta_tilde": f.cert.delta_tilde}
            if Rref is None:
                Rref = R
            else:
                d["dR_fro_rel"] = float(torch.linalg.norm(R - Rref) / torch.linalg.norm(Rref))
                dg = torch.diagonal(Rref)
                d["dR_diag_max_rel"] = float(torch.max(torch.abs(torch.diagonal(R) - dg) / torch.abs(dg)))
            res[order] = d
            del f
            torch.cuda.empty_cache()
        out[name] = res
        del W, theta
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
