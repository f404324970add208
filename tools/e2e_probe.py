"""Timeline of one e2e step (pinned host W -> rbgs() -> R on the host) at
the C2 shape: when the copies and the compute of each block start and end
(torch.profiler device activities)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2111_14641_b200 import sketching, workloads  # noqa: E402
from paper_2111_14641_b200.kernels import COARSE, BlockPartition  # noqa: E402
from paper_2111_14641_b200.rbgs import RbgsConfig, rbgs  # noqa: E402


def main():
    c = bench.CONFIGS["c2"]
    n, m, p, k = c["n"], c["m"], c["p"], c["k"]
    dev = torch.device("cuda", 0)
    W = workloads.trig_device(n, m, bench.SEED_W, 0, n, torch.float32, dev)
    theta = sketching.gaussian_operator(k, n, bench.SEED_THETA)
    theta.device_tables(dev, 0, n)
    cfg = RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)", coarse=COARSE)
    Wh = torch.empty((m, n), dtype=torch.float32).pin_memory().t()
    Wh.copy_(W)
    del W
    torch.cuda.empty_cache()
    for _ in range(2):
        rbgs(Wh, theta, cfg).R.data
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rbgs(Wh, theta, cfg).R.data
    wall = (time.perf_counter() - t0) * 1e3
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        rbgs(Wh, theta, cfg).R.data
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t_min = min(e.time_range.start for e in ev)
    copies = sorted((e.time_range.start - t_min, e.time_range.end - t_min) for e in ev if "Memcpy HtoD" in e.name)
    kern = sorted((e.time_range.start - t_min, e.time_range.end - t_min, e.name[:40]) for e in ev
                  if "Memcpy" not in e.name and "Memset" not in e.name)
    proj = [(round(a / 1e3, 2), round(b / 1e3, 2)) for a, b, nm in kern if "project" in nm]
    out = {"wall_ms_unprofiled": wall,
           "copies_ms": [(round(a / 1e3, 2), round(b / 1e3, 2)) for a, b in copies],
           "first_kernel_ms": round(kern[0][0] / 1e3, 2), "last_kernel_end_ms": round(max(b for _, b, _ in kern) / 1e3, 2),
           "project_ms": proj}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
