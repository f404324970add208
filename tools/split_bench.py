"""The fused gaussian sketch [Theta Q' | Theta W] at the C2 shape (two 1e6 x
40 binary32 inputs, k = 1600): ms per call (CUDA events), the split_planes
pre-pass and gauss_tc_partial device times (torch.profiler), and a hash of
the output bits.  Run once per RB_SPLIT_* setting to compare variants:

    RB_SPLIT_MINB=2 python tools/split_bench.py
"""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_14641_b200 import _device as D  # noqa: E402
from paper_2111_14641_b200 import _lib  # noqa: E402

if os.environ.get("SPLIT_BENCH_LIB"):  # a baseline build of the same C ABI
    _lib.LIB_PATH = os.environ["SPLIT_BENCH_LIB"]
from paper_2111_14641_b200 import sketching, workloads  # noqa: E402


def main():
    n = int(os.environ.get("SB_N", 1_000_000))
    p = int(os.environ.get("SB_P", 40))
    k = int(os.environ.get("SB_K", 1600))
    dev = torch.device("cuda", 0)
    W = workloads.trig_device(n, 2 * p, 7, 0, n, torch.float32, dev)
    g = torch.Generator(device=dev).manual_seed(3)
    W[:, :p] = torch.randn(n, p, device=dev, generator=g) * torch.logspace(0, -6, p, device=dev)
    X1, X2 = W[:, :p], W[:, p:]
    theta = sketching.gaussian_operator(k, n, 11, theta_bits=int(os.environ.get("SB_THETA_BITS", "16")))
    tab = theta.device_tables(dev, 0, n)
    o1 = torch.empty((p, k), dtype=torch.float64, device=dev).t()
    o2 = torch.empty((p, k), dtype=torch.float64, device=dev).t()

    def call():
        D.sketch_gaussian2(X1, X2, tab["theta"], tab["ldt"], k, 1.0, o1, o2,
                           mode=os.environ.get("SB_MODE", "tensor") + ("+q8" if theta.theta_bits == 8 else ""))

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            call()
        torch.cuda.synchronize()
    per = {}
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        for key in ("split_planes", "chunk_max", "encode_planes", "encode_tile", "gauss_tc_partial", "reduce_splits"):
            if key in ev.name:
                d = per.setdefault(key, [0, 0.0])
                d[0] += 1
                d[1] += ev.time_range.elapsed_us() / 1e3
    h = hashlib.sha256(o1.contiguous().cpu().numpy().tobytes() + o2.contiguous().cpu().numpy().tobytes()).hexdigest()
    print(json.dumps({"env": {k2: v for k2, v in os.environ.items() if k2.startswith("RB_")}, "ms_per_call": ms,
                      "kernels_ms_per_launch": {k2: v[1] / v[0] for k2, v in per.items()},
                      "launches_per_call": {k2: v[0] / 5 for k2, v in per.items()}, "sha": h[:16]}))


if __name__ == "__main__":
    main()
