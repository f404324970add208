"""Projection kernel timing (reference order and FMA order) at the C2 and C3
block shapes; RB_PROJECT_RPT picks the rows-per-thread variant.

    RB_PROJECT_RPT=4 python tools/project_bench.py

Prints one JSON object: ms per call and element-steps/s (n * c * p / time;
the reference-order FP32 issue bound on B200 is ~17.1e12, FMUL + FADD).
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_14641_b200 import _device as D  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = "cuda"
    res = {"rpt": os.environ.get("RB_PROJECT_RPT", "default")}
    g = torch.Generator(device=dev).manual_seed(0)
    once = "--once" in sys.argv  # one reference-order C2 call (for ncu)
    shapes = (("C2", 1_000_000, 40, (760,)),) if once else (
        ("C2", 1_000_000, 40, (400, 760)), ("C3", 1 << 24, 32, (480,)))
    for tag, n, p, cs in shapes:
        cmax = max(cs)
        Q = D.empty_cm(n, cmax, torch.float32, dev)
        Q.copy_(torch.randn(n, cmax, generator=g, device=dev))
        X = D.empty_cm(cmax, p, torch.float64, dev)
        X.copy_(torch.randn(cmax, p, generator=g, device=dev, dtype=torch.float64) * 0.01)
        W = D.empty_cm(n, p, torch.float32, dev)
        W.copy_(torch.randn(n, p, generator=g, device=dev))
        out = D.empty_cm(n, p, torch.float32, dev)
        norms = torch.zeros(2, dtype=torch.float64, device=dev)
        for c in cs:
            if once:
                D.project(Q[:, :c], X[:c], W, out, 0, 0, norms)
                torch.cuda.synchronize()
                return
            for order, name in ((0, "ref"), (1, "fma")):
                ms = timeit(lambda: D.project(Q[:, :c], X[:c], W, out, 0, order, norms))
                res[f"{tag}_{name}_c{c}_p{p}"] = dict(ms=round(ms, 4), Tsteps=round(n * c * p / ms / 1e9, 3))
        del Q, X, W, out
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
