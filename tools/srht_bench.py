"""SRHT sketch kernel timing at the C3 shape (n = 2^24, 32 binary32 columns,
k = 1024), warp-per-column kernel vs the CTA-per-tile kernel (RB_SRHT_V1).

    python tools/srht_bench.py [--once]
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_14641_b200 import _device as D  # noqa: E402
from paper_2111_14641_b200 import sketching  # noqa: E402


def main():
    n, cols, k = 1 << 24, 32, 1024
    op = sketching.SketchOperator("srht", k, n, 3)
    X = D.empty_cm(n, cols, torch.float32, "cuda")
    X.copy_(torch.randn(n, cols, device="cuda"))
    out = D.empty_cm(k, cols, torch.float64, "cuda")
    if "--once" in sys.argv:
        sketching.sketch_into(op, X, out)
        torch.cuda.synchronize()
        return
    res = {}
    for name, env in (("warp", None), ("v1", "1")):
        if env:
            os.environ["RB_SRHT_V1"] = env
        else:
            os.environ.pop("RB_SRHT_V1", None)
        for _ in range(2):
            sketching.sketch_into(op, X, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sketching.sketch_into(op, X, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name] = dict(ms=ms, GBps=4.0 * n * cols / ms / 1e6, out_norm=float(out.norm()))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
