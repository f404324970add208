"""Per-kernel timing of the C-ABI entry points at BASELINE shapes (CUDA events).

    python tools/kbench.py [--quick]

Prints one JSON object: ms per call and the achieved algorithmic GB/s or
TFLOP/s of each kernel.  Used to pick kernels and to fill DESIGN.md; the
round's official numbers come from bench.py.
"""

import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_14641_b200 import _device as D  # noqa: E402
from paper_2111_14641_b200 import sketching  # noqa: E402


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
    quick = "--quick" in sys.argv
    dev = "cuda"
    res = {}
    n, p = 1_000_000, 40
    g = torch.Generator(device=dev).manual_seed(0)
    for c in (0, 400, 760):
        Q = D.empty_cm(n, max(c, 1), torch.float32, dev)
        Q.copy_(torch.randn(n, max(c, 1), generator=g, device=dev))
        X = D.empty_cm(max(c, 1), p, torch.float64, dev)
        X.copy_(torch.randn(max(c, 1), p, generator=g, device=dev, dtype=torch.float64) * 0.01)
        W = D.empty_cm(n, p, torch.float32, dev)
        W.copy_(torch.randn(n, p, generator=g, device=dev))
        out = D.empty_cm(n, p, torch.float32, dev)
        norms = torch.zeros(2, dtype=torch.float64, device=dev)
        for order, name in ((0, "ref"), (1, "fma")):
            ms = timeit(lambda: D.project(Q[:, :c] if c else None, X[:c] if c else None, W, out, 0, order, norms))
            byt = 4.0 * n * (c + 2 * p)
            res[f"project_{name}_c{c}_p{p}"] = dict(ms=ms, GBps=byt / ms / 1e6,
                                                   Gelem_steps_per_s=n * c * p / ms / 1e6)
        del Q
    # gaussian dense sketch (C2 per block)
    k = 1600
    op = sketching.gaussian_operator(k, n, 1)
    torch.cuda.synchronize()
    ms_fill = timeit(lambda: op.release_device_tables() or op.device_tables(dev, 0, n), reps=1, warm=1)
    tab = op.device_tables(dev, 0, n)
    Xs = D.empty_cm(n, p, torch.float32, dev)
    Xs.copy_(torch.randn(n, p, generator=g, device=dev))
    S = D.empty_cm(k, p, torch.float64, dev)
    ms = timeit(lambda: sketching.sketch_into(op, Xs, S), reps=3)
    res["gaussian_fill_k1600_n1e6"] = dict(ms=ms_fill)
    res["sketch_gaussian_k1600_p40"] = dict(ms=ms, TFLOPs_fp64=2.0 * k * n * p / ms / 1e9,
                                            GBps_theta=2.0 * k * n / ms / 1e6)
    op.release_device_tables()
    # srht (C3 block)
    ns = 1 << (22 if quick else 24)
    ks, ps = 1024, 32
    op = sketching.SketchOperator("srht", ks, ns, 1)
    Xh = D.empty_cm(ns, ps, torch.float32, dev)
    Xh.copy_(torch.randn(ns, ps, generator=g, device=dev))
    Sh = D.empty_cm(ks, ps, torch.float64, dev)
    ms = timeit(lambda: sketching.sketch_into(op, Xh, Sh), reps=3)
    res[f"sketch_srht_k{ks}_n{ns}_p{ps}"] = dict(ms=ms, GBps=4.0 * ns * ps / ms / 1e6)
    # sparse sign (C4 block)
    op = sketching.sparse_sign_operator(488, ns, 1)
    Xp = Xh[:, :4]
    Sp = D.empty_cm(488, 4, torch.float64, dev)
    ms = timeit(lambda: sketching.sketch_into(op, Xp, Sp), reps=3)
    res[f"sketch_sparse_k488_n{ns}_p4"] = dict(ms=ms, GBps=4.0 * ns * 4 / ms / 1e6)
    del Xh
    # tall trsm (scaling)
    R = torch.eye(p, dtype=torch.float64, device=dev) + 0.01 * torch.triu(torch.randn(p, p, generator=g, device=dev, dtype=torch.float64))
    Rc = D.to_cm(R)
    ms = timeit(lambda: D.trsm_right(W, Rc, out))
    res["trsm_right_n1e6_p40"] = dict(ms=ms, GBps=8.0 * n * p / ms / 1e6)
    # richardson at the last C2 block
    c = 760
    Sd = D.empty_cm(k, c, torch.float64, dev)
    Sd.copy_(torch.randn(k, c, generator=g, device=dev, dtype=torch.float64) / math.sqrt(k))
    P = D.empty_cm(k, p, torch.float64, dev)
    P.copy_(torch.randn(k, p, generator=g, device=dev, dtype=torch.float64))
    Xr = D.empty_cm(c, p, torch.float64, dev)
    T = D.empty_cm(k, p, torch.float64, dev)
    ms = timeit(lambda: D.richardson(Sd, P, 5, Xr, T))
    res["richardson5_k1600_c760_p40"] = dict(ms=ms, GFLOPs=2 * 2 * 5 * k * c * p / ms / 1e6)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
