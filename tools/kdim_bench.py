"""Per-call times of the k-dimensional kernels (CUDA events, 20 reps after
warm-up): rb_ls_richardson, rb_sketched_cholqr_small, rb_certify, and the
tall projection-side kernels for reference.  Prints one JSON line."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_14641_b200 import _device as D  # noqa: E402


def t_ms(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph and
    replayed (the ctypes host path would otherwise be the bound)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    out = {}
    g = torch.Generator(device="cuda").manual_seed(0)
    for k, c, p in [(1600, 760, 40), (1600, 380, 40), (1600, 40, 40), (2048, 960, 64), (400, 190, 10)]:
        S = D.empty_cm(k, c, torch.float64, "cuda")
        S.copy_(torch.randn(k, c, generator=g, device="cuda", dtype=torch.float64) / k ** 0.5)
        P = D.empty_cm(k, p, torch.float64, "cuda")
        P.copy_(torch.randn(k, p, generator=g, device="cuda", dtype=torch.float64))
        X = D.empty_cm(c, p, torch.float64, "cuda")
        T = D.empty_cm(k, p, torch.float64, "cuda")
        R = D.empty_cm(p, p, torch.float64, "cuda")
        So = D.empty_cm(k, p, torch.float64, "cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        outc = torch.zeros(3, dtype=torch.float64, device="cuda")
        key = f"k{k}_c{c}_p{p}"
        out[key] = {
            "richardson5_ms": t_ms(lambda: D.richardson(S, P, 5, X, T)),
            "richardson1_ms": t_ms(lambda: D.richardson(S, P, 1, X, T)),
            "cholqr_ms": t_ms(lambda: D.sketched_cholqr_small(P, R, So, info)),
            "gemm_tn_ms": t_ms(lambda: D.gemm(1, 0, 1.0, S, P, 0.0, X)),
            "gemm_nn_ms": t_ms(lambda: D.gemm(0, 0, -1.0, S, X, 1.0, T)),
        }
        if c >= p:
            Sm = S[:, :c]
            Rm = D.empty_cm(c, c, torch.float64, "cuda")
            Rm.copy_(torch.triu(torch.randn(c, c, generator=g, device="cuda", dtype=torch.float64)))
            out[key]["certify_ms"] = t_ms(lambda: D.certify_sums(Sm, Sm, Rm, outc))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
