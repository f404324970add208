"""Correctness and timing probe of Step 3 on the tensor pipe (RB_ORDER_TC).

    python tools/tc_probe.py check     # small shapes vs a binary64 product
    python tools/tc_probe.py time      # C5 / C3 / C2 shapes, GB/s of the algorithmic bytes

check: every (n, c, p) against W - Q X in binary64; the 3xTF32 bound is a few
2^-22 |Q||X| per product (vs 2^-24 for the binary32 FMA order, also printed).
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_14641_b200 import _device as D  # noqa: E402
from paper_2111_14641_b200._lib import F32  # noqa: E402

ORD = {"reference": 0, "fma": 1, "tc": 3}


def cm(n, m, dtype, dev="cuda"):
    return torch.empty(m, n, dtype=dtype, device=dev).t()


def run(order, Q, X, W):
    n, p = W.shape
    out = cm(n, p, torch.float32)
    norms = torch.zeros(2, dtype=torch.float64, device="cuda")
    D.project(Q, X, W, out, F32, ORD[order], norms)
    return out, norms


def check():
    g = torch.Generator(device="cuda").manual_seed(3)
    ok = True
    for n, c, p in [(128, 32, 16), (512, 32, 64), (640, 64, 64), (1024 + 37, 40, 33), (128 * 300, 96, 48),
                    (128 * 1200 + 5, 960, 64), (128 * 777, 200, 32), (1 << 20, 448, 64)]:
        Q = cm(n, c + 8, torch.float32)
        Q.copy_(torch.randn(n, c + 8, generator=g, device="cuda"))
        Q[:, c:] = float("nan")  # columns past c must never be read
        X = cm(c, p, torch.float64)
        X.copy_(torch.randn(c, p, generator=g, device="cuda", dtype=torch.float64))
        W = cm(n, p, torch.float32)
        W.copy_(torch.randn(n, p, generator=g, device="cuda") * 3)
        ref = W.double() - Q[:, :c].double() @ X.float().double()
        scale = (Q[:, :c].double().abs() @ X.abs()).max().item()
        res = {}
        for o in ("fma", "tc"):
            out, norms = run(o, Q[:, :c], X, W)
            torch.cuda.synchronize()
            err = (out.double() - ref).abs().max().item() / scale
            nq = (norms[1].item() - (out.double() ** 2).sum().item()) / norms[1].item()
            nw = (norms[0].item() - (W.double() ** 2).sum().item()) / norms[0].item()
            res[o] = (err, nq, nw)
        good = res["tc"][0] < 2e-6 and abs(res["tc"][1]) < 1e-12 and abs(res["tc"][2]) < 1e-12
        ok &= good
        print(f"n={n} c={c} p={p}: tc err/|Q||X| {res['tc'][0]:.2e} (fma {res['fma'][0]:.2e}) "
              f"norm defects {res['tc'][1]:.1e} {res['tc'][2]:.1e} {'ok' if good else 'FAIL'}", flush=True)
    print("ALL OK" if ok else "FAILED")
    return 0 if ok else 1


def time_():
    rows = []
    for name, n, p, cs in [("c5", 1 << 24, 64, (64, 512, 960)), ("c3", 1 << 24, 32, (32, 256, 480)),
                           ("c2", 1_000_000, 40, (40, 400, 760))]:
        cmax = max(cs)
        Q = cm(n, cmax, torch.float32)
        Q.normal_()
        W = cm(n, p, torch.float32)
        W.normal_()
        for c in cs:
            X = cm(c, p, torch.float64)
            X.normal_()
            for o in ("tc", "fma", "reference"):
                if o != "tc" and c != cs[1]:
                    continue
                for _ in range(2):
                    run(o, Q[:, :c], X, W)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                reps = 5
                for _ in range(reps):
                    run(o, Q[:, :c], X, W)
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1) / reps
                gb = 4.0 * n * (c + 2 * p) / 1e9
                rows.append(dict(shape=name, n=n, p=p, c=c, order=o, ms=ms, GBps=gb / ms * 1e3))
                print(json.dumps(rows[-1]), flush=True)
        del Q, W
    return 0


def map_():
    """Operand-layout probe: Q[r, k] = (r + 1) + 256 (k + 1), X selects column
    j of Q into output column j, W = 0: -out[r, j] must decode to (r, j)."""
    for n, c, p in [(128, 32, 16), (512, 64, 32)]:
        Q = cm(n, c, torch.float32)
        r = torch.arange(n, device="cuda", dtype=torch.float32)[:, None] % 128
        k = torch.arange(c, device="cuda", dtype=torch.float32)[None, :]
        Q.copy_((r + 1) + 256 * (k + 1))
        X = cm(c, p, torch.float64)
        X.zero_()
        for j in range(p):
            X[(j * 3) % c, j] = 1.0
        W = cm(n, p, torch.float32)
        W.zero_()
        out, _ = run("tc", Q, X, W)
        torch.cuda.synchronize()
        o = (-out).cpu().numpy()
        bad = 0
        for rr in list(range(n)):
            for j in range(p):
                v = o[rr, j]
                want = (rr % 128 + 1) + 256 * ((j * 3) % c + 1)
                if v != want:
                    bad += 1
                    if bad <= 40:
                        kk, r1 = divmod(int(round(v)), 256)
                        print(f"n={n} out[{rr},{j}] = {v} -> (r'={r1 - 1}, k'={kk - 1}) want (r={rr % 128}, k={(j * 3) % c})")
        print(f"n={n} c={c} p={p}: {bad} mismatches of {n * p}", flush=True)
    return 0


def one():
    """python tools/tc_probe.py one N P C [order]: a single shape (for ncu)."""
    n, p, c = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    o = sys.argv[5] if len(sys.argv) > 5 else "tc"
    Q = cm(n, c, torch.float32)
    Q.normal_()
    W = cm(n, p, torch.float32)
    W.normal_()
    X = cm(c, p, torch.float64)
    X.normal_()
    for _ in range(3):
        run(o, Q, X, W)
    torch.cuda.synchronize()
    return 0


if __name__ == "__main__":
    sys.exit({"check": check, "time": time_, "map": map_, "one": one}[sys.argv[1]]())
