"""Co-residency probe: the staged projection (C2 last block: n = 1e6,
c = 760, p = 40) and the lean next-block gaussian sketch (40 columns,
k = 1600), alone and concurrently on two streams (sketch on a high-priority
stream, issued first).  CUDA events around each region; prints JSON."""
import json
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2111_14641_b200 import _device as D, sketching  # noqa: E402


def main():
    n, c, p, k = 1_000_000, 760, 40, 1600
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    Q = D.empty_cm(n, c + p, torch.float32, dev)
    Q.copy_(torch.randn(c + p, n, generator=g, device=dev).t())
    X = D.empty_cm(c, p, torch.float64, dev)
    X.copy_(torch.randn(p, c, generator=g, device=dev, dtype=torch.float64).t() * 0.01)
    W = D.empty_cm(n, p, torch.float32, dev)
    W.copy_(torch.randn(p, n, generator=g, device=dev).t())
    Wn = D.empty_cm(n, p, torch.float32, dev)
    Wn.copy_(torch.randn(p, n, generator=g, device=dev).t())
    out = D.empty_cm(n, p, torch.float32, dev)
    theta = sketching.gaussian_operator(k, n, 11)
    tab = theta.device_tables(dev, 0, n)
    P = D.empty_cm(k, p, torch.float64, dev)
    scale = 1.0 / (sketching.GAUSS_GRID * math.sqrt(k))
    side = torch.cuda.Stream(dev, priority=-1)
    main_s = torch.cuda.current_stream(dev)

    def proj():
        D.project(Q[:, :c], X, W, out, 0, 0)

    def sk(mode):
        D.sketch_gaussian(Wn, tab["theta"], tab["ldt"], k, scale, P, False, mode)

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def both(mode):
        def f():
            side.wait_stream(main_s)
            with torch.cuda.stream(side):
                sk(mode)
            proj()
            main_s.wait_stream(side)
        return f

    res = {"project_ms": timed(proj), "sketch_lean_ms": timed(lambda: sk("lean")),
           "sketch_tensor_ms": timed(lambda: sk("tensor")),
           "both_lean_ms": timed(both("lean")), "both_tensor_ms": timed(both("tensor")),
           "serial_ms": timed(lambda: (sk("tensor"), proj()))}
    # timeline of one concurrent run: events on both streams share one clock
    torch.cuda.synchronize()
    ev = {nm: torch.cuda.Event(enable_timing=True) for nm in ("t0", "sk_end", "pj_end")}
    ev["t0"].record(main_s)
    side.wait_stream(main_s)
    with torch.cuda.stream(side):
        sk("lean")
        ev["sk_end"].record(side)
    proj()
    ev["pj_end"].record(main_s)
    main_s.wait_stream(side)
    torch.cuda.synchronize()
    timeline = {nm: ev["t0"].elapsed_time(e) for nm, e in ev.items()}
    res["timeline_ms"] = timeline
    print(json.dumps(res))


if __name__ == "__main__":
    main()
