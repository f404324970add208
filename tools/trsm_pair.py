"""Tall right TRSM timing and output fingerprint (for A/B of tri_solve_row).

    python tools/trsm_pair.py [out.json]

Times rb_trsm_right (f32 in/out, fp64 solve) at n = 2^24, p in {32, 40, 64}
and n = 1e6, p = 40 with CUDA events; records a hash of the output bytes so
two builds can be compared bit for bit.
"""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_14641_b200 import _device as D  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(7)
res = {}
for n, p in [(1_000_000, 40), (1 << 24, 32), (1 << 24, 40), (1 << 24, 48), (1 << 24, 61), (1 << 24, 64)]:
    B = D.empty_cm(n, p, torch.float32, dev)
    B.copy_(torch.randn(n, p, generator=g, device=dev))
    R = torch.eye(p, dtype=torch.float64, device=dev) + 0.05 * torch.triu(
        torch.randn(p, p, generator=g, device=dev, dtype=torch.float64))
    Rc = D.to_cm(R)
    out = D.empty_cm(n, p, torch.float32, dev)
    for _ in range(3):
        D.trsm_right(B, Rc, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        D.trsm_right(B, Rc, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    h = hashlib.sha256(out.t().contiguous().cpu().numpy().tobytes()).hexdigest()[:16]
    fl = n * p * p  # ~p^2/2 FMA per row = p^2 flops
    res[f"n{n}_p{p}"] = dict(ms=round(ms, 4), TFLOPs=round(fl / ms / 1e9, 2), sha=h)
    del B, out
print(json.dumps(res))
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(json.dumps(res) + "\n")
