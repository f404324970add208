"""Per-kernel device time of one C4 block-GMRES solve (torch profiler).
    python tools/c4_prof.py [full|sketched] [grid]"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2111_14641_b200 import krylov, operators, sketching  # noqa: E402
from paper_2111_14641_b200.rbgs import DeviceConfig, RbgsConfig  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "full"
g = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dev = torch.device("cuda", 0)
A = operators.Poisson3D(g, g, g, device=dev)
gen = torch.Generator(device=dev).manual_seed(7)
B = torch.randn(4, A.n, generator=gen, device=dev, dtype=torch.float64).t()
theta = sketching.sparse_sign_operator(488, A.n, 11, 8)
dc = DeviceConfig(device=dev)


def step():
    return krylov.block_gmres(A, B, theta, 61, restarts=1, cfg=RbgsConfig(), device_cfg=dc, diagnostics=mode)


step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep = step()
    torch.cuda.synchronize()
rows = sorted(prof.key_averages(), key=lambda e: -e.device_time_total)
tot = sum(e.device_time_total for e in rows)
print(f"mode {mode}: total device ms {tot / 1e3:.1f}; rel residual {rep.residual_history[-1][1]:.3e}")
for e in rows[:28]:
    print(f"{e.device_time_total / 1e3:10.2f} ms {e.count:6d}  {e.key[:110]}")
