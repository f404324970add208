"""Small end-to-end cases for compute-sanitizer (tools/sanitize.sh): one RBGS
factorization through the warp-specialised kernels (gauss_tc_partial with the
TMA / mbarrier / TMEM pipeline, project_staged, sumsq3's last-CTA combine,
the cooperative k-dimensional kernels) and one tensor-pipe projection
(project_tc2)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2111_14641_b200 import rbgs as R  # noqa: E402
from paper_2111_14641_b200 import sketching  # noqa: E402
from paper_2111_14641_b200.kernels import BlockPartition  # noqa: E402

g = np.random.Generator(np.random.Philox(5))
n, m, p, k = 2048, 32, 8, 128
W = (g.standard_normal((n, m)) @ np.diag(np.logspace(0, -3, m))).astype(np.float32)
theta = sketching.gaussian_operator(k, n, 11)
for order in ("reference", "tc"):
    cfg = R.RbgsConfig(partition=BlockPartition.uniform(m, p), interblock="sketched_cholqr(1)")
    f = R.rbgs(W, theta, cfg, R.DeviceConfig(projection_order=order))
    torch.cuda.synchronize()
    print(order, "delta", f.cert.delta, flush=True)
f = R.rbgs(W, sketching.SketchOperator("srht", k, n, 3), R.RbgsConfig(partition=BlockPartition.uniform(m, p)))
torch.cuda.synchronize()
print("srht l2_plus_cholqr delta", f.cert.delta)
