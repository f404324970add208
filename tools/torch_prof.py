"""Kernel-time breakdown of one bench step under torch.profiler (CUPTI):

    python tools/torch_prof.py c4|c2|c5shard

Runs bench.py's arm in-process for one warm-up and one profiled step and
prints the top kernels by total device time (no wall-clock claims: the
profiler serialises nothing but adds overhead; use bench.py for numbers)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    sys.argv = ["bench.py", "--config", cfg, "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline"]
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        bench.main()
    rows = []
    for e in prof.key_averages():
        if e.device_time_total > 0:
            rows.append((e.device_time_total / 1e3, e.count, e.key[:90]))
    rows.sort(reverse=True)
    tot = sum(r[0] for r in rows)
    print(f"total device ms (warm-up + 1 step): {tot:.1f}")
    for ms, cnt, key in rows[:30]:
        print(f"{ms:10.2f} ms {cnt:6d}  {key}")


if __name__ == "__main__":
    main()
