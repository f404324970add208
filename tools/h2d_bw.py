"""Host->device bandwidth of the e2e input path (pinned, column-major W of
the C2 shape): one copy vs per-block copies on 1, 2 or 4 streams."""
import json
import time

import torch


def main():
    n, m, p = 1_000_000, 800, 40
    Wh = torch.empty((m, n), dtype=torch.float32).pin_memory()
    Wd = torch.empty((m, n), dtype=torch.float32, device="cuda")
    out = {}
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for b in range(m // p):
                with torch.cuda.stream(streams[b % ns]):
                    Wd[b * p:(b + 1) * p].copy_(Wh[b * p:(b + 1) * p], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        out[f"blocks_{ns}streams_GBps"] = Wh.numel() * 4 / dt / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Wd.copy_(Wh, non_blocking=True)
    torch.cuda.synchronize()
    out["one_copy_GBps"] = Wh.numel() * 4 / (time.perf_counter() - t0) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
