"""R drift of the device factorization against the CPU oracle on an n_s-row
sample of a bench workload, per gaussian sketch mode (tensor / fp64):
    RB_GAUSS_MODE=fp64 python tools/parity_sample.py c2 8192
Test infrastructure: the oracle is the checker."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    n_s = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    cfgd = bench.CONFIGS[name]
    sec, par = bench._oracle_sample(cfgd, n_s, parity=True)
    par["mode"] = os.environ.get("RB_GAUSS_MODE", "auto")
    par["oracle_s"] = sec
    par["config"] = name
    print(json.dumps(par))


if __name__ == "__main__":
    main()
