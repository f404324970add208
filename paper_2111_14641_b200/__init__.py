"""B200-native randomized block Gram-Schmidt (arXiv 2111.14641).

A drop-in for the RBGS hot path of the reference package `sketch_krylov`:
`rbgs`, `RbgsSweep.push_block/finish`, `RbgsConfig`, `certify`,
`sketching.SketchOperator/apply`, `krylov.rbgs_arnoldi/block_gmres`, with
every per-block operation executed by hand-written sm_100a CUDA kernels in
`librbgs_b200.so` (C ABI: include/rbgs_b200.h).  See DESIGN.md.
"""

from . import errors, kernels  # noqa: F401
from .kernels import COARSE, FINE, BlockPartition, Matrix, PrecisionSpec  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # heavy modules (torch-backed) load on first use
    import importlib

    if name in ("rbgs", "sketching", "krylov", "operators", "comm", "workloads"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
