"""ctypes binding of librbgs_b200.so (the C ABI in include/rbgs_b200.h).

Every device computation of the package goes through this module; there is
no CPU fallback.  Importing works without a GPU (so the CPU test suite can
check that the library loads and exports every declared symbol), but any
compute call on a machine without CUDA raises `DeviceUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import re

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librbgs_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "rbgs_b200.h")

F32, F64 = 0, 1
ORDER_REFERENCE, ORDER_FMA, ORDER_REFERENCE_SCALAR, ORDER_TC = 0, 1, 2, 3

_i, _i64, _u64, _sz, _d = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_double
_f = ctypes.c_float
_p = ctypes.c_void_p

# name -> argtypes (all return int unless listed in _RESTYPE)
SIGNATURES = {
    "rb_version": [],
    "rb_last_error": [],
    "rb_launch_count": [],
    "rb_workspace_bytes": [_i64, _i, _i],
    "rb_gauss_prepass_bytes": [_i64, _i, _i, _i],
    "rb_project": [_i, _i, _i, _i, _i64, _i, _i, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _p, _sz, _p],
    "rb_project_trsm": [_i, _i, _i, _i, _i64, _i, _i, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p,
                        _p, _i64, _p, _i64, _i, _p, _sz, _p],
    "rb_gaussian_fill": [_u64, _i, _i64, _i64, _p, _i64, _p],
    "rb_gaussian_fill_bits": [_u64, _i, _i64, _i64, _p, _i64, _i, _p],
    "rb_sketch_gaussian": [_i, _i64, _i, _p, _i64, _p, _i64, _i, _d, _p, _i64, _i, _i, _p, _sz, _p],
    "rb_gauss_prepass": [_i, _p, _i64, _i, _i, _i64, _i, _p, _sz, _p],
    "rb_sketch_gaussian2_pre": [_i, _p, _i64, _i, _i, _p, _i64, _i, _i64, _p, _i64, _i, _d, _p, _i64, _p, _i64, _i, _i,
                                _p, _p, _sz, _p],
    "rb_sketch_gaussian2": [_i, _p, _i64, _i, _i, _p, _i64, _i, _i64, _p, _i64, _i, _d, _p, _i64, _p, _i64, _i, _i,
                            _p, _sz, _p],
    "rb_sketch_srht": [_i, _i64, _i, _p, _i64, _i64, _i64, _p, _p, _i, _d, _p, _i64, _i, _p, _sz, _p],
    "rb_sketch_sparse_sign": [_i, _i64, _i, _p, _i64, _i64, _u64, _i, _i, _p, _i64, _i, _p, _sz, _p],
    "rb_sparse_sign_table": [_u64, _i, _i, _i64, _i64, _p, _p, _p],
    "rb_sketch_sparse_sign_tab": [_i, _i64, _i, _p, _i64, _p, _p, _i, _i, _p, _i64, _i, _p, _sz, _p],
    "rb_sketch_signs": [_i, _i64, _i, _p, _i64, _p, _i64, _i, _d, _p, _i64, _i, _p, _sz, _p],
    "rb_trsm_right": [_i, _i, _i64, _i, _p, _i64, _p, _i64, _p, _i64, _p],
    "rb_gemm_f64": [_i, _i, _i, _i, _i, _d, _p, _i64, _p, _i64, _d, _p, _i64, _p, _sz, _p],
    "rb_gemm_f32": [_i, _i, _i, _i, _i, _f, _p, _i64, _p, _i64, _f, _p, _i64, _p, _sz, _p],
    "rb_certify": [_i, _i, _p, _i64, _p, _i64, _p, _i64, _p, _p, _sz, _p],
    "rb_l2_select": [_i, _i, _p, _p, _p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _p],
    "rb_sumsq3": [_i64, _i, _p, _i64, _i64, _i, _p, _i64, _i64, _i, _p, _i64, _p, _p, _sz, _p],
    "rb_syrk_f64": [_i, _i64, _d, _p, _i64, _d, _p, _i64, _p, _sz, _p],
    "rb_cross": [_i, _i, _i64, _i, _i, _p, _i64, _p, _i64, _p, _i64, _i, _p, _sz, _p],
    "rb_potrf_upper": [_i, _p, _i64, _p, _i64, _p, _p],
    "rb_tsqr_r": [_i, _i64, _i, _p, _i64, _p, _i64, _p, _p, _p, _sz, _p],
    "rb_trsm_left_upper": [_i, _i, _p, _i64, _p, _i64, _p, _p],
    "rb_geqrf_small": [_i, _i, _p, _i64, _p, _i64, _p, _sz, _p],
    "rb_sumsq": [_i, _i64, _i, _p, _i64, _i, _p, _p, _sz, _p],
    "rb_ls_richardson": [_i, _i, _i, _p, _i64, _p, _i64, _i, _p, _i64, _p, _i64, _p, _sz, _p],
    "rb_sketched_cholqr_small": [_i, _i, _p, _i64, _p, _i64, _p, _i64, _p, _p, _sz, _p],
    "rb_stencil7": [_i, _i, _i, _i, _i, _i, _p, _i64, _p, _p, _i64, _p, _i64, _p],
    "rb_csr_spmm": [_i, _i, _i64, _i, _p, _p, _p, _p, _i64, _p, _i64, _p],
    "rb_convert": [_i, _i, _i64, _i, _p, _i64, _p, _i64, _p],
}
_RESTYPE = {"rb_version": ctypes.c_char_p, "rb_last_error": ctypes.c_char_p,
            "rb_workspace_bytes": ctypes.c_size_t, "rb_gauss_prepass_bytes": ctypes.c_size_t,
            "rb_launch_count": ctypes.c_ulonglong}


def launch_count() -> int:
    """Kernels launched by this process through librbgs_b200.so."""
    return int(load().rb_launch_count())


class DeviceUnavailable(RuntimeError):
    """Raised when the CUDA path cannot run (no device or no built library)."""


class KernelError(RuntimeError):
    """A C-ABI call returned an error code."""


_lib = None


def header_symbols():
    """Function names declared in include/rbgs_b200.h."""
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_0-9]+\s*\*?\s+)+\*?(rb_[a-z0-9_]+)\(", text, re.M)))


def load():
    """Load (never build) the shared library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceUnavailable(
            f"{LIB_PATH} is missing: run `python -m paper_2111_14641_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
    _lib = lib
    return lib


def require_cuda():
    if not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device: the RBGS hot path runs only on the GPU "
                                "(no CPU fallback by design)")
    return load()


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def dtype_code(t_or_dtype):
    dt = t_or_dtype.dtype if isinstance(t_or_dtype, torch.Tensor) else t_or_dtype
    if dt == torch.float32:
        return F32
    if dt == torch.float64:
        return F64
    raise TypeError(f"unsupported dtype {dt}")


def call(name, *args):
    """Invoke a C-ABI entry point, raising KernelError on a nonzero return."""
    lib = require_cuda()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.rb_last_error().decode()
        raise KernelError(f"{name} failed ({rc}): {msg}")
    return rc


# ---------------------------------------------------------------------------
# workspace

class Workspace:
    """One growable device scratch buffer per (device, stream) (sketch split
    partials, reduction partials, QR reflectors): calls are asynchronous on
    the caller's stream, so two streams of one device must never share
    scratch (include/rbgs_b200.h, conventions)."""

    _pool = {}

    @classmethod
    def get(cls, nbytes, device):
        idx = torch.device(device).index if torch.device(device).index is not None else torch.cuda.current_device()
        key = (idx, torch.cuda.current_stream(idx).cuda_stream)
        buf = cls._pool.get(key)
        if buf is None or buf.numel() < nbytes:
            nb = max(int(nbytes), 64 << 20)
            if buf is not None:
                # the old buffer may still be read by queued work of its stream
                del cls._pool[key]
            buf = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{idx}")
            cls._pool[key] = buf
        return buf


def ws_for(n, ncols, k, device):
    lib = require_cuda()
    nb = int(lib.rb_workspace_bytes(int(n), int(ncols), int(k)))
    buf = Workspace.get(nb, device)
    return ctypes.c_void_p(buf.data_ptr()), ctypes.c_size_t(buf.numel())
