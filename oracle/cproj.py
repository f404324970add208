"""ctypes loader of oracle/cproj/cproj.c (TEST INFRASTRUCTURE ONLY).

`build()` compiles it with gcc into oracle/cproj/libcproj.so (git-ignored,
travels to the GPU box with the repository snapshot like the product's .so);
`__graft_entry__.build()` calls it.  -ffp-contract=off keeps the Step-3
multiply and subtract separately rounded; the explicit fma() of the TRSM
order is a libm / FMA-instruction fused multiply-add either way.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cproj")
SRC = os.path.join(HERE, "cproj.c")
LIB = os.path.join(HERE, "libcproj.so")
_lib = None


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = ["gcc", "-O3", "-ffp-contract=off", "-fno-fast-math", "-march=x86-64-v3", "-fopenmp", "-shared",
           "-fPIC", "-o", LIB + ".tmp", SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        lib.cproj_project_f32.argtypes = [L, I, I, P, L, P, L, P, L, P, L]
        lib.cproj_project_f32.restype = None
        lib.cproj_trsm_right.argtypes = [L, I, P, L, P, L, P, L]
        lib.cproj_trsm_right.restype = None
        _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def project_f32(Q, X, W):
    """Q' = W - Q X in the reference's order (binary32 in, binary32 out)."""
    Q = np.asfortranarray(Q, dtype=np.float32)
    X = np.asfortranarray(X, dtype=np.float64)
    W = np.asfortranarray(W, dtype=np.float32)
    n, p = W.shape
    c = Q.shape[1] if Q is not None else 0
    assert p <= 64
    out = np.empty((n, p), dtype=np.float32, order="F")
    load().cproj_project_f32(n, c, p, _p(Q), max(n, 1), _p(X), max(c, 1), _p(W), max(n, 1), _p(out), max(n, 1))
    return out


def trsm_right_fma(B, R):
    """X = B R^{-1} in the device kernel's order (binary64)."""
    B = np.asfortranarray(B, dtype=np.float64)
    R = np.asfortranarray(R, dtype=np.float64)
    n, p = B.shape
    assert p <= 64
    out = np.empty((n, p), dtype=np.float64, order="F")
    load().cproj_trsm_right(n, p, _p(B), max(n, 1), _p(R), p, _p(out), max(n, 1))
    return out
