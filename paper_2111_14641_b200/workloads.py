"""Synthetic inputs of the BASELINE.json configs (no dataset is involved).

C1/C2  trig family   W_ij = sin(10 mu_j (x_i+1)) / (cos(100 mu_j (x_i+1)) + 1.1),
                     x_i = i/(n-1), mu_j = 1 + (pi-1) U_j, U from
                     numpy Generator(Philox(seed)).random(m)
C3     W = U diag(sigma) V^T, U, V N(0,1) from seed, sigma logspaced 1..1e-7
C5     W = G diag(logspace(0, -6, m)), G N(0,1) from seed

Host (numpy, fp64) generators feed the parity tests; device generators
(torch on the GPU, fp64 math, rounded to the storage dtype) feed bench.py,
generating each rank's own rows.  Both compute the same formula; sin/cos
may differ by an ulp between libm and CUDA, so parity tests always upload
the host array.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _device as D


def trig_mu(m: int, seed: int) -> np.ndarray:
    return 1.0 + (math.pi - 1.0) * np.random.Generator(np.random.Philox(seed)).random(m)


def trig_host(n: int, m: int, seed: int, rows=None) -> np.ndarray:
    mu = trig_mu(m, seed)
    i = np.arange(n, dtype=np.float64) if rows is None else np.asarray(rows, dtype=np.float64)
    a = np.outer(i / (n - 1) + 1.0, mu)
    return np.asfortranarray(np.sin(10.0 * a) / (np.cos(100.0 * a) + 1.1))


def lowrank_host(n: int, m: int, seed: int, smin: float = 1e-7, orthonormal: bool = False) -> np.ndarray:
    """C3 on the host (parity samples): U diag(sigma) V^T, U n x m and V m x m
    N(0,1) from numpy Generator(Philox(seed)) (as BASELINE.json writes it:
    not orthonormalised), sigma logspaced 1 .. smin.  orthonormal=True gives
    the certified companion of SURVEY.md 8(d) (U, V with orthonormal
    columns, so cond(W) = 1 / smin exactly)."""
    g = np.random.Generator(np.random.Philox(seed))
    U = g.standard_normal((n, m))
    V = g.standard_normal((m, m))
    if orthonormal:
        U = np.linalg.qr(U)[0]
        V = np.linalg.qr(V)[0]
    sig = np.logspace(0.0, math.log10(smin), m)
    return np.asfortranarray((U * sig[None, :]) @ V.T)


def colscaled_host(n: int, m: int, seed: int, lo: float = 1e-6) -> np.ndarray:
    """C5 on the host (parity samples): G diag(logspace(0, log10(lo), m)),
    G N(0,1) from numpy Generator(Philox(seed))."""
    g = np.random.Generator(np.random.Philox(seed))
    return np.asfortranarray(g.standard_normal((n, m)) * np.logspace(0.0, math.log10(lo), m)[None, :])


def trig_device(n: int, m: int, seed: int, row0: int = 0, n_local: int = None, dtype=torch.float32,
                device=None, chunk_cols: int = 64) -> torch.Tensor:
    """Rows row0 .. row0+n_local-1 of the trig family, column-major on device."""
    dev = D.cuda_device(device)
    n_local = n - row0 if n_local is None else n_local
    mu = torch.from_numpy(trig_mu(m, seed)).to(dev)
    x = (torch.arange(row0, row0 + n_local, dtype=torch.float64, device=dev) / (n - 1) + 1.0)
    out = D.empty_cm(n_local, m, dtype, dev)
    for j0 in range(0, m, chunk_cols):
        j1 = min(m, j0 + chunk_cols)
        a = x[:, None] * mu[None, j0:j1]
        out[:, j0:j1].copy_(torch.sin(10.0 * a) / (torch.cos(100.0 * a) + 1.1))
    return out


def colscaled_gaussian_device(n_local: int, m: int, seed: int, lo: float = 1e-6, dtype=torch.float32,
                              device=None, rank: int = 0, out: torch.Tensor = None) -> torch.Tensor:
    """C5: G diag(logspace(0, log10(lo), m)) for this rank's rows (written
    into `out` when given: the in-place bench regenerates W every step)."""
    dev = D.cuda_device(device)
    g = torch.Generator(device=dev).manual_seed(int(seed) * 1000003 + rank)
    if out is None:
        out = D.empty_cm(n_local, m, dtype, dev)
    scale = torch.logspace(0.0, math.log10(lo), m, dtype=torch.float64, device=dev)
    for j0 in range(0, m, 16):
        j1 = min(m, j0 + 16)
        G = torch.randn(j1 - j0, n_local, generator=g, device=dev, dtype=torch.float32)
        out[:, j0:j1].copy_((G.t().double() * scale[None, j0:j1]))
        del G
    return out


def lowrank_device(n_local: int, m: int, seed: int, smin: float = 1e-7, dtype=torch.float32,
                   device=None, rank: int = 0) -> torch.Tensor:
    """C3: U diag(sigma) V^T, U this rank's rows of an N(0,1) n x m, V N(0,1)
    m x m (same on every rank), sigma logspaced 1..smin."""
    dev = D.cuda_device(device)
    gv = torch.Generator(device=dev).manual_seed(int(seed))
    V = torch.randn(m, m, generator=gv, device=dev, dtype=torch.float64)
    sig = torch.logspace(0.0, math.log10(smin), m, dtype=torch.float64, device=dev)
    B = (sig[:, None] * V.t())  # diag(sigma) V^T
    gu = torch.Generator(device=dev).manual_seed(int(seed) * 7919 + 1 + rank)
    out = D.empty_cm(n_local, m, dtype, dev)
    step = 1 << 20
    for r0 in range(0, n_local, step):
        r1 = min(n_local, r0 + step)
        U = torch.randn(r1 - r0, m, generator=gu, device=dev, dtype=torch.float64)
        out[r0:r1].copy_(U @ B)
    return out
