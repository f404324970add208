"""Loader for the committed golden fixtures (tests/golden/*.npz).

The fixtures were produced by `tests/golden/make_golden.py` from the
unmodified reference; this module only reads them (no /root/reference
access), regenerating the few inputs that were stored as generator specs.
"""

from __future__ import annotations

import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def trig_family(n, m, seed):
    """BASELINE.json configs[0]/[1] generator (also used by make_golden.py)."""
    mu = 1.0 + (math.pi - 1.0) * np.random.Generator(np.random.Philox(seed)).random(m)
    x = np.arange(n, dtype=np.float64) / (n - 1)
    a = np.outer(x + 1.0, mu)
    return np.sin(10.0 * a) / (np.cos(100.0 * a) + 1.1)


def oscillatory(n, m):
    """The paper's correlated family as the reference harness builds it
    (`gen_oscillatory`, bench.py:197-211): column j samples
    sin(10(mu+x)) / (cos(100(mu-x)) + 1.1) at mu = j/m, x = 1/n .. 1."""
    x = np.arange(1, n + 1, dtype=np.float64) / n
    mu = np.arange(1, m + 1, dtype=np.float64) / m
    return np.sin(10.0 * (mu[None, :] + x[:, None])) / (
        np.cos(100.0 * (mu[None, :] - x[:, None])) + 1.1)


def rbgs_cases():
    z = load("rbgs")
    out = {}
    for key in z.files:
        nm, field = key.split("/", 1)
        out.setdefault(nm, {})[field] = z[key]
    for nm, c in out.items():
        spec = [str(x) for x in c["spec"]]
        c["kind"], c["k"], c["n"], c["seed"] = spec[0], int(spec[1]), int(spec[2]), int(spec[3])
        cfg = [str(x) for x in c["cfg"]]
        c["widths"] = tuple(int(w) for w in cfg[0].split(","))
        c["ls_solver"], c["interblock"] = cfg[1], cfg[2]
        c["coarse"], c["fine"] = cfg[3], cfg[4]
        c["certify_blocks"], c["resketch"] = bool(int(cfg[5])), bool(int(cfg[6]))
    for nm, c in out.items():
        if "W" in c:
            continue
        if "Wref" in c:
            c["W"] = out[str(c["Wref"])]["W"]
        elif str(c["Wgen"]) == "osc":
            c["W"] = oscillatory(2048, 120)
        else:
            _, n, m, s = str(c["Wgen"]).split(":")
            c["W"] = trig_family(int(n), int(m), int(s))
    return out


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d else 1.0))
