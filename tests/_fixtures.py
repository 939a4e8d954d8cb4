"""Loaders for the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def problems(seed):
    """List of (x, f, noise, xs, lam, mu_ref, var_ref, full_ref|None)."""
    d = load("gpr_problems.npz")
    p = f"s{seed}_"
    n, m, lam = d[p + "n"], d[p + "m"], d[p + "lam"]
    x, f, noise, xs = d[p + "x"], d[p + "f"], d[p + "noise"], d[p + "xs"]
    mu, var = d[p + "mu"], d[p + "var"]
    full = d[p + "full"] if (p + "full") in d.files else None
    out, a, b, q = [], 0, 0, 0
    for i in range(len(n)):
        ni, mi = int(n[i]), int(m[i])
        fr = None
        if full is not None and q < len(full) and i < 8:
            fr = full[q:q + mi * mi].reshape(mi, mi)
            q += mi * mi
        out.append((x[a:a + ni], f[a:a + ni], noise[a:a + ni], xs[b:b + mi],
                    float(lam[i]), mu[b:b + mi], var[b:b + mi], fr))
        a += ni
        b += mi
    return out


def axis_sets():
    d = load("axis.npz")
    offs = np.concatenate([[0], np.cumsum(d["n"])])
    return [(d["points"][offs[i]:offs[i + 1]], int(d["axis"][i]))
            for i in range(len(d["n"]))]


def scan_frames():
    return load("scan_frames.npz")
