"""Seeded BASELINE.json instances (H and shifts) for parity tests and the bench.

The five configurations of BASELINE.json ``configs`` restated as seeded
generators.  H for configs 3-5 comes straight from
``numpy.random.default_rng(seed)`` and is bit-reproducible on any box with the
same numpy; configs 1-2 go through a Hessenberg reduction and are only
reproducible to rounding.  Shifts are LAPACK eigenvalues (scipy.linalg.eigvals)
and are cached under ``data/`` because they take up to ~26 min at n=16000.
"""

from __future__ import annotations

import argparse
import os
import time

import numpy as np

DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data")


def random_hessenberg(n, seed=0):
    """Configs 3/5: triu N(0,1) plus |N(0,1)|+0.1 on the subdiagonal, drawn in that order."""
    rng = np.random.default_rng(seed)
    h = np.triu(rng.standard_normal((n, n)))
    sub = np.abs(rng.standard_normal(n - 1)) + 0.1
    h[np.arange(1, n), np.arange(0, n - 1)] = sub
    return np.asfortranarray(h)


def graded_hessenberg(n, seed=0):
    """Config 4: H = D^-1 G D with d_i = 2^floor(40 i / n), i = 1..n."""
    g = random_hessenberg(n, seed)
    d = np.ldexp(1.0, (40 * np.arange(1, n + 1)) // n)
    return np.asfortranarray(g * (d[None, :] / d[:, None]))


def similarity_hessenberg(n, lam, seed=0):
    """Configs 1/2: Hessenberg form of V diag(lam) V^-1, V ~ N(0,1)."""
    import scipy.linalg as sl

    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, n))
    a = (v * lam[None, :]) @ np.linalg.inv(v)
    h = np.triu(sl.hessenberg(a), -1)
    return np.asfortranarray(h)


def make_h(cfg, seed=0, n=None):
    if cfg == 1:
        n = n or 256
        return similarity_hessenberg(n, np.arange(1, n + 1, dtype=np.float64), seed)
    if cfg == 2:
        n = n or 4000
        return similarity_hessenberg(n, np.arange(1, n + 1) / n + 1.0, seed)
    if cfg == 3:
        return random_hessenberg(n or 4000, seed)
    if cfg == 4:
        return graded_hessenberg(n or 2000, seed)
    if cfg == 5:
        return random_hessenberg(n or 16000, seed)
    raise ValueError(cfg)


def eig_path(cfg, seed=0):
    return os.path.join(DATA, f"cfg{cfg}_seed{seed}_eigs.npy")


def compute_eigs(cfg, seed=0):
    import scipy.linalg as sl

    h = make_h(cfg, seed)
    t0 = time.time()
    ev = sl.eigvals(h, overwrite_a=True, check_finite=False)
    dt = time.time() - t0
    np.save(eig_path(cfg, seed), ev)
    return ev, dt


def shifts(cfg, seed=0):
    """The shift selection each config asks for (BASELINE.json configs)."""
    ev = np.load(eig_path(cfg, seed))
    if cfg == 1:
        return np.sort(ev.real)
    if cfg == 2:
        return np.sort(ev.real)[::4].copy()
    if cfg == 3:
        return ev[ev.imag > 0]
    if cfg == 4:
        sel = ev[ev.imag >= 0]
        return sel * (1.0 + 1e-14)
    if cfg == 5:
        return ev[ev.imag >= 0]
    raise ValueError(cfg)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", type=int, nargs="+")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    os.makedirs(DATA, exist_ok=True)
    for c in a.cfgs:
        ev, dt = compute_eigs(c, a.seed)
        print(f"cfg{c}: {ev.size} eigenvalues, {np.count_nonzero(ev.imag == 0)} real, {dt:.1f}s", flush=True)
