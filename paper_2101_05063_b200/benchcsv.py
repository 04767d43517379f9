"""``hessrq bench`` on the B200 path: runtime decomposition and flop counters
as a ``hessrq-bench-v1`` CSV (the reference's cmd_bench, cli.py:310-377).

    python -m paper_2101_05063_b200.benchcsv --matrix random:n=4000,seed=0 \\
        --shift-count 256 --kind complex --robust both --compare-henry --out b.csv

Same inputs as the reference command: shifts from the reference's generator
spec ``gen:count=C,kind=K,seed=2,radius=1.5`` (cli.py:79-95), right-hand
sides ``ones`` (cli.py:117-122), b_r = min(tile_rows, n).  Same columns, in
the same order: per-task seconds, total_s (wall clock of the dhsrq3/chsrq3
call, host arrays in and out), the exact flop counters and the Table-1
formula counters (what RunStats accumulates), henry_s (henry_rq_solve on the
same shifts, here the GPU single sweep of csrc/hsrq_henry.cuh).

The B200 kernels fuse task types, so the per-task seconds are the measured
fused-kernel times split in proportion to the reference flop model:
ReduceDiag + Solve share the diagonal-sweep kernels' time, ReduceOffdiag +
Update share the panel GEMM and guard-scalar kernels' time, Backtransform is
its own kernel.  The measured kernel times themselves follow in trailing
columns (gpu_*_s), after the reference's schema.  ``backend`` is "b200";
``workers`` is the number of GPUs (1).

Matrix sources: a file in the reference's matrix format (core.py:300-349,
binary or text, as ``hessrq gen`` writes it), or ``random:n=N,seed=S`` (the
config-3 construction) / ``graded:n=N,seed=S`` (config 4).
"""

from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import numpy as np

from . import _lib, flops
from .backsolve import chsrq3, dhsrq3
from .core import ConfigError, HessenbergMatrix
from .henry import henry_rq_solve

BENCH_SCHEMA = "hessrq-bench-v1"
TASK_TYPES = flops.TASK_TYPES
GPU_PHASES = ("diag", "panel", "backtransform", "setup", "scalars")  # hsrq_phase_times order


def _kv(spec):
    out = {}
    for part in spec.split(","):
        if part.strip():
            k, _, v = part.partition("=")
            out[k.strip()] = v.strip()
    return out


def load_matrix(spec):
    kind, _, rest = spec.partition(":")
    if kind in ("random", "graded"):
        kv = _kv(rest)
        n, seed = int(kv.get("n", "1024")), int(kv.get("seed", "0"))
        rng = np.random.default_rng(seed)
        h = np.triu(rng.standard_normal((n, n)))
        h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
        if kind == "graded":  # H = D^-1 G D, d_i = 2^floor(40 i / n) (BASELINE config 4)
            d = np.ldexp(1.0, (40 * np.arange(1, n + 1)) // n)
            h = h * d[None, :] / d[:, None]
        return HessenbergMatrix(h)
    raise ConfigError(f"matrix source {spec!r}: only the random:/graded: generators are "
                      f"supported (the reference's matrix files are out of scope, SURVEY.md §2)")


def gen_shifts(h, count, kind, seed=2, radius=1.5):
    """The reference bench's shift generator (load_shifts "gen:", cli.py:81-95)."""
    rng = np.random.default_rng(seed)
    scale = radius * h.infinity_norm()
    if kind == "real":
        return scale * rng.uniform(1.0, 2.0, count) * rng.choice([-1.0, 1.0], count)
    if kind == "complex":
        ang = rng.uniform(0.15, np.pi - 0.15, count)
        rad = scale * rng.uniform(1.0, 2.0, count)
        return rad * np.exp(1j * ang)
    raise ConfigError(f"unknown shift kind {kind!r}")


def task_seconds(gpu, ex):
    """Per-task-type seconds from the fused kernels' measured times (``gpu``:
    phase -> s) split in proportion to the exact flop counts ``ex``:
    ReduceDiag + Solve share the diagonal sweeps, ReduceOffdiag + Update the
    panel GEMM and guard-scalar kernels; Backtransform is its own kernel."""
    sec = {}
    d = ex["ReduceDiag"] + ex["Solve"]
    for t in ("ReduceDiag", "Solve"):
        sec[t] = gpu["diag"] * ex[t] / d if d else 0.0
    o = ex["ReduceOffdiag"] + ex["Update"]
    for t in ("ReduceOffdiag", "Update"):
        sec[t] = (gpu["panel"] + gpu["scalars"]) * ex[t] / o if o else 0.0
    sec["Backtransform"] = gpu["backtransform"]
    return sec


def header():
    return (["schema", "backend", "n", "m", "kind", "b_r", "b_c", "workers", "robust"]
            + list(TASK_TYPES) + ["total_s"] + [f"flops_{t}" for t in TASK_TYPES]
            + [f"formula_{t}" for t in TASK_TYPES] + ["henry_s"]
            + [f"gpu_{p}_s" for p in GPU_PHASES])


def bench_rows(h, shifts, rhs, tile_rows=128, batch=32, robust_modes=(True,),
               compare_henry=False):
    """One CSV row per robust mode (cli.py:341-365)."""
    import torch

    lib = _lib.load()
    n = h.n
    m = shifts.shape[0]
    cplx = np.iscomplexobj(shifts)
    b_r = min(tile_rows, n)
    fn = chsrq3 if cplx else dhsrq3
    ex, fo = flops.task_flops(n, b_r, m, cplx)
    rows = []
    for robust in robust_modes:
        fn(h, shifts, rhs, b_r=b_r, b_c=batch, robust=robust)  # warm-up (context, H upload)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(h, shifts, rhs, b_r=b_r, b_c=batch, robust=robust)
        total = time.perf_counter() - t0
        lib.hsrq_phase_times(np.zeros(5).ctypes.data)  # drop any stale timings
        lib.hsrq_set_timing(1)
        try:
            fn(h, shifts, rhs, b_r=b_r, b_c=batch, robust=robust)
            ph = (np.zeros(5)).astype(np.float64)
            lib.hsrq_phase_times(ph.ctypes.data)
        finally:
            lib.hsrq_set_timing(0)
        gpu = dict(zip(GPU_PHASES, ph / 1e3))
        sec = task_seconds(gpu, ex)
        henry_s = ""
        if compare_henry:
            henry_rq_solve(h, shifts, rhs)  # warm-up
            t1 = time.perf_counter()
            henry_rq_solve(h, shifts, rhs)
            henry_s = time.perf_counter() - t1
        rows.append([BENCH_SCHEMA, "b200", n, m, "complex" if cplx else "real", tile_rows, batch,
                      1, "on" if robust else "off"]
                     + [sec[t] for t in TASK_TYPES] + [total]
                     + [ex[t] for t in TASK_TYPES] + [fo[t] for t in TASK_TYPES] + [henry_s]
                     + [gpu[p] for p in GPU_PHASES])
        if compare_henry:
            faster = total <= henry_s
            print(f"# smoke: tiled {total:.3f}s vs per-shift single-sweep {henry_s:.3f}s -> "
                  f"tiled {'<=' if faster else '>'} baseline (backend=b200, workers=1)",
                  file=sys.stderr)
    return rows


def write_rows(path, rows):
    out = open(path, "w", newline="") if path else sys.stdout
    try:
        w = csv.writer(out)
        w.writerow(header())
        w.writerows(rows)
    finally:
        if path:
            out.close()


def main(argv=None):
    p = argparse.ArgumentParser(prog="python -m paper_2101_05063_b200.benchcsv",
                                description="runtime decomposition and flop counters (B200)")
    p.add_argument("--matrix", default="random:n=1024,seed=1")
    p.add_argument("--shift-count", type=int, default=64, dest="shift_count")
    p.add_argument("--kind", choices=("real", "complex"), default="real")
    p.add_argument("--tile-rows", type=int, default=128, dest="tile_rows")
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--robust", choices=("on", "off", "both"), default="on")
    p.add_argument("--compare-henry", action="store_true", dest="compare_henry")
    p.add_argument("--out", default=None)
    a = p.parse_args(argv)
    h = load_matrix(a.matrix)
    shifts = gen_shifts(h, a.shift_count, a.kind)
    rhs = np.ones((h.n, a.shift_count), dtype=np.complex128 if a.kind == "complex" else np.float64)
    modes = [True, False] if a.robust == "both" else [a.robust == "on"]
    write_rows(a.out, bench_rows(h, shifts, rhs, a.tile_rows, a.batch, modes, a.compare_henry))
    return 0


if __name__ == "__main__":
    sys.exit(main())
