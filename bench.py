"""Benchmark: eigenvectors/s and fp64 TFLOP/s of the batched shifted-Hessenberg
robust RQ solve (BASELINE.json metric) on BASELINE config 5.

Workload (config 5): n = 16000 random unreduced Hessenberg (seeded, triu
N(0,1) + |N(0,1)|+0.1 subdiagonal), every real eigenvalue plus one member of
every conjugate pair as shifts (3790 real + 6105 complex = 16000 real
columns), b_r = 128, start vector eps*||H||_inf*ones (inviter.py:117-133).
A step = one _solve_group attempt over all shifts: the full tiled reduce +
robust substitution + normalise/backtransform sweep.  Inputs (H 2 GB, X
2 GB) are far larger than L2 (126 MB), so no explicit flush is needed.

  python bench.py [--gpus N --steps K --warmup W]      our B200 path
  python bench.py --impl reference ...                 the CPU oracle port

Under torchrun (N > 1) shifts are partitioned by cost over the ranks (H
replicated), each rank runs its own sweep, and X is gathered to rank 0 with
NCCL inside the timed step (strong scaling: total work fixed).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "eigenvectors/s and fp64 TFLOP/s (% of peak), n=16000, at 1/2/4/8 B200"
FP64_PEAK_FALLBACK = 37.1  # TFLOP/s, DMMA m16n8k4 measured on this pool (profiles/fp64_peak_r01.txt)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = {}
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
    fp64 = d.get("fp64_tflops")
    src = "MEASURED_PEAKS.json" if fp64 else "measured (tools/microbench/fp64_peak.cu, profiles/fp64_peak_r01.txt)"
    return float(fp64 or FP64_PEAK_FALLBACK), src, float(d.get("hbm_gbs", 6469.3))


def workload(cfg, seed=0, n_override=None):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import instances

    n = n_override or {3: 4000, 4: 2000, 5: 16000, 2: 4000, 1: 256}[cfg]
    h = instances.make_h(cfg, seed, n=n)
    if n_override:
        import scipy.linalg as sl

        ev = sl.eigvals(h)
        sel = ev[ev.imag >= 0]
    else:
        sel = instances.shifts(cfg, seed)
    er = np.sort(sel[sel.imag == 0].real)
    ec = sel[sel.imag > 0]
    # the order solver.solve_group runs complex shifts in (sorted by imaginary
    # part: warps of the diagonal sweep then share guard work); the bench drives
    # GroupSolver directly, so it passes them in that order
    ec = ec[np.argsort(ec.imag, kind="stable")]
    b_r = {1: 32, 2: 64}.get(cfg, 128)
    return h, er, ec, b_r


def partition(er, ec, rank, world):
    """This rank's shifts: every world-th shift of each kind (parallel.local_selection:
    equal counts, each rank a representative sample of the spectrum)."""
    return er[rank::world], ec[rank::world]


class ClockSampler:
    """nvidia-smi style clock/throttle sampling during the timed region (pynvml)."""

    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index=0, period=0.1):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_sample(h, er, ec, b_r, n_real=16, n_cplx=16, threads=None):
    """Time the CPU oracle port on a bounded sample of the same workload."""
    from oracle import oracle as O

    O.build()
    try:
        O.use_reference_blas(True)
    except Exception:
        pass
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(1)
    sr = er[rng.choice(er.size, min(n_real, er.size), replace=False)] if er.size else er
    sc = ec[rng.choice(ec.size, min(n_cplx, ec.size), replace=False)] if ec.size else ec
    n = h.shape[0]
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    # one batch per thread (b_c = shifts per thread)
    t0 = time.perf_counter()
    if sr.size:
        bc = max(1, -(-sr.size // threads))
        O.solve(h, sr, np.repeat(rho * np.ones((n, 1)), sr.size, 1), b_r, bc, mode="eigvec",
                nthreads=threads)
    if sc.size:
        bc = max(1, -(-sc.size // threads))
        O.solve(h, sc, np.repeat(rho * np.ones((n, 1)), sc.size, 1).astype(complex), b_r, bc,
                mode="eigvec", nthreads=threads)
    dt = time.perf_counter() - t0
    return (sr.size + sc.size), dt, threads, f"{sr.size} real + {sc.size} complex shifts of the same H"


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available():
    """hessrq (the unmodified reference package, pip-installed --no-deps into
    baseline/_ref) importable with its numba backend."""
    if not os.path.isdir(os.path.join(REF_DIR, "hessrq")):
        return False
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import hessrq

        return hessrq.backend_name() == "numba"
    except Exception:
        return False


class ReferenceCPU:
    """The reference's own CPU path for this seam: hessrq's numba
    ``_solve_group`` (inviter.py:91-106) -- tiled_reduce + robust_tiled_solve
    in eigvec mode, with the reference's thread executor (``workers``) --
    on a bounded sample of the workload's shifts, one attempt, the same start
    vector.  JIT compiled once outside the timed region."""

    def __init__(self, h, er, ec, b_r, n_real, n_cplx, workers=None):
        import hessrq
        from hessrq.core import TileGrid, as_hessenberg
        from hessrq.inviter import InviterConfig, _solve_group

        assert hessrq.backend_name() == "numba"
        self._solve = _solve_group
        self.hm = as_hessenberg(h)
        self.n = self.hm.n
        self.grid = TileGrid(self.n, b_r)
        self.workers = workers or os.cpu_count() or 1
        self.cfg = InviterConfig(b_r=b_r, workers=self.workers)
        rng = np.random.default_rng(1)
        self.sr = er[rng.choice(er.size, min(n_real, er.size), replace=False)] if er.size else er
        self.sc = ec[rng.choice(ec.size, min(n_cplx, ec.size), replace=False)] if ec.size else ec
        self.rho = np.finfo(float).eps * self.hm.infinity_norm()
        # JIT warm-up on a small instance (outside any timing)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import instances

        hs = as_hessenberg(instances.random_hessenberg(200, 1))
        g2 = TileGrid(200, min(b_r, 200))
        for cp, lam in ((False, np.array([0.5, 0.7])), (True, np.array([0.5 + 1j, 0.2 + 0.3j]))):
            _solve_group(hs, g2, lam, np.ones((200, 2), dtype=complex if cp else float),
                         InviterConfig(b_r=min(b_r, 200)), None, cp)
        self.sample = (f"{self.sr.size} real + {self.sc.size} complex shifts of the same H per "
                       f"step: hessrq's numba _solve_group, workers={self.workers}")

    def step(self):
        """One timed sample; returns (shifts attempted, converged, seconds)."""
        n = self.n
        start = self.rho * np.ones((n, 1))
        conv = 0
        t0 = time.perf_counter()
        if self.sr.size:
            r = self._solve(self.hm, self.grid, self.sr, np.repeat(start, self.sr.size, 1), self.cfg,
                            None, False)
            conv += int(np.sum(r.norms > 0.1 / np.sqrt(n)))
        if self.sc.size:
            r = self._solve(self.hm, self.grid, self.sc,
                            np.repeat(start, self.sc.size, 1).astype(complex), self.cfg, None, True)
            conv += int(np.sum(r.norms > 0.1 / np.sqrt(n)))
        return self.sr.size + self.sc.size, conv, time.perf_counter() - t0


def ref_sample(args, nsteps):
    """Shifts of each kind per step of the reference's CPU path: 128 + 128 = 256
    (four full b_c = 32 batches per kind, so the reference's executor and its
    BLAS work at their efficient sizes -- BASELINE.md §5 asks for >= 256; an 8 +
    8 sample runs the same code at half the per-shift rate), reduced in steps
    of 32 when many steps are asked for, so that the whole run stays within a
    few minutes (about 13 s per 256-shift step on 16 host threads)."""
    per = 128 if nsteps <= 10 else min(128, max(32, int(round(1280.0 / nsteps / 32.0)) * 32))
    return (args.ref_real if args.ref_real is not None else per,
            args.ref_cplx if args.ref_cplx is not None else per)


def arm_config(cfg, n, m_r, m_c, b_r, world):
    """The workload description both arms print (bench contract `config`)."""
    return {
        "workload": f"config{cfg}: n={n} random Hessenberg, {m_r} real + {m_c} complex shifts "
                    f"({m_r + 2 * m_c} real columns), b_r={b_r}, one _solve_group attempt "
                    f"(eigvec mode)",
        "parallelism": f"shifts partitioned over {world} GPU(s), H replicated, NCCL gather of X",
        "l2": "inputs (H, X: 2 GB each) exceed L2; no flush needed",
    }


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    on this host's cores -- hessrq's numba _solve_group from baseline/_ref
    when installed (kind "reference"), else the C oracle port (kind "port")."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    h, er, ec, b_r = workload(args.config, n_override=args.n)
    from paper_2101_05063_b200 import flops as F

    n = h.shape[0]
    if reference_available() and not args.port:
        ref = ReferenceCPU(h, er, ec, b_r, *ref_sample(args, args.warmup + args.steps))
        kind, threads, sample = "reference", ref.workers, ref.sample
        dts, att, conv = [], 0, 0
        for i in range(args.warmup + args.steps):
            a, c, dt = ref.step()
            if i >= args.warmup:
                dts.append(dt)
                att, conv = att + a, conv + c
        nr, nc = ref.sr.size, ref.sc.size
        extra = {"converged_fraction": conv / max(1, att),
                 "delivered_value": conv / float(np.sum(dts)),
                 "note": "value counts every attempted shift; the reference's double scale "
                         "factors underflow at n=16000, so only converged_fraction of them "
                         "deliver an eigenvector (SURVEY.md §0 finding 6); delivered_value "
                         "is that rate"}
    else:
        kind, extra = "port", {}
        dts = []
        for i in range(args.warmup + args.steps):
            cnt, dt, threads, sample = cpu_sample(h, er, ec, b_r, args.cpu_real, args.cpu_cplx)
            if i >= args.warmup:
                dts.append(dt)
        att = cnt * args.steps
        nr, nc = min(args.cpu_real, er.size), min(args.cpu_cplx, ec.size)
    t = float(np.mean(dts))
    v = att / float(np.sum(dts))
    fl = F.reference_flops(n, b_r, nr, nc)
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": "eigenvectors/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-5 instance, LAPACK eigenvalues as shifts)",
        "config": arm_config(args.config, n, er.size, ec.size, b_r, args.gpus),
        "cpu_baseline": dict({"value": v, "unit": "eigenvectors/s", "cores": threads, "kind": kind,
                              "sample": sample, "tflops": fl / t / 1e12}, **extra),
        "e2e": {"value": v, "unit": "eigenvectors/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # HSRQ_BENCH_DIST=1 runs the multi-rank code path (NCCL group, collectives,
    # the gather of X) even with one rank: `torchrun --nproc-per-node 1` on a
    # one-GPU box exercises everything but the peer transfers
    dist_on = world > 1 or os.environ.get("HSRQ_BENCH_DIST") == "1"
    if dist_on:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2101_05063_b200 import _lib
    from paper_2101_05063_b200 import flops as F
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    h, er, ec, b_r = workload(args.config, n_override=args.n)
    n = h.shape[0]
    m_total_r, m_total_c = er.size, ec.size
    my_r, my_c = partition(er, ec, rank, world)
    hm = HessenbergMatrix(h)
    rho = np.finfo(float).eps * hm.infinity_norm()
    lib = _lib.load()

    dh = DeviceHessenberg(hm, dev)
    gs = GroupSolver(dh, b_r, my_c.size, my_r.size)
    gs.set_shifts(my_c, my_r)
    start = torch.full((n,), rho, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(timing=False):
        lib.hsrq_set_timing(1 if timing else 0)
        r = gs.launch(start, True, robust=True, mode="eigvec", stream=stream, sync=False)
        return r

    gather_out = None
    if dist_on:
        from paper_2101_05063_b200.parallel import gather_columns

        counts = torch.tensor([gs.ncol], device=dev)
        allc = [torch.zeros_like(counts) for _ in range(world)]
        dist.all_gather(allc, counts)
        counts = [int(c.item()) for c in allc]
        gather_out = torch.empty((sum(counts), n), dtype=torch.float64, device=dev) if rank == 0 else None

    def gather():
        # parallel.gather_columns: every rank's X block to rank 0 over NCCL
        # send/recv, exactly X's bytes once (what hsrq3in_distributed uses)
        if not dist_on:
            return
        gather_columns(gs.X, counts, dst=0, out=gather_out)

    for _ in range(args.warmup):
        step()
        gather()
    torch.cuda.synchronize()
    nf = lib.hsrq_failure_count(ctypes.c_void_p(gs.ws.data_ptr()), ctypes.c_void_p(stream.cuda_stream))
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    phase = np.zeros(5)
    launches = 0
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step(timing=True)
            launches += int(lib.hsrq_last_launch_count())
            gather()
        e1.record(stream)
        torch.cuda.synchronize()
    lib.hsrq_phase_times(ctypes.c_void_p(phase.ctypes.data))  # summed over the K timed steps
    ms = e0.elapsed_time(e1) / args.steps
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist_on:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(t_local.item())
    phase /= args.steps

    # ---- roofline pass: the same K steps with the lookahead off, so each panel
    # launch runs alone on the GPU (with the lookahead the diagonal sweep of the
    # next column shares the SMs with the panel, and the panel's event times
    # include it); the timed region above is the one `value` reports ----
    phase_serial = np.zeros(5)
    ms_serial = None
    if not args.no_serial_pass:
        os.environ["HSRQ_LOOKAHEAD"] = "0"
        try:
            step()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(args.steps):
                step(timing=True)
            s1.record(stream)
            torch.cuda.synchronize()
            lib.hsrq_phase_times(ctypes.c_void_p(phase_serial.ctypes.data))
            phase_serial /= args.steps
            ms_serial = s0.elapsed_time(s1) / args.steps
        finally:
            del os.environ["HSRQ_LOOKAHEAD"]
            lib.hsrq_set_timing(0)

    # ---- e2e through the C ABI with host (pinned) buffers: hsrq_solve_group_host,
    # the reference's calling convention (numpy in/out); H streams to the device
    # in column blocks overlapped with the sweep, X and the scale factors return ----
    e2e = None
    if not args.no_e2e:
        from paper_2101_05063_b200.solver import HostGroupSolver

        hs = HostGroupSolver(n, b_r, my_c.size, my_r.size, dev)
        pin = lambda shape: torch.empty(shape, dtype=torch.float64).pin_memory().numpy()
        h_host = pin((n, n)).T  # column-major (Fortran) view of pinned memory
        h_host[:] = h
        lam = np.concatenate([my_c.astype(np.complex128), my_r.astype(np.complex128)])
        lre_host, lim_host, b_host = pin(lam.size), pin(lam.size), pin(n)
        lre_host[:], lim_host[:] = lam.real, lam.imag
        b_host[:] = rho
        out = hs.new_output(pinned=True)
        h2d = h_host.nbytes + lre_host.nbytes + lim_host.nbytes + b_host.nbytes
        d2h = (out.X.nbytes + out.seg_exp.nbytes + out.alpha_exp.nbytes + out.norms.nbytes
               + out.log2norm.nbytes + out.fail.nbytes + 8)

        def e2e_step():
            hs.launch(h_host, lre_host, lim_host, b_host, True, out, stream=stream)

        # pipelined: two device workspaces and two host output sets, so solve
        # s+1 sweeps while solve s's X downloads (hsrq_solve_group_host_async)
        hsb = [hs, HostGroupSolver(n, b_r, my_c.size, my_r.size, dev)]
        outs = [out, hs.new_output(pinned=True)]

        def e2e_pipelined(k):
            prev = None
            for s_ in range(k):
                t = hsb[s_ % 2].launch(h_host, lre_host, lim_host, b_host, True, outs[s_ % 2],
                                       stream=stream, wait=False)
                if prev is not None:
                    hsb[(s_ - 1) % 2].wait_ticket(prev, outs[(s_ - 1) % 2])
                prev = t
            hsb[(k - 1) % 2].wait_ticket(prev, outs[(k - 1) % 2])
            return outs[(k - 1) % 2]

        e2e_step()
        torch.cuda.synchronize()
        ee0 = torch.cuda.Event(enable_timing=True)
        ee1 = torch.cuda.Event(enable_timing=True)
        ee0.record(stream)
        e2e_step()  # one synchronous solve, for the unpipelined figure
        ee1.record(stream)
        torch.cuda.synchronize()
        ems_sync = ee0.elapsed_time(ee1)
        e2e_pipelined(2)
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        ee0.record(stream)
        out = e2e_pipelined(max(1, args.steps))
        ee1.record(stream)
        torch.cuda.synchronize()
        ems = ee0.elapsed_time(ee1) / max(1, args.steps)
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if dist_on:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        e2e = {"value": (m_total_r + m_total_c) / (ems / 1e3), "unit": "eigenvectors/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": ems, "ms_per_step_unpipelined": ems_sync,
               "api": "hsrq_solve_group_host_async + hsrq_host_wait, two solves in flight "
                      "(host buffers; each rank returns its shard; every step uploads H and "
                      "downloads X)"}
        # the host-buffer entry returns exactly the device entry's result
        e2e["matches_device_entry"] = bool(
            out.nfail == int(nf) and np.array_equal(out.X, gs.X.cpu().numpy())
            and np.array_equal(out.seg_exp, gs.seg_exp.cpu().numpy()))

    # ---- e2e through the drop-in Python API: hsrq3in(H, eigenvalues) with a
    # numpy H and numpy eigenvalues (caller order), numpy eigenvectors out --
    # exactly what a caller of the reference's entry point (inviter.py:186-254)
    # pays: H upload + checks, the solve, the caller-order result assembly ----
    e2e_api = None
    if not args.no_e2e and world == 1:
        import time as _time

        from paper_2101_05063_b200 import InviterConfig, hsrq3in

        sel_api = np.concatenate([ec, er.astype(np.complex128)])
        sel_api = sel_api[np.random.default_rng(0).permutation(sel_api.size)]
        cfg_api = InviterConfig(b_r=b_r, max_restarts=0)
        hf = np.asfortranarray(h)
        r_api = hsrq3in(hf, sel_api, cfg_api)  # warm-up
        conv_api = int(r_api.converged.sum())
        del r_api
        wall = []
        for _ in range(max(1, args.steps)):
            torch.cuda.synchronize()
            t0 = _time.perf_counter()
            r_api = hsrq3in(hf, sel_api, cfg_api)
            wall.append(_time.perf_counter() - t0)
            host_ms = r_api.extras.get("host_ms")
            del r_api
        ams = 1e3 * float(np.mean(wall))
        e2e_api = {"value": sel_api.size / (ams / 1e3), "unit": "eigenvectors/s", "ms_per_step": ams,
                   "h2d_bytes_per_step": int(h.nbytes + sel_api.nbytes),
                   "d2h_bytes_per_step": int(n * sel_api.size * 16),
                   "api": "hsrq3in(H: numpy float64 (n, n) F-order, eigenvalues: numpy complex128 "
                          "in mixed caller order) -> EigvecResult with numpy (n, m) complex128 "
                          "vectors; one attempt (max_restarts=0); host wall clock",
                   "converged": conv_api, "last_call_ms": host_ms}

    # ---- correctness on this rank's shard: convergence of every column and the
    # north_star residual bound on a sample (the last step's X is the result) ----
    norms_all = gs.norms.cpu().numpy()
    conv = int(np.count_nonzero(norms_all > 0.1 / np.sqrt(n)))
    rng = np.random.default_rng(5)
    samp_c = rng.choice(my_c.size, min(6, my_c.size), replace=False) if my_c.size else []
    samp_r = rng.choice(my_r.size, min(6, my_r.size), replace=False) if my_r.size else []
    hf = np.linalg.norm(h, "fro")
    worst = 0.0
    Xs = gs.X
    for i in samp_c:
        x = Xs[2 * i].cpu().numpy() + 1j * Xs[2 * i + 1].cpu().numpy()
        worst = max(worst, np.linalg.norm(h @ x - my_c[i] * x) / (hf * np.linalg.norm(x)))
    for i in samp_r:
        x = Xs[2 * my_c.size + i].cpu().numpy()
        worst = max(worst, np.linalg.norm(h @ x - my_r[i] * x) / (hf * np.linalg.norm(x)))
    check = {"converged": conv, "shifts": int(gs.ms),
             "max_residual_over_n_eps": worst / (n * np.finfo(float).eps),
             "residual_sample": len(samp_c) + len(samp_r),
             "bound": "||Hx-lx||/(||H||_F ||x||) <= 10 n eps"}

    if rank != 0:
        if dist_on:
            dist.destroy_process_group()
        return 0

    peak, peak_src, hbm = load_peaks()
    traffic, traffic_note = None, None
    prof_rel = "profiles/ncu_r02c_k_panel_cl_cfg5_jt84.json"
    prof = os.path.join(ROOT, prof_rel)
    if os.path.exists(prof) and n == 16000:
        with open(prof) as f:
            pj = json.load(f)
        rd = float(pj["dram__bytes_read.sum"].split()[0]) * 1e9
        wr = float(pj["dram__bytes_write.sum"].split()[0]) * 1e9
        traffic = rd + wr
        traffic_note = {"launch": pj["launch"], "algorithmic_bytes": pj["algorithmic_bytes"],
                        "ratio": traffic / pj["algorithmic_bytes"],
                        "source": prof_rel + " (ncu --set full)"}
    nvec = m_total_r + m_total_c
    ref_fl = F.reference_flops(n, b_r, m_total_r, m_total_c)
    exe_fl = F.executed_flops(n, b_r, m_total_r, m_total_c)
    my_ref_fl = F.reference_flops(n, b_r, my_r.size, my_c.size)
    # panel kernel: algorithmic work = reference ReduceOffdiag + Update flops
    N = (n + b_r - 1) // b_r
    pan_alg = my_ref_fl - (my_r.size * (F.per_shift_flops(n, b_r, False) - _offdiag_update(n, b_r, False))
                           + my_c.size * (F.per_shift_flops(n, b_r, True) - _offdiag_update(n, b_r, True)))
    panel_ms = phase_serial[1] if ms_serial is not None else phase[1]
    ach = pan_alg / (panel_ms / 1e3) / 1e12 if panel_ms > 0 else None
    my_exe = F.executed_flops(n, b_r, my_r.size, my_c.size)
    line = {
        "metric": METRIC,
        "value": nvec / (ms / 1e3),
        "unit": "eigenvectors/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded config-5 instance; shifts = LAPACK eigenvalues, cached in data/)",
        "config": arm_config(args.config, n, m_total_r, m_total_c, b_r, world),
        "tflops": ref_fl / (ms / 1e3) / 1e12,
        "tflops_frac_of_fp64_peak": ref_fl / (ms / 1e3) / 1e12 / (peak * world),
        "executed_tflops": exe_fl / (ms / 1e3) / 1e12,
        "eigenvectors_incl_conjugates_per_s": (m_total_r + 2 * m_total_c) / (ms / 1e3),
        "phase_ms": {"diag": phase[0], "scalars": phase[4], "panel": phase[1],
                     "backtransform": phase[2], "setup": phase[3],
                     "note": "timed region (lookahead on: the diag sweep of column jt-1 runs "
                             "beside panel jt, so diag and panel overlap)"},
        "phase_ms_serial": ({"diag": phase_serial[0], "scalars": phase_serial[4],
                             "panel": phase_serial[1], "backtransform": phase_serial[2],
                             "setup": phase_serial[3], "ms_per_step": ms_serial,
                             "note": "second K-step pass with HSRQ_LOOKAHEAD=0 (phases "
                                     "serialised); the roofline is taken from it"}
                            if ms_serial is not None else None),
        "roofline": {
            "bound": "tensor", "kernel": "k_panel_cl / k_panel (DMMA f64 panel update)",
            "achieved": ach, "peak": peak, "unit": "TFLOP/s",
            "frac": (ach / peak) if ach else None, "traffic": traffic, "traffic_detail": traffic_note,
            "peak_source": peak_src,
            "executed_achieved": my_exe / (panel_ms / 1e3) / 1e12 if panel_ms > 0 else None,
            "algorithmic": "reference flop model (hessrq flops.py) ReduceOffdiag+Update flops of "
                           "the panel launches / summed panel-kernel event time",
            "measured_in": ("phase_ms_serial pass (K steps, lookahead off: each panel launch alone "
                            "on the GPU)" if ms_serial is not None else "timed region"),
        },
        "gpu_launches": launches,
        "failed_shifts": int(nf),
        "check": check,
    }
    if e2e:
        line["e2e"] = e2e
    if e2e_api:
        line["e2e_api"] = e2e_api
    if world == 1 and not args.no_shards:
        line["shard_projection"] = shard_projection(dh, b_r, er, ec, start, stream)
    if world == 1 and not args.no_cpu:
        cnt, dt, threads, sample = cpu_sample(h, er, ec, b_r, args.cpu_real, args.cpu_cplx)
        port = {"value": cnt / dt, "unit": "eigenvectors/s", "cores": threads, "kind": "port",
                "sample": sample}
        if reference_available() and not args.port:
            ref = ReferenceCPU(h, er, ec, b_r, *ref_sample(args, 1))
            a, c, dt = ref.step()
            line["cpu_baseline"] = {"value": a / dt, "unit": "eigenvectors/s", "cores": ref.workers,
                                    "kind": "reference", "sample": ref.sample,
                                    "converged_fraction": c / max(1, a), "port": port}
            # BASELINE.md §5 also asks for workers = 1: a small sample (the per-core rate)
            one = ReferenceCPU(h, er, ec, b_r, 8, 8, workers=1)
            a1, _c1, dt1 = one.step()
            line["cpu_baseline"]["single_worker"] = {"value": a1 / dt1, "unit": "eigenvectors/s",
                                                     "cores": 1, "sample": one.sample}
        else:
            line["cpu_baseline"] = port
    clk_s = clk.summary()
    line["clocks"] = clk_s
    print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()
    return 0


def shard_projection(dh, b_r, er, ec, start, stream, worlds=(1, 2, 4, 8), reps=2):
    """Strong-scaling evidence on one GPU: the per-rank time of every rank's
    shard (``partition``: every world-th shift of each kind) for a W-way
    split, each run alone; the projected step time is the slowest rank's.
    Ranks never wait on one another inside the sweep (H replicated, no
    collective until the final gather of X), so this is each rank's compute
    time; the NCCL gather (~2 GB of X into rank 0 over NVLink, a few ms) is
    not included."""
    import torch

    from paper_2101_05063_b200.solver import GroupSolver

    out = {}
    ms1 = None
    for W in worlds:
        times = []
        for r in range(W):
            my_r, my_c = partition(er, ec, r, W)
            gs = GroupSolver(dh, b_r, my_c.size, my_r.size)
            gs.set_shifts(my_c, my_r)
            gs.launch(start, True, stream=stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                gs.launch(start, True, stream=stream, sync=False)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / reps)
            del gs
        torch.cuda.empty_cache()
        t = max(times)
        if W == 1:
            ms1 = t
        out[str(W)] = {"shard": f"{er.size // W}-{-(-er.size // W)} real + "
                                f"{ec.size // W}-{-(-ec.size // W)} complex shifts per rank",
                       "ms_per_step": t, "rank_ms": [round(v, 2) for v in times],
                       "projected_efficiency": ms1 / (W * t)}
    out["note"] = ("every rank's W-way shard measured alone on this GPU, launches pipelined "
                   "without per-phase events; ms_per_step = the slowest rank (W=1 is the base); "
                   "no collective inside the sweep; excludes the final NCCL gather of X")
    return out


def _offdiag_update(n, b_r, cplx):
    """Per-shift reference flops of ReduceOffdiag + Update tasks (the panel's work)."""
    from paper_2101_05063_b200 import flops as F

    ranges = [(s, min(s + b_r, n)) for s in range(0, n, b_r)]
    tot = 0
    for jt in range(len(ranges)):
        k = ranges[jt][1] - ranges[jt][0]
        for i in range(jt):
            ki = ranges[i][1] - ranges[i][0]
            tot += F._reduce_offdiag(ki, k, cplx) + F._update(ki, k, cplx)
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=None, help="override n (debug; eigvals computed live)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-shards", action="store_true", help="skip the 2/4/8-way shard projection")
    ap.add_argument("--no-serial-pass", action="store_true",
                    help="skip the lookahead-off pass the roofline is taken from")
    ap.add_argument("--cpu-real", type=int, default=64)
    ap.add_argument("--cpu-cplx", type=int, default=64)
    ap.add_argument("--ref-real", type=int, default=None,
                    help="reference arm: real shifts per step (default: ref_sample())")
    ap.add_argument("--ref-cplx", type=int, default=None,
                    help="reference arm: complex shifts per step (default: ref_sample())")
    ap.add_argument("--port", action="store_true", help="time the C oracle port, not hessrq")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
