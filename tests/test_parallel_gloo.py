"""World-size-2 run of the sharded driver over gloo on CPU.

The per-rank solve is injected: the CPU oracle stands in for each rank's GPU
(test-only), so this exercises the partition, the ragged all-gather and the
reassembly in caller order that hsrq3in_distributed performs over NCCL.
"""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_solve(h, eigs, config):
    """Per-rank stand-in: one attempt of _solve_group on the CPU oracle."""
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2101_05063_b200.inviter import EigvecResult

    n = h.shape[0]
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    er = eigs[eigs.imag == 0].real
    ec = eigs[eigs.imag != 0]
    vec = np.zeros((n, eigs.size), dtype=np.complex128)
    aexp = np.zeros(eigs.size, dtype=np.int32)
    norms = np.zeros(eigs.size)
    if er.size:
        r = O.solve(h, er, np.repeat(rho * np.ones((n, 1)), er.size, 1), config.b_r, mode="eigvec")
        vec[:, eigs.imag == 0] = r.x
        aexp[eigs.imag == 0] = r.alpha_exp
        norms[eigs.imag == 0] = r.norms
    if ec.size:
        r = O.solve(h, ec, np.repeat(rho * np.ones((n, 1)), ec.size, 1).astype(complex), config.b_r,
                    mode="eigvec")
        vec[:, eigs.imag != 0] = r.x
        aexp[eigs.imag != 0] = r.alpha_exp
        norms[eigs.imag != 0] = r.norms
    conv = norms > 0.1 / np.sqrt(n)
    return EigvecResult(vectors=vec, converged=conv, restarts=np.zeros(eigs.size, np.int64),
                        norms=norms, eigenvalues=eigs, alpha_exp=aexp)


def _worker(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2101_05063_b200 import InviterConfig
    from paper_2101_05063_b200.parallel import hsrq3in_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    n = 40
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    ev = np.linalg.eigvals(h)
    sel = np.concatenate([ev[ev.imag > 0][:3], ev[ev.imag == 0][:4], ev[ev.imag > 0][3:5]])
    res = hsrq3in_distributed(h, sel, InviterConfig(b_r=8), solve=_oracle_solve)
    if rank == 0:
        single = _oracle_solve(h, sel, InviterConfig(b_r=8))
        np.save(out, np.stack([np.abs(res.vectors - single.vectors).max(),
                               float(np.array_equal(res.alpha_exp, single.alpha_exp)),
                               float(res.converged.all())]))
    dist.destroy_process_group()


def test_sharded_solve_matches_single_rank(tmp_path):
    out = str(tmp_path / "r.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    err, same_alpha, conv = np.load(out)
    assert err == 0.0 and same_alpha == 1.0 and conv == 1.0
