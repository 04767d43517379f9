"""Multi-GPU inverse iteration: shifts partitioned, H replicated, X gathered.

Every column of the solve is independent (no kernel couples shifts, and the
restart vectors depend only on the attempt index, inviter.py:76-88), so the
selection shards across ranks with no collective inside the sweep.  One
collective at the end gathers the eigenvectors (plus converged/restarts/
norms/scales) -- NCCL over NVLink on B200 ranks, gloo on CPU in the tests.
(SURVEY.md §8(e).)
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

# flop-model ratio of a complex to a real shift at n=16000, b_r=128
# (1.3330e9 / 6.5329e8, hessrq flops.py)
COMPLEX_COST = 2.04


def shard_bounds(n_real, n_cplx, world):
    """Per-kind shard boundaries: ``(real_cuts, cplx_cuts)``, each ``world + 1`` long.

    Every rank gets an equal share (to one shift) of the real AND of the
    complex shifts, so the flop cost (complex ~2.04 x real at n=16000) and the
    latency-bound diagonal sweeps of both kinds are balanced at once.
    """
    rc = np.array([(n_real * r) // world for r in range(world + 1)], dtype=np.int64)
    cc = np.array([(n_cplx * r) // world for r in range(world + 1)], dtype=np.int64)
    return rc, cc


def local_selection(eigenvalues, rank, world):
    """This rank's shifts (original indices, values) of a mixed selection:
    every world-th shift of each kind, in the order sorted by imaginary part
    -- the same counts as ``shard_bounds`` gives, but each rank a
    representative sample (the guard work of the diagonal sweeps varies along
    the spectrum, and the slowest rank sets the step time)."""
    eigs = np.asarray(eigenvalues, dtype=np.complex128).ravel()
    is_cplx = eigs.imag != 0.0
    ridx = np.nonzero(~is_cplx)[0]
    cidx = np.nonzero(is_cplx)[0]
    cidx = cidx[np.argsort(eigs[cidx].imag, kind="stable")]
    idx = np.concatenate([ridx[rank::world], cidx[rank::world]])
    return idx, eigs[idx]


def _all_gather_rows(t, group, device):
    """all_gather of a (rows, ...) tensor with ragged row counts (pads to the max)."""
    world = dist.get_world_size(group)
    cnt = torch.tensor([t.shape[0]], dtype=torch.int64, device=device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    cnts = [int(c.item()) for c in cnts]
    mx = max(cnts)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
    pad[: t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:c] for o, c in zip(outs, cnts)]


def hsrq3in_distributed(h, eigenvalues, config=None, group=None, solve=None, device=None):
    """hsrq3in (inviter.py:186-254) with the selection sharded over the ranks.

    ``solve(h, eigs_local, config)`` returns an EigvecResult for the local
    shifts (default: this package's hsrq3in on this rank's GPU).  Every rank
    returns the full result in the caller's order.
    """
    if solve is None:
        from .inviter import hsrq3in as solve
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    eigs = np.asarray(eigenvalues, dtype=np.complex128).ravel()
    m = eigs.size
    idx, mine = local_selection(eigs, rank, world)
    if device is None:
        device = (torch.device("cuda", torch.cuda.current_device())
                  if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    n = np.asarray(h.data if hasattr(h, "data") else h).shape[0]
    if mine.size:
        res = solve(h, mine, config)
        vec = np.ascontiguousarray(res.vectors.T)            # (m_local, n) complex
        meta = np.stack([res.converged.astype(np.float64), res.restarts.astype(np.float64),
                         res.norms, np.asarray(res.alpha_exp, dtype=np.float64)], axis=1)
    else:
        vec = np.zeros((0, n), dtype=np.complex128)
        meta = np.zeros((0, 4))
    vt = torch.view_as_real(torch.from_numpy(vec)).to(device)  # (m_local, n, 2)
    mt = torch.from_numpy(meta).to(device)
    it = torch.from_numpy(idx.astype(np.int64)).to(device)
    all_v = _all_gather_rows(vt, group, device)
    all_m = _all_gather_rows(mt, group, device)
    all_i = _all_gather_rows(it, group, device)
    vectors = np.zeros((n, m), dtype=np.complex128)
    conv = np.zeros(m, dtype=bool)
    restarts = np.zeros(m, dtype=np.int64)
    norms = np.zeros(m)
    aexp = np.zeros(m, dtype=np.int32)
    for v, mm, ii in zip(all_v, all_m, all_i):
        ii = ii.cpu().numpy()
        if ii.size == 0:
            continue
        vectors[:, ii] = torch.view_as_complex(v.cpu().contiguous()).numpy().T
        mm = mm.cpu().numpy()
        conv[ii] = mm[:, 0] > 0
        restarts[ii] = mm[:, 1].astype(np.int64)
        norms[ii] = mm[:, 2]
        aexp[ii] = mm[:, 3].astype(np.int32)
    from .inviter import EigvecResult

    return EigvecResult(vectors=vectors, converged=conv, restarts=restarts, norms=norms,
                        eigenvalues=eigs.copy(), alpha=np.ldexp(1.0, aexp), alpha_exp=aexp)
