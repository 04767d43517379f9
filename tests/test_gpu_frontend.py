"""Front end on the GPU: householder_hessenberg
(testprob.py:146-174) via hsrq_hessenberg_reduce against the live
reference's outputs (tests/golden/hessenberg.npz) and the C oracle, the
back-multiplication z = Q x, and the dense pipeline A -> eigenvectors."""

import numpy as np
import pytest

from conftest import golden
from test_oracle_golden import hessenberg_checks

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_reduction_matches_reference_golden():
    from paper_2101_05063_b200.hessenberg import householder_hessenberg

    g = golden("hessenberg")
    tags = list(g["tags"])
    for t in tags:
        a = g[f"{t}_a"]
        h, q = householder_hessenberg(a)
        fwd = t != tags[-1]  # graded case: backward-error bounds only
        hessenberg_checks(a, h, q, g[f"{t}_h"] if fwd else None, g[f"{t}_q"] if fwd else None)
    a = g[f"{tags[9]}_a"]  # already Hessenberg: returned bit for bit, Q = I
    h, q = householder_hessenberg(a)
    assert np.array_equal(h, a) and np.array_equal(q, np.eye(a.shape[0]))


def test_reduction_matches_oracle_multi_panel(oracle):
    """n = 333: five panels of 64 plus a ragged one.  A is block upper
    triangular (blocks 150 + 183), so column 149 is already reduced when the
    sweep reaches it (x = 0): the skip rule fires inside the third panel."""
    from paper_2101_05063_b200.hessenberg import householder_hessenberg

    rng = np.random.default_rng(8)
    a = rng.standard_normal((333, 333))
    a[150:, :150] = 0.0
    h, q = householder_hessenberg(a)
    ho, qo = oracle.householder_hessenberg(a)
    hessenberg_checks(a, h, q, ho, qo)
    assert h[150, 149] == 0.0 and ho[150, 149] == 0.0
    assert np.all(q[150:, :150] == 0.0) and np.all(q[:150, 150:] == 0.0)


def test_backmultiply_and_dense_pipeline():
    """z = Q x against numpy; config-1-like dense A = V diag(1..n) V^-1:
    eigenvectors of A through reduce -> hsrq3in -> back-multiply meet the
    north_star residual bound."""
    from paper_2101_05063_b200 import InviterConfig
    from paper_2101_05063_b200.hessenberg import backmultiply, hsrq3in_dense

    rng = np.random.default_rng(0)
    q = np.linalg.qr(rng.standard_normal((120, 120)))[0]
    x = rng.standard_normal((120, 7)) + 1j * rng.standard_normal((120, 7))
    z = backmultiply(q, x)
    assert np.max(np.abs(z - q @ x)) <= 1e-13 * np.max(np.abs(q @ x))
    n = 256
    V = rng.standard_normal((n, n))
    lam = np.arange(1, n + 1, dtype=float)
    A = V @ np.diag(lam) @ np.linalg.inv(V)
    ev = np.sort(np.linalg.eigvals(A).real)
    res = hsrq3in_dense(A, ev[::8], InviterConfig(b_r=32))
    assert res.converged.all()
    af = np.linalg.norm(A)
    for l, e in enumerate(ev[::8]):
        zl = res.vectors[:, l]
        assert abs(np.linalg.norm(zl) - 1.0) < 1e-12
        r = np.linalg.norm(A @ zl - e * zl) / (af * np.linalg.norm(zl))
        assert r <= 10 * n * np.finfo(float).eps, (l, r)


@pytest.mark.parametrize("ta,tb,M,N,K,beta", [
    (0, 0, 300, 70, 129, 0.0), (0, 1, 257, 190, 64, 1.0), (1, 0, 1000, 64, 3000, 0.0),
    (1, 1, 33, 17, 5, 0.5), (0, 0, 500, 64, 5000, 0.25), (0, 1, 128, 64, 16, -1.0),
    # even leading dimensions: the cp.async-pipelined kernel, ragged tiles and K tails
    (0, 0, 300, 70, 130, 0.0), (0, 1, 258, 190, 66, 1.0), (1, 0, 1000, 64, 3002, 0.0),
    (1, 1, 34, 18, 6, 0.5), (0, 0, 130, 2, 2, 0.0), (1, 0, 64, 200, 17 * 2, -0.5),
    (0, 1, 2, 2, 1000, 2.0)])
def test_front_end_dgemm_matches_fp64_reference(ta, tb, M, N, K, beta):
    """hsrq_dgemm (the front end's DMMA GEMM, csrc/hsrq_blas.cuh) on ragged
    shapes, every transpose combination, beta != 0 (accumulator preload) and
    thin outputs with long K (split-K) vs a torch fp64 product."""
    import ctypes

    from paper_2101_05063_b200 import _lib

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    L = _lib.load()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    # column-major r x c matrices stored as row-major (c, r) tensors
    A = torch.randn((M, K) if ta else (K, M), dtype=torch.float64, device=dev, generator=g)
    B = torch.randn((K, N) if tb else (N, K), dtype=torch.float64, device=dev, generator=g)
    C = torch.randn((N, M), dtype=torch.float64, device=dev, generator=g)
    opA = A if ta else A.t()      # op(A) as a logical M x K tensor
    opB = B if tb else B.t()      # op(B) as K x N
    want = -1.5 * (opA @ opB) + beta * C.t()
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    r = L.hsrq_dgemm(ta, tb, M, N, K, -1.5, P(A), A.shape[1], P(B), B.shape[1], beta, P(C), M,
                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert r == 0
    torch.cuda.synchronize()
    err = (C.t() - want).abs().max().item()
    assert err <= 1e-13 * max(1.0, want.abs().max().item()) * max(1, K) ** 0.5, err


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K,lda,ldb,off", [
    (257, 190, 64, 258, 190, 0),    # 16-byte copies, ragged M and N
    (256, 128, 64, 256, 128, 0),    # exact tiles
    (131, 67, 37, 132, 68, 0),      # partial panel (K < 64), odd extents
    (131, 67, 37, 133, 67, 0),      # odd leading dimensions: 8-byte copies
    (300, 200, 64, 302, 202, 1),    # operands at an odd row offset: 8-byte copies
    (1000, 900, 5, 1000, 900, 0),   # a single K group
])
def test_rank_nb_update_gemm(M, N, K, lda, ldb, off):
    """k_dgemm_nt64 (C -= A B^T, K <= 64: the blocked reduction's trailing and Q
    updates, reached through hsrq_dgemm with alpha = -1, beta = 1) on ragged
    shapes, both copy widths and partial panels vs a torch fp64 product;
    elements outside the M x N block must stay untouched."""
    import ctypes

    from paper_2101_05063_b200 import _lib

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    L = _lib.load()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn((K, lda), dtype=torch.float64, device=dev, generator=g)   # column-major M x K
    B = torch.randn((K, ldb), dtype=torch.float64, device=dev, generator=g)   # column-major N x K
    ldc = M + 3
    C = torch.randn((N + 1, ldc), dtype=torch.float64, device=dev, generator=g)
    C0 = C.clone()
    a = A[:, off:off + M - off]
    b = B[:, off:off + N - off]
    m, n_ = a.shape[1], b.shape[1]
    want = C0[:n_, :m] - b.t() @ a
    P = lambda t, o=0: ctypes.c_void_p(t.data_ptr() + 8 * o)
    r = L.hsrq_dgemm(0, 1, m, n_, K, -1.0, P(A, off), lda, P(B, off), ldb, 1.0, P(C), ldc,
                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert r == 0
    torch.cuda.synchronize()
    err = (C[:n_, :m] - want).abs().max().item()
    assert err <= 1e-13 * max(1.0, want.abs().max().item()) * K ** 0.5, err
    assert torch.equal(C[:n_, m:], C0[:n_, m:]) and torch.equal(C[n_:], C0[n_:])
