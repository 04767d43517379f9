"""Time / check the front end's DMMA GEMM (hsrq_dgemm) on the reduction's
shapes against torch (cuBLAS) -- diagnostics."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_05063_b200 import _lib  # noqa: E402

L = _lib.load()
dev = torch.device("cuda", 0)
P = lambda t: ctypes.c_void_p(t.data_ptr())
SH = [("right NT", 0, 1, 16000, 15000, 64, 1.0), ("W^T TN", 1, 0, 15000, 64, 16000, 0.0),
      ("left NT", 0, 1, 16000, 15000, 64, 1.0), ("Q NN", 0, 0, 16000, 64, 16000, 0.0),
      ("backmul NN", 0, 0, 16000, 16000, 16000, 0.0)]
for name, ta, tb, M, N, K, beta in SH:
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device=dev)  # row-major storage
    B = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device=dev)
    C = torch.randn((M, N), dtype=torch.float64, device=dev)
    # column-major views: a column-major m x k matrix is a row-major k x m tensor
    Acm = A.t().contiguous().t() if False else A  # noqa
    # use transposed storage: column-major X (r x c) == row-major tensor (c x r)
    Ac = torch.randn((K if not ta else M, M if not ta else K), dtype=torch.float64, device=dev)
    Bc = torch.randn((N if not tb else K, K if not tb else N), dtype=torch.float64, device=dev)
    Cc = torch.randn((N, M), dtype=torch.float64, device=dev)
    lda = Ac.shape[1]
    ldb = Bc.shape[1]
    C0 = Cc.clone()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (ta, tb, M, N, K, -1.0, P(Ac), lda, P(Bc), ldb, beta, P(Cc), M, st)
    L.hsrq_dgemm(*args)
    torch.cuda.synchronize()
    # reference: column-major op(A) = (Ac^T if not ta else Ac) ...
    Am = Ac.t() if not ta else Ac  # M x K  (column-major A = Ac^T)
    Am = Ac.t() if not ta else Ac.t().t()
    opA = Ac.t() if not ta else Ac   # column-major A (M x K) stored as row-major (K x M): A = Ac^T; op(A)^T...
    A_cm = Ac.t()  # the column-major matrix as a logical (rows x cols) tensor
    B_cm = Bc.t()
    oa = A_cm.t() if ta else A_cm
    ob = B_cm.t() if tb else B_cm
    want = -1.0 * (oa @ ob) + beta * C0.t()
    err = (Cc.t() - want).abs().max().item() / want.abs().max().item()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        L.hsrq_dgemm(*args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    e0.record()
    for _ in range(reps):
        torch.matmul(oa, ob)
    e1.record()
    torch.cuda.synchronize()
    ms_t = e0.elapsed_time(e1) / reps
    fl = 2.0 * M * N * K
    print(f"{name:12s} M={M} N={N} K={K}: {ms:8.3f} ms {fl / ms / 1e9:7.2f} TF/s  (cuBLAS {ms_t:7.3f} ms "
          f"{fl / ms_t / 1e9:6.2f} TF/s)  rel err {err:.1e}", flush=True)
