// hsrq_hessenberg.cu -- the front end either side of the path (SURVEY §8(f)
// row 2): orthogonal reduction of a dense matrix to upper Hessenberg form,
// H = Q^T A Q (householder_hessenberg, testprob.py:146-174, DGEHRD-
// equivalent), and the back-multiplication of eigenvectors of H into
// eigenvectors of A, z = Q x.
//
// Same reflectors as the reference: for column j, x = A[j+1:, j], tail =
// x[1:].x[1:], skipped when tail == 0 (so a Hessenberg input returns
// unchanged with Q = I, bit for bit), alpha = -sign(x0) * hypot(x0,
// sqrt(tail)), v = (x - alpha e1) / ||x - alpha e1||, P = I - 2 v v^T.
// Applied blocked (the DGEHRD / DLAHR2 scheme): a panel of nb reflectors is
// accumulated as Q_p = I - V T V^T with Y = A V T, so only the panel needs
// the level-2 product A[:, j+1:] v per column (HBM-bound GEMV, the inherent
// cost of the reduction); the trailing two-sided update and the Q update are
// fp64 GEMMs on the tensor cores.  Every dense kernel is this library's own
// (hsrq_blas.cuh: DMMA GEMM, streaming GEMV, the small triangular products);
// nothing links cuBLAS.  The per-column vector work -- the reflector with the
// reference's skip rule and sign convention, the T column -- runs in one
// small kernel per column.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "../../include/hsrq.h"
#include "hsrq_device.cuh"
#include "hsrq_blas.cuh"

namespace {

// k_update_reflect: rows per CTA.  The last CTA's vector phase (n rows) sets
// the time: n = 16000 reduce + Q 3.40 / 3.32 / 3.28 s at 256 / 512 / 1024.
#ifndef UR_THREADS
#define UR_THREADS 1024
#endif
constexpr int HB_NB = 64;  // panel width

thread_local char g_herr[256] = "";

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (threadIdx.x == 0) red[32] = v;
  __syncthreads();
  return red[32];
}

// Left update of column j by the panel's earlier reflectors, a[j0+1:] -=
// V[:, :i] u, fused with the reflector of the column (testprob.py:160-172).
// One thread per row of a[j0+1:] (UR_THREADS-thread CTAs); each CTA adds its rows'
// share of tail = x[1:].x[1:] (x = a[j+1:]) to `rpart`; the CTA that finishes
// last (device counter) adds the shares in CTA order and forms the reflector:
// skipped when tail == 0 (a Hessenberg column stays untouched, bit for bit),
// alpha = -sign(x0) hypot(x0, sqrt(tail)), v = (x - alpha e1) / ||.|| with
// ||.||^2 = v0^2 + tail (numpy's unscaled norm, as the reference).  Writes
// vcol = column i of V (length n: zero above row j+1), a[j+1] = alpha,
// a[j+2:] = 0, tau[i] / ntau[i] = 2 / -2 (0 when skipped), T[i, i] = tau.
__global__ void __launch_bounds__(UR_THREADS) k_update_reflect(
    double* a, int64_t n, int64_t j, int64_t j0, int i, const double* V, int64_t ldv,
    const double* u, double* vcol, double* tau, double* ntau, double* Tii, double* rpart,
    unsigned* counter) {
  __shared__ double red[33];
  __shared__ double us[64];
  __shared__ bool last;
  if (threadIdx.x < i) us[threadIdx.x] = u[threadIdx.x];
  __syncthreads();
  const int64_t r = j0 + 1 + (int64_t)blockIdx.x * UR_THREADS + threadIdx.x;
  double t = 0.0;
  if (r < n) {
    double ar = a[r];
    if (i > 0) {
      const double* vr = V + r;
      double s0 = 0.0, s1 = 0.0;
      int k = 0;
      for (; k + 2 <= i; k += 2) {
        s0 += vr[(int64_t)k * ldv] * us[k];
        s1 += vr[(int64_t)(k + 1) * ldv] * us[k + 1];
      }
      if (k < i) s0 += vr[(int64_t)k * ldv] * us[k];
      ar -= s0 + s1;
      a[r] = ar;
    }
    if (r >= j + 2) t = ar * ar;
  }
  t = block_sum(t, red);
  if (threadIdx.x == 0) {
    rpart[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *counter = 0u;  // ready for the next launch
  double tail = 0.0;
  for (unsigned c = 0; c < gridDim.x; c++) tail += __ldcg(rpart + c);  // CTA order: deterministic
  const double x0 = __ldcg(a + j + 1);
  if (tail == 0.0) {  // column already reduced: identity reflector, a stays as it is
    for (int64_t q = threadIdx.x; q < n; q += blockDim.x) vcol[q] = 0.0;
    if (threadIdx.x == 0) {
      *tau = 0.0;
      *ntau = -0.0;
      *Tii = 0.0;
    }
    return;
  }
  const double nrm = hsrq::ghypot(x0, sqrt(tail));
  const double alpha = x0 >= 0.0 ? -nrm : nrm;
  const double v0 = x0 - alpha;
  const double vn = sqrt(v0 * v0 + tail);
  // (rows written by other CTAs are read past L1; each row is read and rewritten by one thread)
  for (int64_t q = threadIdx.x; q < n; q += blockDim.x) {
    double v = 0.0;
    if (q > j) {
      v = (q == j + 1 ? v0 : __ldcg(a + q)) / vn;
      a[q] = q == j + 1 ? alpha : 0.0;
    }
    vcol[q] = v;
  }
  if (threadIdx.x == 0) {
    *tau = 2.0;
    *ntau = -2.0;
    *Tii = 2.0;
  }
}

__global__ void k_set_identity(double* Q, int64_t n, int64_t ldq) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  const int64_t c = t / n, r = t - c * n;
  Q[c * ldq + r] = r == c ? 1.0 : 0.0;
}

bool cu_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    snprintf(g_herr, sizeof(g_herr), "%s: %s", what, cudaGetErrorString(e));
    return false;
  }
  return true;
}

}  // namespace

extern "C" {

const char* hsrq_hessenberg_last_error(void) { return g_herr; }

size_t hsrq_hessenberg_workspace_bytes(int64_t n) {
  const size_t nb = HB_NB;
  const size_t nchunk = ((size_t)n + hblas::GV_COLS - 1) / hblas::GV_COLS;
  return sizeof(double) * (((size_t)n + 1) * nb * 2 + nb * nb + 5 * nb + 2 * nb * ((size_t)n + 1) + 256 +
                           nchunk * (size_t)n + 1 + hblas::GT_RS_MAX * 64 + 8);
}

int64_t hsrq_hessenberg_reduce(double* A, int64_t lda, double* Q, int64_t ldq, int64_t n,
                               void* ws, size_t ws_bytes, void* stream_) {
  if (n < 1 || lda < n || (Q && ldq < n)) return HSRQ_ERR_CONFIG;
  if (ws_bytes < hsrq_hessenberg_workspace_bytes(n)) return HSRQ_ERR_WORKSPACE;
  cudaStream_t stream = (cudaStream_t)stream_;
  const int nb = HB_NB;
  const int64_t ne = (n + 1) & ~(int64_t)1;  // even leading dimension of V, Y, W2 (16-byte columns)
  const int64_t ldv = ne;
  double* V = (double*)ws;              // n x nb (ldv)
  double* Y = V + (size_t)ldv * nb;     // n x nb (ldv)
  double* T = Y + (size_t)ldv * nb;     // nb x nb (upper, lower triangle kept zero)
  double* tau = T + (size_t)nb * nb;    // nb
  double* ntau = tau + nb;              // nb
  double* u = ntau + nb;                // nb
  double* W = u + nb;                   // n x nb (W^T of the left update; Q V T)
  double* part = W + (size_t)nb * n + 256;  // GEMV partial sums
  double* wv = u + nb;                      // V^T v of the current column (raw), nb
  // n x nb (ne); the partial-sum block is rounded up to an even count to keep W2 16-byte aligned
  double* W2 = part + ((((size_t)n + hblas::GV_COLS - 1) / hblas::GV_COLS * (size_t)n + 1) & ~(size_t)1);
  double* ypart = W2 + (size_t)nb * (n + 1);  // GT_RS_MAX x 64
  unsigned* counter = (unsigned*)(ypart + hblas::GT_RS_MAX * 64);
  int rs_rows = 0;
  if (!cu_ok(hblas::dgemm_nt64_setup(), "gemm attributes")) return HSRQ_ERR_CUDA;
  if (!cu_ok(hblas::dgemm_pipe_setup(), "gemm attributes")) return HSRQ_ERR_CUDA;
  if (!cu_ok(cudaMemsetAsync(counter, 0, sizeof(unsigned), stream), "counter")) return HSRQ_ERR_CUDA;
  if (Q) {
    k_set_identity<<<(unsigned)((n * n + 255) / 256), 256, 0, stream>>>(Q, n, ldq);
    if (!cu_ok(cudaGetLastError(), "identity")) return HSRQ_ERR_CUDA;
  }
  using namespace hblas;
  for (int64_t j0 = 0; j0 < n - 2; j0 += nb) {
    const int pb = (int)std::min<int64_t>(nb, n - 2 - j0);
    const int64_t L = n - j0 - 1;  // rows j0+1 .. n-1 (support of the panel's V)
    // Rows [0, s) lie above the panel: nothing inside the panel reads them, so
    // (as DLAHR2 / DGEHRD do) their part of Y = A V T and of the panel columns'
    // right update is deferred to one GEMM after the panel, and the per-column
    // level-2 product only streams rows [s, n).  s = j0 (even, so the streamed
    // rows keep their 16-byte alignment).
    const int64_t s = j0, Ls = n - s;
    if (!cu_ok(cudaMemsetAsync(T, 0, sizeof(double) * nb * nb, stream), "T"))
      return HSRQ_ERR_CUDA;
    for (int i = 0; i < pb; ++i) {
      const int64_t j = j0 + i;
      double* aj = A + j * lda;
      if (i > 0) {
        // (the right update of column j, rows s..: a_j -= Y[s:, :i] V[j, :i]^T, was
        // applied by the previous column's k_gemv_n_reduce_y, in its pass over Y)
        // left update of rows j0+1.. : a -= V T^T V^T a  (u = T^T V^T a in one launch)
        k_gemv_t_trmv<<<gemv_t_grid((int)L, i, &rs_rows), 256, 0, stream>>>(
            (int)L, i, V + j0 + 1, ldv, aj + j0 + 1, u, T, nb, 1, nullptr, u, counter, ypart, rs_rows);
      }
      // ... a -= V u for rows j0+1.., and the column's reflector, one launch
      double* vi = V + (size_t)i * ldv;
      k_update_reflect<<<(unsigned)((L + UR_THREADS - 1) / UR_THREADS), UR_THREADS, 0, stream>>>(
          aj, n, j, j0, i, V, ldv, u, vi, tau + i, ntau + i, T + (size_t)i * nb + i, part, counter);
      if (!cu_ok(cudaGetLastError(), "reflector")) return HSRQ_ERR_CUDA;
      // Y[s:, i] = tau (A[s:, j+1:] v - Y[s:, :i] (V^T v)); T[:i, i] = -tau T[:i, :i] (V^T v)
      double* yi = Y + (size_t)i * ldv;
      if (i > 0)  // w = V^T v (kept raw for Y) and the T column, one launch
        k_gemv_t_trmv<<<gemv_t_grid((int)L, i, &rs_rows), 256, 0, stream>>>(
            (int)L, i, V + j0 + 1, ldv, vi + j0 + 1, wv, T, nb, 0, ntau + i, T + (size_t)i * nb, counter,
            ypart, rs_rows);
      {  // A[s:, j+1:] v, reduced in chunk order with the Y correction and tau fused
        const int nv = (int)(n - j - 1);
        const int nchunk = (nv + GV_COLS - 1) / GV_COLS;
        if (nchunk > 0)
          k_gemv_n_part<<<dim3((unsigned)((Ls + GV_ROWS - 1) / GV_ROWS), (unsigned)nchunk),
                          GV_THREADS, 0, stream>>>((int)Ls, nv, A + (j + 1) * lda + s, lda,
                                                   vi + j + 1, 1, part);
        const bool nxt = i + 1 < pb;  // the panel's next column takes its right update here
        k_gemv_n_reduce_y<<<(unsigned)((Ls + 31) / 32), 128, 0, stream>>>(
            (int)Ls, nchunk, part, Y + s, ldv, i, wv, tau + i, yi + s,
            nxt ? aj + lda + s : nullptr, V + j + 1, ldv);
      }
    }
    const int64_t c0 = j0 + pb, nc = n - c0;  // trailing columns
    if (s > 0) {
      // the deferred rows: Y[:s] = (A[:s, j0+1:] V) T from the untouched rows, then
      // their right update over the panel's own columns and the trailing ones
      // (V[j, i'] = 0 for i' >= j - j0, so panel column j only sees its earlier reflectors)
      // (K from row / column j0: V's row j0 is zero, and the even offset keeps the
      // operands 16-byte aligned for the pipelined GEMM)
      dgemm(false, false, (int)s, pb, (int)Ls, 1.0, A + s * lda, lda, V + s, ldv, 0.0, W2, ne,
            stream);
      dgemm(false, false, (int)s, pb, pb, 1.0, W2, ne, T, nb, 0.0, Y, ldv, stream);  // (A V) T
      // (columns from j0 = s: V's row j0 is zero, and the even offset keeps 16-byte copies)
      dgemm_nt64_sub((int)s, (int)Ls, pb, Y, ldv, V + s, ldv, A + s * lda, lda, stream);
    }
    if (nc > 0) {
      // right: A[s:, c0:] -= Y[s:] V[c0:, :]^T
      dgemm_nt64_sub((int)Ls, (int)nc, pb, Y + s, ldv, V + c0, ldv, A + c0 * lda + s, lda, stream);
      // left: A[j0+1:, c0:] -= V T^T (V^T A[j0+1:, c0:]), with W^T = A^T V (nc x pb)
      dgemm(true, false, (int)nc, pb, (int)Ls, 1.0, A + c0 * lda + s, lda, V + s, ldv, 0.0, W, ne,
            stream);
      dgemm(false, false, (int)nc, pb, pb, 1.0, W, ne, T, nb, 0.0, W2, ne, stream);  // W T
      // (rows from s = j0: V's row j0 is zero)
      dgemm_nt64_sub((int)Ls, (int)nc, pb, V + s, ldv, W2, ne, A + c0 * lda + s, lda, stream);
    }
    if (Q) {
      // Q[:, j0+1:] -= (Q[:, j0+1:] V T) V^T
      dgemm(false, false, (int)n, pb, (int)Ls, 1.0, Q + s * ldq, ldq, V + s, ldv, 0.0, W, ne,
            stream);
      dgemm(false, false, (int)n, pb, pb, 1.0, W, ne, T, nb, 0.0, W2, ne, stream);  // (Q V) T
      dgemm_nt64_sub((int)n, (int)Ls, pb, W2, ne, V + s, ldv, Q + s * ldq, ldq, stream);
    }
    if (!cu_ok(cudaGetLastError(), "panel kernels")) return HSRQ_ERR_CUDA;
  }
  if (!cu_ok(cudaStreamSynchronize(stream), "sync")) return HSRQ_ERR_CUDA;
  return 0;
}

int64_t hsrq_dgemm(int32_t trans_a, int32_t trans_b, int64_t M, int64_t N, int64_t K,
                   double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double beta, double* C, int64_t ldc, void* stream) {
  if (M < 0 || N < 0 || K < 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    return HSRQ_ERR_CONFIG;
  if (!trans_a && trans_b && alpha == -1.0 && beta == 1.0 && K <= hblas::NT_K) {
    // the reduction's rank-nb update shape: its own kernel (k_dgemm_nt64)
    if (!cu_ok(hblas::dgemm_nt64_setup(), "gemm attributes")) return HSRQ_ERR_CUDA;
    hblas::dgemm_nt64_sub((int)M, (int)N, (int)K, A, lda, B, ldb, C, ldc, (cudaStream_t)stream);
  } else {
    if (!cu_ok(hblas::dgemm_pipe_setup(), "gemm attributes")) return HSRQ_ERR_CUDA;
    hblas::dgemm(trans_a != 0, trans_b != 0, (int)M, (int)N, (int)K, alpha, A, lda, B, ldb, beta,
                 C, ldc, (cudaStream_t)stream);
  }
  return cu_ok(cudaGetLastError(), "dgemm") ? 0 : HSRQ_ERR_CUDA;
}

int64_t hsrq_backmultiply(const double* Q, int64_t ldq, int64_t n, const double* X, int64_t ldx,
                          int64_t ncol, double* Z, int64_t ldz, void* stream_) {
  if (n < 1 || ncol < 0 || ldq < n || ldx < n || ldz < n) return HSRQ_ERR_CONFIG;
  if (ncol == 0) return 0;
  if (!cu_ok(hblas::dgemm_pipe_setup(), "gemm attributes")) return HSRQ_ERR_CUDA;
  hblas::dgemm(false, false, (int)n, (int)ncol, (int)n, 1.0, Q, ldq, X, ldx, 0.0, Z, ldz,
               (cudaStream_t)stream_);
  return cu_ok(cudaGetLastError(), "gemm qx") ? 0 : HSRQ_ERR_CUDA;
}

}  // extern "C"
