// hsrq_blas.cuh -- the fp64 dense kernels of the front end (included by
// hsrq_hessenberg.cu): the DGEMM / DGEMV / DTRMM / DTRMV / DSCAL shapes the
// blocked Householder reduction and the back-multiplication need, written
// for sm_100a instead of calling cuBLAS.
//
//   k_dgemm<TA, TB>  C = alpha op(A) op(B) + beta C (column-major): 128 x 64
//                    CTA tiles, K chunks of 16 staged through shared memory
//                    with a register prefetch of the next chunk, eight warps
//                    of 32 x 32 on fp64 tensor cores (mma.sync m16n8k4 f64 =
//                    DMMA.8x8x4; FP64 has no tcgen05 kind on sm_100a).
//   k_gemv_n         y = alpha A x + beta y: the reduction's level-2 product
//                    A[:, j+1:] v streams the trailing matrix once per column
//                    (HBM-bound, its inherent cost): 256-row x 128-column
//                    blocks, two rows per thread as 16-byte loads, eight
//                    columns in flight, partial sums per column chunk reduced
//                    in a fixed order (deterministic); few columns: a thread
//                    per row.
//   k_gemv_t         y = alpha A^T x + beta y: a CTA per column.
//                    (W T for the panel's triangular factor is k_dgemm too: T is
//                    kept with an explicitly zero lower triangle.)
//   k_trmv_u         x = op(T) x for the panel's small triangular factor.

namespace hblas {

constexpr int GM = 128, GN = 64, GK = 16;

__device__ __forceinline__ void mma_f64(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// op(A)[i][k] and op(B)[k][j] with zero fill outside the matrix
template <bool T>
__device__ __forceinline__ double opa(const double* A, int64_t lda, int M, int K, int i, int k) {
  if (i >= M || k >= K) return 0.0;
  return T ? A[k + (int64_t)i * lda] : A[i + (int64_t)k * lda];
}
template <bool T>
__device__ __forceinline__ double opb(const double* B, int64_t ldb, int K, int N, int k, int j) {
  if (k >= K || j >= N) return 0.0;
  return T ? B[j + (int64_t)k * ldb] : B[k + (int64_t)j * ldb];
}

// C (or, split over K, the partial block blockIdx.z of `part`) = alpha op(A)
// op(B) + beta C over the K range [kz0, kz1).  beta != 0: the accumulators
// start at (beta / alpha) C, loaded before the main loop, so the epilogue is
// stores only (a read-modify-write per element after the loop would expose
// one load latency per element).
template <bool TA, bool TB>
__global__ void __launch_bounds__(256, 2) k_dgemm(int M, int N, int K, double alpha, const double* A,
                                               int64_t lda, const double* B, int64_t ldb,
                                               double beta, double* C, int64_t ldc, int kchunk,
                                               double* part) {
  __shared__ double As[GK][GM + 4];  // [k][m]
  __shared__ double Bs[GN][GK + 4];  // [n][k]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * GM, n0 = blockIdx.y * GN;
  const int kz0 = blockIdx.z * kchunk, kz1 = min(K, kz0 + kchunk);
  const int wm = warp & 3, wn = warp >> 2;
  const int g = lane >> 2, t4 = lane & 3;
  double ra[8], rb[4];
  // thread -> element maps, coalesced along the contiguous index of each operand
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int idx = tid + e * 256;
      int i, k;
      if (TA) {
        i = idx / GK;
        k = idx % GK;
      } else {
        k = idx / GM;
        i = idx % GM;
      }
      ra[e] = opa<TA>(A, lda, M, kz1, m0 + i, k0 + k);
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int idx = tid + e * 256;
      int k, j;
      if (TB) {
        k = idx / GN;
        j = idx % GN;
      } else {
        j = idx / GK;
        k = idx % GK;
      }
      rb[e] = opb<TB>(B, ldb, kz1, N, k0 + k, n0 + j);
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int idx = tid + e * 256;
      int i, k;
      if (TA) {
        i = idx / GK;
        k = idx % GK;
      } else {
        k = idx / GM;
        i = idx % GM;
      }
      As[k][i] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int idx = tid + e * 256;
      int k, j;
      if (TB) {
        k = idx / GN;
        j = idx % GN;
      } else {
        j = idx / GK;
        k = idx % GK;
      }
      Bs[j][k] = rb[e];
    }
  };
  double acc[2][4][4];
  const bool pre = part == nullptr && beta != 0.0;
  const double ba = pre ? beta / alpha : 0.0;
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int r = m0 + wm * 32 + mi * 16 + g + (e >= 2 ? 8 : 0);
        const int cc = n0 + wn * 32 + ni * 8 + 2 * t4 + (e & 1);
        acc[mi][ni][e] = (pre && r < M && cc < N) ? ba * C[r + (int64_t)cc * ldc] : 0.0;
      }
  load(kz0);
  for (int k0 = kz0; k0 < kz1; k0 += GK) {
    __syncthreads();
    store();
    __syncthreads();
    if (k0 + GK < kz1) load(k0 + GK);  // next chunk in flight during the MMAs
#pragma unroll
    for (int kk = 0; kk < GK; kk += 4) {
      double af[2][2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 2; mi++) {
        const int r = wm * 32 + mi * 16 + g;
        af[mi][0] = As[kk + t4][r];
        af[mi][1] = As[kk + t4][r + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ni++) bf[ni] = Bs[wn * 32 + ni * 8 + g][kk + t4];
#pragma unroll
      for (int mi = 0; mi < 2; mi++)
#pragma unroll
        for (int ni = 0; ni < 4; ni++) mma_f64(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
  }
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int r = m0 + wm * 32 + mi * 16 + g + (e >= 2 ? 8 : 0);
        const int cc = n0 + wn * 32 + ni * 8 + 2 * t4 + (e & 1);
        if (r < M && cc < N) {
          if (part)
            part[((int64_t)blockIdx.z * N + cc) * M + r] = acc[mi][ni][e];
          else
            C[r + (int64_t)cc * ldc] = alpha * acc[mi][ni][e];
        }
      }
}

// 16-byte (or zero-filled shorter) asynchronous copy global -> shared
__device__ __forceinline__ void cp_async16_zfill(double* dst, const double* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes));
}

// k_dgemm with the operands staged by a three-stage cp.async pipeline (the
// register-prefetch kernel above exposes one global-load latency per K chunk
// behind two barriers).  Needs 16-byte aligned operand columns (even leading
// dimensions, aligned bases); dgemm() falls back to k_dgemm otherwise.  Each
// operand lands in shared memory in the orientation its memory layout allows
// 16-byte copies for: A [k][m] (not transposed) or [m][k] (transposed),
// B [n][k] (not transposed) or [k][n] (transposed); the row strides (+4) keep
// the fragment reads conflict-free either way.
constexpr int GP_STAGES = 3;
constexpr int GP_A = GM * (GK + 4), GP_B = GN * (GK + 4);  // doubles per stage (the larger orientation)
constexpr size_t GP_SMEM = sizeof(double) * GP_STAGES * (GP_A + GP_B);
template <bool TA, bool TB>
__global__ void __launch_bounds__(256, 2) k_dgemm_pipe(int M, int N, int K, double alpha,
                                                       const double* A, int64_t lda,
                                                       const double* B, int64_t ldb, double beta,
                                                       double* C, int64_t ldc, int kchunk,
                                                       double* part) {
  extern __shared__ __align__(16) double gp_sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * GM, n0 = blockIdx.y * GN;
  const int kz0 = blockIdx.z * kchunk, kz1 = min(K, kz0 + kchunk);
  const int nk = (kz1 - kz0 + GK - 1) / GK;
  const int wm = warp & 3, wn = warp >> 2;
  const int g = lane >> 2, t4 = lane & 3;
  constexpr int LDA_S = TA ? GK + 4 : GM + 4;  // As[m][k] : As[k][m]
  constexpr int LDB_S = TB ? GN + 4 : GK + 4;  // Bs[k][n] : Bs[n][k]
  auto As = [&](int st) { return gp_sm + st * (GP_A + GP_B); };
  auto Bs = [&](int st) { return gp_sm + st * (GP_A + GP_B) + GP_A; };
  auto load = [&](int st, int kc) {
    const int k0 = kz0 + kc * GK;
    double* as = As(st);
    double* bs = Bs(st);
#pragma unroll
    for (int e = 0; e < GM * GK / 2 / 256; e++) {
      const int idx = tid + e * 256;
      if (TA) {  // pairs along k at one row i of op(A)
        const int i = idx / (GK / 2), k = (idx % (GK / 2)) * 2;
        const int left = (m0 + i < M) ? min(2, kz1 - (k0 + k)) : 0;
        const double* src = left > 0 ? A + (k0 + k) + (int64_t)(m0 + i) * lda : A;
        cp_async16_zfill(as + i * LDA_S + k, src, left > 0 ? 8 * left : 0);
      } else {   // pairs along m at one k
        const int k = idx / (GM / 2), i = (idx % (GM / 2)) * 2;
        const int left = (k0 + k < kz1) ? min(2, M - (m0 + i)) : 0;
        const double* src = left > 0 ? A + (m0 + i) + (int64_t)(k0 + k) * lda : A;
        cp_async16_zfill(as + k * LDA_S + i, src, left > 0 ? 8 * left : 0);
      }
    }
#pragma unroll
    for (int e = 0; e < GN * GK / 2 / 256; e++) {
      const int idx = tid + e * 256;
      if (TB) {  // op(B)[k][j] = B[j + k ldb]: pairs along n at one k
        const int k = idx / (GN / 2), j = (idx % (GN / 2)) * 2;
        const int left = (k0 + k < kz1) ? min(2, N - (n0 + j)) : 0;
        const double* src = left > 0 ? B + (n0 + j) + (int64_t)(k0 + k) * ldb : B;
        cp_async16_zfill(bs + k * LDB_S + j, src, left > 0 ? 8 * left : 0);
      } else {   // op(B)[k][j] = B[k + j ldb]: pairs along k at one column j
        const int j = idx / (GK / 2), k = (idx % (GK / 2)) * 2;
        const int left = (n0 + j < N) ? min(2, kz1 - (k0 + k)) : 0;
        const double* src = left > 0 ? B + (k0 + k) + (int64_t)(n0 + j) * ldb : B;
        cp_async16_zfill(bs + j * LDB_S + k, src, left > 0 ? 8 * left : 0);
      }
    }
  };
#pragma unroll
  for (int st = 0; st < GP_STAGES - 1; st++) {
    if (st < nk) load(st, st);
    asm volatile("cp.async.commit_group;");
  }
  double acc[2][4][4];
  const bool pre = part == nullptr && beta != 0.0;
  const double ba = pre ? beta / alpha : 0.0;
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int r = m0 + wm * 32 + mi * 16 + g + (e >= 2 ? 8 : 0);
        const int cc = n0 + wn * 32 + ni * 8 + 2 * t4 + (e & 1);
        acc[mi][ni][e] = (pre && r < M && cc < N) ? ba * C[r + (int64_t)cc * ldc] : 0.0;
      }
  for (int kc = 0; kc < nk; kc++) {
    asm volatile("cp.async.wait_group %0;" ::"n"(GP_STAGES - 2));
    __syncthreads();
    if (kc + GP_STAGES - 1 < nk) load((kc + GP_STAGES - 1) % GP_STAGES, kc + GP_STAGES - 1);
    asm volatile("cp.async.commit_group;");
    const double* as = As(kc % GP_STAGES);
    const double* bs = Bs(kc % GP_STAGES);
#pragma unroll
    for (int kk = 0; kk < GK; kk += 4) {
      double af[2][2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 2; mi++) {
        const int r = wm * 32 + mi * 16 + g;
        af[mi][0] = TA ? as[r * LDA_S + kk + t4] : as[(kk + t4) * LDA_S + r];
        af[mi][1] = TA ? as[(r + 8) * LDA_S + kk + t4] : as[(kk + t4) * LDA_S + r + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ni++) {
        const int cn = wn * 32 + ni * 8 + g;
        bf[ni] = TB ? bs[(kk + t4) * LDB_S + cn] : bs[cn * LDB_S + kk + t4];
      }
#pragma unroll
      for (int mi = 0; mi < 2; mi++)
#pragma unroll
        for (int ni = 0; ni < 4; ni++) mma_f64(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
  }
  asm volatile("cp.async.wait_group 0;");
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int r = m0 + wm * 32 + mi * 16 + g + (e >= 2 ? 8 : 0);
        const int cc = n0 + wn * 32 + ni * 8 + 2 * t4 + (e & 1);
        if (r < M && cc < N) {
          if (part)
            part[((int64_t)blockIdx.z * N + cc) * M + r] = acc[mi][ni][e];
          else
            C[r + (int64_t)cc * ldc] = alpha * acc[mi][ni][e];
        }
      }
}

// C -= A B^T for K <= 64 (the blocked reduction's rank-nb updates: the right
// and left trailing updates and the Q update), A M x K and B N x K column-
// major.  With K this small a K-chunked pipeline is all prologue: here a CTA
// brings its whole 128 x K and 64 x K operand panels into shared memory with
// one burst of cp.async (two commit groups, so the MMAs start on the first K
// half), preloads -C into the accumulators meanwhile, and runs the K loop
// without a barrier; two CTAs per SM (100 KiB each) overlap one's loads and
// stores with the other's DMMAs.  AL: every operand column is 16-byte aligned
// (16-byte copies), otherwise 8-byte copies.
constexpr int NT_K = 64;
constexpr size_t NT_SMEM = sizeof(double) * NT_K * ((GM + 4) + (GN + 4));
__device__ __forceinline__ void cp_async_zfill(double* dst, const double* src, int bytes, int size) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (size == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(bytes));
}
template <bool AL>
__global__ void __launch_bounds__(256, 2) k_dgemm_nt64(int M, int N, int K, const double* A,
                                                       int64_t lda, const double* B, int64_t ldb,
                                                       double* C, int64_t ldc) {
  extern __shared__ __align__(16) double nt_sm[];
  double (*As)[GM + 4] = reinterpret_cast<double (*)[GM + 4]>(nt_sm);                 // [k][m]
  double (*Bs)[GN + 4] = reinterpret_cast<double (*)[GN + 4]>(nt_sm + NT_K * (GM + 4));  // [k][n]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * GM, n0 = blockIdx.y * GN;
  const int wm = warp & 3, wn = warp >> 2;
  const int g = lane >> 2, t4 = lane & 3;
  constexpr int W = AL ? 2 : 1;  // doubles per copy
#pragma unroll
  for (int h = 0; h < 2; h++) {
#pragma unroll
    for (int e = 0; e < (NT_K / 2) * GM / W / 256; e++) {
      const int idx = tid + e * 256;
      const int k = h * (NT_K / 2) + idx / (GM / W), i = (idx % (GM / W)) * W;
      const int left = k < K ? min(W, M - (m0 + i)) : 0;
      const double* src = left > 0 ? A + (m0 + i) + (int64_t)k * lda : A;
      cp_async_zfill(&As[k][i], src, left > 0 ? 8 * left : 0, 8 * W);
    }
#pragma unroll
    for (int e = 0; e < (NT_K / 2) * GN / W / 256; e++) {
      const int idx = tid + e * 256;
      const int k = h * (NT_K / 2) + idx / (GN / W), j = (idx % (GN / W)) * W;
      const int left = k < K ? min(W, N - (n0 + j)) : 0;
      const double* src = left > 0 ? B + (n0 + j) + (int64_t)k * ldb : B;
      cp_async_zfill(&Bs[k][j], src, left > 0 ? 8 * left : 0, 8 * W);
    }
    asm volatile("cp.async.commit_group;");
  }
  double acc[2][4][4];
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int r = m0 + wm * 32 + mi * 16 + g + (e >= 2 ? 8 : 0);
        const int cc = n0 + wn * 32 + ni * 8 + 2 * t4 + (e & 1);
        acc[mi][ni][e] = (r < M && cc < N) ? -C[r + (int64_t)cc * ldc] : 0.0;
      }
#pragma unroll
  for (int h = 0; h < 2; h++) {
    if (h == 0)
      asm volatile("cp.async.wait_group 1;");
    else
      asm volatile("cp.async.wait_group 0;");
    __syncthreads();
    if (h * (NT_K / 2) >= K) break;
#pragma unroll
    for (int kk = h * (NT_K / 2); kk < (h + 1) * (NT_K / 2); kk += 4) {
      double af[2][2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 2; mi++) {
        const int r = wm * 32 + mi * 16 + g;
        af[mi][0] = As[kk + t4][r];
        af[mi][1] = As[kk + t4][r + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ni++) bf[ni] = Bs[kk + t4][wn * 32 + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 2; mi++)
#pragma unroll
        for (int ni = 0; ni < 4; ni++) mma_f64(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
  }
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int r = m0 + wm * 32 + mi * 16 + g + (e >= 2 ? 8 : 0);
        const int cc = n0 + wn * 32 + ni * 8 + 2 * t4 + (e & 1);
        if (r < M && cc < N) C[r + (int64_t)cc * ldc] = -acc[mi][ni][e];
      }
}

// y = alpha A x + beta y, A column-major m x n: partial sums of column chunks
// of 128 into part[chunk][row], then k_gemv_n_reduce in chunk order.
constexpr int GV_THREADS = 128, GV_ROWS = 2 * GV_THREADS, GV_COLS = 128;
// two rows per thread (16-byte loads when the rows are 16-byte aligned), eight
// column loads in flight per thread
__global__ void __launch_bounds__(GV_THREADS) k_gemv_n_part(int m, int n, const double* A,
                                                            int64_t lda, const double* x,
                                                            int64_t incx, double* part) {
  const int r = blockIdx.x * GV_ROWS + 2 * threadIdx.x;
  const int c0 = blockIdx.y * GV_COLS, c1 = min(n, c0 + GV_COLS);
  __shared__ double xs[GV_COLS];
  for (int j = threadIdx.x; j < c1 - c0; j += GV_THREADS) xs[j] = x[(int64_t)(c0 + j) * incx];
  __syncthreads();
  if (r >= m) return;
  const double* a = A + r + (int64_t)c0 * lda;
  const int nc = c1 - c0;
  double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
  const bool vec = r + 1 < m && ((reinterpret_cast<uintptr_t>(a) | (lda * 8)) & 15) == 0;
  int j = 0;
  if (vec) {
    for (; j + 8 <= nc; j += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = *reinterpret_cast<const double2*>(a + (int64_t)(j + u) * lda);
#pragma unroll
      for (int u = 0; u < 8; u++) {
        s0[u & 3] += v[u].x * xs[j + u];
        s1[u & 3] += v[u].y * xs[j + u];
      }
    }
    for (; j < nc; j++) {
      const double2 v = *reinterpret_cast<const double2*>(a + (int64_t)j * lda);
      s0[0] += v.x * xs[j];
      s1[0] += v.y * xs[j];
    }
  } else {  // unaligned rows or the last odd row: scalar loads
    for (; j < nc; j++) {
      s0[0] += a[(int64_t)j * lda] * xs[j];
      if (r + 1 < m) s1[0] += a[(int64_t)j * lda + 1] * xs[j];
    }
  }
  part[(int64_t)blockIdx.y * m + r] = (s0[0] + s0[1]) + (s0[2] + s0[3]);
  if (r + 1 < m) part[(int64_t)blockIdx.y * m + r + 1] = (s1[0] + s1[1]) + (s1[2] + s1[3]);
}
__global__ void k_gemv_n_reduce(int m, int nchunk, const double* part, double alpha, double beta,
                                double* y) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double s = 0.0;
#pragma unroll 8
  for (int c = 0; c < nchunk; c++) s += part[(int64_t)c * m + r];
  y[r] = beta == 0.0 ? alpha * s : alpha * s + beta * y[r];
}

// y = alpha A x + beta y for few columns (n <= 64): one thread per row.
__global__ void k_gemv_n_small(int m, int n, const double* A, int64_t lda, const double* x,
                               int64_t incx, double alpha, double beta, double* y) {
  __shared__ double xs[64];
  if (threadIdx.x < n) xs[threadIdx.x] = x[(int64_t)threadIdx.x * incx];
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double s0 = 0.0, s1 = 0.0;
  int j = 0;
  for (; j + 2 <= n; j += 2) {
    s0 += A[r + (int64_t)j * lda] * xs[j];
    s1 += A[r + (int64_t)(j + 1) * lda] * xs[j + 1];
  }
  if (j < n) s0 += A[r + (int64_t)j * lda] * xs[j];
  const double s = s0 + s1;
  y[r] = beta == 0.0 ? alpha * s : alpha * s + beta * y[r];
}

// y = alpha A^T x + beta y, A column-major m x n: one CTA per column.
__global__ void __launch_bounds__(256) k_gemv_t(int m, int n, const double* A, int64_t lda,
                                                const double* x, double alpha, double beta,
                                                double* y) {
  __shared__ double red[8];
  const int col = blockIdx.x;
  const double* a = A + (int64_t)col * lda;
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += 256) s += a[i] * x[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; w++) t += red[w];
    y[col] = beta == 0.0 ? alpha * t : alpha * t + beta * y[col];
  }
}

// The panel's fused column kernels (one launch where the unfused sequence
// needed two or three; the reduction is launch-bound per column):
//
// k_gemv_t_trmv: y = A^T x (grid: columns x row ranges of rs_rows rows, the
// partial sums of a column added in row-range order), and the CTA that
// finishes last (a device counter) then forms z = s op(T) y for the panel's
// triangular factor T (p x p upper, p <= 64): trans = 1 -> z = T^T y (the
// left update's u), trans = 0 -> z = T y (the T column); s = *scale (a device
// scalar, e.g. -tau) or 1 when scale is NULL.  z may alias y.  ypart:
// GT_RS_MAX x 64 scratch.
constexpr int GT_RS_MAX = 16, GT_RS_ROWS = 1024;
__global__ void __launch_bounds__(256) k_gemv_t_trmv(int m, int n, const double* A, int64_t lda,
                                                     const double* x, double* y, const double* T,
                                                     int64_t ldt, int trans, const double* scale,
                                                     double* z, unsigned* counter, double* ypart,
                                                     int rs_rows) {
  __shared__ double red[8];
  __shared__ bool last;
  const int col = blockIdx.x;
  const int r0 = blockIdx.y * rs_rows, r1 = min(m, r0 + rs_rows);
  const double* a = A + (int64_t)col * lda;
  double s0 = 0.0, s1 = 0.0;
  int i = r0 + threadIdx.x;
  for (; i + 256 < r1; i += 512) {
    s0 += a[i] * x[i];
    s1 += a[i + 256] * x[i + 256];
  }
  if (i < r1) s0 += a[i] * x[i];
  double s = s0 + s1;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; w++) t += red[w];
    ypart[blockIdx.y * 64 + col] = t;
    __threadfence();
    last = atomicAdd(counter, 1u) == (unsigned)n * gridDim.y - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double ys[64];
  if (threadIdx.x < n) {
    double t = 0.0;
    for (unsigned rs = 0; rs < gridDim.y; rs++) t += ypart[rs * 64 + threadIdx.x];
    ys[threadIdx.x] = t;
    y[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x < n) {
    const int i = threadIdx.x;
    double acc = 0.0;
    if (!trans) {
      for (int j = i; j < n; j++) acc += T[i + (int64_t)j * ldt] * ys[j];
    } else {
      for (int j = 0; j <= i; j++) acc += T[j + (int64_t)i * ldt] * ys[j];
    }
    z[i] = scale ? *scale * acc : acc;
  }
  if (threadIdx.x == 0) *counter = 0u;  // ready for the next column
}
inline dim3 gemv_t_grid(int m, int n, int* rs_rows) {
  int rs = std::min(GT_RS_MAX, std::max(1, (m + GT_RS_ROWS - 1) / GT_RS_ROWS));
  *rs_rows = ((m + rs - 1) / rs + 1) & ~1;
  return dim3((unsigned)n, (unsigned)((m + *rs_rows - 1) / *rs_rows));
}

// y = tau * (sum_c part[c] - Y[:, :p] w): the Av GEMV's chunk reduction fused
// with the panel correction and the reflector's scale (DLAHR2's Y column).
// Four lanes per row: lane q adds chunks / columns q, q + 4, ... in order, the
// four sums are combined as (0 + 1) + (2 + 3).  blockDim = 128 (32 rows).
// With anext != NULL the same pass over the row of Y also applies the right
// update of the panel's NEXT column, anext -= Y[:, :p + 1] vnext[:p + 1]^T
// (vnext[k] = V[j + 1, k] at stride ldvn; Y[:, p] is the column just formed),
// which would otherwise be a launch of its own per column.
__global__ void __launch_bounds__(128) k_gemv_n_reduce_y(int m, int nchunk, const double* part,
                                                         const double* Y, int64_t ldy, int p,
                                                         const double* w, const double* tau,
                                                         double* y, double* anext,
                                                         const double* vnext, int64_t ldvn) {
  __shared__ double ws[64], vs[65];
  if (threadIdx.x < p) ws[threadIdx.x] = w[threadIdx.x];
  if (anext && threadIdx.x <= p) vs[threadIdx.x] = vnext[(int64_t)threadIdx.x * ldvn];
  __syncthreads();
  // lanes of a quad differ in lane bits 3..4, so a warp's loads cover 8 consecutive rows
  const int lane = threadIdx.x & 31, q = lane >> 3;
  const int r = blockIdx.x * 32 + (threadIdx.x >> 5) * 8 + (lane & 7);
  double s = 0.0, cor = 0.0, upd = 0.0;
  if (r < m) {
#pragma unroll 4
    for (int c = q; c < nchunk; c += 4) s += part[(int64_t)c * m + r];
    if (anext) {
#pragma unroll 4
      for (int k = q; k < p; k += 4) {
        const double yk = Y[r + (int64_t)k * ldy];
        cor += yk * ws[k];
        upd += yk * vs[k];
      }
    } else {
#pragma unroll 4
      for (int k = q; k < p; k += 4) cor += Y[r + (int64_t)k * ldy] * ws[k];
    }
  }
  s += __shfl_xor_sync(0xffffffffu, s, 8);
  cor += __shfl_xor_sync(0xffffffffu, cor, 8);
  upd += __shfl_xor_sync(0xffffffffu, upd, 8);
  s += __shfl_xor_sync(0xffffffffu, s, 16);
  cor += __shfl_xor_sync(0xffffffffu, cor, 16);
  upd += __shfl_xor_sync(0xffffffffu, upd, 16);
  if (r < m && q == 0) {
    const double yr = *tau * (s - cor);
    y[r] = yr;
    if (anext) anext[r] -= upd + yr * vs[p];
  }
}

// x = T x (trans = 0) or T^T x (trans = 1), T p x p upper (ldt), one block.
__global__ void k_trmv_u(int p, const double* T, int64_t ldt, double* x, int trans) {
  __shared__ double xs[64];
  const int i = threadIdx.x;
  if (i < p) xs[i] = x[i];
  __syncthreads();
  if (i < p) {
    double s = 0.0;
    if (!trans) {
      for (int j = i; j < p; j++) s += T[i + (int64_t)j * ldt] * xs[j];
    } else {
      for (int j = 0; j <= i; j++) s += T[j + (int64_t)i * ldt] * xs[j];
    }
    x[i] = s;
  }
}

// x *= *alpha (a device scalar)
__global__ void k_dscal(int n, const double* alpha, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] *= *alpha;
}

// C = alpha sum_z part[z] + beta C (split-K, summed in z order: deterministic)
__global__ void k_dgemm_splitk_reduce(int M, int N, int S, const double* part, double alpha,
                                      double beta, double* C, int64_t ldc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)M * N) return;
  const int r = (int)(t % M), cc = (int)(t / M);
  double acc = 0.0;
  for (int z = 0; z < S; z++) acc += part[((int64_t)z * N + cc) * M + r];
  double* p = C + r + (int64_t)cc * ldc;
  *p = beta == 0.0 ? alpha * acc : alpha * acc + beta * *p;
}

// ---- host wrappers (stream-ordered, column-major, cuBLAS argument order) ----

// The pipelined kernels need their dynamic shared-memory limit raised on the
// current device; entry points call dgemm_pipe_setup() first (cheap, idempotent).
static thread_local bool g_pipe_ready = false;
inline cudaError_t dgemm_pipe_setup() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_dgemm_pipe<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GP_SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_dgemm_pipe<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GP_SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_dgemm_pipe<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GP_SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_dgemm_pipe<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GP_SMEM)) != cudaSuccess) return e;
  g_pipe_ready = true;
  return cudaSuccess;
}

inline void dgemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                  cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  const dim3 grid2((unsigned)((M + GM - 1) / GM), (unsigned)((N + GN - 1) / GN));
  // Split K when the output has too few tiles to fill the GPU (the reduction's
  // n x 64 products with K = n): partial blocks in stream-ordered scratch.
  int S = 1;
  const long tiles = (long)grid2.x * grid2.y;
  if (tiles < 296 && K >= 8 * GK) S = (int)std::min<long>((296 + tiles - 1) / tiles, K / (4 * GK));
  const int kchunk = S > 1 ? ((K + S - 1) / S + GK - 1) / GK * GK : K;
  S = S > 1 ? (K + kchunk - 1) / kchunk : 1;
  double* part = nullptr;
  if (S > 1 && cudaMallocAsync((void**)&part, sizeof(double) * (size_t)S * M * N, s) != cudaSuccess) {
    part = nullptr;
    S = 1;
  }
  const dim3 grid(grid2.x, grid2.y, (unsigned)S);
  const int kc = S > 1 ? kchunk : K;
  // 16-byte aligned operand columns: the cp.async pipeline (dgemm_pipe_setup() once per device)
  const bool al = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
                    (uintptr_t)(lda * 8) | (uintptr_t)(ldb * 8)) & 15) == 0;
  if (al && g_pipe_ready) {
    if (!ta && !tb)
      k_dgemm_pipe<false, false><<<grid, 256, GP_SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
    else if (!ta && tb)
      k_dgemm_pipe<false, true><<<grid, 256, GP_SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
    else if (ta && !tb)
      k_dgemm_pipe<true, false><<<grid, 256, GP_SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
    else
      k_dgemm_pipe<true, true><<<grid, 256, GP_SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
  } else if (!ta && !tb)
    k_dgemm<false, false><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
  else if (!ta && tb)
    k_dgemm<false, true><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
  else if (ta && !tb)
    k_dgemm<true, false><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
  else
    k_dgemm<true, true><<<grid, 256, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kc, part);
  if (part) {
    const int64_t mn = (int64_t)M * N;
    k_dgemm_splitk_reduce<<<(unsigned)((mn + 255) / 256), 256, 0, s>>>(M, N, S, part, alpha, beta, C,
                                                                       ldc);
    cudaFreeAsync(part, s);
  }
}

// C -= A B^T, K <= 64 (see k_dgemm_nt64)
inline void dgemm_nt64_sub(int M, int N, int K, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double* C, int64_t ldc, cudaStream_t s) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  const dim3 grid((unsigned)((M + GM - 1) / GM), (unsigned)((N + GN - 1) / GN));
  const bool al = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
                    (uintptr_t)(lda * 8) | (uintptr_t)(ldb * 8)) & 15) == 0;
  if (al)
    k_dgemm_nt64<true><<<grid, 256, NT_SMEM, s>>>(M, N, K, A, lda, B, ldb, C, ldc);
  else
    k_dgemm_nt64<false><<<grid, 256, NT_SMEM, s>>>(M, N, K, A, lda, B, ldb, C, ldc);
}
inline cudaError_t dgemm_nt64_setup() {  // per call of the reduction: the attribute is per device
  cudaError_t e = cudaFuncSetAttribute(k_dgemm_nt64<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)NT_SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_dgemm_nt64<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)NT_SMEM);
}

// y = alpha op(A) x + beta y; part: scratch of ceil(n / 128) * m doubles (no-trans only)
inline void dgemv(bool trans, int m, int n, double alpha, const double* A, int64_t lda,
                  const double* x, int64_t incx, double beta, double* y, double* part,
                  cudaStream_t s) {
  if (!trans) {
    if (m <= 0) return;
    if (n <= 64) {  // the panel's few-column products (also n = 0: y = beta y)
      k_gemv_n_small<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, n, A, lda, x, incx, alpha,
                                                                 beta, y);
      return;
    }
    const int nchunk = (n + GV_COLS - 1) / GV_COLS;
    k_gemv_n_part<<<dim3((unsigned)((m + GV_ROWS - 1) / GV_ROWS), (unsigned)nchunk), GV_THREADS, 0,
                    s>>>(m, n, A, lda, x, incx, part);
    k_gemv_n_reduce<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(m, nchunk, part, alpha, beta, y);
  } else {
    if (n <= 0) return;
    k_gemv_t<<<(unsigned)n, 256, 0, s>>>(m, n, A, lda, x, alpha, beta, y);
  }
}

}  // namespace hblas
