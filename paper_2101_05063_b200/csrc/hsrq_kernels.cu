// hsrq_kernels.cu -- B200 (sm_100a) kernels and C ABI for the batched
// shifted-Hessenberg robust RQ solve (arXiv 2101.05063), the path behind
// hessrq's _solve_group (inviter.py:91-106).
//
// One right-to-left sweep over tile columns jt = N-1 .. 0 replaces the
// reference's two DAG phases (tiled_reduce, reduce.py:39-171, then
// _substitute, backsolve.py:62-313):
//
//   k_diag(jt)   one warp per shift: the diagonal tile's Givens sweep
//                (reduce_diag, numba_backend.py:75-106) fused with the robust
//                in-tile backward substitution that recomputes R on the fly
//                (solve_rsolve :133-195; complex: creduce_diag :420-464 +
//                _build_complex_r :530-551 + robust_trsv_complex :493-527),
//                then the update operands for the panel: Z (the rotated
//                solution segment, update_rupdate step 2, :240-253) and
//                W_j = c_j prod_{t<j} s_t (the reduce_offdiag recursion
//                :109-125 written as a linear combination of H columns).
//   k_panel(jt)  the shared off-diagonal work for every tile row above the
//                diagonal as ONE fp64 tensor-core GEMM over all shifts,
//                A = H[0:js, js-1:je-1] times [W | Z] (DMMA via mma.sync f64),
//                with the three ProtectUpdate guards of update_rupdate
//                (:205-311) in its prologue/epilogue (a CTA owns whole tile
//                rows, so every guard is CTA-local), producing the next
//                crossover column and the updated right-hand sides in place.
//   k_backtransform  rbacktransform / crbacktransform (:326-375, :759-822).
//
// Scale factors are carried as int32 log2 exponents (see include/hsrq.h).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <vector>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/hsrq.h"
#include "hsrq_device.cuh"

namespace {
// NVTX range over a host enqueue region (one range per
// solve, per tile-column step, per backtransform).  Without a profiler
// attached nvtxRangePush is a no-op call.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, int v) {
    char buf[64];
    snprintf(buf, sizeof(buf), fmt, v);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace hsrq;

namespace {

constexpr int MAXK = 128;    // largest tile (b_r) supported on the GPU path

// Panel GEMM tiling.
constexpr int BM = 128;      // rows per CTA (whole tile rows)
constexpr int BN = 32;       // data columns per CTA (-> 2*BN accumulator columns)
constexpr int BK = 16;       // K chunk
constexpr int STAGES = 3;
constexpr int APAD = BM + 4; // smem A row stride (k-major), conflict-free frags
constexpr int BPAD = BK + 4; // smem B row stride (n-major)
constexpr int SMAX = 8;      // max tile rows per CTA
constexpr int PANEL_THREADS = 256;
constexpr int KP = 128;      // stride of the B operand (K padded)

// k_panel fast path: prefetch the epilogue tiles to L2 (HSRQ_PANEL_PREFETCH=0 disables)
__device__ __constant__ int g_panel_prefetch = 1;

// Event counters (guard paths taken), read with hsrq_debug_counters().
__device__ unsigned long long g_ctr[32];
#ifdef HSRQ_COUNTERS
#define HSRQ_COUNT(i) atomicAdd(&g_ctr[(i)], 1ULL)
#else
#define HSRQ_COUNT(i) ((void)0)
#endif

struct StepScalars {         // per shift, written by k_diag, read by k_panel
  double rho_re, rho_im;     // s0 * xbelow[0]      (update_rupdate :213)
  double zk_re, zk_im;       // Z[k-1]              (:302)
  double zmax;               // max_{j<k-1} |Z[j]|  (:268-271)
  double P;                  // prod_t s_t          (reduce_offdiag recursion)
  double c0_re, c0_im;       // cross-tile rotation (reduce_diag :94-101)
};

struct Ctx {
  const double* H;
  int64_t ldh, n;
  int b_r, N;
  const double *lam_re, *lam_im;
  int64_t mc, mr, ms, ncol, ncol_pad;
  double* X;
  int64_t ldx;
  double* Cr;            // crossover, n x ncol (ld ldx)
  double *c_re, *c_im, *s;
  int64_t ldc;
  int compact;           // HSRQ_MODE_COMPACT_ROTATIONS: c_re holds the Stewart code t
                         // (real) / t1 (complex), c_im holds t2 of complex shift q < mc,
                         // s is unused (givens.py:90-198)
  double* Rt;            // compact mode: exact rotations of the current tile column,
                         // [c_re | c_im | s] x ms x KP (the panel operands need them)
  int32_t* E;            // N x ms
  double* Bop;           // (2*ncol_pad) x KP
  StepScalars* SS;       // ms
  double* HM0;           // N x N : max |H[tile i rows, js-1]|
  double* RS;            // N x N : max row sum |H[tile i rows, js:je-1]|
  double* HMK;           // N x MAXK : max_{i<kp} |h(i, kp-1)| of each diagonal tile
  double* XB;            // 2 x N x ms: max |X| over each tile's rows (real: exact;
                         // complex: max(|re|+|im|), an upper bound of max |x|) =
                         // the larger of the two halves (k_panel_cl: one per CTA
                         // of the pair; every other writer: [0] = max, [1] = 0)
  int64_t* fail;         // ms
  unsigned long long* nfail;
  int robust, mode;
  double omega;
  int diag_gemm_only;  // diagnostics: panel without epilogue (HSRQ_PANEL_GEMM_ONLY=1)
  unsigned long long* diag_tl;  // HSRQ_TIMELINE: per-CTA phase timestamps
  int diag_tl_jt;
};

__device__ __forceinline__ void col_of_shift(const Ctx& c, int64_t q, bool& cplx, int64_t& col) {
  cplx = q < c.mc;
  col = cplx ? 2 * q : 2 * c.mc + (q - c.mc);
}

__device__ __forceinline__ int64_t pack_fail(int phase, int tile, int row) {
  return ((int64_t)phase << 56) | ((int64_t)tile << 24) | (int64_t)row;
}

// ---------------------------------------------------------------------------
// setup: HM0 / RS tables (per H, b_r), crossover init, X init
// ---------------------------------------------------------------------------

// atomicMax of non-negative doubles into tile-row slots, warp-reduced first
// when the warp's 32 rows share one tile (b_r a multiple of 32): one atomic
// per warp instead of 32 contending on one address (max is order-free).
__device__ __forceinline__ void tile_max2(double* slot_a, double a, double* slot_b, double b,
                                          bool warp_uniform) {
  if (warp_uniform) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if ((threadIdx.x & 31) != 0) return;
  }
  atomicMax((unsigned long long*)slot_a, dkey(a));
  atomicMax((unsigned long long*)slot_b, dkey(b));
}

// HM0[jt][i] = max_{r in tile i} |H[r, js-1]|             (update_rupdate :207-210)
// RS[jt][i]  = max_{r in tile i} sum_{j=1}^{k-1} |htile[r, j]| (:256-262),
// summed left to right like the reference.  One thread per (row, jt).
__global__ void k_tables(Ctx c) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int jt = blockIdx.y + 1;
  if (jt >= c.N) return;
  int64_t js = (int64_t)jt * c.b_r;
  // js is a multiple of b_r: with b_r % 32 == 0 a warp is wholly inside or
  // outside the rows < js, and its rows share one tile
  const bool wu = (c.b_r & 31) == 0 && (blockDim.x & 31) == 0;
  if (r >= js) return;
  int64_t je = js + c.b_r < c.n ? js + c.b_r : c.n;
  int k = (int)(je - js);
  int i = (int)(r / c.b_r);
  double h0 = fabs(c.H[(js - 1) * c.ldh + r]);
  double acc = 0.0;
  for (int j = 1; j < k; j++) acc += fabs(c.H[(js - 1 + j) * c.ldh + r]);
  tile_max2(&c.HM0[(int64_t)jt * c.N + i], h0, &c.RS[(int64_t)jt * c.N + i], acc, wu);
}

// HMK[jt][kp] = max_{i<kp} |H[js+i, js+kp-1]| (the hmax of solve_rsolve :155-163).
__global__ void k_hmk(Ctx c) {
  const int jt = blockIdx.x, kp = threadIdx.x;
  const int64_t js = (int64_t)jt * c.b_r;
  const int64_t je = js + c.b_r < c.n ? js + c.b_r : c.n;
  if (kp < 1 || kp >= (int)(je - js)) return;
  double m = 0.0;
  for (int i = 0; i < kp; i++) {
    const double v = fabs(c.H[(js + kp - 1) * c.ldh + js + i]);
    if (v > m) m = v;
  }
  c.HMK[(int64_t)jt * MAXK + kp] = m;
}

// The tables of one tile column jt (host-feed mode, where H arrives column
// block by column block): HM0[jt][*] / RS[jt][*] as k_tables (blocks over the
// rows < js) and HMK[jt][*] as k_hmk (the last block).
__global__ void k_tables_jt(Ctx c, int jt) {
  const int64_t js = (int64_t)jt * c.b_r;
  const int64_t je = js + c.b_r < c.n ? js + c.b_r : c.n;
  const int k = (int)(je - js);
  if (blockIdx.x == gridDim.x - 1) {  // HMK
    for (int kp = threadIdx.x; kp < MAXK; kp += blockDim.x) {
      if (kp < 1 || kp >= k) continue;
      double m = 0.0;
      for (int i = 0; i < kp; i++) {
        const double v = fabs(c.H[(js + kp - 1) * c.ldh + js + i]);
        if (v > m) m = v;
      }
      c.HMK[(int64_t)jt * MAXK + kp] = m;
    }
    return;
  }
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (jt < 1 || r >= js) return;
  const bool wu = (c.b_r & 31) == 0 && (blockDim.x & 31) == 0;
  const int i = (int)(r / c.b_r);
  const double h0 = fabs(c.H[(js - 1) * c.ldh + r]);
  double acc = 0.0;
  for (int j = 1; j < k; j++) acc += fabs(c.H[(js - 1 + j) * c.ldh + r]);
  tile_max2(&c.HM0[(int64_t)jt * c.N + i], h0, &c.RS[(int64_t)jt * c.N + i], acc, wu);
}

// X = B (or the broadcast start vector), Cr(:, N-1) = H(:, n-1) - lambda e_n
// (reduce.py:66-69, 77-78).
__global__ void k_init(Ctx c, const double* B, int64_t ldb, int b_broadcast) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t col = blockIdx.y;
  const bool valid = r < c.n && col < c.ncol;
  const bool cplx = col < 2 * c.mc;
  const bool im = cplx && (col & 1);
  const int64_t q = cplx ? col / 2 : c.mc + (col - 2 * c.mc);
  double bb = 0.0;
  if (valid) {
    const double b = b_broadcast ? (im ? 0.0 : B[r]) : B[col * ldb + r];
    c.X[col * c.ldx + r] = b;
    bb = fabs(b);
    if (cplx && !im && !b_broadcast) bb = bb + fabs(B[(col + 1) * ldb + r]);
    double h = im ? 0.0 : c.H[(c.n - 1) * c.ldh + r];
    if (r == c.n - 1) h -= im ? c.lam_im[q] : c.lam_re[q];
    c.Cr[col * c.ldx + r] = h;
  }
  if (im) return;  // uniform per block (one column per blockIdx.y)
  // the per-tile bound of max|X| (XB): warp-reduced when a warp's rows share
  // one tile, one atomic per warp instead of 32 on one address
  if ((c.b_r & 31) == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bb = fmax(bb, __shfl_xor_sync(0xffffffffu, bb, o));
    if ((threadIdx.x & 31) != 0) return;
  }
  if (valid) atomicMax((unsigned long long*)&c.XB[(r / c.b_r) * c.ms + q], dkey(bb));
}

__global__ void k_zero_state(Ctx c, int zero_tables) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t ne = (int64_t)c.N * c.ms;
  if (t < ne) {
    c.E[t] = 0;
    c.XB[t] = 0.0;
    c.XB[ne + t] = 0.0;
  }
  if (t < c.ms) c.fail[t] = 0;
  if (zero_tables && t < (int64_t)c.N * c.N) {
    c.HM0[t] = 0.0;
    c.RS[t] = 0.0;
  }
  if (t == 0) *c.nfail = 0;
}

__global__ void k_zero_bop(double* Bop, int64_t count) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < count) Bop[t] = 0.0;
}

#include "hsrq_diag.cuh"
#include "hsrq_diag_ws.cuh"
#include "hsrq_diag_rx.cuh"

#include "hsrq_panel.cuh"
#include "hsrq_panel_cl.cuh"

#include "hsrq_backtransform.cuh"

#include "hsrq_henry.cuh"

// elementwise helpers for parity tests
__global__ void k_protect_batch(const double* b, const double* h, const double* x, double omega,
                                int64_t count, double* out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < count) {
    int e = protect_update_e(b[t], h[t], x[t], omega);
    out[t] = p2(e);
  }
}
__global__ void k_protect_pair_batch(const double* b1, const double* h1, const double* b2,
                                     const double* h2, const double* x, double omega,
                                     int64_t count, double* out1, double* out2) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < count) {
    int e1, e2;
    protect_update_e2(b1[t], h1[t], b2[t], h2[t], x[t], omega, e1, e2);
    out1[t] = p2(e1);
    out2[t] = p2(e2);
  }
}
__global__ void k_compact_encode(int64_t count, int cplx, const double* c_re, const double* c_im,
                                 const double* s, double* t1, double* t2) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  if (cplx)
    compact_encode_cplx(c_re[t], c_im[t], s[t], t1[t], t2[t]);
  else
    t1[t] = compact_encode(c_re[t], s[t]);
}

__global__ void k_compact_decode(int64_t count, int cplx, const double* t1, const double* t2,
                                 double* c_re, double* c_im, double* s) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  if (cplx)
    compact_decode_cplx(t1[t], t2[t], c_re[t], c_im[t], s[t]);
  else
    compact_decode(t1[t], c_re[t], s[t]);
}

// Compact mode: Stewart codes of tile rows [js, js + k) from the tile scratch
// (one thread per (row, shift); failed shifts' rows are encoded too, harmless).
__global__ void k_compact_tile(Ctx c, int64_t js, int k) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)k * c.ms) return;
  const int64_t q = t / k;
  const int row = (int)(t - q * k);
  const double cr = c.Rt[q * KP + row], s = c.Rt[(2 * c.ms + q) * KP + row];
  if (q < c.mc) {
    double t1, t2;
    compact_encode_cplx(cr, c.Rt[(c.ms + q) * KP + row], s, t1, t2);
    c.c_re[q * c.ldc + js + row] = t1;
    c.c_im[q * c.ldc + js + row] = t2;
  } else {
    c.c_re[q * c.ldc + js + row] = compact_encode(cr, s);
  }
}

__global__ void k_hypot_batch(const double* x, const double* y, int64_t count, double* out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < count) out[t] = ghypot(x[t], y[t]);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

thread_local char g_err[512] = "";
thread_local int64_t g_launches = 0;
int g_timing = 0;
unsigned long long* g_tl = nullptr;
double g_phase_ms[5] = {0, 0, 0, 0, 0};
// Timed solves whose events have not been read yet (hsrq_phase_times).
// Per solve: ev[0] start, ev[1] after setup, per column jt the six events
// 2 + 6 jt + {diag start, diag end, scalars start/end, panel start/end},
// ev[nev - 3] / ev[nev - 2] around the backtransform.
struct PendingTiming {
  cudaEvent_t* ev;
  int nev, N;
};
std::vector<PendingTiming> g_pending;

void drain_timing(double* acc) {
  for (PendingTiming& pt : g_pending) {
    cudaEvent_t* ev = pt.ev;
    const int nev = pt.nev;
    auto tev = [&](int jt, int slot) { return ev[2 + 6 * jt + slot]; };
    cudaEventSynchronize(ev[nev - 2]);
    float t;
    for (int jt = pt.N - 1; jt >= 0; --jt) {
      cudaEventElapsedTime(&t, tev(jt, 0), tev(jt, 1));
      acc[0] += t;
      if (jt == 0) continue;
      cudaEventElapsedTime(&t, tev(jt, 2), tev(jt, 3));
      acc[4] += t;
      cudaEventElapsedTime(&t, tev(jt, 4), tev(jt, 5));
      acc[1] += t;
    }
    cudaEventElapsedTime(&t, ev[nev - 3], ev[nev - 2]);
    acc[2] += t;
    cudaEventElapsedTime(&t, ev[0], ev[1]);
    acc[3] += t;
    cudaEventElapsedTime(&t, ev[1], tev(pt.N - 1, 0));
    acc[3] += t;
    for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
    delete[] ev;
  }
  g_pending.clear();
}

bool ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return false;
  }
  return true;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int g_panel_fast = 1;  // HSRQ_PANEL_FAST=0 forces the general epilogue (testing)
int g_panel_cluster = 1;  // HSRQ_PANEL_CLUSTER=0: the 256-thread k_panel fast path instead of k_panel_cl

// Diagonal-kernel variants: DP lanes per shift and DW warps per CTA, chosen
// per kind (real / complex) from the number of shifts in the launch.  The
// sweeps are latency-bound (a serial 128-step recurrence per shift), so the
// best DP is the one that just fills the GPU: many shifts (one GPU, all of
// config 5) -> few lanes per shift and more rows per lane; few shifts (a
// rank's shard at 4 or 8 GPUs) -> more lanes per shift, shorter row loops.
// Measured (tools/shard_time.py, config-5 shards): complex 6105 -> DP 4,
// 3052 -> 8, 1526 and 763 -> 16/32.  HSRQ_DIAG="DP,DWR,DWC" forces one
// (DP, real DW, complex DW) triple (tuning).
struct DiagVariant {
  int dp, dw;
};
DiagVariant g_force_r = {0, 0}, g_force_c = {0, 0};
int g_diag_ws = -1;    // complex sweep warp pairs per CTA (k_diag_cplx_ws); 0 = off
int g_diag_ws_r = -1;  // real sweep warp pairs per CTA (k_diag_real_ws); 0 = off
int g_diag_rx = -1;    // rotation-ahead complex sweep (k_diag_cplx_rx): pairs per CTA, 0 = off,
                       // -1 = automatic (DP-16 pairs, 8 per CTA, where one warp per shift is picked)

template <int DP, int NP>
size_t diag_ws_smem() {
  return sizeof(double) * (MAXK + NP * (4 * MAXK * (32 / DP) + 3 * MAXK + 32 * (32 / DP)));
}
template <int DP, int NP>
size_t diag_ws_smem_r() {
  return sizeof(double) * (MAXK + NP * (2 * MAXK * (32 / DP) + 3 * MAXK + 16 * (32 / DP)));
}
#define HSRQ_DIAG_WS(X) X(4, 1) X(4, 2) X(4, 3) X(8, 2) X(8, 3) X(8, 4) X(16, 2) X(16, 4) X(32, 4) X(32, 8)
#define HSRQ_DIAG_RX(X) X(16, 4) X(16, 8) X(32, 4) X(32, 8)
#define HSRQ_DIAG_WSR(X) X(4, 2) X(4, 3) X(4, 4) X(8, 2) X(8, 4) X(16, 2) X(16, 4) X(32, 4) X(32, 8)

template <int DP, int DW, bool CPLX>
size_t diag_smem() {
  return sizeof(double) * (MAXK + DW * ((CPLX ? 4 : 2) * MAXK * (32 / DP) + 2 * MAXK));
}

#define HSRQ_DIAG_REAL(X) X(2, 2) X(4, 2) X(4, 4) X(4, 8) X(8, 6) X(16, 8) X(32, 8) X(16, 16) X(32, 16)
#define HSRQ_DIAG_CPLX(X) X(2, 1) X(4, 1) X(4, 2) X(4, 4) X(8, 4) X(16, 8) X(32, 8) X(16, 16) X(32, 16)

// Function attributes (raised dynamic shared-memory limits) and __device__
// symbols are per device: the one-shot setup below runs once per device
// ordinal, under a mutex (a process may drive several GPUs from several
// host threads).
constexpr int MAX_DEVICES = 64;
std::mutex g_setup_mu;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

bool diag_attrs() {
  static bool done[MAX_DEVICES] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= MAX_DEVICES) return false;
  std::lock_guard<std::mutex> lock(g_setup_mu);
  if (done[dev]) return true;
#ifdef HSRQ_FUZZ
  if (const char* m = getenv("HSRQ_FUZZ_MASK")) {
    const unsigned v = (unsigned)strtoul(m, nullptr, 0);
    cudaMemcpyToSymbol(g_fuzz_mask, &v, sizeof(v));
  }
#endif
  const char* pf = getenv("HSRQ_PANEL_FAST");
  if (pf) g_panel_fast = atoi(pf);
  if (const char* pcl = getenv("HSRQ_PANEL_CLUSTER")) g_panel_cluster = atoi(pcl);
  const char* pp = getenv("HSRQ_PANEL_PREFETCH");
  if (pp) {
    int v = atoi(pp);
    cudaMemcpyToSymbol(g_panel_prefetch, &v, sizeof(int));
  }
  const char* e = getenv("HSRQ_DIAG");
  if (e) {
    int dp, dwr, dwc, d4;
    const int got = sscanf(e, "%d,%d,%d,%d", &dp, &dwr, &dwc, &d4);
    if (got == 4) {  // "DPR,DWR,DPC,DWC": separate lanes per shift
      g_force_r = DiagVariant{dp, dwr};
      g_force_c = DiagVariant{dwc, d4};
    } else if (got == 3) {
      g_force_r = DiagVariant{dp, dwr};
      g_force_c = DiagVariant{dp, dwc};
    }
  }
  bool ok = true;
#define HSRQ_ATTR_R(DP, DW)                                                                       ok = ok && ck(cudaFuncSetAttribute(k_diag_real<DP, DW>,                                                                            cudaFuncAttributeMaxDynamicSharedMemorySize,                                                    (int)diag_smem<DP, DW, false>()), "attr diag r");
#define HSRQ_ATTR_C(DP, DW)                                                                       ok = ok && ck(cudaFuncSetAttribute(k_diag_cplx<DP, DW>,                                                                            cudaFuncAttributeMaxDynamicSharedMemorySize,                                                    (int)diag_smem<DP, DW, true>()), "attr diag c");
#define HSRQ_ATTR_W(DP, NP)                                                                \
  ok = ok && ck(cudaFuncSetAttribute(k_diag_cplx_ws<DP, NP>,                               \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                     (int)diag_ws_smem<DP, NP>()),                         \
                "attr diag ws");
  HSRQ_DIAG_REAL(HSRQ_ATTR_R)
  HSRQ_DIAG_CPLX(HSRQ_ATTR_C)
  HSRQ_DIAG_WS(HSRQ_ATTR_W)
#define HSRQ_ATTR_WR(DP, NP)                                                               \
  ok = ok && ck(cudaFuncSetAttribute(k_diag_real_ws<DP, NP>,                               \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                     (int)diag_ws_smem_r<DP, NP>()),                       \
                "attr diag wsr");
  HSRQ_DIAG_WSR(HSRQ_ATTR_WR)
#undef HSRQ_ATTR_WR
#define HSRQ_ATTR_RX(DP, NP)                                                               \
  ok = ok && ck(cudaFuncSetAttribute(k_diag_cplx_rx<DP, NP>,                               \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                     (int)diag_rx_smem<DP, NP>()),                         \
                "attr diag rx");
  HSRQ_DIAG_RX(HSRQ_ATTR_RX)
#undef HSRQ_ATTR_RX
  if (const char* w = getenv("HSRQ_DIAG_RX")) g_diag_rx = atoi(w);
#undef HSRQ_ATTR_R
#undef HSRQ_ATTR_C
#undef HSRQ_ATTR_W
  if (const char* w = getenv("HSRQ_DIAG_WS")) g_diag_ws = atoi(w);
  if (const char* w = getenv("HSRQ_DIAG_WSR")) g_diag_ws_r = atoi(w);
  done[dev] = ok;
  return ok;
}

// Automatic choice: lanes per shift so that count * DP / 32 warps roughly
// fill the machine (~6 warps per SM: the smem-limited residency of the
// complex kernel at DP 4), rounded down to a power of two in [4, 32].
DiagVariant diag_pick(bool cplx, int64_t count) {
  const DiagVariant f = cplx ? g_force_c : g_force_r;
  if (f.dp) return f;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double want = 32.0 * 6.0 * sms / (double)(count > 0 ? count : 1);
  int dp = 4;
  while (dp < 32 && 2 * dp <= want) dp *= 2;
  switch (dp) {
    case 4: return cplx ? DiagVariant{4, 2} : DiagVariant{4, 4};
    case 8: return cplx ? DiagVariant{8, 4} : DiagVariant{8, 6};
    // few shifts: the lookahead runs the sweep beside the panel; 16-warp CTAs
    // pack it onto fewer SMs (a complex CTA then fills its SM's registers),
    // leaving the other SMs to the panel at its full two-CTA rate
    case 16: return DiagVariant{16, 16};
    default: return DiagVariant{32, 16};
  }
}

template <int DP, int DW>
void diag_launch_r(const Ctx& c, const DiagArgs& a, cudaStream_t s) {
  const int per = DW * (32 / DP);
  k_diag_real<DP, DW><<<(unsigned)((a.count + per - 1) / per), DW * 32,
                        diag_smem<DP, DW, false>(), s>>>(c, a);
}
template <int DP, int DW>
void diag_launch_c(const Ctx& c, const DiagArgs& a, cudaStream_t s) {
  const int per = DW * (32 / DP);
  k_diag_cplx<DP, DW><<<(unsigned)((a.count + per - 1) / per), DW * 32,
                        diag_smem<DP, DW, true>(), s>>>(c, a);
}

template <int DP, int NP>
void diag_launch_ws_r(const Ctx& c, const DiagArgs& a, cudaStream_t s) {
  const int per = NP * (32 / DP);
  k_diag_real_ws<DP, NP><<<(unsigned)((a.count + per - 1) / per), NP * 64,
                           diag_ws_smem_r<DP, NP>(), s>>>(c, a);
}
template <int DP, int NP>
void diag_launch_ws(const Ctx& c, const DiagArgs& a, cudaStream_t s) {
  const int per = NP * (32 / DP);
  k_diag_cplx_ws<DP, NP><<<(unsigned)((a.count + per - 1) / per), NP * 64, diag_ws_smem<DP, NP>(),
                           s>>>(c, a);
}

template <int DP, int NP>
void diag_launch_rx(const Ctx& c, const DiagArgs& a, cudaStream_t s) {
  const int per = NP * (32 / DP);
  k_diag_cplx_rx<DP, NP><<<(unsigned)((a.count + per - 1) / per), NP * 64, diag_rx_smem<DP, NP>(),
                           s>>>(c, a);
}

void diag_launch(bool cplx, const Ctx& c, const DiagArgs& a, cudaStream_t s) {
  const DiagVariant v = diag_pick(cplx, a.count);
  // Rotation-ahead pairs (k_diag_cplx_rx).  Automatic where the pick is one
  // warp per shift (the 1/8 shards of config 5): pairs at 16 lanes per shift,
  // 8 per CTA -- the same 16 shifts per SM as the one-warp sweep, the
  // rotation chain beside the solution chain (1/8 shard: 96.7 -> 89.8 ms).
  if (cplx && !a.tile_mode) {
    if (g_diag_rx < 0 && v.dp == 32 && g_force_c.dp == 0) {
      diag_launch_rx<16, 8>(c, a, s);
      return;
    }
#define HSRQ_LAUNCH_RX(DP, NP)        \
  if (v.dp == DP && g_diag_rx == NP) { \
    diag_launch_rx<DP, NP>(c, a, s);  \
    return;                           \
  }
    if (g_diag_rx > 0) {
      HSRQ_DIAG_RX(HSRQ_LAUNCH_RX)
    }
#undef HSRQ_LAUNCH_RX
  }
  // warp-specialised complex sweep: automatic at DP 4 (all of config 5 on
  // one GPU: 506 -> 495 ms); measured no gain at DP >= 8 (the lookahead
  // shards), where the sweep runs beside the panel
  const int np = g_diag_ws >= 0 ? g_diag_ws : (g_force_c.dp == 0 && v.dp == 4 ? 2 : 0);
  if (cplx && np > 0) {
#define HSRQ_LAUNCH_W(DP, NP)         \
  if (v.dp == DP && np == NP) {       \
    diag_launch_ws<DP, NP>(c, a, s);  \
    return;                           \
  }
    HSRQ_DIAG_WS(HSRQ_LAUNCH_W)
#undef HSRQ_LAUNCH_W
  }
  // real: only for groups without complex shifts (real-only config 5: 128 ->
  // 122 ms; beside the complex sweep the extra warps cost more than they save)
  const int npr = g_diag_ws_r >= 0 ? g_diag_ws_r
                                   : (c.mc == 0 && g_force_r.dp == 0 && v.dp <= 16 ? 2 : 0);
  if (!cplx && npr > 0) {
#define HSRQ_LAUNCH_WR(DP, NP)          \
  if (v.dp == DP && npr == NP) {        \
    diag_launch_ws_r<DP, NP>(c, a, s);  \
    return;                             \
  }
    HSRQ_DIAG_WSR(HSRQ_LAUNCH_WR)
#undef HSRQ_LAUNCH_WR
  }
#define HSRQ_LAUNCH_R(DP, DW)         \
  if (v.dp == DP && v.dw == DW) {     \
    diag_launch_r<DP, DW>(c, a, s);   \
    return;                           \
  }
#define HSRQ_LAUNCH_C(DP, DW)         \
  if (v.dp == DP && v.dw == DW) {     \
    diag_launch_c<DP, DW>(c, a, s);   \
    return;                           \
  }
  if (cplx) {
    HSRQ_DIAG_CPLX(HSRQ_LAUNCH_C)
    diag_launch_c<4, 2>(c, a, s);
  } else {
    HSRQ_DIAG_REAL(HSRQ_LAUNCH_R)
    diag_launch_r<4, 4>(c, a, s);
  }
#undef HSRQ_LAUNCH_R
#undef HSRQ_LAUNCH_C
}

struct WsLayout {
  size_t cr, bop, ss, hm0, rs, hmk, xb, rsc, rt, nfail, total;
};

WsLayout ws_layout(int64_t n, int b_r, int64_t mc, int64_t mr) {
  const int64_t ncol = 2 * mc + mr;
  const int64_t ncol_pad = (ncol + BN - 1) / BN * BN;
  const int64_t N = (n + b_r - 1) / b_r;
  const int64_t ms = mc + mr;
  WsLayout L;
  size_t off = 0;
  L.nfail = off;  // first, so hsrq_failure_count(ws) can find it
  off = 256;
  L.cr = off;
  off = align_up(off + sizeof(double) * (size_t)n * ncol, 256);
  L.bop = off;  // two buffers (column parity, see the lookahead in solve_impl)
  off = align_up(off + 2 * sizeof(double) * (size_t)(2 * ncol_pad) * KP, 256);
  L.ss = off;   // two buffers
  off = align_up(off + 2 * sizeof(StepScalars) * (size_t)ms, 256);
  L.hm0 = off;
  off = align_up(off + sizeof(double) * (size_t)N * N, 256);
  L.rs = off;
  off = align_up(off + sizeof(double) * (size_t)N * N, 256);
  L.hmk = off;
  off = align_up(off + sizeof(double) * (size_t)N * MAXK, 256);
  L.xb = off;  // two halves (the cluster panel writes one per CTA of a pair)
  off = align_up(off + 2 * sizeof(double) * (size_t)N * ms, 256);
  L.rsc = off;
  off = align_up(off + 64 * (size_t)N * ms, 256);
  L.rt = off;
  off = align_up(off + sizeof(double) * 3 * (size_t)KP * ms, 256);
  L.total = off;
  return L;
}

// Host-feed mode (hsrq_solve_group_host): H is copied from host memory on a
// copy stream in column blocks, right to left -- the order the sweep
// consumes it -- so the transfer overlaps the sweep.  Block b holds columns
// [b*b_r - 1, (b+1)*b_r - 1) (block N: the rest); blk[b] is recorded when it
// has landed.  Tile column jt needs blocks jt..N.
struct HostFeed {
  const double* H_host;  // column-major, leading dimension ldh_host
  int64_t ldh_host;
  double* X_host;        // solution destination (column-major, ldx_host), or null
  int64_t ldx_host;
  cudaStream_t copy;     // H2D copy stream (also runs the per-block table kernels)
  cudaEvent_t* blk;      // N + 2 events: blk[b] = block b copied and tabulated; blk[N + 1] entry
  cudaStream_t d2h;      // D2H stream for X (its own copy engine: overlaps the next H2D)
  int wait_on_stream;    // 1: `stream` waits for X on the host at the end (synchronous entry)
  int early;             // 1: the copy stream starts at once (async entry: the caller
                         // guarantees the workspace is idle), else after prior work on `stream`
  int chunks;            // backtransform / X download chunks: a chunk below one wave of
                         // warps costs a full per-warp latency (~4.5 ms at n = 16000), so
                         // 4 for the synchronous entry (D2H of chunk c behind chunk c+1)
                         // and 1 for the async one (the next solve hides the download)
};

// Raised dynamic shared-memory limits of the panel and diagonal kernels,
// once per device (diag_attrs does the diagonal ones).
int64_t ensure_attrs() {
  static bool attr_done[MAX_DEVICES] = {};
  const size_t panel_smem = sizeof(PanelSmem);
  const int cur_dev = current_device();
  if (cur_dev < 0 || cur_dev >= MAX_DEVICES) return HSRQ_ERR_CONFIG;
  if (!diag_attrs()) return HSRQ_ERR_CUDA;
  std::unique_lock<std::mutex> setup_lock(g_setup_mu);
  if (!attr_done[cur_dev]) {
    if (
        !ck(cudaFuncSetAttribute(k_panel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel") ||
        !ck(cudaFuncSetAttribute(k_panel<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel") ||
        !ck(cudaFuncSetAttribute(k_panel<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel") ||
        !ck(cudaFuncSetAttribute(k_panel<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel") ||
        !ck(cudaFuncSetAttribute(k_panel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel fast") ||
        !ck(cudaFuncSetAttribute(k_panel_cl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(PanelClSmem)), "attr panel cluster"))
      return HSRQ_ERR_CUDA;
    attr_done[cur_dev] = true;
  }
  return 0;
}

int64_t solve_impl(const double* H, int64_t ldh, int64_t n, int32_t b_r, const double* lam_re,
                   const double* lam_im, int64_t mc, int64_t mr, const double* B, int64_t ldb,
                   int32_t b_broadcast, double* X, int64_t ldx, double* c_re, double* c_im,
                   double* s, int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                   double* log2norm, int64_t* fail, int32_t robust, int32_t mode, void* ws,
                   size_t ws_bytes, cudaStream_t stream, const HostFeed* feed = nullptr,
                   double omega_in = 0.0) {
  g_launches = 0;
  NvtxRange nv_solve("hsrq solve_group");
  if (n < 1 || b_r < 1 || b_r > MAXK || b_r > n || mc < 0 || mr < 0 || mc + mr < 1 || ldx < n ||
      ldh < n || ldc < n) {
    snprintf(g_err, sizeof(g_err), "bad configuration (n=%lld b_r=%d)", (long long)n, b_r);
    return HSRQ_ERR_CONFIG;
  }
  WsLayout L = ws_layout(n, b_r, mc, mr);
  if (ws_bytes < L.total) return HSRQ_ERR_WORKSPACE;
  unsigned char* w = (unsigned char*)ws;
  Ctx c;
  c.H = H;
  c.ldh = ldh;
  c.n = n;
  c.b_r = b_r;
  c.N = (int)((n + b_r - 1) / b_r);
  c.lam_re = lam_re;
  c.lam_im = lam_im;
  c.mc = mc;
  c.mr = mr;
  c.ms = mc + mr;
  c.ncol = 2 * mc + mr;
  c.ncol_pad = (c.ncol + BN - 1) / BN * BN;
  c.X = X;
  c.ldx = ldx;
  c.Cr = (double*)(w + L.cr);
  c.c_re = const_cast<double*>(c_re);
  c.c_im = const_cast<double*>(c_im);
  c.s = const_cast<double*>(s);
  c.ldc = ldc;
  c.E = seg_exp;
  c.Bop = (double*)(w + L.bop);
  c.SS = (StepScalars*)(w + L.ss);
  c.HM0 = (double*)(w + L.hm0);
  c.RS = (double*)(w + L.rs);
  c.XB = (double*)(w + L.xb);
  c.HMK = (double*)(w + L.hmk);
  c.fail = fail;
  c.nfail = (unsigned long long*)(w + L.nfail);
  c.robust = robust;
  c.mode = mode & 1;
  c.compact = (mode & HSRQ_MODE_COMPACT_ROTATIONS) ? 1 : 0;
  c.Rt = (double*)(w + L.rt);
  c.diag_gemm_only = getenv("HSRQ_PANEL_GEMM_ONLY") ? atoi(getenv("HSRQ_PANEL_GEMM_ONLY")) : 0;
  c.diag_tl = nullptr;
  c.diag_tl_jt = -1;
  if (getenv("HSRQ_TIMELINE")) {
    static unsigned long long* tl = nullptr;
    if (!tl) cudaMalloc(&tl, 8192 * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(tl, 0, 8192 * 8 * sizeof(unsigned long long), stream);
    c.diag_tl = tl;
    c.diag_tl_jt = atoi(getenv("HSRQ_TIMELINE"));
    g_tl = tl;
  }
  // OverflowBudget.for_grid (overflow.py:41-47) unless the caller passes
  // its own budget (dhsrq3 / chsrq3 budget=, backsolve.py:342-346)
  c.omega = robust ? (omega_in > 0.0 ? omega_in : (1.7976931348623157e308 / 2.0) / (double)b_r)
                   : HUGE_VAL;
  // the crossover block shares X's leading dimension
  if (ldx != n) {
    snprintf(g_err, sizeof(g_err), "ldx must equal n in this build");
    return HSRQ_ERR_CONFIG;
  }

  const size_t panel_smem = sizeof(PanelSmem);
  if (const int64_t r = ensure_attrs(); r != 0) return r;
  // Optional per-launch timing: events around every launch, one sync at the end.
  const int nev = 6 * c.N + 6;
  cudaEvent_t* ev = nullptr;
  if (g_timing) {
    ev = new cudaEvent_t[nev];
    for (int i = 0; i < nev; i++) cudaEventCreate(&ev[i]);
    cudaEventRecord(ev[0], stream);
  }
  const int64_t nzero = std::max<int64_t>((int64_t)c.N * c.ms, (int64_t)c.N * c.N) + c.ms + 1;
  k_zero_state<<<(unsigned)((nzero + 255) / 256), 256, 0, stream>>>(c, feed ? 0 : 1);
  g_launches++;
  const int64_t nbop = 4 * c.ncol_pad * KP;  // both buffers
  k_zero_bop<<<(unsigned)((nbop + 255) / 256), 256, 0, stream>>>(c.Bop, nbop);
  g_launches++;
  if (!feed) {
    if (c.N > 1) {
      dim3 gt((unsigned)((n + 255) / 256), (unsigned)(c.N - 1));
      k_tables<<<gt, 256, 0, stream>>>(c);
      g_launches++;
    }
    k_hmk<<<(unsigned)c.N, MAXK, 0, stream>>>(c);
    g_launches++;
  } else {
    // H arrives block by block on the copy stream (after prior work on
    // `stream` released the buffers); each block's table kernel follows its
    // copy there, off the sweep's critical path
    cudaStream_t cp = feed->copy;
    if (!feed->early) {
      cudaEventRecord(feed->blk[c.N + 1], stream);
      cudaStreamWaitEvent(cp, feed->blk[c.N + 1], 0);
    }
    if (!ck(cudaMemsetAsync(c.HM0, 0, sizeof(double) * (size_t)c.N * c.N, cp), "memset") ||
        !ck(cudaMemsetAsync(c.RS, 0, sizeof(double) * (size_t)c.N * c.N, cp), "memset"))
      return HSRQ_ERR_CUDA;
    for (int64_t b = c.N; b >= 0; --b) {
      const int64_t c0 = std::min<int64_t>(n, std::max<int64_t>(0, b * b_r - 1));
      const int64_t c1 = b == c.N ? n : std::min<int64_t>(n, (b + 1) * b_r - 1);
      if (c1 > c0 &&
          !ck(cudaMemcpy2DAsync(const_cast<double*>(H) + c0 * ldh, sizeof(double) * ldh,
                                feed->H_host + c0 * feed->ldh_host,
                                sizeof(double) * feed->ldh_host, sizeof(double) * n,
                                (size_t)(c1 - c0), cudaMemcpyHostToDevice, cp),
              "H2D H"))
        return HSRQ_ERR_CUDA;
      if (b < c.N) {
        const unsigned nb = (unsigned)((b * b_r + 255) / 256) + 1;
        k_tables_jt<<<nb, 256, 0, cp>>>(c, (int)b);
        g_launches++;
      }
      cudaEventRecord(feed->blk[b], cp);
    }
    // k_init needs column n - 1
    cudaStreamWaitEvent(stream, feed->blk[c.N], 0);
    cudaStreamWaitEvent(stream, feed->blk[c.N - 1], 0);
  }
  {
    dim3 gi((unsigned)((n + 255) / 256), (unsigned)c.ncol);
    k_init<<<gi, 256, 0, stream>>>(c, B, ldb, b_broadcast);
    g_launches++;
  }
  if (g_timing) cudaEventRecord(ev[1], stream);
  const bool a16 = (ldh % 2 == 0) && (b_r % 2 == 0);
  const int S = std::min(SMAX, std::max(1, BM / b_r));
  // Streams (one set per host thread and device): `side` runs the real
  // diagonal kernel concurrently with the complex one; `dstr` (+ `dside` for
  // the real shifts) carries the lookahead diagonal sweep of column jt-1
  // while the panel of column jt finishes the rows above it -- high
  // priority, so the latency-bound sweep's CTAs are scheduled ahead of the
  // remaining panel CTAs.
  thread_local cudaStream_t side = nullptr, dstr = nullptr, dside = nullptr;
  thread_local int side_dev = -1;
  thread_local cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_bot = nullptr,
                           ev_diag = nullptr;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    if (side_dev != dev) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (!ck(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo), "side stream") ||
          !ck(cudaStreamCreateWithPriority(&dstr, cudaStreamNonBlocking, hi), "diag stream") ||
          !ck(cudaStreamCreateWithPriority(&dside, cudaStreamNonBlocking, hi), "diag side") ||
          !ck(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "fork event") ||
          !ck(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "join event") ||
          !ck(cudaEventCreateWithFlags(&ev_bot, cudaEventDisableTiming), "bottom event") ||
          !ck(cudaEventCreateWithFlags(&ev_diag, cudaEventDisableTiming), "diag event"))
        return HSRQ_ERR_CUDA;
      side_dev = dev;
    }
  }
  // Lookahead: the diagonal sweep of column jt-1 only needs tile row jt-1 of
  // panel jt, so that row goes first and the sweep overlaps the rest of the
  // panel.  HSRQ_LOOKAHEAD=0/1 forces it off/on (default on).
  // Measured (tools/shard_time.py, config-5 shards, ms per solve, off -> on):
  // 1 GPU 515 -> 514, 1/2 shard 291 -> 261, 1/4 175 -> 162, 1/8 116 -> 105
  // (round 1); with the 2-CTA cluster panel, all of config 5 on one GPU:
  // 464.0 -> 452.3 ms (tools/profile_solve.py).  The panel's launch times
  // then include the concurrent sweep, so bench.py takes the roofline from a
  // second timed pass with HSRQ_LOOKAHEAD=0.
  bool lookahead = true;
  if (const char* e = getenv("HSRQ_LOOKAHEAD")) lookahead = atoi(e) != 0;
  // Bop / SS are double-buffered by column parity: the lookahead sweep of
  // jt-1 writes its panel operands while panel jt still reads its own.
  Ctx cb[2] = {c, c};
  cb[1].Bop = c.Bop + 2 * c.ncol_pad * KP;
  cb[1].SS = c.SS + c.ms;
  const int kt = 6;  // timing events per column
  auto tev = [&](int jt, int slot) { return ev[2 + kt * jt + slot]; };

  // diagonal sweep of column jd on stream sd (real shifts forked onto `side`)
  auto run_diag = [&](int jd, cudaStream_t sd, cudaStream_t sside) -> bool {
    DiagArgs a;
    memset(&a, 0, sizeof(a));
    a.jt = jd;
    a.js = (int64_t)jd * b_r;
    const int64_t je = a.js + b_r < n ? a.js + b_r : n;
    a.k = (int)(je - a.js);
    a.has_left = jd > 0;
    if (feed) cudaStreamWaitEvent(sd, feed->blk[jd], 0);  // this column's H block + tables
    if (g_timing) cudaEventRecord(tev(jd, 0), sd);
    const bool fork = mc > 0 && mr > 0;
    if (fork) {
      cudaEventRecord(ev_fork, sd);
      cudaStreamWaitEvent(sside, ev_fork, 0);
    }
    // Compact rotation storage: the diagonal kernels record the tile's exact
    // rotations into the tile scratch Rt (the panel operands need them), and
    // k_compact_tile writes their Stewart codes into the tables.
    Ctx cd = cb[jd & 1];
    a.rot_off = a.js;
    if (c.compact) {
      cd.c_re = c.Rt;
      cd.c_im = c.Rt + c.ms * KP;
      cd.s = c.Rt + 2 * c.ms * KP;
      cd.ldc = KP;
      a.rot_off = 0;
    }
    // complex first: its sweep is the longer one (the critical path), so its
    // CTAs should be resident before the real kernel's fill the rest
    if (mc > 0) {
      a.q0 = 0;
      a.count = mc;
      diag_launch(true, cd, a, sd);
      g_launches++;
    }
    if (mr > 0) {
      a.q0 = mc;
      a.count = mr;
      diag_launch(false, cd, a, fork ? sside : sd);
      g_launches++;
    }
    if (fork) {
      cudaEventRecord(ev_join, sside);
      cudaStreamWaitEvent(sd, ev_join, 0);
    }
    if (c.compact) {
      const int64_t cnt = (int64_t)a.k * c.ms;
      k_compact_tile<<<(unsigned)((cnt + 255) / 256), 256, 0, sd>>>(c, a.js, a.k);
      g_launches++;
    }
    if (g_timing) cudaEventRecord(tev(jd, 1), sd);
    return true;
  };
  // panel GEMM of column jt over tile rows [t0, t1)
  const bool seg16 = (b_r % 16) == 0;
  RowScalars* rsc = (RowScalars*)(w + L.rsc);
  auto run_panel = [&](int jt, int t0, int t1) {
    if (t1 <= t0) return;
    PanelArgs p;
    p.jt = jt;
    p.js = (int64_t)jt * b_r;
    p.k = (int)(std::min<int64_t>(p.js + b_r, n) - p.js);
    p.S = S;
    p.t0 = t0;
    p.t1 = t1;
    const Ctx& cj = cb[jt & 1];
    if (const char* e = getenv("HSRQ_PANEL_EXP")) {  // diagnostics: 64-row 4-warp GEMM only
      const int st = atoi(e);
      dim3 g64((unsigned)(2 * (t1 - t0)), (unsigned)(c.ncol_pad / BN));
      if (st == 3) {
        static bool a3 = false;
        if (!a3) cudaFuncSetAttribute(k_panel64_gemm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(Gemm64Smem<3>));
        a3 = true;
        k_panel64_gemm<3><<<g64, 128, sizeof(Gemm64Smem<3>), stream>>>(cj, p);
      } else {
        static bool a2 = false;
        if (!a2) cudaFuncSetAttribute(k_panel64_gemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(Gemm64Smem<2>));
        a2 = true;
        k_panel64_gemm<2><<<g64, 128, sizeof(Gemm64Smem<2>), stream>>>(cj, p);
      }
      g_launches++;
      return;
    }
    // b_r = 128 with full K chunks: the 2-CTA cluster form (HSRQ_PANEL_CLUSTER=0: k_panel)
    if (a16 && b_r == BM && g_panel_fast && g_panel_cluster && p.k == BM && !c.diag_gemm_only &&
        !c.diag_tl) {
      dim3 gcl((unsigned)(2 * (t1 - t0)), (unsigned)(c.ncol_pad / BN));
      k_panel_cl<<<gcl, CL_THREADS, sizeof(PanelClSmem), stream>>>(cj, p, rsc);
      g_launches++;
      return;
    }
    dim3 gp((unsigned)((t1 - t0 + S - 1) / S), (unsigned)(c.ncol_pad / BN));
    if (a16 && b_r == BM && g_panel_fast)
      k_panel<true, true, true><<<gp, PANEL_THREADS, panel_smem, stream>>>(cj, p, rsc);
    else if (a16 && seg16)
      k_panel<true, true, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(cj, p, rsc);
    else if (a16)
      k_panel<true, false, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(cj, p, rsc);
    else if (seg16)
      k_panel<false, true, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(cj, p, rsc);
    else
      k_panel<false, false, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(cj, p, rsc);
    g_launches++;
  };

  // Diagnostics / tests (HSRQ_STOP_AT=s): end the sweep after column s's
  // panel -- X then holds the solved tiles >= s and the updated right-hand
  // sides below, E the segment exponents -- without the backtransform.
  int stop_at = -1;
  if (const char* e = getenv("HSRQ_STOP_AT")) stop_at = atoi(e);
  bool stopped = stop_at == c.N - 1 && c.N - 1 == 0;
  {
    NvtxRange nv("hsrq diag tile %d", c.N - 1);
    run_diag(c.N - 1, stream, side);
  }
  for (int jt = c.N - 1; jt >= 1 && !stopped; --jt) {
    NvtxRange nv("hsrq tile column %d", jt);
    PanelArgs p;
    p.jt = jt;
    p.js = (int64_t)jt * b_r;
    p.k = (int)(std::min<int64_t>(p.js + b_r, n) - p.js);
    p.S = S;
    p.t0 = 0;
    p.t1 = jt;
    if (g_timing) cudaEventRecord(tev(jt, 2), stream);
    const int64_t nsc = (int64_t)jt * c.ms;
    k_scalars<<<(unsigned)((nsc + 127) / 128), 128, 0, stream>>>(cb[jt & 1], p, rsc);
    g_launches++;
    if (g_timing) {
      cudaEventRecord(tev(jt, 3), stream);
      cudaEventRecord(tev(jt, 4), stream);
    }
    if (jt == stop_at) {
      run_panel(jt, 0, jt);
      stopped = true;
      break;
    }
    if (lookahead) {
      run_panel(jt, jt - 1, jt);  // tile row jt-1: all the next sweep needs
      cudaEventRecord(ev_bot, stream);
      cudaStreamWaitEvent(dstr, ev_bot, 0);
      run_diag(jt - 1, dstr, dside);
      cudaEventRecord(ev_diag, dstr);
      run_panel(jt, 0, jt - 1);
      if (g_timing) cudaEventRecord(tev(jt, 5), stream);
      cudaStreamWaitEvent(stream, ev_diag, 0);
    } else {
      run_panel(jt, 0, jt);
      if (g_timing) cudaEventRecord(tev(jt, 5), stream);
      run_diag(jt - 1, stream, side);
    }
  }
  if (g_timing) cudaEventRecord(ev[nev - 3], stream);
  NvtxRange nv_bt("hsrq backtransform");
  if (stopped) {
    // (timing of a stopped sweep is not recorded)
  } else if (!feed || !feed->X_host) {
    bt_launch(c, alpha_exp, norms, log2norm, 0, c.ms, c.ms, stream);
    g_launches++;
  } else {
    // host feed: backtransform in shift chunks; each chunk's columns of X go
    // to the host on the copy stream while the next chunk is transformed
    const int nch = feed->chunks;
    for (int ch = 0; ch < nch; ch++) {
      const int64_t q0 = c.ms * ch / nch, q1 = c.ms * (ch + 1) / nch;
      if (q1 <= q0) continue;
      bt_launch(c, alpha_exp, norms, log2norm, q0, q1, c.ms, stream);
      g_launches++;
      // (the block events are free again: every wait on them is already enqueued)
      cudaEvent_t e = feed->blk[ch % (c.N + 1)];
      cudaEventRecord(e, stream);
      cudaStreamWaitEvent(feed->d2h, e, 0);
      // columns of shifts [q0, q1): complex part then real part
      const int64_t cq1 = std::min<int64_t>(q1, c.mc), rq0 = std::max<int64_t>(q0, c.mc);
      if (cq1 > q0 &&
          !ck(cudaMemcpy2DAsync(feed->X_host + 2 * q0 * feed->ldx_host,
                                sizeof(double) * feed->ldx_host, c.X + 2 * q0 * c.ldx,
                                sizeof(double) * c.ldx, sizeof(double) * n,
                                (size_t)(2 * (cq1 - q0)), cudaMemcpyDeviceToHost, feed->d2h),
              "D2H X"))
        return HSRQ_ERR_CUDA;
      if (q1 > rq0 &&
          !ck(cudaMemcpy2DAsync(feed->X_host + (2 * c.mc + rq0 - c.mc) * feed->ldx_host,
                                sizeof(double) * feed->ldx_host,
                                c.X + (2 * c.mc + rq0 - c.mc) * c.ldx, sizeof(double) * c.ldx,
                                sizeof(double) * n, (size_t)(q1 - rq0), cudaMemcpyDeviceToHost,
                                feed->d2h),
              "D2H X"))
        return HSRQ_ERR_CUDA;
    }
    if (feed->wait_on_stream) {
      cudaEventRecord(feed->blk[c.N + 1], feed->d2h);
      cudaStreamWaitEvent(stream, feed->blk[c.N + 1], 0);  // X is on the host
    }
  }
  if (g_timing && stopped) {  // a stopped sweep leaves later columns' events unrecorded
    for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
    delete[] ev;
  } else if (g_timing) {
    // read back lazily (hsrq_phase_times): no host sync inside a timed solve
    cudaEventRecord(ev[nev - 2], stream);
    g_pending.push_back(PendingTiming{ev, nev, c.N});
  }
  if (!ck(cudaGetLastError(), "launch")) return HSRQ_ERR_CUDA;
  return 0;
}

// Device workspace of the host-buffer entry point (hsrq_solve_group_host).
struct HostLayout {
  int64_t ldh;  // device H leading dimension (even)
  size_t h, x, cre, cim, s, lre, lim, b, seg, aexp, norms, l2, fail, ws, total;
};
HostLayout host_layout(int64_t n, int b_r, int64_t mc, int64_t mr) {
  HostLayout L;
  const int64_t ncol = 2 * mc + mr, ms = mc + mr, N = (n + b_r - 1) / b_r;
  L.ldh = n + (n & 1);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align_up(off + bytes, 256);
    return at;
  };
  L.h = take(sizeof(double) * (size_t)L.ldh * n);
  L.x = take(sizeof(double) * (size_t)n * ncol);
  L.cre = take(sizeof(double) * (size_t)n * ms);
  L.cim = take(sizeof(double) * (size_t)n * ms);
  L.s = take(sizeof(double) * (size_t)n * ms);
  L.lre = take(sizeof(double) * (size_t)ms);
  L.lim = take(sizeof(double) * (size_t)ms);
  L.b = take(sizeof(double) * (size_t)n);
  L.seg = take(sizeof(int32_t) * (size_t)N * ms);
  L.aexp = take(sizeof(int32_t) * (size_t)ms);
  L.norms = take(sizeof(double) * (size_t)ms);
  L.l2 = take(sizeof(double) * (size_t)ms);
  L.fail = take(sizeof(int64_t) * (size_t)ms);
  L.ws = take(ws_layout(n, b_r, mc, mr).total);
  L.total = off;
  return L;
}

// ---------------------------------------------------------------------------
// Henry's single sweep (hsrq_henry.cuh)
// ---------------------------------------------------------------------------

struct HenryLayout {
  size_t v, c, s, st, first, total;
};
HenryLayout henry_layout(int64_t n, int64_t m, int cplx) {
  HenryLayout L;
  const size_t w = cplx ? 2 : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align_up(off + bytes, 256);
    return at;
  };
  L.v = take(sizeof(double) * w * (size_t)n * m);
  L.c = take(sizeof(double) * w * (size_t)n * m);
  L.s = take(sizeof(double) * (size_t)n * m);
  L.st = take(sizeof(int64_t) * (size_t)m);
  L.first = take(sizeof(unsigned long long));
  L.total = off;
  return L;
}
}  // namespace

extern "C" {

const char* hsrq_version(void) { return "hsrq_b200 0.1.0 (sm_100a)"; }
const char* hsrq_last_error(void) { return g_err; }

size_t hsrq_workspace_bytes(int64_t n, int32_t b_r, int64_t m_cplx, int64_t m_real) {
  if (n < 1 || b_r < 1) return 0;
  return ws_layout(n, b_r, m_cplx, m_real).total;
}

int64_t hsrq_solve_group_async(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                               const double* lam_re, const double* lam_im, int64_t m_cplx,
                               int64_t m_real, const double* B, int64_t ldb,
                               int32_t b_broadcast, double* X, int64_t ldx, double* c_re,
                               double* c_im, double* s, int64_t ldc, int32_t* seg_exp,
                               int32_t* alpha_exp, double* norms, double* log2norm,
                               int64_t* fail, int32_t robust, int32_t mode, void* ws,
                               size_t ws_bytes, void* stream) {
  return solve_impl(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb, b_broadcast, X, ldx,
                    c_re, c_im, s, ldc, seg_exp, alpha_exp, norms, log2norm, fail, robust, mode,
                    ws, ws_bytes, (cudaStream_t)stream);
}

int64_t hsrq_graph_capture(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                           const double* lam_re, const double* lam_im, int64_t m_cplx,
                           int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                           double* X, int64_t ldx, double* c_re, double* c_im, double* s,
                           int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                           double* log2norm, int64_t* fail, int32_t robust, int32_t mode, void* ws,
                           size_t ws_bytes, void* stream_, void** graph_out) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!graph_out || g_timing) return HSRQ_ERR_CONFIG;
  // one eager solve first: the per-thread side streams, events and kernel
  // attributes are created outside the capture
  int64_t r = solve_impl(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb, b_broadcast, X,
                         ldx, c_re, c_im, s, ldc, seg_exp, alpha_exp, norms, log2norm, fail,
                         robust, mode, ws, ws_bytes, stream);
  if (r < 0) return r;
  // capture on a private stream (the legacy default stream cannot capture)
  cudaStream_t cap = nullptr;
  if (!ck(cudaStreamSynchronize(stream), "sync") ||
      !ck(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream") ||
      !ck(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture")) {
    if (cap) cudaStreamDestroy(cap);
    return HSRQ_ERR_CUDA;
  }
  r = solve_impl(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb, b_broadcast, X, ldx,
                 c_re, c_im, s, ldc, seg_exp, alpha_exp, norms, log2norm, fail, robust, mode, ws,
                 ws_bytes, cap);
  cudaGraph_t graph = nullptr;
  const bool ended = ck(cudaStreamEndCapture(cap, &graph), "end capture");
  cudaStreamDestroy(cap);
  if (r < 0 || !ended) {
    if (graph) cudaGraphDestroy(graph);
    return r < 0 ? r : HSRQ_ERR_CUDA;
  }
  cudaGraphExec_t exec = nullptr;
  const bool ok = ck(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
  cudaGraphDestroy(graph);
  if (!ok) return HSRQ_ERR_CUDA;
  *graph_out = (void*)exec;
  return 0;
}

int64_t hsrq_graph_launch(void* graph, void* stream) {
  if (!graph) return HSRQ_ERR_CONFIG;
  return ck(cudaGraphLaunch((cudaGraphExec_t)graph, (cudaStream_t)stream), "graph launch")
             ? 0
             : HSRQ_ERR_CUDA;
}

void hsrq_graph_destroy(void* graph) {
  if (graph) cudaGraphExecDestroy((cudaGraphExec_t)graph);
}

int64_t hsrq_failure_count(void* ws, void* stream) {
  unsigned long long nf = 0;
  if (!ck(cudaMemcpyAsync(&nf, ws, sizeof(nf), cudaMemcpyDeviceToHost, (cudaStream_t)stream),
          "copy nfail") ||
      !ck(cudaStreamSynchronize((cudaStream_t)stream), "sync"))
    return HSRQ_ERR_CUDA;
  return (int64_t)nf;
}

int64_t hsrq_solve_group(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                         const double* lam_re, const double* lam_im, int64_t m_cplx,
                         int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                         double* X, int64_t ldx, double* c_re, double* c_im, double* s,
                         int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                         double* log2norm, int64_t* fail, int32_t robust, int32_t mode, void* ws,
                         size_t ws_bytes, void* stream) {
  return hsrq_solve_group_omega(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb,
                                b_broadcast, X, ldx, c_re, c_im, s, ldc, seg_exp, alpha_exp, norms,
                                log2norm, fail, robust, mode, 0.0, ws, ws_bytes, stream);
}

int64_t hsrq_solve_group_omega(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                               const double* lam_re, const double* lam_im, int64_t m_cplx,
                               int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                               double* X, int64_t ldx, double* c_re, double* c_im, double* s,
                               int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                               double* log2norm, int64_t* fail, int32_t robust, int32_t mode,
                               double omega, void* ws, size_t ws_bytes, void* stream) {
  if (!(omega >= 0.0) || omega > 1.7976931348623157e308 / 2.0) {
    snprintf(g_err, sizeof(g_err), "omega=%g outside (0, maxfloat/2]", omega);
    return HSRQ_ERR_CONFIG;
  }
  int64_t r = solve_impl(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb, b_broadcast, X,
                         ldx, c_re, c_im, s, ldc, seg_exp, alpha_exp, norms, log2norm, fail,
                         robust, mode, ws, ws_bytes, (cudaStream_t)stream, nullptr, omega);
  if (r < 0) return r;
  WsLayout L = ws_layout(n, b_r, m_cplx, m_real);
  unsigned long long nf = 0;
  if (!ck(cudaMemcpyAsync(&nf, (unsigned char*)ws + L.nfail, sizeof(nf), cudaMemcpyDeviceToHost,
                          (cudaStream_t)stream),
          "copy nfail"))
    return HSRQ_ERR_CUDA;
  if (!ck(cudaStreamSynchronize((cudaStream_t)stream), "sync")) return HSRQ_ERR_CUDA;
  return (int64_t)nf;
}

size_t hsrq_host_workspace_bytes(int64_t n, int32_t b_r, int64_t m_cplx, int64_t m_real) {
  if (n < 1 || b_r < 1) return 0;
  return host_layout(n, b_r, m_cplx, m_real).total;
}

namespace {
// Tickets of asynchronous host-buffer solves: the event after the last D2H of
// the solve, and where its per-shift failure codes land.
struct HostTicket {
  cudaEvent_t done = nullptr;
  const int64_t* fail = nullptr;
  int64_t ms = 0;
  int live = 0;
};
constexpr int NTICKET = 16;
thread_local HostTicket g_tickets[NTICKET];
thread_local int64_t g_ticket_seq = 0;

int64_t host_enqueue(const double* H, int64_t ldh, int64_t n, int32_t b_r, const double* lam_re,
                     const double* lam_im, int64_t m_cplx, int64_t m_real, const double* B,
                     int64_t ldb, int32_t b_broadcast, double* X, int64_t ldx, int32_t* seg_exp,
                     int32_t* alpha_exp, double* norms, double* log2norm, int64_t* fail,
                     int32_t robust, int32_t mode, void* dev_ws, size_t dev_ws_bytes,
                     cudaStream_t stream, int early) {
  if (n < 1 || b_r < 1 || b_r > MAXK || b_r > n || m_cplx < 0 || m_real < 0 ||
      m_cplx + m_real < 1 || ldh < n || ldx < n || (!b_broadcast && ldb < n)) {
    snprintf(g_err, sizeof(g_err), "bad configuration (n=%lld b_r=%d)", (long long)n, b_r);
    return HSRQ_ERR_CONFIG;
  }
  const HostLayout L = host_layout(n, b_r, m_cplx, m_real);
  if (dev_ws_bytes < L.total) return HSRQ_ERR_WORKSPACE;
  unsigned char* w = (unsigned char*)dev_ws;
  double* Hd = (double*)(w + L.h);
  double* Xd = (double*)(w + L.x);
  const int64_t ms = m_cplx + m_real, ncol = 2 * m_cplx + m_real, N = (n + b_r - 1) / b_r;
  // per-thread copy streams (H2D, D2H: separate copy engines) and event pool
  thread_local cudaStream_t copy = nullptr, d2h = nullptr;
  thread_local int copy_dev = -1;
  thread_local std::vector<cudaEvent_t> evs;
  int dev = 0;
  cudaGetDevice(&dev);
  if (copy_dev != dev) {
    if (!ck(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking), "copy stream") ||
        !ck(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking), "d2h stream"))
      return HSRQ_ERR_CUDA;
    for (auto e : evs) cudaEventDestroy(e);
    evs.clear();
    copy_dev = dev;
  }
  while ((int64_t)evs.size() < N + 2) {
    cudaEvent_t e;
    if (!ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event")) return HSRQ_ERR_CUDA;
    evs.push_back(e);
  }
  // shifts and right-hand sides on the compute stream
  double* lre = (double*)(w + L.lre);
  double* lim = (double*)(w + L.lim);
  if (!ck(cudaMemcpyAsync(lre, lam_re, sizeof(double) * ms, cudaMemcpyHostToDevice, stream),
          "H2D lam"))
    return HSRQ_ERR_CUDA;
  if (lam_im) {
    if (!ck(cudaMemcpyAsync(lim, lam_im, sizeof(double) * ms, cudaMemcpyHostToDevice, stream),
            "H2D lam"))
      return HSRQ_ERR_CUDA;
  } else if (!ck(cudaMemsetAsync(lim, 0, sizeof(double) * ms, stream), "memset lam")) {
    return HSRQ_ERR_CUDA;
  }
  const double* Bd;
  int64_t ldbd;
  if (b_broadcast) {
    double* bd = (double*)(w + L.b);
    if (!ck(cudaMemcpyAsync(bd, B, sizeof(double) * n, cudaMemcpyHostToDevice, stream), "H2D B"))
      return HSRQ_ERR_CUDA;
    Bd = bd;
    ldbd = 0;
  } else {  // B lands in X (k_init reads and writes each entry in one thread)
    if (!ck(cudaMemcpy2DAsync(Xd, sizeof(double) * n, B, sizeof(double) * ldb,
                              sizeof(double) * n, (size_t)ncol, cudaMemcpyHostToDevice, stream),
            "H2D B"))
      return HSRQ_ERR_CUDA;
    Bd = Xd;
    ldbd = n;
  }
  HostFeed feed{H, ldh, X, ldx, copy, evs.data(), d2h, 0, early, early ? 1 : 4};
  if (const char* e = getenv("HSRQ_HOST_CHUNKS")) feed.chunks = std::max(1, atoi(e));
  int32_t* segd = (int32_t*)(w + L.seg);
  int32_t* aexpd = (int32_t*)(w + L.aexp);
  double* normsd = (double*)(w + L.norms);
  double* l2d = (double*)(w + L.l2);
  int64_t* faild = (int64_t*)(w + L.fail);
  void* wsd = w + L.ws;
  const int64_t r = solve_impl(Hd, L.ldh, n, b_r, lre, lim, m_cplx, m_real, Bd, ldbd, b_broadcast,
                               Xd, n, (double*)(w + L.cre), (double*)(w + L.cim),
                               (double*)(w + L.s), n, segd, aexpd, normsd, l2d, faild, robust, mode,
                               wsd, ws_layout(n, b_r, m_cplx, m_real).total, stream, &feed);
  if (r < 0) return r;
  // the small per-shift outputs follow X on the D2H stream, after the sweep
  HostTicket& t = g_tickets[g_ticket_seq % NTICKET];
  if (t.live) cudaEventSynchronize(t.done);  // ring slot reuse: that solve is long done
  if (!t.done && !ck(cudaEventCreateWithFlags(&t.done, cudaEventDisableTiming), "ticket event"))
    return HSRQ_ERR_CUDA;
  cudaEvent_t swept = evs[N + 1];
  cudaEventRecord(swept, stream);
  cudaStreamWaitEvent(d2h, swept, 0);
  if (!ck(cudaMemcpyAsync(seg_exp, segd, sizeof(int32_t) * N * ms, cudaMemcpyDeviceToHost, d2h),
          "D2H seg") ||
      !ck(cudaMemcpyAsync(alpha_exp, aexpd, sizeof(int32_t) * ms, cudaMemcpyDeviceToHost, d2h),
          "D2H alpha") ||
      !ck(cudaMemcpyAsync(norms, normsd, sizeof(double) * ms, cudaMemcpyDeviceToHost, d2h),
          "D2H norms") ||
      !ck(cudaMemcpyAsync(log2norm, l2d, sizeof(double) * ms, cudaMemcpyDeviceToHost, d2h),
          "D2H log2norm") ||
      !ck(cudaMemcpyAsync(fail, faild, sizeof(int64_t) * ms, cudaMemcpyDeviceToHost, d2h),
          "D2H fail"))
    return HSRQ_ERR_CUDA;
  cudaEventRecord(t.done, d2h);
  t.fail = fail;
  t.ms = ms;
  t.live = 1;
  return g_ticket_seq++;
}
}  // namespace

int64_t hsrq_host_wait(int64_t ticket) {
  if (ticket < 0 || ticket >= g_ticket_seq || ticket < g_ticket_seq - NTICKET) return HSRQ_ERR_CONFIG;
  HostTicket& t = g_tickets[ticket % NTICKET];
  if (!ck(cudaEventSynchronize(t.done), "wait")) return HSRQ_ERR_CUDA;
  int64_t nf = 0;
  for (int64_t q = 0; q < t.ms; q++) nf += t.fail[q] != 0;
  return nf;
}

int64_t hsrq_solve_group_host_async(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                                    const double* lam_re, const double* lam_im, int64_t m_cplx,
                                    int64_t m_real, const double* B, int64_t ldb,
                                    int32_t b_broadcast, double* X, int64_t ldx, int32_t* seg_exp,
                                    int32_t* alpha_exp, double* norms, double* log2norm,
                                    int64_t* fail, int32_t robust, int32_t mode, void* dev_ws,
                                    size_t dev_ws_bytes, void* stream) {
  return host_enqueue(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb, b_broadcast, X, ldx,
                      seg_exp, alpha_exp, norms, log2norm, fail, robust, mode, dev_ws,
                      dev_ws_bytes, (cudaStream_t)stream, 1);
}

int64_t hsrq_solve_group_host(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                              const double* lam_re, const double* lam_im, int64_t m_cplx,
                              int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                              double* X, int64_t ldx, int32_t* seg_exp, int32_t* alpha_exp,
                              double* norms, double* log2norm, int64_t* fail, int32_t robust,
                              int32_t mode, void* dev_ws, size_t dev_ws_bytes, void* stream) {
  const int64_t t = host_enqueue(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb,
                                 b_broadcast, X, ldx, seg_exp, alpha_exp, norms, log2norm, fail,
                                 robust, mode, dev_ws, dev_ws_bytes, (cudaStream_t)stream, 0);
  if (t < 0) return t;
  return hsrq_host_wait(t);
}

int64_t hsrq_last_launch_count(void) { return g_launches; }

int64_t hsrq_debug_timeline(unsigned long long* out_host) {
  if (!g_tl) return -1;
  cudaDeviceSynchronize();
  return cudaMemcpy(out_host, g_tl, 8192 * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? 0
             : HSRQ_ERR_CUDA;
}

int64_t hsrq_debug_stepprof(int64_t* out_host, int32_t reset) {
#ifdef HSRQ_STEPPROF
  unsigned long long v[16];
  if (cudaMemcpyFromSymbol(v, g_stepprof, sizeof(v)) != cudaSuccess) return HSRQ_ERR_CUDA;
  for (int i = 0; i < 16; i++) out_host[i] = (int64_t)v[i];
  if (reset) {
    unsigned long long z[16] = {0};
    if (cudaMemcpyToSymbol(g_stepprof, z, sizeof(z)) != cudaSuccess) return HSRQ_ERR_CUDA;
  }
  return 16;
#else
  (void)out_host;
  (void)reset;
  return 0;
#endif
}

int64_t hsrq_debug_counters(int64_t* out_host, int32_t reset) {
  unsigned long long v[32];
  if (cudaMemcpyFromSymbol(v, g_ctr, sizeof(v)) != cudaSuccess) return HSRQ_ERR_CUDA;
  for (int i = 0; i < 32; i++) out_host[i] = (int64_t)v[i];
  if (reset) {
    unsigned long long z[32] = {0};
    if (cudaMemcpyToSymbol(g_ctr, z, sizeof(z)) != cudaSuccess) return HSRQ_ERR_CUDA;
  }
  return 0;
}
void hsrq_set_timing(int32_t enable) { g_timing = enable; }

int32_t hsrq_tune_diag(int32_t dp, int32_t dwr, int32_t dwc, int32_t wsr, int32_t wsc) {
  diag_attrs();  // reads the environment once; the explicit setting wins
  g_force_r = DiagVariant{dp, dwr};
  g_force_c = DiagVariant{dp, dwc};
  if (dp == 0) g_force_r = g_force_c = DiagVariant{0, 0};
  g_diag_ws_r = wsr;
  g_diag_ws = wsc;
  return 0;
}
int32_t hsrq_tune_panel(int32_t cluster) {
  diag_attrs();  // reads the environment once; the explicit setting wins
  g_panel_cluster = cluster != 0;
  return g_panel_cluster;
}
int32_t hsrq_tune_diag_rx(int32_t np) {
  diag_attrs();  // reads the environment once; the explicit setting wins
  g_diag_rx = (np == 4 || np == 8) ? np : (np < 0 ? -1 : 0);
  return g_diag_rx;
}
void hsrq_phase_times(double* out_host) {
  for (int i = 0; i < 5; i++) g_phase_ms[i] = 0.0;
  drain_timing(g_phase_ms);
  for (int i = 0; i < 5; i++) out_host[i] = g_phase_ms[i];
}

int64_t hsrq_tile_diag(int32_t k, int32_t b, const double* hdiag, const double* hleft,
                       int32_t has_left, const double* lam_re, const double* lam_im,
                       const double* rright, double* x, double* c_re, double* c_im, double* s,
                       int32_t* beta_exp, int64_t* status, int32_t robust, double omega,
                       void* stream) {
  if (k < 1 || k > MAXK || b < 1) return HSRQ_ERR_CONFIG;
  Ctx c;
  memset(&c, 0, sizeof(c));
  c.lam_re = lam_re;
  c.lam_im = lam_im;
  c.mc = lam_im ? 1 : 0;  // tile mode: kind flag only
  c.robust = robust;
  c.omega = omega;
  DiagArgs a;
  memset(&a, 0, sizeof(a));
  a.tile_mode = 1;
  a.k = k;
  a.has_left = has_left;
  a.t_hdiag = hdiag;
  a.t_rright = rright;
  a.t_x = x;
  a.t_cre = c_re;
  a.t_cim = c_im;
  a.t_s = s;
  a.t_beta = beta_exp;
  a.t_status = status;
  a.t_b = b;
  a.t_hleft = hleft;
  a.q0 = 0;
  a.count = b;
  if (!diag_attrs()) return HSRQ_ERR_CUDA;
  if (!ck(cudaMemsetAsync(status, 0, sizeof(int64_t) * b, (cudaStream_t)stream), "memset"))
    return HSRQ_ERR_CUDA;
  diag_launch(lam_im != nullptr, c, a, (cudaStream_t)stream);
  if (!ck(cudaGetLastError(), "launch") || !ck(cudaStreamSynchronize((cudaStream_t)stream), "sync"))
    return HSRQ_ERR_CUDA;
  return 0;
}

int64_t hsrq_tile_backtransform(int64_t n, int32_t b_r, int32_t b, int32_t cplx,
                                const double* c_re, const double* c_im, const double* s,
                                const int32_t* seg_exp, double* x, double* norms,
                                int32_t* alpha_exp, int32_t mode, double omega, void* stream_) {
  if (n < 1 || b_r < 1 || b < 1) return HSRQ_ERR_CONFIG;
  cudaStream_t stream = (cudaStream_t)stream_;
  Ctx c;
  memset(&c, 0, sizeof(c));
  c.n = n;
  c.b_r = b_r;
  c.N = (int)((n + b_r - 1) / b_r);
  c.mc = cplx ? b : 0;
  c.mr = cplx ? 0 : b;
  c.ms = b;
  c.ncol = cplx ? 2 * b : b;
  c.X = x;
  c.ldx = n;
  c.c_re = const_cast<double*>(c_re);
  c.c_im = const_cast<double*>(c_im);
  c.s = const_cast<double*>(s);
  c.ldc = n;
  c.E = const_cast<int32_t*>(seg_exp);
  c.robust = 1;
  c.mode = mode;
  c.omega = omega;
  int64_t* fail = nullptr;
  double* l2 = nullptr;
  if (!ck(cudaMallocAsync(&fail, sizeof(int64_t) * b, stream), "alloc") ||
      !ck(cudaMallocAsync(&l2, sizeof(double) * b, stream), "alloc") ||
      !ck(cudaMemsetAsync(fail, 0, sizeof(int64_t) * b, stream), "memset"))
    return HSRQ_ERR_CUDA;
  c.fail = fail;
  bt_launch(c, alpha_exp, norms, l2, 0, b, b, stream);
  const bool ok = ck(cudaGetLastError(), "launch");
  cudaFreeAsync(fail, stream);
  cudaFreeAsync(l2, stream);
  if (!ok || !ck(cudaStreamSynchronize(stream), "sync")) return HSRQ_ERR_CUDA;
  return 0;
}

int64_t hsrq_protect_update_batch(const double* bnorm, const double* hnorm, const double* xnorm,
                                  double omega, int64_t count, double* out, void* stream) {
  if (count <= 0) return 0;
  k_protect_batch<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      bnorm, hnorm, xnorm, omega, count, out);
  return ck(cudaGetLastError(), "launch") ? 0 : HSRQ_ERR_CUDA;
}

int64_t hsrq_protect_update_pair_batch(const double* b1, const double* h1, const double* b2,
                                       const double* h2, const double* xnorm, double omega,
                                       int64_t count, double* out1, double* out2, void* stream) {
  if (count <= 0) return 0;
  k_protect_pair_batch<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      b1, h1, b2, h2, xnorm, omega, count, out1, out2);
  return ck(cudaGetLastError(), "launch") ? 0 : HSRQ_ERR_CUDA;
}

int64_t hsrq_hypot_batch(const double* x, const double* y, int64_t count, double* out,
                         void* stream) {
  if (count <= 0) return 0;
  k_hypot_batch<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, y, count, out);
  return ck(cudaGetLastError(), "launch") ? 0 : HSRQ_ERR_CUDA;
}

size_t hsrq_henry_workspace_bytes(int64_t n, int64_t m, int32_t cplx) {
  return henry_layout(n, m, cplx).total;
}

int64_t hsrq_henry_solve(const double* H, int64_t ldh, int64_t n, const double* lam, int64_t m,
                         int32_t cplx, double* X, int64_t ldx, int64_t* status, void* ws,
                         size_t ws_bytes, void* stream_) {
  if (n < 1 || m < 1 || ldh < n || ldx < n || n >= (1 << 21) || m >= (1 << 21))
    return HSRQ_ERR_CONFIG;
  const HenryLayout L = henry_layout(n, m, cplx);
  if (ws_bytes < L.total || ws == nullptr) return HSRQ_ERR_WORKSPACE;
  cudaStream_t stream = (cudaStream_t)stream_;
  char* w = (char*)ws;
  HenryArgs a;
  a.H = H;
  a.ldh = ldh;
  a.n = n;
  a.m = m;
  a.lam = lam;
  a.X = X;
  a.ldx = ldx;
  a.V = (double*)(w + L.v);
  a.C = (double*)(w + L.c);
  a.S = (double*)(w + L.s);
  a.status = status ? status : (int64_t*)(w + L.st);
  a.first = (unsigned long long*)(w + L.first);
  if (!ck(cudaMemsetAsync(a.first, 0, sizeof(unsigned long long), stream), "memset"))
    return HSRQ_ERR_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // threads: whole warps covering n rows, at most HENRY_THREADS
  const int T = (int)std::min<int64_t>(HENRY_THREADS, ((n + 31) / 32) * 32);
  // resident CTAs: keep the working set (v, x, c: 3 n-vectors per shift) under
  // ~half the L2 so the row traffic stays on chip (HSRQ_HENRY_CTAS overrides)
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cplx ? (const void*)k_henry_cplx
                                                           : (const void*)k_henry_real, T, 0);
  const double per_shift = 3.0 * 8.0 * (cplx ? 2 : 1) * (double)n;
  int per_sm = (int)std::max(1.0, std::floor(60.0e6 / (per_shift * sms)));
  per_sm = std::min(per_sm, std::max(1, occ));
  if (const char* e = getenv("HSRQ_HENRY_CTAS")) per_sm = std::max(1, atoi(e));
  const int64_t grid = std::min<int64_t>(m, (int64_t)sms * per_sm);
  if (cplx)
    k_henry_cplx<<<(unsigned)grid, T, 0, stream>>>(a);
  else
    k_henry_real<<<(unsigned)grid, T, 0, stream>>>(a);
  int64_t* first = (int64_t*)(w + L.first);  // reuse the key slot for the packed status
  k_henry_first<<<1, 1, 0, stream>>>(a.first, first);
  g_launches = 2;
  int64_t st = 0;
  if (!ck(cudaGetLastError(), "launch") ||
      !ck(cudaMemcpyAsync(&st, first, sizeof(int64_t), cudaMemcpyDeviceToHost, stream), "d2h") ||
      !ck(cudaStreamSynchronize(stream), "sync"))
    return HSRQ_ERR_CUDA;
  return st;
}

int64_t hsrq_compact_encode(int64_t count, int32_t cplx, const double* c_re, const double* c_im,
                            const double* s, double* t1, double* t2, void* stream) {
  if (count <= 0) return 0;
  k_compact_encode<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      count, cplx, c_re, c_im, s, t1, t2);
  return ck(cudaGetLastError(), "launch") ? 0 : HSRQ_ERR_CUDA;
}

int64_t hsrq_compact_decode(int64_t count, int32_t cplx, const double* t1, const double* t2,
                            double* c_re, double* c_im, double* s, void* stream) {
  if (count <= 0) return 0;
  k_compact_decode<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      count, cplx, t1, t2, c_re, c_im, s);
  return ck(cudaGetLastError(), "launch") ? 0 : HSRQ_ERR_CUDA;
}

}  // extern "C"

#include "hsrq_hostio.cuh"
#include "hsrq_tile_update.cuh"
