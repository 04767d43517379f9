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
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstring>

#include "../../include/hsrq.h"
#include "hsrq_device.cuh"

using namespace hsrq;

namespace {

constexpr int MAXK = 128;    // largest tile (b_r) supported on the GPU path
constexpr int SLOTS = 4;     // rows per lane in the diagonal kernel (MAXK / 32)
constexpr int DIAG_WARPS = 8;

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
  int32_t* E;            // N x ms
  double* Bop;           // (2*ncol_pad) x KP
  StepScalars* SS;       // ms
  double* HM0;           // N x N : max |H[tile i rows, js-1]|
  double* RS;            // N x N : max row sum |H[tile i rows, js:je-1]|
  double* XB;            // N x ms: max |X| over each tile's rows (real: exact;
                         // complex: max(|re|+|im|), an upper bound of max |x|)
  int64_t* fail;         // ms
  unsigned long long* nfail;
  int robust, mode;
  double omega;
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

// HM0[jt][i] = max_{r in tile i} |H[r, js-1]|             (update_rupdate :207-210)
// RS[jt][i]  = max_{r in tile i} sum_{j=1}^{k-1} |htile[r, j]| (:256-262),
// summed left to right like the reference.  One thread per (row, jt).
__global__ void k_tables(Ctx c) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int jt = blockIdx.y + 1;
  if (jt >= c.N) return;
  int64_t js = (int64_t)jt * c.b_r;
  if (r >= js) return;
  int64_t je = js + c.b_r < c.n ? js + c.b_r : c.n;
  int k = (int)(je - js);
  int i = (int)(r / c.b_r);
  double h0 = fabs(c.H[(js - 1) * c.ldh + r]);
  double acc = 0.0;
  for (int j = 1; j < k; j++) acc += fabs(c.H[(js - 1 + j) * c.ldh + r]);
  atomicMax((unsigned long long*)&c.HM0[(int64_t)jt * c.N + i], dkey(h0));
  atomicMax((unsigned long long*)&c.RS[(int64_t)jt * c.N + i], dkey(acc));
}

// X = B (or the broadcast start vector), Cr(:, N-1) = H(:, n-1) - lambda e_n
// (reduce.py:66-69, 77-78).
__global__ void k_init(Ctx c, const double* B, int64_t ldb, int b_broadcast) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t col = blockIdx.y;
  if (r >= c.n || col >= c.ncol) return;
  bool cplx = col < 2 * c.mc;
  bool im = cplx && (col & 1);
  int64_t q = cplx ? col / 2 : c.mc + (col - 2 * c.mc);
  double b = b_broadcast ? (im ? 0.0 : B[r]) : B[col * ldb + r];
  c.X[col * c.ldx + r] = b;
  if (!im) {
    double bb = fabs(b);
    if (cplx && !b_broadcast) bb = bb + fabs(B[(col + 1) * ldb + r]);
    atomicMax((unsigned long long*)&c.XB[(r / c.b_r) * c.ms + q], dkey(bb));
  }
  double h = im ? 0.0 : c.H[(c.n - 1) * c.ldh + r];
  if (r == c.n - 1) h -= im ? c.lam_im[q] : c.lam_re[q];
  c.Cr[col * c.ldx + r] = h;
}

__global__ void k_zero_state(Ctx c) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t ne = (int64_t)c.N * c.ms;
  if (t < ne) {
    c.E[t] = 0;
    c.XB[t] = 0.0;
  }
  if (t < c.ms) c.fail[t] = 0;
  if (t < (int64_t)c.N * c.N) {
    c.HM0[t] = 0.0;
    c.RS[t] = 0.0;
  }
  if (t == 0) *c.nfail = 0;
}

__global__ void k_zero_bop(double* Bop, int64_t count) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < count) Bop[t] = 0.0;
}

// ---------------------------------------------------------------------------
// k_diag: diagonal tile (one warp per shift)
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ T sel(const T (&a)[SLOTS], int j) {
  T r = a[0];
#pragma unroll
  for (int t = 1; t < SLOTS; t++)
    if (j == t) r = a[t];
  return r;
}
template <typename T>
__device__ __forceinline__ void put(T (&a)[SLOTS], int j, T v) {
#pragma unroll
  for (int t = 0; t < SLOTS; t++)
    if (j == t) a[t] = v;
}

struct DiagSmem {
  double hs[MAXK * (MAXK + 1) / 2 + MAXK];  // packed tile columns 0..k-2, rows 0..t+1
  double hmax[MAXK];                        // max_{i<kp} |h(i, kp-1)|
  double cs_c[DIAG_WARPS][MAXK];
  double cs_ci[DIAG_WARPS][MAXK];
  double cs_s[DIAG_WARPS][MAXK];
};

__device__ __forceinline__ int hs_off(int t) { return t * (t + 3) / 2; }

struct DiagArgs {
  int jt;
  int64_t js;
  int k;
  int has_left;
  // tile-level mode (hsrq_tile_diag): explicit tile buffers instead of the sweep state
  int tile_mode;
  const double* t_hdiag;   // k x (k-1) row-major
  const double* t_hleft;
  const double* t_rright;  // k x b / 2b row-major
  double* t_x;
  double *t_cre, *t_cim, *t_s;
  int32_t* t_beta;
  int64_t* t_status;
  int t_b;
};

__device__ __forceinline__ void record_fail(const Ctx& c, int64_t q, int phase, int tile, int row,
                                            const DiagArgs& a) {
  if (a.tile_mode) {
    a.t_status[q] = (int64_t)(phase) * (1LL << 42) + (int64_t)row;
    return;
  }
  if (c.fail[q] == 0) {
    c.fail[q] = pack_fail(phase, tile, row);
    atomicAdd(c.nfail, 1ULL);
  }
}

// Real shift: reduce_diag + solve_rsolve fused (same v recurrence, identical
// arithmetic), then the panel operands.
__device__ void diag_real(const Ctx& c, const DiagArgs& a, DiagSmem& sm, int64_t q, int64_t col,
                          int warp, double hleft0) {
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  const double lam = c.lam_re[q];
  const double omega = c.omega;
  const bool robust = c.robust;
  double v[SLOTS], x[SLOTS];
#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < k) {
      if (a.tile_mode) {
        v[j] = a.t_rright[(int64_t)i * a.t_b + q];
        x[j] = a.t_x[(int64_t)i * a.t_b + q];
      } else {
        v[j] = c.Cr[col * c.ldx + a.js + i];
        x[j] = c.X[col * c.ldx + a.js + i];
      }
    } else {
      v[j] = 0.0;
      x[j] = 0.0;
    }
  }
  double* csc = sm.cs_c[warp];
  double* css = sm.cs_s[warp];
  int gexp = 0;
  bool failed = false;
  for (int kp = k - 1; kp >= 1; --kp) {
    const int o = kp & 31, sl = kp >> 5;
    double vk = __shfl_sync(0xffffffffu, sel(v, sl), o);
    double xk = __shfl_sync(0xffffffffu, sel(x, sl), o);
    const double* hcol = sm.hs + hs_off(kp - 1);
    const double av = hcol[kp];
    double r = ghypot(av, vk);
    if (r == 0.0) {
      if (lane == 0) record_fail(c, q, HSRQ_KIND_DEGENERATE, a.jt, kp, a);
      failed = true;
      break;
    }
    const double cc = vk / r, ss = -av / r;
    if (lane == 0) {
      csc[kp] = cc;
      css[kp] = ss;
    }
    const double phi = vk * cc - av * ss;
    if (phi == 0.0) {
      if (lane == 0) record_fail(c, q, HSRQ_KIND_SINGULAR, a.jt, kp, a);
      failed = true;
      break;
    }
    if (robust) {
      double aphi = fabs(phi), ax = fabs(xk);
      if (aphi < 1.0 && ax > aphi * omega) {
        int e = pow2floor_e(aphi * omega / ax);
        double xi = p2(e);
#pragma unroll
        for (int j = 0; j < SLOTS; j++) x[j] *= xi;
        xk *= xi;
        gexp += e;
      }
    }
    xk = xk / phi;
    if (robust) {
      double xm = 0.0, vm = 0.0;
#pragma unroll
      for (int j = 0; j < SLOTS; j++) {
        int i = lane + 32 * j;
        if (i < kp) {
          double ax = fabs(x[j]), avv = fabs(v[j]);
          if (ax > xm) xm = ax;
          if (avv > vm) vm = avv;
        }
      }
      xm = warp_max(xm);
      vm = warp_max(vm);
      int e = protect_update_e(xm, vm + sm.hmax[kp] + fabs(lam), fabs(xk), omega);
      if (e < 0) {
        double xi = p2(e);
#pragma unroll
        for (int j = 0; j < SLOTS; j++) x[j] *= xi;
        xk *= xi;
        gexp += e;
      }
    }
    if (lane == o) put(x, sl, xk);
    const double tau1 = ss * xk, tau2 = cc * xk;
#pragma unroll
    for (int j = 0; j < SLOTS; j++) {
      int i = lane + 32 * j;
      if (i < kp - 1) {
        double hi = hcol[i];
        x[j] = (x[j] - tau2 * v[j]) + tau1 * hi;
        v[j] = cc * hi + ss * v[j];
      } else if (i == kp - 1) {
        double hd = hcol[i] - lam;
        x[j] = (x[j] - tau2 * v[j]) + tau1 * hd;
        v[j] = cc * hd + ss * v[j];
      }
    }
  }
  if (failed) return;
  // cross-tile rotation (reduce_diag :94-105) and the last pivot (:178-192)
  double v0 = __shfl_sync(0xffffffffu, v[0], 0);
  double x0 = __shfl_sync(0xffffffffu, x[0], 0);
  double c0 = 1.0, s0 = 0.0, piv = v0;
  if (a.has_left) {
    double al = hleft0;
    double r = ghypot(al, v0);
    if (r == 0.0) {
      if (lane == 0) record_fail(c, q, HSRQ_KIND_DEGENERATE, a.jt, 0, a);
      return;
    }
    c0 = v0 / r;
    s0 = -al / r;
    piv = v0 * c0 - al * s0;
  }
  if (lane == 0) {
    csc[0] = c0;
    css[0] = s0;
  }
  if (piv == 0.0) {
    if (lane == 0) record_fail(c, q, HSRQ_KIND_SINGULAR, a.jt, 0, a);
    return;
  }
  if (robust) {
    double avv = fabs(piv), ax = fabs(x0);
    if (avv < 1.0 && ax > avv * omega) {
      int e = pow2floor_e(avv * omega / ax);
      double xi = p2(e);
#pragma unroll
      for (int j = 0; j < SLOTS; j++) x[j] *= xi;
      x0 *= xi;
      gexp += e;
    }
  }
  x0 = x0 / piv;
  if (lane == 0) x[0] = x0;
  __syncwarp();

  // outputs: solution tile, rotations, scale exponent
#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < k) {
      if (a.tile_mode) {
        a.t_x[(int64_t)i * a.t_b + q] = x[j];
        a.t_cre[(int64_t)i * a.t_b + q] = csc[i];
        a.t_s[(int64_t)i * a.t_b + q] = css[i];
        if (a.t_cim) a.t_cim[(int64_t)i * a.t_b + q] = 0.0;
      } else {
        c.X[col * c.ldx + a.js + i] = x[j];
        c.c_re[q * c.ldc + a.js + i] = csc[i];
        c.s[q * c.ldc + a.js + i] = css[i];
        if (c.c_im) c.c_im[q * c.ldc + a.js + i] = 0.0;
      }
    }
  }
  if (a.tile_mode) {
    if (lane == 0) a.t_beta[q] += gexp;
    return;
  }
  if (lane == 0) c.E[(int64_t)a.jt * c.ms + q] += gexp;
  if (a.jt == 0) return;

  // ---- panel operands ----
  // W_j = c_j prod_{t<j} s_t, P = prod_t s_t; Z: update_rupdate :246-253.
  double w[SLOTS], z[SLOTS];
#pragma unroll
  for (int j = 0; j < SLOTS; j++) w[j] = z[j] = 0.0;
  double pre = 1.0;
  double carry = c0 * __shfl_sync(0xffffffffu, x[0], 0);  // Z[0] = c[0] * Z[0]
  for (int j = 0; j < k; j++) {
    const double cj = csc[j], sj = css[j];
    const int oj = j & 31, slj = j >> 5;
    if (lane == oj) put(w, slj, cj * pre);
    pre = pre * sj;
    if (j >= 1) {
      double t2 = __shfl_sync(0xffffffffu, sel(x, slj), oj);
      double t1 = carry;
      double zf = cj * t1 - sj * t2;  // final Z[j-1]
      carry = sj * t1 + cj * t2;
      const int om = (j - 1) & 31, slm = (j - 1) >> 5;
      if (lane == om) put(z, slm, zf);
    }
  }
  // zmax over Z[0:k-1]
  double zm = 0.0;
#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < k - 1 && fabs(z[j]) > zm) zm = fabs(z[j]);
  }
  zm = warp_max(zm);
  // B operand: column 2*col = W, 2*col+1 = [0, Z[0..k-2]]
  double* bw = c.Bop + (2 * col) * KP;
  double* bz = c.Bop + (2 * col + 1) * KP;
#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < KP) {
      bw[i] = i < k ? w[j] : 0.0;
      // Zs[i+1] = Z[i]
      if (i + 1 < KP) bz[i + 1] = (i < k - 1) ? z[j] : 0.0;
    }
  }
  if (lane == 0) {
    bz[0] = 0.0;
    StepScalars st;
    st.rho_re = s0 * x0;
    st.rho_im = 0.0;
    st.zk_re = carry;
    st.zk_im = 0.0;
    st.zmax = zm;
    st.P = pre;
    st.c0_re = c0;
    st.c0_im = 0.0;
    c.SS[q] = st;
  }
}

// Complex shift: creduce_diag + _build_complex_r + robust_trsv_complex,
// with R's column kp formed and consumed at step kp.
__device__ void diag_cplx(const Ctx& c, const DiagArgs& a, DiagSmem& sm, int64_t q, int64_t col,
                          int warp, double hleft0) {
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  const double lre = c.lam_re[q], lim = c.lam_im[q];
  const double omega = c.omega;
  const bool robust = c.robust;
  cplx v[SLOTS], x[SLOTS];
#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < k) {
      if (a.tile_mode) {
        int64_t b2 = 2 * (int64_t)a.t_b;
        v[j] = mk(a.t_rright[i * b2 + 2 * q], a.t_rright[i * b2 + 2 * q + 1]);
        x[j] = mk(a.t_x[i * b2 + 2 * q], a.t_x[i * b2 + 2 * q + 1]);
      } else {
        v[j] = mk(c.Cr[col * c.ldx + a.js + i], c.Cr[(col + 1) * c.ldx + a.js + i]);
        x[j] = mk(c.X[col * c.ldx + a.js + i], c.X[(col + 1) * c.ldx + a.js + i]);
      }
    } else {
      v[j] = mk(0.0, 0.0);
      x[j] = mk(0.0, 0.0);
    }
  }
  double* csc = sm.cs_c[warp];
  double* csi = sm.cs_ci[warp];
  double* css = sm.cs_s[warp];
  int gexp = 0;
  for (int kp = k - 1; kp >= 1; --kp) {
    const int o = kp & 31, sl = kp >> 5;
    cplx vsel = sel(v, sl), xsel = sel(x, sl);
    cplx vk = mk(__shfl_sync(0xffffffffu, vsel.re, o), __shfl_sync(0xffffffffu, vsel.im, o));
    cplx xk = mk(__shfl_sync(0xffffffffu, xsel.re, o), __shfl_sync(0xffffffffu, xsel.im, o));
    const double* hcol = sm.hs + hs_off(kp - 1);
    const double av = hcol[kp];
    double absv = ghypot(vk.re, vk.im);
    double r = ghypot(av, absv);
    if (r == 0.0) {
      if (lane == 0) record_fail(c, q, HSRQ_KIND_DEGENERATE, a.jt, kp, a);
      return;
    }
    const double cr = vk.re / r, ci = vk.im / r, sv = -av / r;
    if (lane == 0) {
      csc[kp] = cr;
      csi[kp] = ci;
      css[kp] = sv;
    }
    const cplx cc = mk(cr, ci), ccj = mk(cr, -ci), svc = mk(sv, 0.0);
    // R column kp: r_i = conj(c) v_i - s t_i  (i <= kp)
    cplx rcol[SLOTS];
#pragma unroll
    for (int j = 0; j < SLOTS; j++) {
      int i = lane + 32 * j;
      cplx t = mk(i <= kp ? hcol[i] : 0.0, 0.0);
      if (i == kp - 1) t = csub(t, mk(lre, lim));
      rcol[j] = csub(cmul(ccj, v[j]), cmul(svc, t));
    }
    const cplx d = csub(cmul(ccj, vk), cmul(svc, mk(av, 0.0)));
    if (d.re == 0.0 && d.im == 0.0) {
      if (lane == 0) record_fail(c, q, HSRQ_KIND_SINGULAR, a.jt, kp, a);
      return;
    }
    if (robust) {
      double ad = cabs_(d), ax = cabs_(xk);
      if (ad < 1.0 && ax > ad * omega) {
        int e = pow2floor_e(ad * omega / ax);
        cplx xi = mk(p2(e), 0.0);
#pragma unroll
        for (int j = 0; j < SLOTS; j++) x[j] = cmul(x[j], xi);
        xk = cmul(xk, xi);
        gexp += e;
      }
    }
    xk = cdiv(xk, d);
    if (robust) {
      // upper bounds first (|z| <= (|re|+|im|)(1+2^-50)); exact hypots only if needed
      double rb = 0.0, bb = 0.0;
#pragma unroll
      for (int j = 0; j < SLOTS; j++) {
        int i = lane + 32 * j;
        if (i < kp) {
          double q1 = fabs(rcol[j].re) + fabs(rcol[j].im);
          double q2 = fabs(x[j].re) + fabs(x[j].im);
          if (q1 > rb) rb = q1;
          if (q2 > bb) bb = q2;
        }
      }
      rb = warp_max(rb) * (1.0 + 0x1p-50);
      bb = warp_max(bb) * (1.0 + 0x1p-50);
      double axk = cabs_(xk);
      if (!protect_update_is_one(bb, rb, axk, omega)) {
        double rm = 0.0, bm = 0.0;
#pragma unroll
        for (int j = 0; j < SLOTS; j++) {
          int i = lane + 32 * j;
          if (i < kp) {
            double q1 = cabs_(rcol[j]), q2 = cabs_(x[j]);
            if (q1 > rm) rm = q1;
            if (q2 > bm) bm = q2;
          }
        }
        rm = warp_max(rm);
        bm = warp_max(bm);
        int e = protect_update_e(bm, rm, axk, omega);
        if (e < 0) {
          cplx xi = mk(p2(e), 0.0);
#pragma unroll
          for (int j = 0; j < SLOTS; j++) x[j] = cmul(x[j], xi);
          xk = cmul(xk, xi);
          gexp += e;
        }
      }
    }
    if (lane == o) put(x, sl, xk);
#pragma unroll
    for (int j = 0; j < SLOTS; j++) {
      int i = lane + 32 * j;
      if (i < kp) {
        x[j] = csub(x[j], cmul(xk, rcol[j]));
        if (i < kp - 1) {
          double hi = hcol[i];
          v[j] = mk(cr * hi + sv * v[j].re, ci * hi + sv * v[j].im);
        } else {
          double tre = hcol[i] - lre, tim = -lim;
          v[j] = mk((cr * tre - ci * tim) + sv * v[j].re, (cr * tim + ci * tre) + sv * v[j].im);
        }
      }
    }
  }
  // j = 0: cross-tile rotation (creduce_diag :449-463) and R[0,0] (:546-550)
  cplx v0 = mk(__shfl_sync(0xffffffffu, v[0].re, 0), __shfl_sync(0xffffffffu, v[0].im, 0));
  cplx x0 = mk(__shfl_sync(0xffffffffu, x[0].re, 0), __shfl_sync(0xffffffffu, x[0].im, 0));
  double c0r = 1.0, c0i = 0.0, s0 = 0.0;
  cplx d = v0;
  if (a.has_left) {
    double al = hleft0;
    double absv = ghypot(v0.re, v0.im);
    double r = ghypot(al, absv);
    if (r == 0.0) {
      if (lane == 0) record_fail(c, q, HSRQ_KIND_DEGENERATE, a.jt, 0, a);
      return;
    }
    c0r = v0.re / r;
    c0i = v0.im / r;
    s0 = -al / r;
    d = csub(cmul(mk(c0r, -c0i), v0), cmul(mk(s0, 0.0), mk(al, 0.0)));
  }
  if (lane == 0) {
    csc[0] = c0r;
    csi[0] = c0i;
    css[0] = s0;
  }
  if (d.re == 0.0 && d.im == 0.0) {
    if (lane == 0) record_fail(c, q, HSRQ_KIND_SINGULAR, a.jt, 0, a);
    return;
  }
  if (robust) {
    double ad = cabs_(d), ax = cabs_(x0);
    if (ad < 1.0 && ax > ad * omega) {
      int e = pow2floor_e(ad * omega / ax);
      cplx xi = mk(p2(e), 0.0);
#pragma unroll
      for (int j = 0; j < SLOTS; j++) x[j] = cmul(x[j], xi);
      x0 = cmul(x0, xi);
      gexp += e;
    }
  }
  x0 = cdiv(x0, d);
  if (lane == 0) x[0] = x0;
  __syncwarp();

#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < k) {
      if (a.tile_mode) {
        int64_t b2 = 2 * (int64_t)a.t_b;
        a.t_x[i * b2 + 2 * q] = x[j].re;
        a.t_x[i * b2 + 2 * q + 1] = x[j].im;
        a.t_cre[(int64_t)i * a.t_b + q] = csc[i];
        a.t_cim[(int64_t)i * a.t_b + q] = csi[i];
        a.t_s[(int64_t)i * a.t_b + q] = css[i];
      } else {
        c.X[col * c.ldx + a.js + i] = x[j].re;
        c.X[(col + 1) * c.ldx + a.js + i] = x[j].im;
        c.c_re[q * c.ldc + a.js + i] = csc[i];
        c.c_im[q * c.ldc + a.js + i] = csi[i];
        c.s[q * c.ldc + a.js + i] = css[i];
      }
    }
  }
  if (a.tile_mode) {
    if (lane == 0) a.t_beta[q] += gexp;
    return;
  }
  if (lane == 0) c.E[(int64_t)a.jt * c.ms + q] += gexp;
  if (a.jt == 0) return;

  // ---- panel operands (cupdate_crupdate :645-666; W complex, P real) ----
  cplx w[SLOTS], z[SLOTS];
#pragma unroll
  for (int j = 0; j < SLOTS; j++) w[j] = z[j] = mk(0.0, 0.0);
  double pre = 1.0;
  cplx carry = mk(c0r * x0.re + c0i * x0.im, c0r * x0.im - c0i * x0.re);
  for (int j = 0; j < k; j++) {
    const double cr = csc[j], ci = csi[j], sj = css[j];
    const int oj = j & 31, slj = j >> 5;
    if (lane == oj) put(w, slj, mk(cr * pre, ci * pre));
    pre = pre * sj;
    if (j >= 1) {
      cplx xs = sel(x, slj);
      cplx t2 = mk(__shfl_sync(0xffffffffu, xs.re, oj), __shfl_sync(0xffffffffu, xs.im, oj));
      cplx t1 = carry;
      cplx zf = mk((cr * t1.re - ci * t1.im) - sj * t2.re, (cr * t1.im + ci * t1.re) - sj * t2.im);
      carry = mk(sj * t1.re + (cr * t2.re + ci * t2.im), sj * t1.im + (cr * t2.im - ci * t2.re));
      const int om = (j - 1) & 31, slm = (j - 1) >> 5;
      if (lane == om) put(z, slm, zf);
    }
  }
  double zm = 0.0;
#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < k - 1) {
      double qz = cabs_(z[j]);
      if (qz > zm) zm = qz;
    }
  }
  zm = warp_max(zm);
  double* bw_re = c.Bop + (2 * col) * KP;
  double* bz_re = c.Bop + (2 * col + 1) * KP;
  double* bw_im = c.Bop + (2 * (col + 1)) * KP;
  double* bz_im = c.Bop + (2 * (col + 1) + 1) * KP;
#pragma unroll
  for (int j = 0; j < SLOTS; j++) {
    int i = lane + 32 * j;
    if (i < KP) {
      bw_re[i] = i < k ? w[j].re : 0.0;
      bw_im[i] = i < k ? w[j].im : 0.0;
      if (i + 1 < KP) {
        bz_re[i + 1] = (i < k - 1) ? z[j].re : 0.0;
        bz_im[i + 1] = (i < k - 1) ? z[j].im : 0.0;
      }
    }
  }
  if (lane == 0) {
    bz_re[0] = 0.0;
    bz_im[0] = 0.0;
    StepScalars st;
    st.rho_re = s0 * x0.re;
    st.rho_im = s0 * x0.im;
    st.zk_re = carry.re;
    st.zk_im = carry.im;
    st.zmax = zm;
    st.P = pre;
    st.c0_re = c0r;
    st.c0_im = c0i;
    c.SS[q] = st;
  }
}

__global__ void __launch_bounds__(DIAG_WARPS * 32) k_diag(Ctx c, DiagArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DiagSmem& sm = *reinterpret_cast<DiagSmem*>(smem_raw);
  const int k = a.k;
  // stage the diagonal tile (columns 0..k-2, rows 0..t+1) and per-kp maxima
  for (int t = 0; t + 1 < k; t++) {
    for (int i = threadIdx.x; i <= t + 1; i += blockDim.x) {
      double h = a.tile_mode ? a.t_hdiag[(int64_t)i * (k - 1) + t]
                             : c.H[(a.js + t) * c.ldh + a.js + i];
      sm.hs[hs_off(t) + i] = h;
    }
  }
  __syncthreads();
  for (int kp = 1 + threadIdx.x; kp < k; kp += blockDim.x) {
    const double* hcol = sm.hs + hs_off(kp - 1);
    double m = 0.0;
    for (int i = 0; i < kp; i++)
      if (fabs(hcol[i]) > m) m = fabs(hcol[i]);
    sm.hmax[kp] = m;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * DIAG_WARPS + warp;
  const int64_t ms = a.tile_mode ? a.t_b : c.ms;
  if (q >= ms) return;
  bool cplx;
  int64_t col;
  if (a.tile_mode) {
    cplx = c.mc != 0;
    col = 0;
  } else {
    col_of_shift(c, q, cplx, col);
    if (c.fail[q] != 0) return;
  }
  double hleft0 = 0.0;
  if (a.has_left) hleft0 = a.tile_mode ? a.t_hleft[0] : c.H[(a.js - 1) * c.ldh + a.js];
  if (cplx)
    diag_cplx(c, a, sm, q, col, warp, hleft0);
  else
    diag_real(c, a, sm, q, col, warp, hleft0);
}

#include "hsrq_panel.cuh"

#include "hsrq_backtransform.cuh"

// elementwise helpers for parity tests
__global__ void k_protect_batch(const double* b, const double* h, const double* x, double omega,
                                int64_t count, double* out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < count) {
    int e = protect_update_e(b[t], h[t], x[t], omega);
    out[t] = p2(e);
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
double g_phase_ms[4] = {0, 0, 0, 0};

bool ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return false;
  }
  return true;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct WsLayout {
  size_t cr, bop, ss, hm0, rs, xb, rsc, nfail, total;
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
  L.bop = off;
  off = align_up(off + sizeof(double) * (size_t)(2 * ncol_pad) * KP, 256);
  L.ss = off;
  off = align_up(off + sizeof(StepScalars) * (size_t)ms, 256);
  L.hm0 = off;
  off = align_up(off + sizeof(double) * (size_t)N * N, 256);
  L.rs = off;
  off = align_up(off + sizeof(double) * (size_t)N * N, 256);
  L.xb = off;
  off = align_up(off + sizeof(double) * (size_t)N * ms, 256);
  L.rsc = off;
  off = align_up(off + 64 * (size_t)N * ms, 256);
  L.total = off;
  return L;
}

int64_t solve_impl(const double* H, int64_t ldh, int64_t n, int32_t b_r, const double* lam_re,
                   const double* lam_im, int64_t mc, int64_t mr, const double* B, int64_t ldb,
                   int32_t b_broadcast, double* X, int64_t ldx, double* c_re, double* c_im,
                   double* s, int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                   double* log2norm, int64_t* fail, int32_t robust, int32_t mode, void* ws,
                   size_t ws_bytes, cudaStream_t stream) {
  g_launches = 0;
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
  c.c_re = c_re;
  c.c_im = c_im;
  c.s = s;
  c.ldc = ldc;
  c.E = seg_exp;
  c.Bop = (double*)(w + L.bop);
  c.SS = (StepScalars*)(w + L.ss);
  c.HM0 = (double*)(w + L.hm0);
  c.RS = (double*)(w + L.rs);
  c.XB = (double*)(w + L.xb);
  c.fail = fail;
  c.nfail = (unsigned long long*)(w + L.nfail);
  c.robust = robust;
  c.mode = mode;
  c.omega = robust ? (1.7976931348623157e308 / 2.0) / (double)b_r
                   : HUGE_VAL;
  // the crossover block shares X's leading dimension
  if (ldx != n) {
    snprintf(g_err, sizeof(g_err), "ldx must equal n in this build");
    return HSRQ_ERR_CONFIG;
  }

  static bool attr_done = false;
  const size_t diag_smem = sizeof(DiagSmem);
  const size_t panel_smem = sizeof(PanelSmem);
  if (!attr_done) {
    if (!ck(cudaFuncSetAttribute(k_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)diag_smem),
            "attr diag") ||
        !ck(cudaFuncSetAttribute(k_panel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel") ||
        !ck(cudaFuncSetAttribute(k_panel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel") ||
        !ck(cudaFuncSetAttribute(k_panel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel") ||
        !ck(cudaFuncSetAttribute(k_panel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem), "attr panel"))
      return HSRQ_ERR_CUDA;
    attr_done = true;
  }
  // Optional per-launch timing: events around every launch, one sync at the end.
  const int nev = 2 * c.N + 4;
  cudaEvent_t* ev = nullptr;
  if (g_timing) {
    ev = new cudaEvent_t[nev];
    for (int i = 0; i < nev; i++) cudaEventCreate(&ev[i]);
    cudaEventRecord(ev[0], stream);
  }
  const int64_t nzero = std::max<int64_t>((int64_t)c.N * c.ms, (int64_t)c.N * c.N) + c.ms + 1;
  k_zero_state<<<(unsigned)((nzero + 255) / 256), 256, 0, stream>>>(c);
  g_launches++;
  const int64_t nbop = 2 * c.ncol_pad * KP;
  k_zero_bop<<<(unsigned)((nbop + 255) / 256), 256, 0, stream>>>(c.Bop, nbop);
  g_launches++;
  if (c.N > 1) {
    dim3 gt((unsigned)((n + 255) / 256), (unsigned)(c.N - 1));
    k_tables<<<gt, 256, 0, stream>>>(c);
    g_launches++;
  }
  {
    dim3 gi((unsigned)((n + 255) / 256), (unsigned)c.ncol);
    k_init<<<gi, 256, 0, stream>>>(c, B, ldb, b_broadcast);
    g_launches++;
  }
  if (g_timing) cudaEventRecord(ev[1], stream);
  const bool a16 = (ldh % 2 == 0) && (b_r % 2 == 0);
  const int S = std::min(SMAX, std::max(1, BM / b_r));
  for (int jt = c.N - 1; jt >= 0; --jt) {
    DiagArgs a;
    memset(&a, 0, sizeof(a));
    a.jt = jt;
    a.js = (int64_t)jt * b_r;
    int64_t je = a.js + b_r < n ? a.js + b_r : n;
    a.k = (int)(je - a.js);
    a.has_left = jt > 0;
    unsigned gd = (unsigned)((c.ms + DIAG_WARPS - 1) / DIAG_WARPS);
    k_diag<<<gd, DIAG_WARPS * 32, diag_smem, stream>>>(c, a);
    g_launches++;
    if (g_timing) cudaEventRecord(ev[2 + 2 * jt], stream);
    if (jt > 0) {
      PanelArgs p;
      p.jt = jt;
      p.js = a.js;
      p.k = a.k;
      p.S = S;
      RowScalars* rsc = (RowScalars*)(w + L.rsc);
      const int64_t nsc = (int64_t)jt * c.ms;
      k_scalars<<<(unsigned)((nsc + 127) / 128), 128, 0, stream>>>(c, p, rsc);
      g_launches++;
      dim3 gp((unsigned)(c.ncol_pad / BN), (unsigned)((jt + S - 1) / S));
      const bool seg16 = (b_r % 16) == 0;
      if (a16 && seg16)
        k_panel<true, true><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
      else if (a16)
        k_panel<true, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
      else if (seg16)
        k_panel<false, true><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
      else
        k_panel<false, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
      g_launches++;
    }
    if (g_timing) cudaEventRecord(ev[3 + 2 * jt], stream);
  }
  k_backtransform<<<(unsigned)((c.ms + BT_WARPS - 1) / BT_WARPS), BT_WARPS * 32, 0, stream>>>(
      c, alpha_exp, norms, log2norm);
  g_launches++;
  if (g_timing) {
    cudaEventRecord(ev[nev - 2], stream);
    cudaEventSynchronize(ev[nev - 2]);
    float t;
    double t_diag = 0, t_panel = 0;
    // launch order: ev[1] | diag(N-1) ev[2+2(N-1)] panel ev[3+2(N-1)] | diag(N-2) ...
    int prev = 1;
    for (int jt = c.N - 1; jt >= 0; --jt) {
      cudaEventElapsedTime(&t, ev[prev], ev[2 + 2 * jt]);
      t_diag += t;
      cudaEventElapsedTime(&t, ev[2 + 2 * jt], ev[3 + 2 * jt]);
      t_panel += t;
      prev = 3 + 2 * jt;
    }
    cudaEventElapsedTime(&t, ev[prev], ev[nev - 2]);
    g_phase_ms[2] = t;
    cudaEventElapsedTime(&t, ev[0], ev[1]);
    g_phase_ms[3] = t;
    g_phase_ms[0] = t_diag;
    g_phase_ms[1] = t_panel;
    for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
    delete[] ev;
  }
  if (!ck(cudaGetLastError(), "launch")) return HSRQ_ERR_CUDA;
  return 0;
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
  int64_t r = solve_impl(H, ldh, n, b_r, lam_re, lam_im, m_cplx, m_real, B, ldb, b_broadcast, X,
                         ldx, c_re, c_im, s, ldc, seg_exp, alpha_exp, norms, log2norm, fail,
                         robust, mode, ws, ws_bytes, (cudaStream_t)stream);
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

int64_t hsrq_last_launch_count(void) { return g_launches; }
void hsrq_set_timing(int32_t enable) { g_timing = enable; }
void hsrq_phase_times(double* out_host) {
  for (int i = 0; i < 4; i++) out_host[i] = g_phase_ms[i];
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
  const size_t diag_smem = sizeof(DiagSmem);
  if (!ck(cudaFuncSetAttribute(k_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)diag_smem),
          "attr"))
    return HSRQ_ERR_CUDA;
  if (!ck(cudaMemsetAsync(status, 0, sizeof(int64_t) * b, (cudaStream_t)stream), "memset"))
    return HSRQ_ERR_CUDA;
  k_diag<<<(b + DIAG_WARPS - 1) / DIAG_WARPS, DIAG_WARPS * 32, diag_smem, (cudaStream_t)stream>>>(c, a);
  if (!ck(cudaGetLastError(), "launch") || !ck(cudaStreamSynchronize((cudaStream_t)stream), "sync"))
    return HSRQ_ERR_CUDA;
  return 0;
}

int64_t hsrq_protect_update_batch(const double* bnorm, const double* hnorm, const double* xnorm,
                                  double omega, int64_t count, double* out, void* stream) {
  if (count <= 0) return 0;
  k_protect_batch<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      bnorm, hnorm, xnorm, omega, count, out);
  return ck(cudaGetLastError(), "launch") ? 0 : HSRQ_ERR_CUDA;
}

int64_t hsrq_hypot_batch(const double* x, const double* y, int64_t count, double* out,
                         void* stream) {
  if (count <= 0) return 0;
  k_hypot_batch<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, y, count, out);
  return ck(cudaGetLastError(), "launch") ? 0 : HSRQ_ERR_CUDA;
}

}  // extern "C"
