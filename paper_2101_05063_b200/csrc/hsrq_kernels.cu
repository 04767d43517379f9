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
  double h = im ? 0.0 : c.H[(c.n - 1) * c.ldh + r];
  if (r == c.n - 1) h -= im ? c.lam_im[q] : c.lam_re[q];
  c.Cr[col * c.ldx + r] = h;
}

__global__ void k_zero_state(Ctx c) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t ne = (int64_t)c.N * c.ms;
  if (t < ne) c.E[t] = 0;
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

// ---------------------------------------------------------------------------
// k_panel: fused reduction + guarded update GEMM on DMMA
// ---------------------------------------------------------------------------

struct PanelArgs {
  int jt;
  int64_t js;
  int k;            // width of tile column jt (K)
  int S;            // tile rows per CTA
};

struct PanelSmem {
  union {
    struct {
      double A[STAGES][BK][APAD];
      double B[STAGES][2 * BN][BPAD];
    } pipe;
    double C[2 * BN][APAD];  // accumulators, [acc col][row]
  } u;
  unsigned long long red[2][SMAX][BN];
  double fb[SMAX][BN], rr[SMAX][BN], ri[SMAX][BN], fx[SMAX][BN], xi2[SMAX][BN];
  double zkr[SMAX][BN], zki[SMAX][BN], xi3[SMAX][BN];
  int dexp[SMAX][BN];
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void mma_f64(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Loads one K chunk of A (rows row0.., H columns js-1+kc*BK..) and B.
template <bool A16>
__device__ __forceinline__ void panel_load(const Ctx& c, const PanelArgs& p, PanelSmem& sm,
                                           int stage, int kc, int64_t row0, int rows_valid,
                                           int64_t col0) {
  const int tid = threadIdx.x;
  // A: BK columns x BM rows
  if (A16) {
#pragma unroll
    for (int it = 0; it < (BK * BM / 2) / PANEL_THREADS; it++) {
      int e = tid + it * PANEL_THREADS;  // 16-byte chunk index
      int kk = e / (BM / 2);
      int m2 = (e % (BM / 2)) * 2;
      int kglob = kc * BK + kk;
      bool valid = kglob < p.k && m2 < rows_valid;
      const double* src = c.H + (p.js - 1 + (valid ? kglob : 0)) * c.ldh + row0 + (valid ? m2 : 0);
      cp_async16(&sm.u.pipe.A[stage][kk][m2], src, valid);
    }
  } else {
#pragma unroll
    for (int it = 0; it < (BK * BM) / PANEL_THREADS; it++) {
      int e = tid + it * PANEL_THREADS;
      int kk = e / BM;
      int m = e % BM;
      int kglob = kc * BK + kk;
      bool valid = kglob < p.k && m < rows_valid;
      const double* src = c.H + (p.js - 1 + (valid ? kglob : 0)) * c.ldh + row0 + (valid ? m : 0);
      cp_async8(&sm.u.pipe.A[stage][kk][m], src, valid);
    }
  }
  // B: 2*BN accumulator columns x BK
#pragma unroll
  for (int it = 0; it < (2 * BN * BK / 2) / PANEL_THREADS; it++) {
    int e = tid + it * PANEL_THREADS;
    int nn = e / (BK / 2);
    int k2 = (e % (BK / 2)) * 2;
    const double* src = c.Bop + (2 * col0 + nn) * KP + kc * BK + k2;
    cp_async16(&sm.u.pipe.B[stage][nn][k2], src, true);
  }
}

// Column bookkeeping for a data column of this CTA.
struct ColInfo {
  bool valid, cplx, im;
  int64_t col, partner, q;
};
__device__ __forceinline__ ColInfo col_info(const Ctx& c, int64_t col) {
  ColInfo ci;
  ci.col = col;
  ci.valid = col < c.ncol;
  ci.cplx = col < 2 * c.mc;
  ci.im = ci.cplx && (col & 1);
  ci.partner = ci.cplx ? (col ^ 1) : col;
  ci.q = ci.cplx ? col / 2 : c.mc + (col - 2 * c.mc);
  return ci;
}

template <bool A16>
__global__ void __launch_bounds__(PANEL_THREADS, 2) k_panel(Ctx c, PanelArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PanelSmem& sm = *reinterpret_cast<PanelSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int S = p.S;
  const int tile0 = blockIdx.y * S;                  // first tile row of this CTA
  const int ntiles = min(S, p.jt - tile0);           // tile rows here (all above jt)
  const int64_t row0 = (int64_t)tile0 * c.b_r;
  const int rows_valid = ntiles * c.b_r;
  const int64_t col0 = (int64_t)blockIdx.x * BN;
  const int nk = (p.k + BK - 1) / BK;
  const int jt = p.jt;
  const double omega = c.omega;
  const bool robust = c.robust;

  // start the pipeline
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nk) panel_load<A16>(c, p, sm, s, s, row0, rows_valid, col0);
    cp_commit();
  }

  // ---------------- prologue: update steps 1 and 2 guards ----------------
  // thread -> (data column cl = tid / 8, row part rp = tid % 8: rows rp + 8*j)
  const int cl = tid >> 3, rp = tid & 7;
  const ColInfo ci = col_info(c, col0 + cl);
  for (int e = tid; e < 2 * SMAX * BN; e += PANEL_THREADS) (&sm.red[0][0][0])[e] = 0ULL;
  __syncthreads();
  if (ci.valid) {
    // step-1 bmax (update_rupdate :214-217 / cupdate :609-613)
    double lm = 0.0;
    int seg = -1;
    for (int r = rp; r < rows_valid; r += 8) {
      int sg = r / c.b_r;
      if (sg != seg) {
        if (seg >= 0) atomicMax(&sm.red[0][seg][cl], dkey(lm));
        seg = sg;
        lm = 0.0;
      }
      double xv = c.X[ci.col * c.ldx + row0 + r];
      double q = ci.cplx ? ghypot(c.X[(ci.col & ~1LL) * c.ldx + row0 + r],
                                  c.X[(ci.col | 1LL) * c.ldx + row0 + r])
                         : fabs(xv);
      if (q > lm) lm = q;
    }
    if (seg >= 0) atomicMax(&sm.red[0][seg][cl], dkey(lm));
  }
  __syncthreads();
  // per (segment, column) step-1 scalars
  for (int e = tid; e < S * BN; e += PANEL_THREADS) {
    int sg = e / BN, cc = e % BN;
    ColInfo cj = col_info(c, col0 + cc);
    if (!cj.valid || sg >= ntiles) continue;
    int it = tile0 + sg;
    const StepScalars st = c.SS[cj.q];
    const int ae = c.E[(int64_t)jt * c.ms + cj.q];
    const int be = c.E[(int64_t)it * c.ms + cj.q];
    const bool shifted = it == jt - 1;
    double fbv = 1.0, fxv = 1.0, rre = st.rho_re, rim = st.rho_im;
    int d = 0;
    if (robust) {
      const int g = ae < be ? ae : be;
      const double bmax = dval(sm.red[0][sg][cc]);
      const double alam = shifted ? (cj.cplx ? ghypot(c.lam_re[cj.q], c.lam_im[cj.q])
                                             : fabs(c.lam_re[cj.q]))
                                  : 0.0;
      const double hm0 = c.HM0[(int64_t)jt * c.N + it];
      const double arho = cj.cplx ? ghypot(rre, rim) : fabs(rre);
      const int xe = protect_update_e(p2(g - be) * bmax, hm0 + alam, arho, omega);
      d = xe + g;
      fbv = p2(d - be);
      fxv = p2(d - ae);
      if (fxv != 1.0) {
        rre = fxv * rre;
        rim = fxv * rim;
      }
    }
    sm.fb[sg][cc] = fbv;
    sm.fx[sg][cc] = fxv;
    sm.rr[sg][cc] = rre;
    sm.ri[sg][cc] = rim;
    sm.dexp[sg][cc] = d;
  }
  __syncthreads();
  // step-1 application and the step-2 bmax (:224-231, :264-267)
  if (ci.valid && robust) {
    double lm = 0.0;
    int seg = -1;
    for (int r = rp; r < rows_valid; r += 8) {
      int sg = r / c.b_r;
      if (sg != seg) {
        if (seg >= 0) atomicMax(&sm.red[1][seg][cl], dkey(lm));
        seg = sg;
        lm = 0.0;
      }
      const int64_t grow = row0 + r;
      const double h0 = c.H[(p.js - 1) * c.ldh + grow];
      const bool last = ((r + 1) % c.b_r == 0) && (tile0 + sg == jt - 1);
      const double fbv = sm.fb[sg][cl];
      double q;
      if (ci.cplx) {
        const int64_t cr_ = ci.col & ~1LL;
        double xr = c.X[cr_ * c.ldx + grow], xi = c.X[(cr_ + 1) * c.ldx + grow];
        if (fbv != 1.0) {
          xr *= fbv;
          xi *= fbv;
        }
        const double rre = sm.rr[sg][cl], rim = sm.ri[sg][cl];
        xr += rre * h0;
        xi += rim * h0;
        if (last) {
          const double lr = c.lam_re[ci.q], li = c.lam_im[ci.q];
          xr -= lr * rre - li * rim;
          xi -= lr * rim + li * rre;
        }
        q = ghypot(xr, xi);
      } else {
        double xv = c.X[ci.col * c.ldx + grow];
        if (fbv != 1.0) xv *= fbv;
        const double rho = sm.rr[sg][cl];
        xv += rho * h0;
        if (last) xv -= c.lam_re[ci.q] * rho;
        q = fabs(xv);
      }
      if (q > lm) lm = q;
    }
    if (seg >= 0) atomicMax(&sm.red[1][seg][cl], dkey(lm));
  }
  __syncthreads();
  for (int e = tid; e < S * BN; e += PANEL_THREADS) {
    int sg = e / BN, cc = e % BN;
    ColInfo cj = col_info(c, col0 + cc);
    if (!cj.valid || sg >= ntiles) continue;
    int it = tile0 + sg;
    const StepScalars st = c.SS[cj.q];
    const double fxv = sm.fx[sg][cc];
    double zr = st.zk_re, zi = st.zk_im;
    if (fxv != 1.0) {
      zr *= fxv;
      zi *= fxv;
    }
    double x2 = 1.0;
    if (robust && p.k > 1) {
      const double zmax = fxv != 1.0 ? fxv * st.zmax : st.zmax;
      const int xe = protect_update_e(dval(sm.red[1][sg][cc]), c.RS[(int64_t)jt * c.N + it], zmax,
                                      omega);
      if (xe < 0) {
        x2 = p2(xe);
        sm.dexp[sg][cc] += xe;
        zr *= x2;
        zi *= x2;
      }
    }
    sm.xi2[sg][cc] = x2;
    sm.zkr[sg][cc] = zr;
    sm.zki[sg][cc] = zi;
  }
  // (the __syncthreads of the main loop orders these before the epilogue)

  // ---------------- main loop: acc = A * [W | Zs] on DMMA ----------------
  const int wm = warp & 3, wn = warp >> 2;  // 4 x 2 warps, warp tile 32 rows x 32 acc cols
  const int g = lane >> 2, t4 = lane & 3;
  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int e = 0; e < 4; e++) acc[i][j][e] = 0.0;

  for (int kc = 0; kc < nk; kc++) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = kc + STAGES - 1;
      if (nxt < nk) panel_load<A16>(c, p, sm, nxt % STAGES, nxt, row0, rows_valid, col0);
      cp_commit();
    }
    const int st = kc % STAGES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[2][2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 2; mi++) {
        int r = wm * 32 + mi * 16 + g;
        af[mi][0] = sm.u.pipe.A[st][kk + t4][r];
        af[mi][1] = sm.u.pipe.A[st][kk + t4][r + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ni++) bf[ni] = sm.u.pipe.B[st][wn * 32 + ni * 8 + g][kk + t4];
#pragma unroll
      for (int mi = 0; mi < 2; mi++)
#pragma unroll
        for (int ni = 0; ni < 4; ni++) mma_f64(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  // stage accumulators: C[acc col][row]
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++) {
      int r = wm * 32 + mi * 16 + g;
      int cc = wn * 32 + ni * 8 + 2 * t4;
      sm.u.C[cc][r] = acc[mi][ni][0];
      sm.u.C[cc + 1][r] = acc[mi][ni][1];
      sm.u.C[cc][r + 8] = acc[mi][ni][2];
      sm.u.C[cc + 1][r + 8] = acc[mi][ni][3];
    }
  for (int e = tid; e < 2 * SMAX * BN; e += PANEL_THREADS) (&sm.red[0][0][0])[e] = 0ULL;
  __syncthreads();

  // ---------------- epilogue ----------------
  // X'' = xi2 * X' - (fx xi2) (A Z);  guards of step 3 need max|X''| and max|Cr_old|.
  constexpr int RPT = BM / 8;  // rows per thread
  double xo[RPT];  // X'' (own part) kept across the step-3 reduction
  if (ci.valid) {
    double lmb = 0.0, lmr = 0.0;
    int seg = -1;
#pragma unroll
    for (int j = 0; j < RPT; j++) {
      int r = rp + 8 * j;
      xo[j] = 0.0;
      if (r >= rows_valid) continue;
      int sg = r / c.b_r;
      if (sg != seg) {
        if (seg >= 0) {
          atomicMax(&sm.red[0][seg][cl], dkey(lmb));
          atomicMax(&sm.red[1][seg][cl], dkey(lmr));
        }
        seg = sg;
        lmb = lmr = 0.0;
      }
      const int64_t grow = row0 + r;
      const double h0 = c.H[(p.js - 1) * c.ldh + grow];
      const bool last = ((r + 1) % c.b_r == 0) && (tile0 + sg == jt - 1);
      const double fbv = sm.fb[sg][cl], x2 = sm.xi2[sg][cl];
      const double pz = sm.fx[sg][cl] * x2;
      if (ci.cplx) {
        const int64_t cre_ = ci.col & ~1LL;
        const int cl_re = cl & ~1;
        double xr = c.X[cre_ * c.ldx + grow], xi = c.X[(cre_ + 1) * c.ldx + grow];
        if (fbv != 1.0) {
          xr *= fbv;
          xi *= fbv;
        }
        const double rre = sm.rr[sg][cl], rim = sm.ri[sg][cl];
        xr += rre * h0;
        xi += rim * h0;
        if (last) {
          const double lr = c.lam_re[ci.q], li = c.lam_im[ci.q];
          xr -= lr * rre - li * rim;
          xi -= lr * rim + li * rre;
        }
        if (x2 < 1.0) {
          xr *= x2;
          xi *= x2;
        }
        xr -= pz * sm.u.C[2 * cl_re + 1][r];
        xi -= pz * sm.u.C[2 * (cl_re + 1) + 1][r];
        const double cr_r = c.Cr[cre_ * c.ldx + grow], cr_i = c.Cr[(cre_ + 1) * c.ldx + grow];
        xo[j] = ci.im ? xi : xr;
        double qb = ghypot(xr, xi), qr = ghypot(cr_r, cr_i);
        if (qb > lmb) lmb = qb;
        if (qr > lmr) lmr = qr;
      } else {
        double xv = c.X[ci.col * c.ldx + grow];
        if (fbv != 1.0) xv *= fbv;
        const double rho = sm.rr[sg][cl];
        xv += rho * h0;
        if (last) xv -= c.lam_re[ci.q] * rho;
        if (x2 < 1.0) xv *= x2;
        xv -= pz * sm.u.C[2 * cl + 1][r];
        const double crv = c.Cr[ci.col * c.ldx + grow];
        xo[j] = xv;
        if (fabs(xv) > lmb) lmb = fabs(xv);
        if (fabs(crv) > lmr) lmr = fabs(crv);
      }
    }
    if (seg >= 0) {
      atomicMax(&sm.red[0][seg][cl], dkey(lmb));
      atomicMax(&sm.red[1][seg][cl], dkey(lmr));
    }
  }
  __syncthreads();
  // step 3 guard (:287-301) and the new beta
  for (int e = tid; e < S * BN; e += PANEL_THREADS) {
    int sg = e / BN, cc = e % BN;
    ColInfo cj = col_info(c, col0 + cc);
    if (!cj.valid || sg >= ntiles) continue;
    double zr = sm.zkr[sg][cc], zi = sm.zki[sg][cc];
    double x3 = 1.0;
    if (robust) {
      const double az = cj.cplx ? ghypot(zr, zi) : fabs(zr);
      const int xe = protect_update_e(dval(sm.red[0][sg][cc]), dval(sm.red[1][sg][cc]), az, omega);
      if (xe < 0) {
        x3 = p2(xe);
        sm.dexp[sg][cc] += xe;
        zr *= x3;
        zi *= x3;
      }
      if (!cj.im) c.E[(int64_t)(tile0 + sg) * c.ms + cj.q] = sm.dexp[sg][cc];
    }
    sm.xi3[sg][cc] = x3;
    sm.zkr[sg][cc] = zr;
    sm.zki[sg][cc] = zi;
  }
  __syncthreads();
  if (ci.valid) {
    const StepScalars st = c.SS[ci.q];
#pragma unroll
    for (int j = 0; j < RPT; j++) {
      int r = rp + 8 * j;
      if (r >= rows_valid) continue;
      int sg = r / c.b_r;
      const int64_t grow = row0 + r;
      const double x3 = sm.xi3[sg][cl];
      const double zr = sm.zkr[sg][cl], zi = sm.zki[sg][cl];
      double xv = xo[j];
      if (x3 < 1.0) xv *= x3;
      double crn;
      const bool lastrow = (grow == p.js - 1);
      if (ci.cplx) {
        const int64_t cre_ = ci.col & ~1LL;
        const double crr = c.Cr[cre_ * c.ldx + grow], cri = c.Cr[(cre_ + 1) * c.ldx + grow];
        if (ci.im)
          xv -= crr * zi + cri * zr;
        else
          xv -= crr * zr - cri * zi;
        crn = sm.u.C[2 * cl][r] + st.P * (ci.im ? cri : crr);
        if (lastrow) {
          const double lr = c.lam_re[ci.q], li = c.lam_im[ci.q];
          crn -= ci.im ? (st.c0_re * li + st.c0_im * lr) : (st.c0_re * lr - st.c0_im * li);
        }
      } else {
        const double crv = c.Cr[ci.col * c.ldx + grow];
        xv -= crv * zr;
        crn = sm.u.C[2 * cl][r] + st.P * crv;
        if (lastrow) crn -= st.c0_re * c.lam_re[ci.q];
      }
      c.X[ci.col * c.ldx + grow] = xv;
      c.Cr[ci.col * c.ldx + grow] = crn;
    }
  }
}

// ---------------------------------------------------------------------------
// k_backtransform: rbacktransform / crbacktransform, one thread per shift
// ---------------------------------------------------------------------------
__global__ void k_backtransform(Ctx c, int32_t* alpha_exp, double* norms, double* log2norm) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= c.ms) return;
  bool cplx;
  int64_t col;
  col_of_shift(c, q, cplx, col);
  const int64_t n = c.n;
  double* xr = c.X + col * c.ldx;
  double* xi = cplx ? c.X + (col + 1) * c.ldx : nullptr;
  const double* cr = c.c_re + q * c.ldc;
  const double* ci = cplx ? c.c_im + q * c.ldc : nullptr;
  const double* ss = c.s + q * c.ldc;
  if (c.fail[q] != 0) {
    norms[q] = __longlong_as_double(0x7ff8000000000000LL);
    log2norm[q] = norms[q];
    alpha_exp[q] = 0;
    return;
  }
  if (!c.robust) {  // backtransform / cbacktransform (:314-323, :739-756)
    norms[q] = __longlong_as_double(0x7ff8000000000000LL);
    log2norm[q] = norms[q];
    alpha_exp[q] = 0;
  } else {
    int amin = c.E[q];
    for (int t = 1; t < c.N; t++) {
      int e = c.E[(int64_t)t * c.ms + q];
      if (e < amin) amin = e;
    }
    for (int t = 0; t < c.N; t++) {
      double f = p2(amin - c.E[(int64_t)t * c.ms + q]);
      if (f != 1.0) {
        int64_t s0 = (int64_t)t * c.b_r, s1 = s0 + c.b_r < n ? s0 + c.b_r : n;
        for (int64_t i = s0; i < s1; i++) {
          xr[i] *= f;
          if (cplx) xi[i] *= f;
        }
      }
    }
    double xmax = 0.0;
    for (int64_t i = 0; i < n; i++) {
      double qv = cplx ? ghypot(xr[i], xi[i]) : fabs(xr[i]);
      if (qv > xmax) xmax = qv;
    }
    if (xmax == 0.0) {
      norms[q] = 0.0;
      log2norm[q] = -__longlong_as_double(0x7ff0000000000000LL);
      alpha_exp[q] = amin;
      return;
    }
    double tsum = 0.0;
    for (int64_t i = 0; i < n; i++) {
      if (cplx) {
        double qr = xr[i] / xmax, qi = xi[i] / xmax;
        tsum += qr * qr + qi * qi;
      } else {
        double qv = xr[i] / xmax;
        tsum += qv * qv;
      }
    }
    double rt = sqrt(tsum);
    norms[q] = ldexp(xmax, -amin) * rt;
    log2norm[q] = log2(xmax) + log2(rt) - (double)amin;
    alpha_exp[q] = amin;
    if (c.mode == 1) {
      for (int64_t i = 0; i < n; i++) {
        xr[i] /= xmax;
        if (cplx) xi[i] /= xmax;
      }
      for (int64_t i = 0; i < n; i++) {
        xr[i] /= rt;
        if (cplx) xi[i] /= rt;
      }
    } else {
      double qq = c.omega / xmax;
      if (rt > qq) {
        int e = pow2floor_e(qq / rt);
        double f = p2(e);
        for (int64_t i = 0; i < n; i++) {
          xr[i] *= f;
          if (cplx) xi[i] *= f;
        }
        alpha_exp[q] = amin + e;
      }
    }
  }
  // rotation sweep
  if (cplx) {
    double t1r = xr[0], t1i = xi[0];
    for (int64_t i = 1; i < n; i++) {
      double c_r = cr[i], c_i = ci[i], sv = ss[i];
      double t2r = xr[i], t2i = xi[i];
      xr[i - 1] = (c_r * t1r - c_i * t1i) - sv * t2r;
      xi[i - 1] = (c_r * t1i + c_i * t1r) - sv * t2i;
      double nr = sv * t1r + (c_r * t2r + c_i * t2i);
      double ni = sv * t1i + (c_r * t2i - c_i * t2r);
      t1r = nr;
      t1i = ni;
    }
    xr[n - 1] = t1r;
    xi[n - 1] = t1i;
  } else {
    double t1 = xr[0];
    for (int64_t i = 1; i < n; i++) {
      double t2 = xr[i];
      xr[i - 1] = cr[i] * t1 - ss[i] * t2;
      t1 = cr[i] * t2 + ss[i] * t1;
    }
    xr[n - 1] = t1;
  }
}

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
  size_t cr, bop, ss, hm0, rs, nfail, total;
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
            "attr diag"))
      return HSRQ_ERR_CUDA;
    if (!ck(cudaFuncSetAttribute(k_panel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem),
            "attr panel"))
      return HSRQ_ERR_CUDA;
    if (!ck(cudaFuncSetAttribute(k_panel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)panel_smem),
            "attr panel8"))
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
      dim3 gp((unsigned)(c.ncol_pad / BN), (unsigned)((jt + S - 1) / S));
      if (a16)
        k_panel<true><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p);
      else
        k_panel<false><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p);
      g_launches++;
    }
    if (g_timing) cudaEventRecord(ev[3 + 2 * jt], stream);
  }
  k_backtransform<<<(unsigned)((c.ms + 127) / 128), 128, 0, stream>>>(c, alpha_exp, norms, log2norm);
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
