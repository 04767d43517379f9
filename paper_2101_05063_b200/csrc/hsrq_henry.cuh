// hsrq_henry.cuh -- Henry's single-sweep RQ solve (henry_solve_real /
// henry_solve_complex, _kernels/numba_backend.py:830-923, driven by
// henry_rq_solve, reference.py:21-60): the level-2 baseline the tiled
// algorithm of the paper is measured against (included by hsrq_kernels.cu).
//
// One CTA per shift (persistent over the shift list).  Row i of the shift's
// working vectors v and x is owned by thread i % HENRY_THREADS for the whole
// sweep -- as a regular row (i < kp - 1) and as the shifted row kp - 1 -- so
// the only cross-thread value per step is the pivot pair (v[kp], x[kp]),
// handed over through shared memory with one __syncthreads.  Every thread
// evaluates the step's rotation redundantly from that pair, so the step
// scalars need no second barrier.  v and x live in global memory (L2: the
// launch keeps the resident working set under the L2 size, and CTAs that
// start together walk H's columns in near lock step, so a column of H is
// read from HBM once per wave).  The row arithmetic is the reference's,
// expression for expression (-fmad=false), so x is bit-identical.
//
// After the sweep warp 0 runs the ordered rotation sweep (backtransform,
// :314-323, or the complex loop inside henry_solve_complex :915-923): 32
// rows are loaded coalesced, their values broadcast lane by lane, and every
// lane runs the same scalar recurrence; lane j keeps output row base + j.

#undef HSRQ_FUZZ_FILE
#define HSRQ_FUZZ_FILE 8u
constexpr int HENRY_THREADS = 512;

struct HenryArgs {
  const double* H;
  int64_t ldh, n, m;
  const double* lam;   // real: m; complex: m (re, im) pairs
  double* X;           // real: n x m (ldx); complex: n x m double2 (ldx in complex elements)
  int64_t ldx;
  double* V;           // working v: n x m (double or double2), ld n
  double* C;           // rotations c: n x m (double or double2), ld n
  double* S;           // rotations s: n x m, ld n
  int64_t* status;     // per shift packed status (kind << 42 | q << 21 | row), 0 ok
  unsigned long long* first;  // max over shifts of henry_key (first failure)
};

// Reference failure order: kp descending (row 0 = the final pivot loop), then
// the shift index ascending (numba_backend.py:845-873).
__device__ __forceinline__ unsigned long long henry_key(int kind, int64_t q, int64_t row) {
  return ((unsigned long long)row << 34) | ((0xFFFFFFFFull - (unsigned long long)q) << 2) |
         (unsigned long long)kind;
}

__device__ __forceinline__ void henry_fail(const HenryArgs& a, int kind, int64_t q, int64_t row) {
  a.status[q] = ((int64_t)kind << 42) | (q << 21) | row;
  atomicMax(a.first, henry_key(kind, q, row));
}

__global__ void __launch_bounds__(HENRY_THREADS) k_henry_real(HenryArgs a) {
  __shared__ double piv[2][2];  // [parity][v, x]
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31;
  const int64_t n = a.n;
  for (int64_t q = blockIdx.x; q < a.m; q += gridDim.x) {
    const double lam = a.lam[q];
    double* x = a.X + q * a.ldx;
    double* v = a.V + q * n;
    double* cc = a.C + q * n;
    double* cs = a.S + q * n;
    const double* hl = a.H + (n - 1) * a.ldh;
    for (int64_t i = tid; i < n - 1; i += T) v[i] = hl[i];
    if (tid == (int)((n - 1) % T)) {
      piv[0][0] = hl[n - 1] - lam;  // v[n-1] -= lam
      piv[0][1] = x[n - 1];
    }
    if (tid == 0) {
      cc[0] = 1.0;
      cs[0] = 0.0;
      a.status[q] = 0;
    }
    HSRQ_SYNCTHREADS();
    int p = 0;
    bool ok = true;
    for (int64_t kp = n - 1; kp >= 1; --kp) {
      const double vk = piv[p][0];
      double xk = piv[p][1];
      const double* hc = a.H + (kp - 1) * a.ldh;
      const double av = hc[kp];
      const double r = ghypot(av, vk);
      if (r == 0.0) {
        if (tid == 0) henry_fail(a, HSRQ_KIND_DEGENERATE, q, kp);
        ok = false;
        break;
      }
      const double c = vk / r, s = -av / r;
      const double phi = vk * c - av * s;
      if (phi == 0.0) {
        if (tid == 0) henry_fail(a, HSRQ_KIND_SINGULAR, q, kp);
        ok = false;
        break;
      }
      xk /= phi;
      if (tid == (int)(kp % T)) {
        x[kp] = xk;
        cc[kp] = c;
        cs[kp] = s;
      }
      const double tau1 = s * xk, tau2 = c * xk;
      int64_t i = tid;
#pragma unroll 4
      for (; i < kp - 1; i += T) {
        const double hi = hc[i];
        const double vi = v[i];
        x[i] = (x[i] - tau2 * vi) + tau1 * hi;
        v[i] = c * hi + s * vi;
      }
      if (i == kp - 1) {  // this thread owns the shifted row kp - 1
        const double hdl = hc[kp - 1] - lam;
        const double vi = v[kp - 1];
        piv[p ^ 1][1] = (x[kp - 1] - tau2 * vi) + tau1 * hdl;
        piv[p ^ 1][0] = c * hdl + s * vi;
      }
      p ^= 1;
      HSRQ_SYNCTHREADS();
    }
    if (ok) {
      const double v0 = piv[p][0];
      if (v0 == 0.0) {
        if (tid == 0) henry_fail(a, HSRQ_KIND_SINGULAR, q, 0);
        ok = false;
      } else if (tid == 0) {
        x[0] = piv[p][1] / v0;
      }
    }
    HSRQ_SYNCTHREADS();
    if (ok && tid < 32) {  // backtransform (numba_backend.py:314-323)
      double t1 = x[0];
      for (int64_t base = 0; base < n - 1; base += 32) {
        const int64_t i = base + 1 + lane;
        double ci = 0.0, si = 0.0, xi = 0.0;
        if (i < n) {
          ci = cc[i];
          si = cs[i];
          xi = x[i];
        }
        double out = 0.0;
        const int cnt = (int)(n - 1 - base < 32 ? n - 1 - base : 32);
        for (int j = 0; j < cnt; ++j) {
          const double c = __shfl_sync(0xffffffffu, ci, j);
          const double s = __shfl_sync(0xffffffffu, si, j);
          const double t2 = __shfl_sync(0xffffffffu, xi, j);
          const double o = c * t1 - s * t2;
          t1 = c * t2 + s * t1;
          if (lane == j) out = o;
        }
        if (lane < cnt) x[base + lane] = out;
      }
      if (lane == 0) x[n - 1] = t1;
    }
    HSRQ_SYNCTHREADS();
  }
}

__global__ void __launch_bounds__(HENRY_THREADS) k_henry_cplx(HenryArgs a) {
  __shared__ double piv[2][4];  // [parity][v.re, v.im, x.re, x.im]
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31;
  const int64_t n = a.n;
  for (int64_t q = blockIdx.x; q < a.m; q += gridDim.x) {
    const cplx lam = mk(a.lam[2 * q], a.lam[2 * q + 1]);
    double2* x = reinterpret_cast<double2*>(a.X) + q * a.ldx;
    double2* v = reinterpret_cast<double2*>(a.V) + q * n;
    double2* cc = reinterpret_cast<double2*>(a.C) + q * n;
    double* cs = a.S + q * n;
    const double* hl = a.H + (n - 1) * a.ldh;
    for (int64_t i = tid; i < n - 1; i += T) v[i] = make_double2(hl[i], 0.0);
    if (tid == (int)((n - 1) % T)) {
      const cplx v0 = csub(mk(hl[n - 1], 0.0), lam);  // v[n-1] -= lam
      const double2 x0 = x[n - 1];
      piv[0][0] = v0.re;
      piv[0][1] = v0.im;
      piv[0][2] = x0.x;
      piv[0][3] = x0.y;
    }
    if (tid == 0) {
      cc[0] = make_double2(1.0, 0.0);
      cs[0] = 0.0;
      a.status[q] = 0;
    }
    HSRQ_SYNCTHREADS();
    int p = 0;
    bool ok = true;
    for (int64_t kp = n - 1; kp >= 1; --kp) {
      const cplx vk = mk(piv[p][0], piv[p][1]);
      cplx xk = mk(piv[p][2], piv[p][3]);
      const double* hc = a.H + (kp - 1) * a.ldh;
      const double av = hc[kp];
      const double r = ghypot(av, cabs_(vk));
      if (r == 0.0) {
        if (tid == 0) henry_fail(a, HSRQ_KIND_DEGENERATE, q, kp);
        ok = false;
        break;
      }
      const cplx c = cdiv(vk, mk(r, 0.0));
      const double s = -av / r;
      const cplx cj = mk(c.re, -c.im);
      const cplx phi = csub(cmul(cj, vk), mk(av * s, 0.0));
      if (phi.re == 0.0 && phi.im == 0.0) {
        if (tid == 0) henry_fail(a, HSRQ_KIND_SINGULAR, q, kp);
        ok = false;
        break;
      }
      xk = cdiv(xk, phi);
      if (tid == (int)(kp % T)) {
        x[kp] = make_double2(xk.re, xk.im);
        cc[kp] = make_double2(c.re, c.im);
        cs[kp] = s;
      }
      const cplx sc = mk(s, 0.0);
      const cplx tau1 = cmul(sc, xk), tau2 = cmul(cj, xk);
      int64_t i = tid;
#pragma unroll 2
      for (; i < kp - 1; i += T) {
        const cplx hi = mk(hc[i], 0.0);
        const double2 vv = v[i], xx = x[i];
        const cplx vi = mk(vv.x, vv.y);
        const cplx xn = cadd(csub(mk(xx.x, xx.y), cmul(tau2, vi)), cmul(tau1, hi));
        const cplx vn = cadd(cmul(c, hi), cmul(sc, vi));
        x[i] = make_double2(xn.re, xn.im);
        v[i] = make_double2(vn.re, vn.im);
      }
      if (i == kp - 1) {  // the shifted row kp - 1
        const cplx hdl = csub(mk(hc[kp - 1], 0.0), lam);
        const double2 vv = v[kp - 1], xx = x[kp - 1];
        const cplx vi = mk(vv.x, vv.y);
        const cplx xn = cadd(csub(mk(xx.x, xx.y), cmul(tau2, vi)), cmul(tau1, hdl));
        const cplx vn = cadd(cmul(c, hdl), cmul(sc, vi));
        piv[p ^ 1][0] = vn.re;
        piv[p ^ 1][1] = vn.im;
        piv[p ^ 1][2] = xn.re;
        piv[p ^ 1][3] = xn.im;
      }
      p ^= 1;
      HSRQ_SYNCTHREADS();
    }
    if (ok) {
      const cplx v0 = mk(piv[p][0], piv[p][1]);
      if (v0.re == 0.0 && v0.im == 0.0) {
        if (tid == 0) henry_fail(a, HSRQ_KIND_SINGULAR, q, 0);
        ok = false;
      } else if (tid == 0) {
        const cplx x0 = cdiv(mk(piv[p][2], piv[p][3]), v0);
        x[0] = make_double2(x0.re, x0.im);
      }
    }
    HSRQ_SYNCTHREADS();
    if (ok && tid < 32) {  // rotation sweep of henry_solve_complex (:915-923)
      const double2 x0 = x[0];
      cplx t1 = mk(x0.x, x0.y);
      for (int64_t base = 0; base < n - 1; base += 32) {
        const int64_t i = base + 1 + lane;
        double2 ci = make_double2(0.0, 0.0), xi = make_double2(0.0, 0.0);
        double si = 0.0;
        if (i < n) {
          ci = cc[i];
          si = cs[i];
          xi = x[i];
        }
        double2 out = make_double2(0.0, 0.0);
        const int cnt = (int)(n - 1 - base < 32 ? n - 1 - base : 32);
        for (int j = 0; j < cnt; ++j) {
          const cplx c = mk(__shfl_sync(0xffffffffu, ci.x, j), __shfl_sync(0xffffffffu, ci.y, j));
          const cplx s = mk(__shfl_sync(0xffffffffu, si, j), 0.0);
          const cplx t2 = mk(__shfl_sync(0xffffffffu, xi.x, j), __shfl_sync(0xffffffffu, xi.y, j));
          const cplx o = csub(cmul(c, t1), cmul(s, t2));
          t1 = cadd(cmul(s, t1), cmul(mk(c.re, -c.im), t2));
          if (lane == j) out = make_double2(o.re, o.im);
        }
        if (lane < cnt) x[base + lane] = out;
      }
      if (lane == 0) x[n - 1] = make_double2(t1.re, t1.im);
    }
    HSRQ_SYNCTHREADS();
  }
}

__global__ void k_henry_first(const unsigned long long* first, int64_t* out) {
  const unsigned long long k = *first;
  if (k == 0) {
    *out = 0;
    return;
  }
  const int64_t kind = (int64_t)(k & 3ull);
  const int64_t q = (int64_t)(0xFFFFFFFFull - ((k >> 2) & 0xFFFFFFFFull));
  const int64_t row = (int64_t)(k >> 34);
  *out = (kind << 42) + (q << 21) + row;  // _pack (numba_backend.py:33-34)
}
