// hsrq_device.cuh -- scalar device arithmetic shared by the kernels.
//
// Everything here is written so that, compiled with -fmad=false (no FMA
// contraction, matching numba's LLVM output, _kernels/numba_backend.py:1-7),
// it reproduces the reference's scalar arithmetic bit for bit:
//   * ghypot: glibc 2.39's hypot (the libm routine numba's math.hypot binds,
//     numba/cpython/mathimpl.py hypot_float_impl), i.e. the non-FMA kernel of
//     sysdeps/ieee754/dbl-64/e_hypot.c (Borges' algorithm).  CUDA's own hypot
//     differs by an ulp on ~0.03 % of inputs, which would perturb rotations.
//   * pow2floor / protect_update: numba_backend.py:37-67, with the result
//     carried as a log2 exponent.
//   * complex ops: numba's lowering ((a+bi)(c+di) = (ac-bd)+(ad+bc)i, reals
//     promoted to (x, 0), CPython's _Py_c_quot division, abs = hypot).
#pragma once
#include <cstdint>

namespace hsrq {

constexpr int EXP_ZERO = -1075;  // exponent of a scale that halved to 0

// Schedule fuzzing (race check; compute-sanitizer is not available on the GPU
// pool).  The diagnostics build `-DHSRQ_FUZZ` (libhsrq_b200_fuzz.so,
// tools/race_fuzz.py) makes a pseudo-random subset of threads sleep up to
// ~2 us right after every warp / pair / CTA barrier of the diagonal sweeps,
// the panel and k_scalars, so a shared-memory value read without the barrier
// that orders it behind its write (or overwritten before its last reader is
// done) changes the result, which the fuzz run then compares bitwise with
// the production build.  The production build compiles these to plain barriers.
#ifdef HSRQ_FUZZ
// bit per source file (HSRQ_FUZZ_FILE at the point of use): 1 hsrq_diag.cuh,
// 2 hsrq_diag_ws.cuh, 4 hsrq_panel.cuh, 8 hsrq_henry.cuh; HSRQ_FUZZ_MASK
// (environment, read at the first solve) selects which files are fuzzed
__device__ unsigned g_fuzz_mask = 0xffffffffu;
__device__ __forceinline__ void fuzz_delay(unsigned site) {
  if (!(g_fuzz_mask & (site >> 16))) return;
  unsigned h = (blockIdx.x * 0x9E3779B1u) ^ (threadIdx.x * 0x85EBCA77u) ^ (site * 0xC2B2AE3Du) ^
               (unsigned)clock();
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep((h >> 16) & 2047u);
}
#define HSRQ_SYNCWARP() (__syncwarp(), ::hsrq::fuzz_delay(__LINE__ | (HSRQ_FUZZ_FILE << 16)))
#define HSRQ_SYNCTHREADS() (__syncthreads(), ::hsrq::fuzz_delay(__LINE__ | (HSRQ_FUZZ_FILE << 16)))
#else
#define HSRQ_SYNCWARP() __syncwarp()
#define HSRQ_SYNCTHREADS() __syncthreads()
#endif

struct cplx {
  double re, im;
};

__device__ __forceinline__ cplx mk(double re, double im) { return cplx{re, im}; }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  double ac = a.re * b.re, bd = a.im * b.im, ad = a.re * b.im, bc = a.im * b.re;
  return cplx{ac - bd, ad + bc};
}
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }

// Exact 2^e for e in [-1075, 1023] (0 below -1074).
__device__ __forceinline__ double p2(int e) {
  if (e >= -1022) return __longlong_as_double((long long)(e + 1023) << 52);
  if (e >= -1074) return __longlong_as_double(1LL << (e + 1074));
  return 0.0;
}

// glibc 2.39 e_hypot.c kernel (no __FP_FAST_FMA on x86_64).
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

__device__ __forceinline__ double ghypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000LL);
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay / 0x1p-54) return ax + ay;
    return hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
  }
  if (ay <= ax * 0x1p-54) return ax + ay;
  return hypot_kernel(ax, ay);
}

__device__ __forceinline__ double cabs_(cplx a) { return ghypot(a.re, a.im); }

// CPython _Py_c_quot as lowered by numba (numba/cpython/numbers.py).
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  double areal = a.re, aimag = a.im, breal = b.re, bimag = b.im;
  if (fabs(breal) >= fabs(bimag)) {
    if (breal == 0.0) return cplx{__longlong_as_double(0x7ff8000000000000LL),
                                  __longlong_as_double(0x7ff8000000000000LL)};
    double ratio = bimag / breal;
    double denom = breal + bimag * ratio;
    return cplx{(areal + aimag * ratio) / denom, (aimag - areal * ratio) / denom};
  }
  double ratio = breal / bimag;
  double denom = breal * ratio + bimag;
  return cplx{(areal * ratio + aimag) / denom, (aimag * ratio - areal) / denom};
}

// floor(log2(x)) for positive normal x; -2000 for 0 / subnormal, 2000 for inf/NaN.
__device__ __forceinline__ int ilogb_pos(double x) {
  const int b = (int)((__double_as_longlong(x) >> 52) & 0x7ff);
  if (b == 0) return -2000;
  if (b == 0x7ff) return 2000;
  return b - 1023;
}

// pow2floor (numba_backend.py:37-44) as an exponent.
__device__ __forceinline__ int pow2floor_e(double x) {
  if (x <= 0.0 || x != x) return -1074;
  if (isinf(x)) return 0;
  int e;
  frexp(x, &e);
  return e - 1;
}

// protect_update (numba_backend.py:47-67); returns log2(xi): 0 when xi == 1,
// EXP_ZERO when the halving loop reached 0.
__device__ __forceinline__ int protect_update_e(double bnorm, double hnorm, double xnorm,
                                             double omega) {
  double cand;
  if (xnorm <= 1.0) {
    if (bnorm + hnorm * xnorm <= omega) return 0;
    cand = (omega * 0.5) / (bnorm * 0.5 + (hnorm * xnorm) * 0.5);
  } else {
    if (bnorm <= omega && hnorm <= (omega - bnorm) / xnorm) return 0;
    double u = bnorm / xnorm;
    cand = ((omega * 0.5) / (u * 0.5 + hnorm * 0.5)) / xnorm;
  }
  if (!(cand > 0.0)) cand = 0x1p-1074;
  if (cand > 1.0) cand = 1.0;
  int e = pow2floor_e(cand);
  double xi = p2(e);
  for (int it = 0; it < 200; it++) {
    if (xi * bnorm + hnorm * (xi * xnorm) <= omega) break;
    xi *= 0.5;
    e -= 1;
  }
  if (xi == 0.0) e = EXP_ZERO;
  return e;
}

// protect_update_e at two argument pairs with the same xnorm (the guard-2
// interval ends), evaluated side by side so the two division chains and
// halving loops overlap; each result equals protect_update_e's.
__device__ __forceinline__ void protect_update_e2(double bn1, double hn1, double bn2, double hn2,
                                                  double xnorm, double omega, int& r1, int& r2) {
  bool z1, z2;
  double c1, c2;
  if (xnorm <= 1.0) {
    z1 = bn1 + hn1 * xnorm <= omega;
    z2 = bn2 + hn2 * xnorm <= omega;
    c1 = (omega * 0.5) / (bn1 * 0.5 + (hn1 * xnorm) * 0.5);
    c2 = (omega * 0.5) / (bn2 * 0.5 + (hn2 * xnorm) * 0.5);
  } else {
    z1 = bn1 <= omega && hn1 <= (omega - bn1) / xnorm;
    z2 = bn2 <= omega && hn2 <= (omega - bn2) / xnorm;
    const double u1 = bn1 / xnorm, u2 = bn2 / xnorm;
    c1 = ((omega * 0.5) / (u1 * 0.5 + hn1 * 0.5)) / xnorm;
    c2 = ((omega * 0.5) / (u2 * 0.5 + hn2 * 0.5)) / xnorm;
  }
  if (!(c1 > 0.0)) c1 = 0x1p-1074;
  if (c1 > 1.0) c1 = 1.0;
  if (!(c2 > 0.0)) c2 = 0x1p-1074;
  if (c2 > 1.0) c2 = 1.0;
  int e1 = pow2floor_e(c1), e2 = pow2floor_e(c2);
  double x1 = p2(e1), x2 = p2(e2);
  bool d1 = z1, d2 = z2;
  for (int it = 0; it < 200 && !(d1 && d2); it++) {
    if (!d1) {
      if (x1 * bn1 + hn1 * (x1 * xnorm) <= omega) {
        d1 = true;
      } else {
        x1 *= 0.5;
        e1 -= 1;
      }
    }
    if (!d2) {
      if (x2 * bn2 + hn2 * (x2 * xnorm) <= omega) {
        d2 = true;
      } else {
        x2 *= 0.5;
        e2 -= 1;
      }
    }
  }
  r1 = z1 ? 0 : (x1 == 0.0 ? EXP_ZERO : e1);
  r2 = z2 ? 0 : (x2 == 0.0 ? EXP_ZERO : e2);
}

// Cheap test "protect_update would return 1" from upper bounds of the norms;
// protect_update is monotone in each argument (overflow.py:50-57), so a pass
// here is exact.  A fail means "evaluate the exact norms".
__device__ __forceinline__ bool protect_update_is_one(double bnorm, double hnorm, double xnorm,
                                                      double omega) {
  if (xnorm <= 1.0) return bnorm + hnorm * xnorm <= omega;
  return bnorm <= omega && hnorm <= (omega - bnorm) / xnorm;
}

// Max of non-negative doubles across a warp (NaN never wins, matching the
// reference's `if abs(v) > vmax` scans).
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Non-negative double <-> ordered uint64 for atomicMax reductions.
__device__ __forceinline__ unsigned long long dkey(double v) {
  return (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ double dval(unsigned long long k) { return __longlong_as_double((long long)k); }


// ---------------------------------------------------------------------------
// Stewart compact rotation storage (givens.py:90-198): one real per real
// rotation, two per complex rotation.  The smaller component is stored, the
// window offset (0/2/4/6) records which one and the sign of the other.
// Expression for expression the reference's, so encode and decode are
// bit-identical to compact_encode / compact_decode (IEEE add/sqrt/div).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double compact_encode(double c, double s) {
  if (fabs(s) <= fabs(c)) {
    const double base = c >= 0.0 ? 0.0 : 2.0;
    return s != 0.0 ? copysign(fabs(s) + base, s) : base;
  }
  const double base = s >= 0.0 ? 4.0 : 6.0;
  return c != 0.0 ? copysign(fabs(c) + base, c) : base;
}

__device__ __forceinline__ double pmax0(double u) { return u > 0.0 ? u : 0.0; }  // max(0.0, u)

__device__ __forceinline__ void compact_decode(double t, double& c, double& s) {
  const double at = fabs(t);
  if (at <= 1.0) {
    s = t;
    c = __dsqrt_rn(pmax0(1.0 - s * s));
  } else if (at <= 3.0) {
    s = at != 2.0 ? copysign(at - 2.0, t) : 0.0;
    c = -__dsqrt_rn(pmax0(1.0 - s * s));
  } else if (at <= 5.0) {
    c = at != 4.0 ? copysign(at - 4.0, t) : 0.0;
    s = __dsqrt_rn(pmax0(1.0 - c * c));
  } else {
    c = at != 6.0 ? copysign(at - 6.0, t) : 0.0;
    s = -__dsqrt_rn(pmax0(1.0 - c * c));
  }
}

// compact_encode_complex: (|c|, s) and the unit direction of c.
__device__ __forceinline__ void compact_encode_cplx(double cr, double ci, double s, double& t1,
                                                    double& t2) {
  const double ac = ghypot(cr, ci);
  t1 = compact_encode(ac, s);
  t2 = ac == 0.0 ? compact_encode(1.0, 0.0) : compact_encode(cr / ac, ci / ac);
}

__device__ __forceinline__ void compact_decode_cplx(double t1, double t2, double& cr, double& ci,
                                                    double& s) {
  double ac, dc, ds;
  compact_decode(t1, ac, s);
  compact_decode(t2, dc, ds);
  cr = ac * dc;
  ci = ac * ds;
}

}  // namespace hsrq
