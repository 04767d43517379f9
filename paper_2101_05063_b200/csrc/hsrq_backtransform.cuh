// hsrq_backtransform.cuh -- rbacktransform / crbacktransform
// (numba_backend.py:326-375, :759-822) and the unguarded backtransform
// (:314-323, :739-756); one warp per shift (included by hsrq_kernels.cu).
//
// Row chunks of 32 are loaded coalesced (lane = row).  The two inherently
// ordered parts -- the sum of squares for the 2-norm and the rotation sweep
// -- are evaluated in the reference's row order: the chunk's values are
// broadcast lane by lane and every lane runs the same scalar recurrence, so
// norms and vectors come out bit-identical to the oracle.

// The ordered rotation sweep x[i-1] = c_i t1 - s_i t2, t1 = s_i t1 + c_i' t2
// (rbacktransform :366-375 / crbacktransform :810-822).  Rows are loaded 32
// at a time (lane = row), normalised / guarded, and their (x, c, s) are
// broadcast lane by lane; the 32-step chunk is fully unrolled so the
// shuffles issue ahead of the dependent t1 chain.  Lane t-1 keeps output row
// base + t - 1; row base - 1 (the previous chunk's last) is written by lane 0.
template <bool CP>
__device__ __forceinline__ void bt_sweep(double* xr, double* xi, const double* cr,
                                         const double* ci, const double* ss, int64_t n, int lane,
                                         bool normalize, bool do_scale, double xmax, double rt,
                                         double sc, int compact) {
  double t1r = 0.0, t1i = 0.0;
  // raw values of the next chunk, loaded one chunk ahead (latency hiding)
  double ra = 0.0, rb = 0.0, rc = 1.0, rci = 0.0, rs = 0.0;
  auto fetch = [&](int64_t i) {
    if (i < n) {
      ra = xr[i];
      if (CP) rb = xi[i];
      rc = cr[i];
      if (CP) rci = ci[i];
      if (!compact) rs = ss[i];
    }
  };
  fetch(lane);
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t i = base + lane;
    double a = ra, b = rb, cc = 1.0, cim = 0.0, sv = 0.0;
    const double c0 = rc, c1 = rci, c2 = rs;
    fetch(base + 32 + lane);
    if (i < n) {
      if (normalize) {
        a /= xmax;
        a /= rt;
        if (CP) {
          b /= xmax;
          b /= rt;
        }
      } else if (do_scale) {
        a *= sc;
        if (CP) b *= sc;
      }
      if (compact) {  // Stewart codes (givens.py:107-124, :144-149)
        if (CP)
          compact_decode_cplx(c0, c1, cc, cim, sv);
        else
          compact_decode(c0, cc, sv);
      } else {
        cc = c0;
        sv = c2;
        if (CP) cim = c1;
      }
    } else {
      a = 0.0;
      b = 0.0;
    }
    const int cnt = (int)(n - base < 32 ? n - base : 32);
    if (base == 0) {  // t1 = x[0]
      t1r = __shfl_sync(0xffffffffu, a, 0);
      if (CP) t1i = __shfl_sync(0xffffffffu, b, 0);
    }
    double outr = 0.0, outi = 0.0;
#pragma unroll
    for (int t = 0; t < 32; t++) {
      const double t2r = __shfl_sync(0xffffffffu, a, t);
      const double t2i = CP ? __shfl_sync(0xffffffffu, b, t) : 0.0;
      const double c_r = __shfl_sync(0xffffffffu, cc, t);
      const double s_ = __shfl_sync(0xffffffffu, sv, t);
      const double c_i = CP ? __shfl_sync(0xffffffffu, cim, t) : 0.0;
      if (t < cnt && (t > 0 || base > 0)) {
        double pr, pi = 0.0, nr, ni = 0.0;
        if (CP) {
          pr = (c_r * t1r - c_i * t1i) - s_ * t2r;
          pi = (c_r * t1i + c_i * t1r) - s_ * t2i;
          nr = s_ * t1r + (c_r * t2r + c_i * t2i);
          ni = s_ * t1i + (c_r * t2i - c_i * t2r);
        } else {
          pr = c_r * t1r - s_ * t2r;
          nr = c_r * t2r + s_ * t1r;
        }
        if (t == 0) {
          if (lane == 0) {
            xr[base - 1] = pr;
            if (CP) xi[base - 1] = pi;
          }
        } else if (lane == t - 1) {
          outr = pr;
          outi = pi;
        }
        t1r = nr;
        t1i = ni;
      }
    }
    // lanes 0..cnt-2 hold final rows base..base+cnt-2
    if (lane < cnt - 1) {
      xr[base + lane] = outr;
      if (CP) xi[base + lane] = outi;
    }
  }
  if (lane == 0) {
    xr[n - 1] = t1r;
    if (CP) xi[n - 1] = t1i;
  }
}

constexpr int BT_WARPS = 4;

__global__ void __launch_bounds__(BT_WARPS * 32) k_backtransform(Ctx c, int32_t* alpha_exp,
                                                                 double* norms, double* log2norm,
                                                                 int64_t q_begin, int64_t q_end) {
  const int lane = threadIdx.x & 31;
  const int64_t q = q_begin + (int64_t)blockIdx.x * BT_WARPS + (threadIdx.x >> 5);
  if (q >= q_end) return;
  bool cplx;
  int64_t col;
  col_of_shift(c, q, cplx, col);
  const int64_t n = c.n;
  double* xr = c.X + col * c.ldx;
  double* xi = cplx ? c.X + (col + 1) * c.ldx : nullptr;
  const double* cr = c.c_re + q * c.ldc;
  const double* ci = cplx ? c.c_im + q * c.ldc : nullptr;
  const double* ss = c.compact ? nullptr : c.s + q * c.ldc;
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  if (c.fail[q] != 0) {
    if (lane == 0) {
      norms[q] = qnan;
      log2norm[q] = qnan;
      alpha_exp[q] = 0;
    }
    return;
  }
  double xmax = 0.0, rt = 1.0;
  bool normalize = false, do_scale = false;
  double sc = 1.0;
  if (!c.robust) {
    if (lane == 0) {
      norms[q] = qnan;
      log2norm[q] = qnan;
      alpha_exp[q] = 0;
    }
  } else {
    // alpha_min and the consistency scaling (:330-342)
    int amin = 0x7fffffff;
    for (int t = lane; t < c.N; t += 32) amin = min(amin, c.E[(int64_t)t * c.ms + q]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amin = min(amin, __shfl_xor_sync(0xffffffffu, amin, o));
    double lm = 0.0;
    for (int64_t base = 0; base < n; base += 32) {
      const int64_t i = base + lane;
      if (i < n) {
        const int t = (int)(i / c.b_r);
        const double f = p2(amin - c.E[(int64_t)t * c.ms + q]);
        double a = xr[i];
        double b = cplx ? xi[i] : 0.0;
        if (f != 1.0) {
          a *= f;
          xr[i] = a;
          if (cplx) {
            b *= f;
            xi[i] = b;
          }
        }
        const double qv = cplx ? ghypot(a, b) : fabs(a);
        if (qv > lm) lm = qv;
      }
    }
    xmax = warp_max(lm);
    if (xmax == 0.0) {
      if (lane == 0) {
        norms[q] = 0.0;
        log2norm[q] = -__longlong_as_double(0x7ff0000000000000LL);
        alpha_exp[q] = amin;
      }
      return;  // zero column: no backtransform (:347-350)
    }
    // sum of squares in row order (:351-355)
    double tsum = 0.0;
    double pa = 0.0, pb = 0.0;  // next chunk, loaded one chunk ahead
    if (lane < n) {
      pa = xr[lane];
      if (cplx) pb = xi[lane];
    }
    for (int64_t base = 0; base < n; base += 32) {
      const int64_t i = base + lane;
      const double ca = pa, cb = pb;
      if (i + 32 < n) {
        pa = xr[i + 32];
        if (cplx) pb = xi[i + 32];
      }
      double sq = 0.0;
      if (i < n) {
        if (cplx) {
          const double qr = ca / xmax, qi = cb / xmax;
          sq = qr * qr + qi * qi;
        } else {
          const double qv = ca / xmax;
          sq = qv * qv;
        }
      }
      // rows >= n contribute +0.0: exact (tsum >= +0), so the chunk loop is
      // fully unrolled and its shuffles issue ahead of the dependent adds
#pragma unroll
      for (int t = 0; t < 32; t++) tsum += __shfl_sync(0xffffffffu, sq, t);
    }
    rt = sqrt(tsum);
    int aout = amin;
    if (c.mode == 1) {
      normalize = true;
    } else {
      const double qq = c.omega / xmax;
      if (rt > qq) {
        const int e = pow2floor_e(qq / rt);
        sc = p2(e);
        do_scale = true;
        aout = amin + e;
      }
    }
    if (lane == 0) {
      norms[q] = ldexp(xmax, -amin) * rt;
      log2norm[q] = log2(xmax) + log2(rt) - (double)amin;
      alpha_exp[q] = aout;
    }
  }
  // normalise / guard and the rotation sweep, chunk by chunk (:358-375)
  if (cplx)
    bt_sweep<true>(xr, xi, cr, ci, ss, n, lane, normalize, do_scale, xmax, rt, sc, c.compact);
  else
    bt_sweep<false>(xr, xi, cr, ci, ss, n, lane, normalize, do_scale, xmax, rt, sc, c.compact);
}
