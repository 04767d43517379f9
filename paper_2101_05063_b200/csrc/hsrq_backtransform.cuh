// hsrq_backtransform.cuh -- rbacktransform / crbacktransform
// (numba_backend.py:326-375, :759-822) and the unguarded backtransform
// (:314-323, :739-756); one warp per shift (included by hsrq_kernels.cu).
//
// Row chunks of 32 are loaded coalesced (lane = row).  The two inherently
// ordered parts -- the sum of squares for the 2-norm and the rotation sweep
// -- are evaluated in the reference's row order: the chunk's values are
// broadcast lane by lane and every lane runs the same scalar recurrence, so
// norms and vectors come out bit-identical to the oracle.

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
    for (int64_t base = 0; base < n; base += 32) {
      const int64_t i = base + lane;
      double sq = 0.0;
      if (i < n) {
        if (cplx) {
          const double qr = xr[i] / xmax, qi = xi[i] / xmax;
          sq = qr * qr + qi * qi;
        } else {
          const double qv = xr[i] / xmax;
          sq = qv * qv;
        }
      }
      const int cnt = (int)(n - base < 32 ? n - base : 32);
      for (int t = 0; t < cnt; t++) tsum += __shfl_sync(0xffffffffu, sq, t);
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
  double t1r = 0.0, t1i = 0.0;
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t i = base + lane;
    double a = 0.0, b = 0.0, cc = 1.0, cim = 0.0, sv = 0.0;
    if (i < n) {
      a = xr[i];
      if (cplx) b = xi[i];
      if (normalize) {
        a /= xmax;
        a /= rt;
        if (cplx) {
          b /= xmax;
          b /= rt;
        }
      } else if (do_scale) {
        a *= sc;
        if (cplx) b *= sc;
      }
      if (c.compact) {  // Stewart codes (givens.py:107-124, :144-149)
        if (cplx)
          compact_decode_cplx(cr[i], ci[i], cc, cim, sv);
        else
          compact_decode(cr[i], cc, sv);
      } else {
        cc = cr[i];
        sv = ss[i];
        if (cplx) cim = ci[i];
      }
    }
    const int cnt = (int)(n - base < 32 ? n - base : 32);
    double outr = 0.0, outi = 0.0;
    for (int t = 0; t < cnt; t++) {
      const double t2r = __shfl_sync(0xffffffffu, a, t);
      const double t2i = cplx ? __shfl_sync(0xffffffffu, b, t) : 0.0;
      if (base + t == 0) {  // t1 = x[0]
        t1r = t2r;
        t1i = t2i;
        continue;
      }
      const double c_r = __shfl_sync(0xffffffffu, cc, t);
      const double s_ = __shfl_sync(0xffffffffu, sv, t);
      double nr, ni, pr, pi;
      if (cplx) {
        const double c_i = __shfl_sync(0xffffffffu, cim, t);
        pr = (c_r * t1r - c_i * t1i) - s_ * t2r;
        pi = (c_r * t1i + c_i * t1r) - s_ * t2i;
        nr = s_ * t1r + (c_r * t2r + c_i * t2i);
        ni = s_ * t1i + (c_r * t2i - c_i * t2r);
      } else {
        pr = c_r * t1r - s_ * t2r;
        pi = 0.0;
        nr = c_r * t2r + s_ * t1r;
        ni = 0.0;
      }
      // x[i-1] = pr: row base+t-1 belongs to lane t-1 of this chunk, or to
      // lane 31 of the previous chunk (written directly)
      if (t == 0) {
        if (lane == 0) {
          xr[base - 1] = pr;
          if (cplx) xi[base - 1] = pi;
        }
      } else if (lane == t - 1) {
        outr = pr;
        outi = pi;
      }
      t1r = nr;
      t1i = ni;
    }
    // lanes 0..cnt-2 hold final rows base..base+cnt-2
    if (lane < cnt - 1) {
      xr[base + lane] = outr;
      if (cplx) xi[base + lane] = outi;
    }
  }
  if (lane == 0) {
    xr[n - 1] = t1r;
    if (cplx) xi[n - 1] = t1i;
  }
}
