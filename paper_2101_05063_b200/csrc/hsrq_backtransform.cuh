// hsrq_backtransform.cuh -- rbacktransform / crbacktransform
// (numba_backend.py:326-375, :759-822) and the unguarded backtransform
// (:314-323, :739-756); G lanes per shift, 32/G shifts per warp (included
// by hsrq_kernels.cu).
//
// Row chunks of G are loaded coalesced (lane = row within the shift's lane
// group).  The two inherently ordered parts -- the sum of squares for the
// 2-norm and the rotation sweep -- are evaluated in the reference's row
// order: the chunk's values are broadcast lane by lane within the group and
// every lane of the group runs the same scalar recurrence, so norms and
// vectors come out bit-identical to the oracle.  The recurrence costs one
// warp instruction per step whatever G is, so packing 32/G shifts into a warp
// divides the instruction count by 32/G (G = 32: 9.2e9 warp instructions per
// config-5 solve, issue-bound).  Shuffles use the group's own member mask:
// groups of one warp may take different paths (real / complex, failed).

// The ordered rotation sweep x[i-1] = c_i t1 - s_i t2, t1 = s_i t1 + c_i' t2
// (rbacktransform :366-375 / crbacktransform :810-822).  Rows are loaded G
// at a time, normalised / guarded, and their (x, c, s) are broadcast lane by
// lane; the G-step chunk is fully unrolled so the shuffles issue ahead of the
// dependent t1 chain.  Lane t-1 of the group keeps output row base + t - 1;
// row base - 1 (the previous chunk's last) is written by the group's lane 0.
template <int G, bool CP>
__device__ __forceinline__ void bt_sweep(double* xr, double* xi, const double* cr,
                                         const double* ci, const double* ss, int64_t n, int gl,
                                         int gb, unsigned gm, bool normalize, bool do_scale,
                                         double xmax, double rt, double sc, int compact) {
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
  fetch(gl);
  for (int64_t base = 0; base < n; base += G) {
    const int64_t i = base + gl;
    double a = ra, b = rb, cc = 1.0, cim = 0.0, sv = 0.0;
    const double c0 = rc, c1 = rci, c2 = rs;
    fetch(base + G + gl);
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
    const int cnt = (int)(n - base < G ? n - base : G);
    if (base == 0) {  // t1 = x[0]
      t1r = __shfl_sync(gm, a, gb);
      if (CP) t1i = __shfl_sync(gm, b, gb);
    }
    double outr = 0.0, outi = 0.0;
#pragma unroll
    for (int t = 0; t < G; t++) {
      const double t2r = __shfl_sync(gm, a, gb + t);
      const double t2i = CP ? __shfl_sync(gm, b, gb + t) : 0.0;
      const double c_r = __shfl_sync(gm, cc, gb + t);
      const double s_ = __shfl_sync(gm, sv, gb + t);
      const double c_i = CP ? __shfl_sync(gm, cim, gb + t) : 0.0;
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
          if (gl == 0) {
            xr[base - 1] = pr;
            if (CP) xi[base - 1] = pi;
          }
        } else if (gl == t - 1) {
          outr = pr;
          outi = pi;
        }
        t1r = nr;
        t1i = ni;
      }
    }
    // group lanes 0..cnt-2 hold final rows base..base+cnt-2
    if (gl < cnt - 1) {
      xr[base + gl] = outr;
      if (CP) xi[base + gl] = outi;
    }
  }
  if (gl == 0) {
    xr[n - 1] = t1r;
    if (CP) xi[n - 1] = t1i;
  }
}

constexpr int BT_THREADS = 128;

template <int G>
__device__ __forceinline__ double group_max(double v, unsigned gm) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(gm, v, o);
    v = w > v ? w : v;
  }
  return v;
}

template <int G>
__global__ void __launch_bounds__(BT_THREADS) k_backtransform(Ctx c, int32_t* alpha_exp,
                                                              double* norms, double* log2norm,
                                                              int64_t q_begin, int64_t q_end) {
  const int lane = threadIdx.x & 31;
  const int gl = lane % G, gb = lane - gl;
  const unsigned gm = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << gb);
  const int64_t q = q_begin + ((int64_t)blockIdx.x * BT_THREADS + threadIdx.x) / G;
  if (q >= q_end) return;  // whole groups leave together
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
    if (gl == 0) {
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
    if (gl == 0) {
      norms[q] = qnan;
      log2norm[q] = qnan;
      alpha_exp[q] = 0;
    }
  } else {
    // alpha_min and the consistency scaling (:330-342)
    int amin = 0x7fffffff;
    for (int t = gl; t < c.N; t += G) amin = min(amin, c.E[(int64_t)t * c.ms + q]);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) amin = min(amin, __shfl_xor_sync(gm, amin, o));
    double lm = 0.0;
    for (int64_t base = 0; base < n; base += G) {
      const int64_t i = base + gl;
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
    xmax = group_max<G>(lm, gm);
    if (xmax == 0.0) {
      if (gl == 0) {
        norms[q] = 0.0;
        log2norm[q] = -__longlong_as_double(0x7ff0000000000000LL);
        alpha_exp[q] = amin;
      }
      return;  // zero column: no backtransform (:347-350)
    }
    // sum of squares in row order (:351-355)
    double tsum = 0.0;
    double pa = 0.0, pb = 0.0;  // next chunk, loaded one chunk ahead
    if (gl < n) {
      pa = xr[gl];
      if (cplx) pb = xi[gl];
    }
    for (int64_t base = 0; base < n; base += G) {
      const int64_t i = base + gl;
      const double ca = pa, cb = pb;
      if (i + G < n) {
        pa = xr[i + G];
        if (cplx) pb = xi[i + G];
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
      for (int t = 0; t < G; t++) tsum += __shfl_sync(gm, sq, gb + t);
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
    if (gl == 0) {
      norms[q] = ldexp(xmax, -amin) * rt;
      log2norm[q] = log2(xmax) + log2(rt) - (double)amin;
      alpha_exp[q] = aout;
    }
  }
  // normalise / guard and the rotation sweep, chunk by chunk (:358-375)
  if (cplx)
    bt_sweep<G, true>(xr, xi, cr, ci, ss, n, gl, gb, gm, normalize, do_scale, xmax, rt, sc,
                      c.compact);
  else
    bt_sweep<G, false>(xr, xi, cr, ci, ss, n, gl, gb, gm, normalize, do_scale, xmax, rt, sc,
                       c.compact);
}

// Launch for shifts [q0, q1) of a group of ms shifts.  Lanes per shift G:
// enough warps to keep ~16 per SM busy (the recurrence is latency-bound per
// warp), otherwise as few lanes as possible (issue-bound): measured at config
// 5, G = 32 -> 8 takes the backtransform from 12.4 to 10.6 ms, while a 1/8
// shard needs G = 32 (3.4 vs 9.9 ms at G = 8).  HSRQ_BT_G overrides.
inline void bt_launch(const Ctx& c, int32_t* alpha_exp, double* norms, double* log2norm,
                      int64_t q0, int64_t q1, int64_t ms, cudaStream_t s) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double want = 32.0 * 16.0 * sms / (double)(ms > 0 ? ms : 1);
  int g = 4;
  while (g < 32 && g < want) g *= 2;
  if (const char* e = getenv("HSRQ_BT_G")) g = atoi(e);
  const unsigned blocks = (unsigned)(((q1 - q0) * g + BT_THREADS - 1) / BT_THREADS);
  if (g == 4)
    k_backtransform<4><<<blocks, BT_THREADS, 0, s>>>(c, alpha_exp, norms, log2norm, q0, q1);
  else if (g == 8)
    k_backtransform<8><<<blocks, BT_THREADS, 0, s>>>(c, alpha_exp, norms, log2norm, q0, q1);
  else if (g == 16)
    k_backtransform<16><<<blocks, BT_THREADS, 0, s>>>(c, alpha_exp, norms, log2norm, q0, q1);
  else
    k_backtransform<32><<<(unsigned)(((q1 - q0) * 32 + BT_THREADS - 1) / BT_THREADS), BT_THREADS,
                          0, s>>>(c, alpha_exp, norms, log2norm, q0, q1);
}
