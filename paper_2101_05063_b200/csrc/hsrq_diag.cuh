// hsrq_diag.cuh -- the diagonal-tile kernels (included by hsrq_kernels.cu).
//
// Per shift, one tile column's Givens sweep (reduce_diag, numba_backend.py:
// 75-106; creduce_diag :420-464) fused with the robust in-tile backward
// substitution that recomputes R on the fly (solve_rsolve :133-195; complex:
// _build_complex_r :530-551 + robust_trsv_complex :493-527 consuming R's
// column kp at step kp), then the panel operands W, Zs and the step scalars.
// The arithmetic is the reference's, operation for operation (compiled with
// -fmad=false), so c, s, x and the scale exponents are bit-identical.
//
// Layout: DP = 4 lanes per shift, DG = 8 shifts per warp.  The tile's v and
// x live in shared memory ([row][shift], lane-owned rows i = pl + 4t), so
// the long dependent chain of each step -- hypot, three divisions, the
// pivot -- is executed once per 4 lanes instead of once per 32, and the
// O(kp) row updates are spread over 32 lanes.  The guard-2 maxima over rows
// < kp are accumulated in the previous step's update loop; the complex
// guards are evaluated from cheap monotone bounds first and exactly only
// when a bound cannot prove protect_update == 1.

// Lanes per shift (DP) and warps per CTA are template parameters; the host
// picks the variant (see diag_launch in hsrq_kernels.cu).
#undef HSRQ_FUZZ_FILE
#define HSRQ_FUZZ_FILE 1u
constexpr double DSLACK = 1.0 + 0x1p-46;
constexpr unsigned FULL = 0xffffffffu;

// Per-step phase profile (diagnostics build -DHSRQ_STEPPROF, read with
// hsrq_debug_stepprof): clock64 marks inside the one-warp complex sweep's
// step, summed over the steps of warp 0 of every CTA.
#ifdef HSRQ_STEPPROF
__device__ unsigned long long g_stepprof[16];
#define SP_DECL long long sp_t0 = 0, sp_acc[12] = {0}; int sp_i = 0;
#define SP_START() (sp_t0 = clock64(), sp_i = 0)
#define SP_MARK() { const long long t_ = clock64(); sp_acc[sp_i++] += t_ - sp_t0; sp_t0 = t_; }
#define SP_FLUSH(n) if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) == 0) { \
    for (int i_ = 0; i_ < (n); i_++) atomicAdd(&g_stepprof[i_], (unsigned long long)sp_acc[i_]); \
    atomicAdd(&g_stepprof[15], 1ULL); }
#else
#define SP_DECL
#define SP_START() ((void)0)
#define SP_MARK() ((void)0)
#define SP_FLUSH(n) ((void)0)
#endif

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

struct DiagArgs {
  int jt;
  int64_t js;
  int k;
  int has_left;
  int64_t q0, count;  // shifts [q0, q0 + count) handled by this launch
  int64_t rot_off;    // row offset of this tile in the rotation table (js; 0 when the
                      // diag launch records into the compact mode's tile scratch)
  // tile-level mode (hsrq_tile_diag): explicit buffers, shifts 0..t_b-1
  int tile_mode;
  const double* t_hdiag;   // k x (k-1) row-major
  const double* t_hleft;
  const double* t_rright;  // k x b (real) / k x 2b (complex interleaved) row-major
  double* t_x;
  double *t_cre, *t_cim, *t_s;
  int32_t* t_beta;
  int64_t* t_status;
  int t_b;
};

__device__ __forceinline__ double hget(const Ctx& c, const DiagArgs& a, int i, int t) {
  return a.tile_mode ? a.t_hdiag[(int64_t)i * (a.k - 1) + t] : c.H[(a.js + t) * c.ldh + a.js + i];
}

// Copy rows 0..nrows-1 of diagonal-tile column t into a warp-private smem
// buffer (cp.async, one commit group); the next step's column is prefetched
// while the current step runs.
__device__ __forceinline__ void fill_col(const Ctx& c, const DiagArgs& a, double* buf, int t,
                                         int nrows, int lane) {
  if (!a.tile_mode && ((c.ldh | a.js) & 1) == 0) {
    // contiguous, 16-byte aligned column segment: two rows per cp.async
    const double* src = c.H + (a.js + t) * c.ldh + a.js;
    for (int i = 2 * lane; i < nrows; i += 64) {
      if (i + 1 < nrows)
        cp_async16(&buf[i], src + i, true);
      else
        cp_async8(&buf[i], src + i, true);
    }
  } else {
    for (int i = lane; i < nrows; i += 32) {
      const double* src = a.tile_mode ? &a.t_hdiag[(int64_t)i * (a.k - 1) + t]
                                      : &c.H[(a.js + t) * c.ldh + a.js + i];
      cp_async8(&buf[i], src, true);
    }
  }
  cp_commit();
}

template <int DP>
__device__ __forceinline__ double gmax(double v) {  // max over the DP lanes of a group
#pragma unroll
  for (int o = 1; o < DP; o <<= 1) {
    const double w = __shfl_xor_sync(FULL, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Whole warp (DP = 32): two integer REDUX ops on the bit pattern instead of a
// five-level shuffle chain.  Every gmax operand is a non-negative double
// (fabs / squares / moduli), for which the bit pattern orders like the
// value, so the result equals the shuffle chain's.
__device__ __forceinline__ double gmax_redux(double v, unsigned mask) {
  const unsigned long long k = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
  const unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  const unsigned mh = __reduce_max_sync(mask, hi);
  const unsigned ml = __reduce_max_sync(mask, hi == mh ? lo : 0u);
  return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}
template <>
__device__ __forceinline__ double gmax<32>(double v) {
  return gmax_redux(v, FULL);
}
// (DP = 16 with per-half-warp member masks is correct but measured slower:
// 146.6 -> 152.5 ms per 1/4 shard)

__device__ __forceinline__ void record_fail(const Ctx& c, const DiagArgs& a, int64_t q, int phase,
                                            int row) {
  if (a.tile_mode) {
    a.t_status[q] = (int64_t)phase * (1LL << 42) + (int64_t)row;
    return;
  }
  if (c.fail[q] == 0) {
    c.fail[q] = pack_fail(phase, a.jt, row);
    atomicAdd(c.nfail, 1ULL);
  }
}

// hmax[kp] = max_{i<kp} |h(i, kp-1)| (solve_rsolve :155-163), per tile column.
__device__ __forceinline__ void load_hmax(const Ctx& c, const DiagArgs& a, double* hmax) {
  for (int kp = 1 + threadIdx.x; kp < a.k; kp += blockDim.x) {
    double m;
    if (a.tile_mode) {
      m = 0.0;
      for (int i = 0; i < kp; i++) {
        double v = fabs(hget(c, a, i, kp - 1));
        if (v > m) m = v;
      }
    } else {
      m = c.HMK[(int64_t)a.jt * MAXK + kp];
    }
    hmax[kp] = m;
  }
  HSRQ_SYNCTHREADS();
}

__device__ __forceinline__ void put_rot(const Ctx& c, const DiagArgs& a, int64_t q, int row,
                                        double cr, double ci, double s) {
  if (a.tile_mode) {
    a.t_cre[(int64_t)row * a.t_b + q] = cr;
    if (a.t_cim) a.t_cim[(int64_t)row * a.t_b + q] = ci;
    a.t_s[(int64_t)row * a.t_b + q] = s;
  } else {
    c.c_re[q * c.ldc + a.rot_off + row] = cr;
    if (c.c_im) c.c_im[q * c.ldc + a.rot_off + row] = ci;
    c.s[q * c.ldc + a.rot_off + row] = s;
  }
}

template <int DP>
__device__ __forceinline__ void diag_real_operands(const Ctx& c, const DiagArgs& a, int64_t q,
                                                   int64_t col, bool live, int pl, int grp, int k,
                                                   double* V, double* Xs, double c0, double s0,
                                                   double x0);

// The last step of a real shift's sweep -- cross-tile rotation
// (reduce_diag :94-105) and the last pivot (:178-192) -- the write-back of
// x and the panel operands (update_rupdate :246-253); shared by k_diag_real
// and the chain warp of k_diag_real_ws.
template <int DP>
__device__ __forceinline__ void diag_real_tail(const Ctx& c, const DiagArgs& a, int64_t q,
                                               int64_t col, bool live, int pl, int grp, int k,
                                               double* V, double* Xs, int gexp, bool robust) {
  constexpr int DG = 32 / DP;
  const double omega = c.omega;
#define VV(i) V[(i) * DG + grp]
#define XX(i) Xs[(i) * DG + grp]
  const double v0 = VV(0);
  double x0 = XX(0);
  // every lane has read row 0 before lane 0 may rescale / overwrite it below
  // (found by the schedule-fuzzing race check, tools/race_fuzz.py)
  HSRQ_SYNCWARP();
  double c0 = 1.0, s0 = 0.0, piv = v0;
  double hleft0 = 0.0;
  if (a.has_left) {
    hleft0 = a.tile_mode ? a.t_hleft[0] : c.H[(a.js - 1) * c.ldh + a.js];
    const double r = ghypot(hleft0, v0);
    if (live && r == 0.0) {
      if (pl == 0) record_fail(c, a, q, HSRQ_KIND_DEGENERATE, 0);
      live = false;
    }
    c0 = v0 / r;
    s0 = -hleft0 / r;
    piv = v0 * c0 - hleft0 * s0;
  }
  if (live && pl == 0) put_rot(c, a, q, 0, c0, 0.0, s0);
  if (live && piv == 0.0) {
    if (pl == 0) record_fail(c, a, q, HSRQ_KIND_SINGULAR, 0);
    live = false;
  }
  if (robust && live) {
    const double avv = fabs(piv), ax = fabs(x0);
    if (avv < 1.0 && ax > avv * omega) {
      const int e = pow2floor_e(avv * omega / ax);
      const double xi = p2(e);
      for (int i = pl; i < k; i += DP) XX(i) *= xi;
      x0 *= xi;
      gexp += e;
    }
  }
  x0 = x0 / piv;
  if (pl == 0) XX(0) = x0;
  HSRQ_SYNCWARP();
  // (no early return: dead or padding groups keep executing so that warp
  // shuffles stay convergent; their writes are masked by `live`)
  if (live) {
    for (int i = pl; i < k; i += DP) {
      if (a.tile_mode)
        a.t_x[(int64_t)i * a.t_b + q] = XX(i);
      else
        c.X[col * c.ldx + a.js + i] = XX(i);
    }
  }
  if (a.tile_mode) {
    if (live && pl == 0) a.t_beta[q] += gexp;
    return;
  }
  if (live && pl == 0) c.E[(int64_t)a.jt * c.ms + q] += gexp;
  if (a.jt == 0) return;
  diag_real_operands<DP>(c, a, q, col, live, pl, grp, k, V, Xs, c0, s0, x0);
#undef VV
#undef XX
}

// Panel operands of a real shift after its sweep (update_rupdate :246-253,
// reduce_offdiag :109-125 as a linear map): W_j = c_j prod_{t<j} s_t, P, the
// rotated solution Z and the step scalars -- from the tile's recorded
// rotations (c_re / s at rot_off) and its final x in shared memory.  Shared
// by k_diag_real, the chain warp of k_diag_real_ws and the tile-level update
// entry (k_tile_operands).
template <int DP>
__device__ __forceinline__ void diag_real_operands(const Ctx& c, const DiagArgs& a, int64_t q,
                                                   int64_t col, bool live, int pl, int grp, int k,
                                                   double* V, double* Xs, double c0, double s0,
                                                   double x0) {
  constexpr int DG = 32 / DP;
#define VV(i) V[(i) * DG + grp]
#define XX(i) Xs[(i) * DG + grp]
  // ---- panel operands: W_j = c_j prod_{t<j} s_t, P; Z (update_rupdate :246-253) ----
  double* bw = c.Bop + (2 * col) * KP;
  double* bz = c.Bop + (2 * col + 1) * KP;
  const double* crow = c.c_re + (live ? q : 0) * c.ldc + a.rot_off;
  const double* srow = c.s + (live ? q : 0) * c.ldc + a.rot_off;
  double pre = 1.0;
  double carry = c0 * x0;  // Z[0] = c[0] * Z[0]
  // rotations j = jb + pl loaded by lane pl one chunk of DP ahead and
  // broadcast within the group: the serial carry chain no longer waits on
  // an L2 round trip per j
  const int gb = grp * DP;
  double lc = 1.0, ls = 0.0;
  if (pl < k) {
    lc = crow[pl];
    ls = srow[pl];
  }
  for (int jb = 0; jb < k; jb += DP) {
    double nc = 1.0, ns = 0.0;
    if (jb + DP + pl < k) {
      nc = crow[jb + DP + pl];
      ns = srow[jb + DP + pl];
    }
#pragma unroll(DP > 8 ? 8 : DP)
    for (int t = 0; t < DP; t++) {
      const int j = jb + t;
      const double cj = __shfl_sync(FULL, lc, gb + t), sj = __shfl_sync(FULL, ls, gb + t);
      if (j < k) {
        if (live && pl == t) bw[j] = cj * pre;
        pre = pre * sj;
        if (j >= 1) {
          const double t2 = XX(j), t1 = carry;
          const double zf = cj * t1 - sj * t2;  // final Z[j-1]
          carry = sj * t1 + cj * t2;
          if (pl == t) {
            if (live) bz[j] = zf;
            VV(j - 1) = zf;  // keep Z for zmax
          }
        }
      }
    }
    lc = nc;
    ls = ns;
  }
  HSRQ_SYNCWARP();
  double zm = 0.0;
  for (int i = pl; i < k - 1; i += DP) {
    const double z = fabs(VV(i));
    if (z > zm) zm = z;
  }
  zm = gmax<DP>(zm);
  if (live) {
    for (int j = k + pl; j < KP; j += DP) {
      bw[j] = 0.0;
      bz[j] = 0.0;
    }
    if (pl == 0) {
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
#undef VV
#undef XX
}

// ---------------------------------------------------------------------------
// real shifts
// ---------------------------------------------------------------------------
template <int DP, int DW>
__global__ void __launch_bounds__(DW * 32) k_diag_real(Ctx c, DiagArgs a) {
  constexpr int DG = 32 / DP;
  extern __shared__ __align__(16) double dsm[];
  double* hmax = dsm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / DP, pl = lane % DP;
  double* V = dsm + MAXK + warp * (2 * MAXK * DG + 2 * MAXK);
  double* Xs = V + MAXK * DG;
  double* hb = Xs + MAXK * DG;  // [2][MAXK] column buffers
  const int k = a.k;
  load_hmax(c, a, hmax);
  const int64_t q = a.q0 + ((int64_t)blockIdx.x * DW + warp) * DG + grp;
  bool live = q < a.q0 + a.count;
  if (live && !a.tile_mode && c.fail[q] != 0) live = false;
  const int64_t col = a.tile_mode ? 0 : 2 * c.mc + (q - c.mc);
  const double lam = live ? c.lam_re[q] : 0.0;
  const double omega = c.omega;
  const bool robust = c.robust;
#define VV(i) V[(i) * DG + grp]
#define XX(i) Xs[(i) * DG + grp]
  double xm = 0.0, vm = 0.0;  // partial maxima over own rows < kp (for the next step)
  for (int i = pl; i < k; i += DP) {
    double vv = 0.0, xx = 0.0;
    if (live) {
      if (a.tile_mode) {
        vv = a.t_rright[(int64_t)i * a.t_b + q];
        xx = a.t_x[(int64_t)i * a.t_b + q];
      } else {
        vv = c.Cr[col * c.ldx + a.js + i];
        xx = c.X[col * c.ldx + a.js + i];
      }
    }
    VV(i) = vv;
    XX(i) = xx;
    if (i < k - 1) {
      if (fabs(xx) > xm) xm = fabs(xx);
      if (fabs(vv) > vm) vm = fabs(vv);
    }
  }
  int cur = 0;
  if (k >= 2) {
    fill_col(c, a, hb, k - 2, k, lane);
    cp_wait<0>();
  }
  HSRQ_SYNCWARP();
  int gexp = 0;
  for (int kp = k - 1; kp >= 1; --kp) {
    const double* hcol = hb + cur * MAXK;  // column kp-1, rows 0..kp
    if (kp >= 2) fill_col(c, a, hb + (cur ^ 1) * MAXK, kp - 2, kp, lane);
    const double vk = VV(kp);
    double xk = XX(kp);
    const double av = hcol[kp];
    const double r = ghypot(av, vk);
    if (live && r == 0.0) {
      if (pl == 0) record_fail(c, a, q, HSRQ_KIND_DEGENERATE, kp);
      live = false;
    }
    const double cc = vk / r, ss = -av / r;
    if (live && pl == 0) put_rot(c, a, q, kp, cc, 0.0, ss);
    const double phi = vk * cc - av * ss;
    if (live && phi == 0.0) {
      if (pl == 0) record_fail(c, a, q, HSRQ_KIND_SINGULAR, kp);
      live = false;
    }
    xm = gmax<DP>(xm);
    vm = gmax<DP>(vm);
    if (robust && live) {
      const double aphi = fabs(phi), ax = fabs(xk);
      if (aphi < 1.0 && ax > aphi * omega) {  // guard 1 (:144-151)
        if (pl == 0) HSRQ_COUNT(0);
        const int e = pow2floor_e(aphi * omega / ax);
        const double xi = p2(e);
        for (int i = pl; i < k; i += DP) XX(i) *= xi;
        xk *= xi;
        xm *= xi;
        gexp += e;
      }
    }
    xk = xk / phi;
    if (robust && live) {  // guard 2 (:153-168)
      const int e = protect_update_e(xm, vm + hmax[kp] + fabs(lam), fabs(xk), omega);
      if (pl == 0) HSRQ_COUNT(6);
      if (e < 0) {
        if (pl == 0) HSRQ_COUNT(1);
        const double xi = p2(e);
        for (int i = pl; i < k; i += DP) XX(i) *= xi;
        xk *= xi;
        gexp += e;
      }
    }
    if (pl == (kp % DP)) XX(kp) = xk;
    const double tau1 = ss * xk, tau2 = cc * xk;
    double nxm = 0.0, nvm = 0.0;
#pragma unroll 1
    for (int i = pl; i < kp - 1; i += DP) {
      const double hi = hcol[i];
      double vv = VV(i), xx = XX(i);
      xx = (xx - tau2 * vv) + tau1 * hi;
      vv = cc * hi + ss * vv;
      if (fabs(xx) > nxm) nxm = fabs(xx);
      if (fabs(vv) > nvm) nvm = fabs(vv);
      VV(i) = vv;
      XX(i) = xx;
    }
    if (pl == (kp - 1) % DP) {  // the shifted row (diagonal entry h - lambda)
      const int i = kp - 1;
      const double hd = hcol[i] - lam;
      const double vv = VV(i), xx = XX(i);
      XX(i) = (xx - tau2 * vv) + tau1 * hd;
      VV(i) = cc * hd + ss * vv;
    }
    xm = nxm;
    vm = nvm;
    cp_wait<0>();
    HSRQ_SYNCWARP();
    cur ^= 1;
  }
  diag_real_tail<DP>(c, a, q, col, live, pl, grp, k, V, Xs, gexp, robust);
#undef VV
#undef XX
}

// Panel operands of a complex shift after its sweep (cupdate_crupdate
// :645-666; W complex, P real): W_j, Z, the step scalars (chain-warp /
// whole-warp code shared by k_diag_cplx and k_diag_cplx_ws).
template <int DP>
__device__ __forceinline__ void diag_cplx_operands(const Ctx& c, const DiagArgs& a, int64_t q,
                                                   int64_t col, bool live, int pl, int grp, int k,
                                                   double* Xr, double* Xi, double* Vr, double* Vi,
                                                   double c0r, double c0i, double s0, cplx x0) {
  constexpr int DG = 32 / DP;
#define IX(i) ((i) * DG + grp)
  double* bw_re = c.Bop + (2 * col) * KP;
  double* bz_re = c.Bop + (2 * col + 1) * KP;
  double* bw_im = c.Bop + (2 * (col + 1)) * KP;
  double* bz_im = c.Bop + (2 * (col + 1) + 1) * KP;
  const int64_t qs = live ? q : 0;
  const double* crow = c.c_re + qs * c.ldc + a.rot_off;
  const double* cirow = c.c_im + qs * c.ldc + a.rot_off;
  const double* srow = c.s + qs * c.ldc + a.rot_off;
  double pre = 1.0;
  cplx carry = mk(c0r * x0.re + c0i * x0.im, c0r * x0.im - c0i * x0.re);
  // rotations prefetched one chunk ahead by lane pl (j = jb + pl) and
  // broadcast within the group (see diag_real_tail)
  const int gb = grp * DP;
  double lc = 1.0, lci = 0.0, ls = 0.0;
  if (pl < k) {
    lc = crow[pl];
    lci = cirow[pl];
    ls = srow[pl];
  }
  for (int jb = 0; jb < k; jb += DP) {
    double nc = 1.0, nci = 0.0, ns = 0.0;
    if (jb + DP + pl < k) {
      nc = crow[jb + DP + pl];
      nci = cirow[jb + DP + pl];
      ns = srow[jb + DP + pl];
    }
#pragma unroll(DP > 8 ? 8 : DP)
    for (int t = 0; t < DP; t++) {
      const int j = jb + t;
      const double cr = __shfl_sync(FULL, lc, gb + t), ci = __shfl_sync(FULL, lci, gb + t);
      const double sj = __shfl_sync(FULL, ls, gb + t);
      if (j < k) {
        if (live && pl == t) {
          bw_re[j] = cr * pre;
          bw_im[j] = ci * pre;
        }
        pre = pre * sj;
        if (j >= 1) {
          const cplx t2 = mk(Xr[IX(j)], Xi[IX(j)]), t1 = carry;
          const cplx zf = mk((cr * t1.re - ci * t1.im) - sj * t2.re,
                             (cr * t1.im + ci * t1.re) - sj * t2.im);
          carry = mk(sj * t1.re + (cr * t2.re + ci * t2.im), sj * t1.im + (cr * t2.im - ci * t2.re));
          if (pl == t) {
            if (live) {
              bz_re[j] = zf.re;
              bz_im[j] = zf.im;
            }
            Vr[IX(j - 1)] = zf.re;
            Vi[IX(j - 1)] = zf.im;
          }
        }
      }
    }
    lc = nc;
    lci = nci;
    ls = ns;
  }
  HSRQ_SYNCWARP();
  double zm = 0.0;
  for (int i = pl; i < k - 1; i += DP) {
    const double z = cabs_(mk(Vr[IX(i)], Vi[IX(i)]));
    if (z > zm) zm = z;
  }
  zm = gmax<DP>(zm);
  if (live) {
    for (int j = k + pl; j < KP; j += DP) {
      bw_re[j] = bw_im[j] = 0.0;
      bz_re[j] = bz_im[j] = 0.0;
    }
    if (pl == 0) {
      bz_re[0] = bz_im[0] = 0.0;
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
#undef IX
}

// ---------------------------------------------------------------------------
// complex shifts (Im > 0), interleaved re/im columns 2q, 2q+1
// ---------------------------------------------------------------------------
template <int DP, int DW>
__global__ void __launch_bounds__(DW * 32) k_diag_cplx(Ctx c, DiagArgs a) {
  constexpr int DG = 32 / DP;
  extern __shared__ __align__(16) double dsm[];
  double* hmax = dsm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / DP, pl = lane % DP;
  double* Vr = dsm + MAXK + warp * (4 * MAXK * DG + 2 * MAXK);
  double* Vi = Vr + MAXK * DG;
  double* Xr = Vi + MAXK * DG;
  double* Xi = Xr + MAXK * DG;
  double* hb = Xi + MAXK * DG;  // [2][MAXK] column buffers
  const int k = a.k;
  load_hmax(c, a, hmax);
  const int64_t q = a.q0 + ((int64_t)blockIdx.x * DW + warp) * DG + grp;
  bool live = q < a.q0 + a.count;
  if (live && !a.tile_mode && c.fail[q] != 0) live = false;
  const int64_t col = a.tile_mode ? 0 : 2 * q;
  const double lre = live ? c.lam_re[q] : 0.0, lim = live ? c.lam_im[q] : 0.0;
  const double omega = c.omega;
  const bool robust = c.robust;
#define IX(i) ((i) * DG + grp)
  double xb = 0.0, vb = 0.0;  // bounds (|re|+|im|) over own rows < kp
  for (int i = pl; i < k; i += DP) {
    double vr = 0.0, vi = 0.0, xr = 0.0, xi = 0.0;
    if (live) {
      if (a.tile_mode) {
        const int64_t b2 = 2 * (int64_t)a.t_b;
        vr = a.t_rright[i * b2 + 2 * q];
        vi = a.t_rright[i * b2 + 2 * q + 1];
        xr = a.t_x[i * b2 + 2 * q];
        xi = a.t_x[i * b2 + 2 * q + 1];
      } else {
        vr = c.Cr[col * c.ldx + a.js + i];
        vi = c.Cr[(col + 1) * c.ldx + a.js + i];
        xr = c.X[col * c.ldx + a.js + i];
        xi = c.X[(col + 1) * c.ldx + a.js + i];
      }
    }
    Vr[IX(i)] = vr;
    Vi[IX(i)] = vi;
    Xr[IX(i)] = xr;
    Xi[IX(i)] = xi;
    if (i < k - 1) {
      const double bx = fabs(xr) + fabs(xi), bv = fabs(vr) + fabs(vi);
      if (bx > xb) xb = bx;
      if (bv > vb) vb = bv;
    }
  }
  int cur = 0;
  if (k >= 2) {
    fill_col(c, a, hb, k - 2, k, lane);
    cp_wait<0>();
  }
  HSRQ_SYNCWARP();
  int gexp = 0;
  SP_DECL
  for (int kp = k - 1; kp >= 1; --kp) {
    SP_START();
    const double* hcol = hb + cur * MAXK;  // column kp-1, rows 0..kp
    if (kp >= 2) fill_col(c, a, hb + (cur ^ 1) * MAXK, kp - 2, kp, lane);
    const cplx vk = mk(Vr[IX(kp)], Vi[IX(kp)]);
    cplx xk = mk(Xr[IX(kp)], Xi[IX(kp)]);
    const double av = hcol[kp];
    SP_MARK();  // 0: column prefetch issue, row kp reads
    const double absv = ghypot(vk.re, vk.im);
    const double r = ghypot(av, absv);
    SP_MARK();  // 1: two glibc hypots
    if (live && r == 0.0) {
      if (pl == 0) record_fail(c, a, q, HSRQ_KIND_DEGENERATE, kp);
      live = false;
    }
    const double cr = vk.re / r, ci = vk.im / r, sv = -av / r;
    if (live && pl == 0) put_rot(c, a, q, kp, cr, ci, sv);
    const cplx ccj = mk(cr, -ci), svc = mk(sv, 0.0);
    const cplx d = csub(cmul(ccj, vk), cmul(svc, mk(av, 0.0)));  // R[kp, kp]
    if (live && d.re == 0.0 && d.im == 0.0) {
      if (pl == 0) record_fail(c, a, q, HSRQ_KIND_SINGULAR, kp);
      live = false;
    }
    SP_MARK();  // 2: three divisions, pivot, rotation store
    xb = gmax<DP>(xb);
    vb = gmax<DP>(vb);
    if (robust && live) {  // guard 1 (robust_trsv_complex :501-508)
      const double adlo = fmax(fabs(d.re), fabs(d.im));
      if (adlo < 1.0 && (fabs(xk.re) + fabs(xk.im)) * DSLACK > adlo * omega) {
        const double ad = cabs_(d), ax = cabs_(xk);
        if (pl == 0) HSRQ_COUNT(2);
        if (ad < 1.0 && ax > ad * omega) {
          if (pl == 0) HSRQ_COUNT(3);
          const int e = pow2floor_e(ad * omega / ax);
          const cplx xi = mk(p2(e), 0.0);
          for (int i = pl; i < k; i += DP) {
            const cplx t = cmul(mk(Xr[IX(i)], Xi[IX(i)]), xi);
            Xr[IX(i)] = t.re;
            Xi[IX(i)] = t.im;
          }
          xk = cmul(xk, xi);
          xb = xb * xi.re + 0x1p-1070;
          gexp += e;
        }
      }
    }
    SP_MARK();  // 3: group maxima, guard 1
    xk = cdiv(xk, d);
    SP_MARK();  // 4: complex pivot division
    // guard 2 (:510-523): protect_update(max|x_i|, max|r_i|, |x_kp|), i < kp
    bool exact2 = false;
    double rb = 0.0;
    if (robust && live) {
      rb = ((fabs(cr) + fabs(ci)) * vb + fabs(sv) * (hmax[kp] + fabs(lre) + fabs(lim))) * DSLACK;
      exact2 = !protect_update_is_one(xb * DSLACK, rb, (fabs(xk.re) + fabs(xk.im)) * DSLACK, omega);
      if (pl == 0) HSRQ_COUNT(7);
      if (pl == 0 && exact2) HSRQ_COUNT(4);
    }
    SP_MARK();  // 5: guard-2 bound test
#ifdef HSRQ_EXP_NOEXACT2
    exact2 = false;  // timing experiment only: results are wrong
#endif
    if (__any_sync(FULL, exact2)) {
      // The bounds could not prove xi = 1.  Certify protect_update's exponent
      // from an interval around the two maxima instead of evaluating glibc
      // moduli row by row: scaled squared moduli (one pass, no hypot) give
      // max|.| to within 2^-47; protect_update_e is monotone in both norms
      // (hsrq_device.cuh), so equal exponents at both interval ends are the
      // exact exponent.  Otherwise (a binade edge, or bounds too loose to
      // scale by) fall back to the exact maxima.
      if (lane == 0) HSRQ_COUNT(12);
      const int ex = ilogb_pos(xb), er = ilogb_pos(rb);
      const double sx = p2(-max(-1000, min(1020, ex))), sr = p2(-max(-1000, min(1020, er)));
      double tx = 0.0, tr = 0.0;
#pragma unroll 1
      for (int i = pl; i < kp; i += DP) {
        const cplx t = i == kp - 1 ? csub(mk(hcol[i], 0.0), mk(lre, lim)) : mk(hcol[i], 0.0);
        const cplx ri = csub(cmul(ccj, mk(Vr[IX(i)], Vi[IX(i)])), cmul(svc, t));
        const double a1 = ri.re * sr, b1 = ri.im * sr;
        const double a2 = Xr[IX(i)] * sx, b2 = Xi[IX(i)] * sx;
        const double t1 = a1 * a1 + b1 * b1, t2 = a2 * a2 + b2 * b2;
        tr = t1 > tr ? t1 : tr;
        tx = t2 > tx ? t2 : tx;
      }
      tr = gmax<DP>(tr);
      tx = gmax<DP>(tx);
      bool full = false;
      int e = 0;
#ifdef HSRQ_COUNTERS
      // what-if: which tighter cheap bounds would have passed the guard-2 test
      if (exact2 && pl == 0 && tx > 0.0 && tr > 0.0) {
        const double xbm = sqrt(tx) * p2(ex) * (1.0 + 0x1p-40);
        const double rbm = sqrt(tr) * p2(er) * (1.0 + 0x1p-40);
        const double ax1 = (fabs(xk.re) + fabs(xk.im)) * DSLACK, axm = cabs_(xk);
        if (protect_update_is_one(xbm, rb, ax1, omega)) HSRQ_COUNT(16);
        if (protect_update_is_one(xb * DSLACK, rbm, ax1, omega)) HSRQ_COUNT(17);
        if (protect_update_is_one(xbm, rbm, ax1, omega)) HSRQ_COUNT(18);
        if (protect_update_is_one(xbm, rbm, axm, omega)) HSRQ_COUNT(19);
        if (protect_update_is_one(xb * DSLACK, rb, axm, omega)) HSRQ_COUNT(20);
        if (xbm > omega) HSRQ_COUNT(22);
        if (rbm * axm > omega) HSRQ_COUNT(23);
        if (axm > 1.0) HSRQ_COUNT(24);
      }
#endif
      if (exact2) {
        const double ax = cabs_(xk);
        if (ex > -1000 && ex < 1020 && er > -1000 && er < 1020 && tx >= 0x1p-960 &&
            tr >= 0x1p-960 && tx <= 16.0 && tr <= 16.0) {
          const double qx = sqrt(tx), qr = sqrt(tr);
          const double bl = (qx - qx * 0x1p-47) * p2(ex), bh = (qx + qx * 0x1p-47) * p2(ex);
          const double rl = (qr - qr * 0x1p-47) * p2(er), rh = (qr + qr * 0x1p-47) * p2(er);
          e = protect_update_e(bl, rl, ax, omega);
          full = e != protect_update_e(bh, rh, ax, omega);
          if (full && pl == 0) HSRQ_COUNT(14);
        } else {
          full = true;
          if (pl == 0) HSRQ_COUNT(15);
#ifdef HSRQ_COUNTERS
          if (pl == 0 && lane == 0 && blockIdx.x == 0 && kp == 100)
            printf("jt %d ex %d er %d tx %g tr %g xb %g rb %g\n", a.jt, ex, er, tx, tr, xb, rb);
#endif
        }
      }
      if (__any_sync(FULL, full)) {  // exact glibc moduli (rare)
        if (lane == 0) HSRQ_COUNT(13);
        double rm = 0.0, bm = 0.0;
        for (int i = pl; i < kp; i += DP) {
          cplx t = mk(hcol[i], 0.0);
          if (i == kp - 1) t = csub(t, mk(lre, lim));
          const cplx ri = csub(cmul(ccj, mk(Vr[IX(i)], Vi[IX(i)])), cmul(svc, t));
          const double q1 = cabs_(ri), q2 = cabs_(mk(Xr[IX(i)], Xi[IX(i)]));
          if (q1 > rm) rm = q1;
          if (q2 > bm) bm = q2;
        }
        rm = gmax<DP>(rm);
        bm = gmax<DP>(bm);
        if (full) e = protect_update_e(bm, rm, cabs_(xk), omega);
      }
#ifdef HSRQ_COUNTERS
      if (exact2 && e == 0 && pl == 0) HSRQ_COUNT(21);
#endif
      if (exact2 && e < 0) {
        if (pl == 0) HSRQ_COUNT(5);
        const cplx xi = mk(p2(e), 0.0);
        for (int i = pl; i < k; i += DP) {
          const cplx t = cmul(mk(Xr[IX(i)], Xi[IX(i)]), xi);
          Xr[IX(i)] = t.re;
          Xi[IX(i)] = t.im;
        }
        xk = cmul(xk, xi);
        gexp += e;
      }
    }
    SP_MARK();  // 6: guard-2 certification / exact maxima / rescale
    if (pl == (kp % DP)) {
      Xr[IX(kp)] = xk.re;
      Xi[IX(kp)] = xk.im;
    }
    double nxb = 0.0, nvb = 0.0;
#pragma unroll 1
    for (int i = pl; i < kp - 1; i += DP) {
      const double hi = hcol[i];
      const cplx v = mk(Vr[IX(i)], Vi[IX(i)]);
      cplx x = mk(Xr[IX(i)], Xi[IX(i)]);
      const cplx ri = csub(cmul(ccj, v), cmul(svc, mk(hi, 0.0)));  // R[i, kp]
      x = csub(x, cmul(xk, ri));
      const cplx vn = mk(cr * hi + sv * v.re, ci * hi + sv * v.im);
      const double bx = fabs(x.re) + fabs(x.im), bv = fabs(vn.re) + fabs(vn.im);
      if (bx > nxb) nxb = bx;
      if (bv > nvb) nvb = bv;
      Vr[IX(i)] = vn.re;
      Vi[IX(i)] = vn.im;
      Xr[IX(i)] = x.re;
      Xi[IX(i)] = x.im;
    }
    SP_MARK();  // 7: row update
    if (pl == (kp - 1) % DP) {  // the shifted row (diagonal entry h - lambda)
      const int i = kp - 1;
      const double hi = hcol[i];
      const cplx v = mk(Vr[IX(i)], Vi[IX(i)]);
      cplx x = mk(Xr[IX(i)], Xi[IX(i)]);
      const cplx ri = csub(cmul(ccj, v), cmul(svc, csub(mk(hi, 0.0), mk(lre, lim))));
      x = csub(x, cmul(xk, ri));
      const double tre = hi - lre, tim = -lim;
      const cplx vn = mk((cr * tre - ci * tim) + sv * v.re, (cr * tim + ci * tre) + sv * v.im);
      Vr[IX(i)] = vn.re;
      Vi[IX(i)] = vn.im;
      Xr[IX(i)] = x.re;
      Xi[IX(i)] = x.im;
    }
    xb = nxb;
    vb = nvb;
    SP_MARK();  // 8: shifted row
    cp_wait<0>();
    HSRQ_SYNCWARP();
    SP_MARK();  // 9: column prefetch wait, warp barrier
    cur ^= 1;
  }
  SP_FLUSH(10);
  // j = 0: cross-tile rotation (creduce_diag :449-463) and R[0,0] (:546-550)
  const cplx v0 = mk(Vr[IX(0)], Vi[IX(0)]);
  cplx x0 = mk(Xr[IX(0)], Xi[IX(0)]);
  HSRQ_SYNCWARP();  // row 0 read by every lane before lane 0 rescales / overwrites it
  double c0r = 1.0, c0i = 0.0, s0 = 0.0;
  cplx d = v0;
  if (a.has_left) {
    const double al = a.tile_mode ? a.t_hleft[0] : c.H[(a.js - 1) * c.ldh + a.js];
    const double absv = ghypot(v0.re, v0.im);
    const double r = ghypot(al, absv);
    if (live && r == 0.0) {
      if (pl == 0) record_fail(c, a, q, HSRQ_KIND_DEGENERATE, 0);
      live = false;
    }
    c0r = v0.re / r;
    c0i = v0.im / r;
    s0 = -al / r;
    d = csub(cmul(mk(c0r, -c0i), v0), cmul(mk(s0, 0.0), mk(al, 0.0)));
  }
  if (live && pl == 0) put_rot(c, a, q, 0, c0r, c0i, s0);
  if (live && d.re == 0.0 && d.im == 0.0) {
    if (pl == 0) record_fail(c, a, q, HSRQ_KIND_SINGULAR, 0);
    live = false;
  }
  if (robust && live) {
    const double ad = cabs_(d), ax = cabs_(x0);
    if (ad < 1.0 && ax > ad * omega) {
      const int e = pow2floor_e(ad * omega / ax);
      const cplx xi = mk(p2(e), 0.0);
      for (int i = pl; i < k; i += DP) {
        const cplx t = cmul(mk(Xr[IX(i)], Xi[IX(i)]), xi);
        Xr[IX(i)] = t.re;
        Xi[IX(i)] = t.im;
      }
      x0 = cmul(x0, xi);
      gexp += e;
    }
  }
  x0 = cdiv(x0, d);
  if (pl == 0) {
    Xr[IX(0)] = x0.re;
    Xi[IX(0)] = x0.im;
  }
  HSRQ_SYNCWARP();
  if (live) {
    for (int i = pl; i < k; i += DP) {
      if (a.tile_mode) {
        const int64_t b2 = 2 * (int64_t)a.t_b;
        a.t_x[i * b2 + 2 * q] = Xr[IX(i)];
        a.t_x[i * b2 + 2 * q + 1] = Xi[IX(i)];
      } else {
        c.X[col * c.ldx + a.js + i] = Xr[IX(i)];
        c.X[(col + 1) * c.ldx + a.js + i] = Xi[IX(i)];
      }
    }
  }
  if (a.tile_mode) {
    if (live && pl == 0) a.t_beta[q] += gexp;
    return;
  }
  if (live && pl == 0) c.E[(int64_t)a.jt * c.ms + q] += gexp;
  if (a.jt == 0) return;

  diag_cplx_operands<DP>(c, a, q, col, live, pl, grp, k, Xr, Xi, Vr, Vi, c0r, c0i, s0, x0);
#undef IX
}
