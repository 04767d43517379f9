// hsrq_panel_cl.cuh -- k_panel for b_r = 128 as 2-CTA clusters (included by
// hsrq_kernels.cu after hsrq_panel.cuh).
//
// Same arithmetic as k_panel's fast path (epilogue_b128), bit for bit: the
// GEMM acc = A [W | Zs] on DMMA in the same K order, then update steps 1 and
// 3 and the crossover.  What changes is the shape: a tile row (128 rows) is
// split over a cluster of two 64-row, 4-warp CTAs, so four CTAs share an SM
// instead of two 8-warp ones, and while one of them runs its guarded
// epilogue three keep the DMMA pipe fed (two 8-warp CTAs: the lone GEMM CTA
// reached 71 % of the pair's rate, which exposed ~90 ms of epilogue per
// config-5 solve).  Step 3's guard needs maxima over the whole tile row:
// each CTA reduces its 64 rows and PUSHES them into its peer's shared memory
// (distributed shared memory stores, one cluster barrier), and both evaluate
// the identical guard from local memory -- the rare exact-moduli path
// likewise.  Nothing reads remote memory after a barrier, so a CTA may exit
// while its peer still works: no trailing cluster barriers.  The next
// column's XB bound is written per half (c.XB / c.XB + N ms), its reader
// (k_scalars) takes the larger.

#undef HSRQ_FUZZ_FILE
#define HSRQ_FUZZ_FILE 4u

namespace cg = cooperative_groups;

constexpr int CL_BM = 64;                 // rows per CTA (half a tile row)
constexpr int CL_THREADS = 128;           // 4 warps: 2 (M) x 2 (N) warp tiles of 32 x 32
constexpr int CL_STAGES = 2;
constexpr int CL_ROWS = 8;                // epilogue: threads per column pair
constexpr int CL_RPT = CL_BM / CL_ROWS;   // rows per thread (8)
// C row stride: the epilogue's four column pairs per warp read rows 4 apart;
// 4 * 66 doubles = 16 banks mod 32, so they pair up on the two 128-byte
// wavefronts a 64-bit warp read needs anyway (stride 68: all four collide)
constexpr int CL_CPAD = CL_BM + 2;
#ifndef CL_MINB
#define CL_MINB 4  // resident CTAs per SM the register budget is sized for
#endif

struct PanelClSmem {
  union {
    struct {
      double A[CL_STAGES][BK][CL_BM + 4];
      double B[CL_STAGES][2 * BN][BPAD];
    } pipe;
    double C[2 * BN][CL_CPAD];  // accumulators, [acc col][row]
  } u;
  RowScalars rsc[BN];
  unsigned long long red[2][BN];    // pass-1 maxima of this CTA's rows
  unsigned long long redp[2][BN];   // ... of the peer's rows (written by the peer)
  unsigned long long hred[2][BN];   // exact glibc-moduli maxima (rare path)
  unsigned long long hredp[2][BN];  // ... of the peer's rows (written by the peer)
  double x3[BN], z3r[BN], z3i[BN];
  int dex[BN];
  int need[BN];
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CL_THREADS, CL_MINB)
    k_panel_cl(Ctx c, PanelArgs p, const RowScalars* __restrict__ RSc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PanelClSmem& sm = *reinterpret_cast<PanelClSmem*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();  // 0: rows 0..63 of the tile row, 1: rows 64..127
  PanelClSmem& peer = *cluster.map_shared_rank(&sm, rank ^ 1u);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile0 = p.t0 + (int)(blockIdx.x >> 1);
  const int64_t row0 = (int64_t)tile0 * BM + rank * CL_BM;
  const int64_t col0 = (int64_t)blockIdx.y * BN;
  const int nk = BK == 0 ? 0 : p.k / BK;  // p.k == 128 on this path
  const int jt = p.jt;
  const bool robust = c.robust;

  // ---- operand loads: 16-byte cp.async, 4 A + 4 B copies per thread per K chunk ----
  const int kk0 = tid / 32, m2 = (tid % 32) * 2;
  const double* a0 = c.H + (p.js - 1 + kk0) * c.ldh + row0 + m2;
  const int nn = tid / 8, k2 = (tid % 8) * 2;
  const double* b0 = c.Bop + (2 * col0 + nn) * KP + k2;
  auto load = [&](int stage, int kc) {
    const double* a = a0 + (int64_t)kc * BK * c.ldh;
#pragma unroll
    for (int i = 0; i < 4; i++)
      cp_async16(&sm.u.pipe.A[stage][kk0 + 4 * i][m2], a + (int64_t)4 * i * c.ldh, true);
    const double* b = b0 + kc * BK;
#pragma unroll
    for (int i = 0; i < 4; i++)
      cp_async16(&sm.u.pipe.B[stage][nn + 16 * i][k2], b + 16 * i * KP, true);
  };
  // Remote shared memory may only be touched once the peer CTA is known to
  // run: arrive at the cluster barrier now, wait for it right before the
  // push of the maxima (long satisfied by then, so the wait costs nothing).
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  load(0, 0);
  cp_commit();
  if (g_panel_prefetch) {  // this CTA's epilogue tiles (X, Cr: 32 columns x 64 rows) towards L2
    for (int L = tid; L < 2 * BN * (CL_BM / 16); L += CL_THREADS) {
      const int arr = L / (BN * (CL_BM / 16)), cc = (L / (CL_BM / 16)) % BN, seg = L % (CL_BM / 16);
      const int64_t col = col0 + cc;
      if (col < c.ncol) {
        const double* a = (arr ? c.Cr : c.X) + col * c.ldx + row0 + seg * 16;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      }
    }
  }
  for (int cc = tid; cc < BN; cc += CL_THREADS) {
    const int64_t col = col0 + cc;
    if (col < c.ncol) {
      const int64_t q = col < 2 * c.mc ? col / 2 : c.mc + (col - 2 * c.mc);
      sm.rsc[cc] = RSc[(int64_t)tile0 * c.ms + q];
    }
    sm.need[cc] = 0;
  }

  // ---------------- main loop: acc = A [W | Zs] on DMMA ----------------
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, t4 = lane & 3;
  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int e = 0; e < 4; e++) acc[i][j][e] = 0.0;
  for (int kc = 0; kc < nk; kc++) {
    cp_wait<CL_STAGES - 2>();
    HSRQ_SYNCTHREADS();
    if (kc + 1 < nk) load((kc + 1) % CL_STAGES, kc + 1);
    cp_commit();
    const int st = kc % CL_STAGES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[2][2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 2; mi++) {
        const int r = wm * 32 + mi * 16 + g;
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
  HSRQ_SYNCTHREADS();
#pragma unroll
  for (int mi = 0; mi < 2; mi++)
#pragma unroll
    for (int ni = 0; ni < 4; ni++) {
      const int r = wm * 32 + mi * 16 + g;
      const int cc = wn * 32 + ni * 8 + 2 * t4;
      sm.u.C[cc][r] = acc[mi][ni][0];
      sm.u.C[cc + 1][r] = acc[mi][ni][1];
      sm.u.C[cc][r + 8] = acc[mi][ni][2];
      sm.u.C[cc + 1][r + 8] = acc[mi][ni][3];
    }
  HSRQ_SYNCTHREADS();

  // ---------------- epilogue (epilogue_b128 on 64 rows, guards cluster-wide) ----------------
  const int pc = tid / CL_ROWS, rp = tid % CL_ROWS;
  const int cl0 = 2 * pc;
  const int64_t gc0 = col0 + cl0;
  const bool cplx = gc0 < 2 * c.mc;
  const bool v0 = gc0 < c.ncol, v1 = gc0 + 1 < c.ncol;
  const int64_t q0 = cplx ? gc0 / 2 : c.mc + (gc0 - 2 * c.mc);
  const int64_t q1 = cplx ? q0 : q0 + 1;
  // shifted tile (i = jt-1): its last row (rank 1, rp 7, j 7) carries the lambda terms
  const int jlast = (tile0 == jt - 1 && rank == 1 && rp == CL_ROWS - 1) ? CL_RPT - 1 : -1;
  double* __restrict__ X0 = c.X + gc0 * c.ldx + row0;
  double* __restrict__ C0 = c.Cr + gc0 * c.ldx + row0;
  const double* __restrict__ H0 = c.H + (p.js - 1) * c.ldh + row0;
  double xa[CL_RPT], xb[CL_RPT], ca[CL_RPT], cb[CL_RPT], hh[CL_RPT];
#pragma unroll
  for (int j = 0; j < CL_RPT; j++) {
    const int r = rp + CL_ROWS * j;
    xa[j] = v0 ? X0[r] : 0.0;
    xb[j] = v1 ? X0[c.ldx + r] : 0.0;
    ca[j] = v0 ? C0[r] : 0.0;
    cb[j] = v1 ? C0[c.ldx + r] : 0.0;
    hh[j] = H0[r];
  }
  const StepScalars st0 = c.SS[v0 ? q0 : 0];
  const StepScalars st1 = c.SS[v1 ? q1 : 0];
  const double lr0 = v0 ? c.lam_re[q0] : 0.0, li0 = (v0 && cplx) ? c.lam_im[q0] : 0.0;
  const double lr1 = v1 ? c.lam_re[q1] : 0.0;
  const RowScalars s0 = sm.rsc[cl0], s1 = sm.rsc[cl0 + 1];
  const double pz0 = s0.fx * s0.x2, pz1 = s1.fx * s1.x2;
  const double* Z0 = sm.u.C[2 * cl0 + 1];
  const double* Z1 = sm.u.C[2 * cl0 + 3];
  // ---- pass 1: X'' and the step-3 maxima ----
  double mb0 = 0.0, mb1 = 0.0, mr0 = 0.0, mr1 = 0.0;
  if (cplx) {
    const double fb = s0.fb, rr = s0.rr, ri = s0.ri, x2 = s0.x2;
#pragma unroll
    for (int j = 0; j < CL_RPT; j++) {
      const int r = rp + CL_ROWS * j;
      double xr = xa[j], xi = xb[j];
      if (fb != 1.0) {
        xr *= fb;
        xi *= fb;
      }
      xr += rr * hh[j];
      xi += ri * hh[j];
      if (j == jlast) {
        xr -= lr0 * rr - li0 * ri;
        xi -= lr0 * ri + li0 * rr;
      }
      if (x2 < 1.0) {
        xr *= x2;
        xi *= x2;
      }
      xr -= pz0 * Z0[r];
      xi -= pz1 * Z1[r];
      xa[j] = xr;
      xb[j] = xi;
      mb0 = fmax(mb0, fabs(xr) + fabs(xi));
      mr0 = fmax(mr0, fabs(ca[j]) + fabs(cb[j]));
    }
    mb1 = mb0;
    mr1 = mr0;
  } else {
#pragma unroll
    for (int j = 0; j < CL_RPT; j++) {
      const int r = rp + CL_ROWS * j;
      double x0 = xa[j], x1 = xb[j];
      if (s0.fb != 1.0) x0 *= s0.fb;
      if (s1.fb != 1.0) x1 *= s1.fb;
      x0 += s0.rr * hh[j];
      x1 += s1.rr * hh[j];
      if (j == jlast) {
        x0 -= lr0 * s0.rr;
        x1 -= lr1 * s1.rr;
      }
      if (s0.x2 < 1.0) x0 *= s0.x2;
      if (s1.x2 < 1.0) x1 *= s1.x2;
      x0 -= pz0 * Z0[r];
      x1 -= pz1 * Z1[r];
      xa[j] = x0;
      xb[j] = x1;
      mb0 = fmax(mb0, fabs(x0));
      mb1 = fmax(mb1, fabs(x1));
      mr0 = fmax(mr0, fabs(ca[j]));
      mr1 = fmax(mr1, fabs(cb[j]));
    }
  }
#pragma unroll
  for (int o = 1; o < CL_ROWS; o <<= 1) {
    mb0 = fmax(mb0, __shfl_xor_sync(0xffffffffu, mb0, o));
    mb1 = fmax(mb1, __shfl_xor_sync(0xffffffffu, mb1, o));
    mr0 = fmax(mr0, __shfl_xor_sync(0xffffffffu, mr0, o));
    mr1 = fmax(mr1, __shfl_xor_sync(0xffffffffu, mr1, o));
  }
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // the peer CTA has started
  if (rp == 0) {
    sm.red[0][cl0] = peer.redp[0][cl0] = dkey(mb0);
    sm.red[0][cl0 + 1] = peer.redp[0][cl0 + 1] = dkey(mb1);
    sm.red[1][cl0] = peer.redp[1][cl0] = dkey(mr0);
    sm.red[1][cl0 + 1] = peer.redp[1][cl0 + 1] = dkey(mr1);
  }
  cluster.sync();  // both halves' maxima in both CTAs (pushed through distributed shared memory)
  // ---- step 3 guard (:287-301), one thread per column, on the tile row's maxima ----
  int my_need = 0;
  if (tid < BN) {
    const int cc = tid;
    const int64_t col = col0 + cc;
    if (col < c.ncol) {
      const RowScalars& s = sm.rsc[cc];
      double zr = s.zkr, zi = s.zki, x3 = 1.0;
      int dx = s.dexp;
      if (robust) {
        const unsigned long long kb = sm.red[0][cc] > sm.redp[0][cc] ? sm.red[0][cc] : sm.redp[0][cc];
        const unsigned long long kr = sm.red[1][cc] > sm.redp[1][cc] ? sm.red[1][cc] : sm.redp[1][cc];
        const double bb = dval(kb), rb = dval(kr);
        if (col < 2 * c.mc) {
          if (!protect_update_is_one(bb * BOUND_SLACK, rb * BOUND_SLACK,
                                     (fabs(zr) + fabs(zi)) * BOUND_SLACK, c.omega)) {
            sm.need[cc] = 1;
            my_need = 1;
          }
        } else {
          const int xe = protect_update_e(bb, rb, fabs(zr), c.omega);
          if (xe < 0) {
            x3 = p2(xe);
            dx += xe;
            zr *= x3;
          }
        }
      }
      sm.x3[cc] = x3;
      sm.z3r[cc] = zr;
      sm.z3i[cc] = zi;
      sm.dex[cc] = dx;
    }
  }
  // identical decisions in both CTAs (same maxima), so both take this branch
  if (__syncthreads_or(my_need)) {  // rare: exact glibc moduli for flagged complex columns
    double hb = 0.0, hr = 0.0;
    if (cplx && v0) {
#pragma unroll
      for (int j = 0; j < CL_RPT; j++) {
        hb = fmax(hb, ghypot(xa[j], xb[j]));
        hr = fmax(hr, ghypot(ca[j], cb[j]));
      }
    }
#pragma unroll
    for (int o = 1; o < CL_ROWS; o <<= 1) {
      hb = fmax(hb, __shfl_xor_sync(0xffffffffu, hb, o));
      hr = fmax(hr, __shfl_xor_sync(0xffffffffu, hr, o));
    }
    if (rp == 0 && cplx) {
      sm.hred[0][cl0] = peer.hredp[0][cl0] = dkey(hb);
      sm.hred[1][cl0] = peer.hredp[1][cl0] = dkey(hr);
    }
    cluster.sync();
    if (tid < BN && sm.need[tid]) {
      const int cc = tid, ccr = cc & ~1;
      const unsigned long long kb = sm.hred[0][ccr] > sm.hredp[0][ccr] ? sm.hred[0][ccr] : sm.hredp[0][ccr];
      const unsigned long long kr = sm.hred[1][ccr] > sm.hredp[1][ccr] ? sm.hred[1][ccr] : sm.hredp[1][ccr];
      const double zr = sm.z3r[cc], zi = sm.z3i[cc];
      const int xe = protect_update_e(dval(kb), dval(kr), ghypot(zr, zi), c.omega);
      if (xe < 0) {
        const double x3 = p2(xe);
        sm.x3[cc] = x3;
        sm.dex[cc] += xe;
        sm.z3r[cc] = zr * x3;
        sm.z3i[cc] = zi * x3;
      }
    }
    HSRQ_SYNCTHREADS();
  }
  // ---- pass 2: X''' = x3 X'' - Cr_old zk ; Cr_new = A W + P Cr_old - c0 lambda e_{js-1} ----
  const double* W0 = sm.u.C[2 * cl0];
  const double* W1 = sm.u.C[2 * cl0 + 2];
  mb0 = mb1 = 0.0;
  if (cplx) {
    const double x3 = sm.x3[cl0];
    const double zr = sm.z3r[cl0], zi = sm.z3i[cl0];
    const double zr1 = sm.z3r[cl0 + 1], zi1 = sm.z3i[cl0 + 1];
    const double P = st0.P, c0r = st0.c0_re, c0i = st0.c0_im;
#pragma unroll
    for (int j = 0; j < CL_RPT; j++) {
      const int r = rp + CL_ROWS * j;
      double x0 = xa[j], x1 = xb[j];
      if (x3 < 1.0) {
        x0 *= x3;
        x1 *= x3;
      }
      x0 -= ca[j] * zr - cb[j] * zi;
      x1 -= ca[j] * zi1 + cb[j] * zr1;
      double n0 = W0[r] + P * ca[j];
      double n1 = W1[r] + P * cb[j];
      if (j == jlast) {
        n0 -= c0r * lr0 - c0i * li0;
        n1 -= c0r * li0 + c0i * lr0;
      }
      if (v0) {
        X0[r] = x0;
        C0[r] = n0;
        X0[c.ldx + r] = x1;
        C0[c.ldx + r] = n1;
      }
      mb0 = fmax(mb0, fabs(x0) + fabs(x1));
    }
    mb1 = mb0;
  } else {
    const double x30 = sm.x3[cl0], x31 = sm.x3[cl0 + 1];
    const double z0 = sm.z3r[cl0], z1 = sm.z3r[cl0 + 1];
#pragma unroll
    for (int j = 0; j < CL_RPT; j++) {
      const int r = rp + CL_ROWS * j;
      double x0 = xa[j], x1 = xb[j];
      if (x30 < 1.0) x0 *= x30;
      if (x31 < 1.0) x1 *= x31;
      x0 -= ca[j] * z0;
      x1 -= cb[j] * z1;
      double n0 = W0[r] + st0.P * ca[j];
      double n1 = W1[r] + st1.P * cb[j];
      if (j == jlast) {
        n0 -= st0.c0_re * lr0;
        n1 -= st1.c0_re * lr1;
      }
      if (v0) {
        X0[r] = x0;
        C0[r] = n0;
      }
      if (v1) {
        X0[c.ldx + r] = x1;
        C0[c.ldx + r] = n1;
      }
      mb0 = fmax(mb0, fabs(x0));
      mb1 = fmax(mb1, fabs(x1));
    }
  }
#pragma unroll
  for (int o = 1; o < CL_ROWS; o <<= 1) {
    mb0 = fmax(mb0, __shfl_xor_sync(0xffffffffu, mb0, o));
    mb1 = fmax(mb1, __shfl_xor_sync(0xffffffffu, mb1, o));
  }
  // new beta (rank 0) and this half's share of the step-1 bound for the next tile column
  if (rp == 0) {
    const int64_t half = (int64_t)rank * c.N * c.ms;
    const int64_t ix0 = (int64_t)tile0 * c.ms + q0;
    if (v0) {
      if (robust && rank == 0) c.E[ix0] = sm.dex[cl0];
      c.XB[half + ix0] = mb0;
    }
    if (v1 && !cplx) {
      const int64_t ix1 = (int64_t)tile0 * c.ms + q1;
      if (robust && rank == 0) c.E[ix1] = sm.dex[cl0 + 1];
      c.XB[half + ix1] = mb1;
    }
  }
}
