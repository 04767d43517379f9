// hsrq_diag_ws.cuh -- warp-specialised complex diagonal sweep (included by
// hsrq_kernels.cu after hsrq_diag.cuh).
//
// Same arithmetic as k_diag_cplx (creduce_diag numba_backend.py:420-464 +
// robust_trsv_complex :493-527, bit-identical), but each group of 32/DP
// shifts is run by a PAIR of warps sharing the tile's v / x in shared memory:
//
//   chain warp (role 0): the pivot chain of step kp -- hypot, the three
//     divisions, R[kp,kp], the provisional x_kp -- then, after the step's
//     guards, the store of x_kp and the shifted row kp-1;
//   bulk warp (role 1): the O(kp) row update of step kp+1 (rows < kp) and
//     the guard-2 maxima it produces, while the chain warp works on step kp.
//
// The row update of step kp+1 only touches rows < kp and the chain of step kp
// only reads row kp (the previous shifted row), so the two overlap; they meet
// at one pair barrier per step (P).  After P both warps evaluate the guards
// from the same shared values (the decisions are identical, so the barriers
// they gate are taken by both), split the rare exact passes and rescalings
// by rows, and carry on.  Exchange slots written in one step and read in the
// next are double-buffered by the step's parity.  Column buffers are
// triple-buffered: the chain warp prefetches column kp-2 while the bulk warp
// still reads column kp.

#undef HSRQ_FUZZ_FILE
#define HSRQ_FUZZ_FILE 2u
__device__ __forceinline__ void pair_sync(int id) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory");
#ifdef HSRQ_FUZZ
  fuzz_delay((unsigned)id | (HSRQ_FUZZ_FILE << 16));
#endif
}

template <int DP, int NP>
__global__ void __launch_bounds__(NP * 64) k_diag_cplx_ws(Ctx c, DiagArgs a) {
  constexpr int DG = 32 / DP;
  constexpr int PAIR = 4 * MAXK * DG + 3 * MAXK + 32 * DG;
  extern __shared__ __align__(16) double dsm[];
  double* hmax = dsm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;
  const int bar = 1 + pair;
  const int grp = lane / DP, pl = lane % DP;
  double* Vr = dsm + MAXK + pair * PAIR;
  double* Vi = Vr + MAXK * DG;
  double* Xr = Vi + MAXK * DG;
  double* Xi = Xr + MAXK * DG;
  double* hb = Xi + MAXK * DG;  // [3][MAXK] column buffers, column t in slot t % 3
  double* ex = hb + 3 * MAXK;   // [32][DG] exchange slots
#define IX(i) ((i) * DG + grp)
#define CH(p, s) ex[((p) * 10 + (s)) * DG + grp]   // chain results of step kp, p = kp & 1
#define XB(p, s) ex[(20 + (p) * 2 + (s)) * DG + grp]  // guard-2 maxima for step kp
#define E2(s, r) ex[(24 + (s) * 2 + (r)) * DG + grp]  // exact-pass partial maxima
  const int k = a.k;
  load_hmax(c, a, hmax);
  const int64_t q = a.q0 + ((int64_t)blockIdx.x * NP + pair) * DG + grp;
  bool live = q < a.q0 + a.count;
  if (live && !a.tile_mode && c.fail[q] != 0) live = false;
  const int64_t col = a.tile_mode ? 0 : 2 * q;
  const double lre = live ? c.lam_re[q] : 0.0, lim = live ? c.lam_im[q] : 0.0;
  const double omega = c.omega;
  const bool robust = c.robust;
  auto HB = [&](int t) { return hb + (t % 3) * MAXK; };

  if (role == 1) {  // tile load and the first step's bounds
    double xb = 0.0, vb = 0.0;
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
    xb = gmax<DP>(xb);
    vb = gmax<DP>(vb);
    if (pl == 0 && k >= 2) {
      XB((k - 1) & 1, 0) = xb;
      XB((k - 1) & 1, 1) = vb;
    }
  } else if (k >= 2) {
    fill_col(c, a, HB(k - 2), k - 2, k, lane);
  }
  pair_sync(bar);

  int gexp = 0;
  cplx bxk = mk(0.0, 0.0);  // bulk warp: step kp+1's x_kp and rotation
  double bcr = 0.0, bci = 0.0, bsv = 0.0;
  for (int kp = k - 1; kp >= 1; --kp) {
    const int p = kp & 1;
    if (role == 0) {
      // ---- chain of step kp (column kp-1; row kp = the last shifted row) ----
      if (kp >= 2) {
        fill_col(c, a, HB(kp - 2), kp - 2, kp, lane);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      HSRQ_SYNCWARP();
      const double* hcol = HB(kp - 1);
      const cplx vk = mk(Vr[IX(kp)], Vi[IX(kp)]);
      const cplx xk = mk(Xr[IX(kp)], Xi[IX(kp)]);
      const double av = hcol[kp];
      const double absv = ghypot(vk.re, vk.im);
      const double r = ghypot(av, absv);
      if (live && r == 0.0) {
        if (pl == 0) record_fail(c, a, q, HSRQ_KIND_DEGENERATE, kp);
        live = false;
      }
      const double cr = vk.re / r, ci = vk.im / r, sv = -av / r;
      if (live && pl == 0) put_rot(c, a, q, kp, cr, ci, sv);
      const cplx d = csub(cmul(mk(cr, -ci), vk), cmul(mk(sv, 0.0), mk(av, 0.0)));
      if (live && d.re == 0.0 && d.im == 0.0) {
        if (pl == 0) record_fail(c, a, q, HSRQ_KIND_SINGULAR, kp);
        live = false;
      }
      const cplx xq = cdiv(xk, d);
      if (pl == 0) {
        CH(p, 0) = cr;
        CH(p, 1) = ci;
        CH(p, 2) = sv;
        CH(p, 3) = d.re;
        CH(p, 4) = d.im;
        CH(p, 5) = xk.re;
        CH(p, 6) = xk.im;
        CH(p, 7) = xq.re;
        CH(p, 8) = xq.im;
        CH(p, 9) = live ? 1.0 : 0.0;
      }
    } else if (kp < k - 1) {
      // ---- row update of step kp+1 (column kp, rows < kp) ----
      const double* hcol = HB(kp);
      const cplx ccj = mk(bcr, -bci), svc = mk(bsv, 0.0);
      double nxb = 0.0, nvb = 0.0;
#pragma unroll 1
      for (int i = pl; i < kp; i += DP) {
        const double hi = hcol[i];
        const cplx v = mk(Vr[IX(i)], Vi[IX(i)]);
        cplx x = mk(Xr[IX(i)], Xi[IX(i)]);
        const cplx ri = csub(cmul(ccj, v), cmul(svc, mk(hi, 0.0)));  // R[i, kp+1]
        x = csub(x, cmul(bxk, ri));
        const cplx vn = mk(bcr * hi + bsv * v.re, bci * hi + bsv * v.im);
        const double bx = fabs(x.re) + fabs(x.im), bv = fabs(vn.re) + fabs(vn.im);
        if (bx > nxb) nxb = bx;
        if (bv > nvb) nvb = bv;
        Vr[IX(i)] = vn.re;
        Vi[IX(i)] = vn.im;
        Xr[IX(i)] = x.re;
        Xi[IX(i)] = x.im;
      }
      nxb = gmax<DP>(nxb);
      nvb = gmax<DP>(nvb);
      if (pl == 0) {
        XB(p, 0) = nxb;
        XB(p, 1) = nvb;
      }
    }
    pair_sync(bar);  // P: chain of kp and rows of kp+1 done

    // ---- guards of step kp, evaluated identically by both warps ----
    const double cr = CH(p, 0), ci = CH(p, 1), sv = CH(p, 2);
    const cplx d = mk(CH(p, 3), CH(p, 4)), xk0 = mk(CH(p, 5), CH(p, 6));
    cplx xk = mk(CH(p, 7), CH(p, 8));
    const bool lv = CH(p, 9) != 0.0;
    double xb = XB(p, 0), vb = XB(p, 1);
    const double* hcol = HB(kp - 1);
    bool g1 = false;
    int e1 = 0;
    if (robust && lv) {  // guard 1 (robust_trsv_complex :501-508)
      const double adlo = fmax(fabs(d.re), fabs(d.im));
      if (adlo < 1.0 && (fabs(xk0.re) + fabs(xk0.im)) * DSLACK > adlo * omega) {
        const double ad = cabs_(d), ax = cabs_(xk0);
        if (ad < 1.0 && ax > ad * omega) {
          g1 = true;
          e1 = pow2floor_e(ad * omega / ax);
        }
      }
    }
    if (__any_sync(FULL, g1)) {
      if (g1) {
        const cplx xi = mk(p2(e1), 0.0);
        for (int i = pl + DP * role; i < k; i += 2 * DP) {
          const cplx t = cmul(mk(Xr[IX(i)], Xi[IX(i)]), xi);
          Xr[IX(i)] = t.re;
          Xi[IX(i)] = t.im;
        }
        xk = cdiv(cmul(xk0, xi), d);
        xb = xb * xi.re + 0x1p-1070;
        gexp += e1;
      }
      pair_sync(bar);
    }
    // guard 2 (:510-523), certified as in k_diag_cplx, rows split over the pair
    bool exact2 = false;
    double rb = 0.0;
    if (robust && lv) {
      rb = ((fabs(cr) + fabs(ci)) * vb + fabs(sv) * (hmax[kp] + fabs(lre) + fabs(lim))) * DSLACK;
      exact2 = !protect_update_is_one(xb * DSLACK, rb, (fabs(xk.re) + fabs(xk.im)) * DSLACK, omega);
    }
    if (__any_sync(FULL, exact2)) {
      const cplx ccj = mk(cr, -ci), svc = mk(sv, 0.0);
      const int ex_ = ilogb_pos(xb), er_ = ilogb_pos(rb);
      const double sx = p2(-max(-1000, min(1020, ex_))), sr = p2(-max(-1000, min(1020, er_)));
      // |x_kp| for the certification, issued ahead of the row pass
      const double ax = exact2 ? cabs_(xk) : 0.0;
      double tx = 0.0, tr = 0.0;
#pragma unroll 1
      for (int i = pl + DP * role; i < kp; i += 2 * DP) {
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
      if (pl == 0) {
        E2(0, role) = tx;
        E2(1, role) = tr;
      }
      pair_sync(bar);
      {
        const double x0 = E2(0, 0), x1 = E2(0, 1), r0 = E2(1, 0), r1 = E2(1, 1);
        tx = x1 > x0 ? x1 : x0;
        tr = r1 > r0 ? r1 : r0;
      }
      bool full = false;
      int e = 0;
      if (exact2) {
        if (ex_ > -1000 && ex_ < 1020 && er_ > -1000 && er_ < 1020 && tx >= 0x1p-960 &&
            tr >= 0x1p-960 && tx <= 16.0 && tr <= 16.0) {
          const double qx = sqrt(tx), qr = sqrt(tr);
          const double bl = (qx - qx * 0x1p-47) * p2(ex_), bh = (qx + qx * 0x1p-47) * p2(ex_);
          const double rl = (qr - qr * 0x1p-47) * p2(er_), rh = (qr + qr * 0x1p-47) * p2(er_);
          int eh;
          protect_update_e2(bl, rl, bh, rh, ax, omega, e, eh);
          full = e != eh;
        } else {
          full = true;
        }
      }
      if (__any_sync(FULL, full)) {  // exact glibc moduli (rare)
        double rm = 0.0, bm = 0.0;
        for (int i = pl + DP * role; i < kp; i += 2 * DP) {
          cplx t = mk(hcol[i], 0.0);
          if (i == kp - 1) t = csub(t, mk(lre, lim));
          const cplx ri = csub(cmul(ccj, mk(Vr[IX(i)], Vi[IX(i)])), cmul(svc, t));
          const double q1 = cabs_(ri), q2 = cabs_(mk(Xr[IX(i)], Xi[IX(i)]));
          if (q1 > rm) rm = q1;
          if (q2 > bm) bm = q2;
        }
        rm = gmax<DP>(rm);
        bm = gmax<DP>(bm);
        if (pl == 0) {
          E2(2, role) = rm;
          E2(3, role) = bm;
        }
        pair_sync(bar);
        const double r0 = E2(2, 0), r1 = E2(2, 1), b0 = E2(3, 0), b1 = E2(3, 1);
        rm = r1 > r0 ? r1 : r0;
        bm = b1 > b0 ? b1 : b0;
        if (full) e = protect_update_e(bm, rm, ax, omega);
      }
      const bool g2 = exact2 && e < 0;
      if (__any_sync(FULL, g2)) {
        if (g2) {
          const cplx xi = mk(p2(e), 0.0);
          for (int i = pl + DP * role; i < k; i += 2 * DP) {
            const cplx t = cmul(mk(Xr[IX(i)], Xi[IX(i)]), xi);
            Xr[IX(i)] = t.re;
            Xi[IX(i)] = t.im;
          }
          xk = cmul(xk, xi);
          gexp += e;
        }
        pair_sync(bar);
      }
    }
    if (role == 0) {
      if (pl == (kp % DP)) {
        Xr[IX(kp)] = xk.re;
        Xi[IX(kp)] = xk.im;
      }
      if (pl == (kp - 1) % DP) {  // the shifted row (diagonal entry h - lambda)
        const int i = kp - 1;
        const double hi = hcol[i];
        const cplx v = mk(Vr[IX(i)], Vi[IX(i)]);
        cplx x = mk(Xr[IX(i)], Xi[IX(i)]);
        const cplx ri = csub(cmul(mk(cr, -ci), v), cmul(mk(sv, 0.0), csub(mk(hi, 0.0), mk(lre, lim))));
        x = csub(x, cmul(xk, ri));
        const double tre = hi - lre, tim = -lim;
        const cplx vn = mk((cr * tre - ci * tim) + sv * v.re, (cr * tim + ci * tre) + sv * v.im);
        Vr[IX(i)] = vn.re;
        Vi[IX(i)] = vn.im;
        Xr[IX(i)] = x.re;
        Xi[IX(i)] = x.im;
      }
      HSRQ_SYNCWARP();
    } else {
      bxk = xk;
      bcr = cr;
      bci = ci;
      bsv = sv;
    }
  }
  if (role == 1) return;  // the rest is per shift, sequential: chain warp only

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
#undef CH
#undef XB
#undef E2
}

// Real shifts, same pairing (reduce_diag :75-106 + solve_rsolve :133-195).
// Guard 1 depends only on the pivot and x_kp, so the chain warp resolves it
// before the barrier and passes the final x_kp / phi and the exponent; guard
// 2 is protect_update on the bulk warp's exact maxima.
template <int DP, int NP>
__global__ void __launch_bounds__(NP * 64) k_diag_real_ws(Ctx c, DiagArgs a) {
  constexpr int DG = 32 / DP;
  constexpr int PAIR = 2 * MAXK * DG + 3 * MAXK + 16 * DG;
  extern __shared__ __align__(16) double dsm[];
  double* hmax = dsm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;
  const int bar = 1 + pair;
  const int grp = lane / DP, pl = lane % DP;
  double* V = dsm + MAXK + pair * PAIR;
  double* Xs = V + MAXK * DG;
  double* hb = Xs + MAXK * DG;  // [3][MAXK]
  double* ex = hb + 3 * MAXK;   // [16][DG]
#define VV(i) V[(i) * DG + grp]
#define XX(i) Xs[(i) * DG + grp]
#define CH(p, s) ex[((p) * 5 + (s)) * DG + grp]
#define XB(p, s) ex[(10 + (p) * 2 + (s)) * DG + grp]
  const int k = a.k;
  load_hmax(c, a, hmax);
  const int64_t q = a.q0 + ((int64_t)blockIdx.x * NP + pair) * DG + grp;
  bool live = q < a.q0 + a.count;
  if (live && !a.tile_mode && c.fail[q] != 0) live = false;
  const int64_t col = a.tile_mode ? 0 : 2 * c.mc + (q - c.mc);
  const double lam = live ? c.lam_re[q] : 0.0;
  const double omega = c.omega;
  const bool robust = c.robust;
  auto HB = [&](int t) { return hb + (t % 3) * MAXK; };

  if (role == 1) {
    double xm = 0.0, vm = 0.0;
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
    xm = gmax<DP>(xm);
    vm = gmax<DP>(vm);
    if (pl == 0 && k >= 2) {
      XB((k - 1) & 1, 0) = xm;
      XB((k - 1) & 1, 1) = vm;
    }
  } else if (k >= 2) {
    fill_col(c, a, HB(k - 2), k - 2, k, lane);
  }
  pair_sync(bar);

  int gexp = 0;
  double bcc = 0.0, bss = 0.0, bxk = 0.0;  // bulk warp: step kp+1's rotation and x
  for (int kp = k - 1; kp >= 1; --kp) {
    const int p = kp & 1;
    if (role == 0) {
      if (kp >= 2) {
        fill_col(c, a, HB(kp - 2), kp - 2, kp, lane);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      HSRQ_SYNCWARP();
      const double* hcol = HB(kp - 1);
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
      int e1 = 0;
      if (robust && live) {  // guard 1 (:144-151)
        const double aphi = fabs(phi), ax = fabs(xk);
        if (aphi < 1.0 && ax > aphi * omega) {
          e1 = pow2floor_e(aphi * omega / ax);
          xk *= p2(e1);
        }
      }
      xk = xk / phi;
      if (pl == 0) {
        CH(p, 0) = cc;
        CH(p, 1) = ss;
        CH(p, 2) = xk;
        CH(p, 3) = (double)e1;
        CH(p, 4) = live ? 1.0 : 0.0;
      }
    } else if (kp < k - 1) {
      // row update of step kp+1 (column kp, rows < kp)
      const double* hcol = HB(kp);
      const double tau1 = bss * bxk, tau2 = bcc * bxk;
      double nxm = 0.0, nvm = 0.0;
#pragma unroll 1
      for (int i = pl; i < kp; i += DP) {
        const double hi = hcol[i];
        double vv = VV(i), xx = XX(i);
        xx = (xx - tau2 * vv) + tau1 * hi;
        vv = bcc * hi + bss * vv;
        if (fabs(xx) > nxm) nxm = fabs(xx);
        if (fabs(vv) > nvm) nvm = fabs(vv);
        VV(i) = vv;
        XX(i) = xx;
      }
      nxm = gmax<DP>(nxm);
      nvm = gmax<DP>(nvm);
      if (pl == 0) {
        XB(p, 0) = nxm;
        XB(p, 1) = nvm;
      }
    }
    pair_sync(bar);  // P

    const double cc = CH(p, 0), ss = CH(p, 1);
    double xk = CH(p, 2);
    const int e1 = (int)CH(p, 3);
    const bool lv = CH(p, 4) != 0.0;
    double xm = XB(p, 0);
    const double vm = XB(p, 1);
    if (__any_sync(FULL, e1 != 0)) {  // guard 1's rescaling of the other rows
      if (e1 != 0) {
        const double xi = p2(e1);
        for (int i = pl + DP * role; i < k; i += 2 * DP) XX(i) *= xi;
        xm *= xi;
        gexp += e1;
      }
      pair_sync(bar);
    }
    int e2 = 0;
    if (robust && lv) e2 = protect_update_e(xm, vm + hmax[kp] + fabs(lam), fabs(xk), omega);
    if (__any_sync(FULL, e2 < 0)) {  // guard 2 (:153-168)
      if (e2 < 0) {
        const double xi = p2(e2);
        for (int i = pl + DP * role; i < k; i += 2 * DP) XX(i) *= xi;
        xk *= xi;
        gexp += e2;
      }
      pair_sync(bar);
    }
    if (role == 0) {
      if (pl == (kp % DP)) XX(kp) = xk;
      if (pl == (kp - 1) % DP) {  // the shifted row (diagonal entry h - lambda)
        const int i = kp - 1;
        const double hd = HB(kp - 1)[i] - lam;
        const double vv = VV(i), xx = XX(i);
        XX(i) = (xx - (cc * xk) * vv) + (ss * xk) * hd;
        VV(i) = cc * hd + ss * vv;
      }
      HSRQ_SYNCWARP();
    } else {
      bcc = cc;
      bss = ss;
      bxk = xk;
    }
  }
  if (role == 1) return;
  diag_real_tail<DP>(c, a, q, col, live, pl, grp, k, V, Xs, gexp, robust);
#undef VV
#undef XX
#undef CH
#undef XB
}
