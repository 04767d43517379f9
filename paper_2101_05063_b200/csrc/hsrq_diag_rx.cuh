// hsrq_diag_rx.cuh -- complex diagonal sweep with the rotation chain run one
// step ahead of the solution chain (included by hsrq_kernels.cu after
// hsrq_diag_ws.cuh).  For few shifts per GPU (DP = 32: one shift per warp,
// the 1/4 - 1/8 shards of config 5), where the sweep is a latency chain.
//
// Same arithmetic as k_diag_cplx (creduce_diag numba_backend.py:420-464 +
// _build_complex_r :530-551 + robust_trsv_complex :493-527), bit for bit.
// The step-kp recurrence splits into two chains that meet only through R's
// column kp:
//
//   R-warp (role 0): rotation kp from the shifted row v_kp and h(kp, kp-1)
//     (two glibc hypots, three divisions), the pivot d = R[kp, kp], R's
//     column kp (r_i = conj(c) v_i - s h_i, i < kp, with h - lambda on the
//     shifted row) and the v update of rows < kp -- it never reads x;
//   X-warp (role 1): the solution chain of step kp -- guard 1, the complex
//     pivot division, guard 2 (bound test, interval certification from the
//     squared moduli, exact glibc moduli at a binade edge), x_kp and the x
//     update x_i -= x_kp r_i -- reading R's column from shared memory.
//
// At loop iteration kp the R-warp computes step kp while the X-warp
// finishes step kp + 1; one pair barrier per iteration.  R's column and the
// step scalars are double-buffered by step parity.  The scaled maximum of
// |r_i|^2 the guard-2 certification needs is formed by the R-warp in the
// same pass as the column (its scale 2^-ilogb(rb) depends only on R-side
// values), so the X-warp's certification reads it instead of recomputing R.

#undef HSRQ_FUZZ_FILE
#define HSRQ_FUZZ_FILE 16u

template <int DP, int NP>
__host__ __device__ constexpr int diag_rx_pair() {
  return (8 * (32 / DP) + 2) * MAXK + 32 * (32 / DP);
}
template <int DP, int NP>
size_t diag_rx_smem() {
  return sizeof(double) * (MAXK + NP * diag_rx_pair<DP, NP>());
}

// DP lanes per shift (16 or 32: 32 / DP shifts per warp pair), NP pairs per CTA.
template <int DP, int NP>
__global__ void __launch_bounds__(NP * 64) k_diag_cplx_rx(Ctx c, DiagArgs a) {
  constexpr int DG = 32 / DP;
  constexpr int PAIR = diag_rx_pair<DP, NP>();
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
  double* hb = Xi + MAXK * DG;  // [2][MAXK] H columns (R-warp)
  double* Rs = hb + 2 * MAXK;   // [2][2][MAXK][DG] R's column, re / im, by step parity
  double* Ss = Rs + 4 * MAXK * DG;  // [2][16][DG] step scalars by parity
#define IX(i) ((i) * DG + grp)
#define RRE(p, i) Rs[(((p) * 2) * MAXK + (i)) * DG + grp]
#define RIM(p, i) Rs[(((p) * 2 + 1) * MAXK + (i)) * DG + grp]
#define SC(p, s) Ss[((p) * 16 + (s)) * DG + grp]
  const int k = a.k;
  load_hmax(c, a, hmax);
  const int64_t q = a.q0 + ((int64_t)blockIdx.x * NP + pair) * DG + grp;
  bool live = q < a.q0 + a.count;
  if (live && c.fail[q] != 0) live = false;
  const int64_t col = 2 * q;
  const double lre = live ? c.lam_re[q] : 0.0, lim = live ? c.lam_im[q] : 0.0;
  const double omega = c.omega;
  const bool robust = c.robust;

  // ---- tile load: each warp its own state and the first step's bound ----
  double bnd = 0.0;
  for (int i = pl; i < k; i += DP) {
    double re = 0.0, im = 0.0;
    if (live) {
      const double* src = role == 0 ? c.Cr : c.X;
      re = src[col * c.ldx + a.js + i];
      im = src[(col + 1) * c.ldx + a.js + i];
    }
    if (role == 0) {
      Vr[IX(i)] = re;
      Vi[IX(i)] = im;
    } else {
      Xr[IX(i)] = re;
      Xi[IX(i)] = im;
    }
    if (i < k - 1) {
      const double b = fabs(re) + fabs(im);
      if (b > bnd) bnd = b;
    }
  }
  bnd = gmax<DP>(bnd);  // R-warp: vb, X-warp: xb (rows < k-1)
  int cur = 0;
  if (role == 0 && k >= 2) {
    fill_col(c, a, hb, k - 2, k, lane);
    cp_wait<0>();
  }
  HSRQ_SYNCWARP();

  int gexp = 0;     // X-warp
  bool lv = live;   // X-warp: the step's liveness as the R-warp left it
#ifdef HSRQ_STEPPROF
  long long sp_t0 = clock64(), sp_acc[6] = {0};
#define RX_MARK(j) { const long long t_ = clock64(); sp_acc[j] += t_ - sp_t0; sp_t0 = t_; }
#else
#define RX_MARK(j) ((void)0)
#endif
  for (int kp = k - 1; kp >= 0; --kp) {
    if (role == 0) {
      if (kp >= 1) {
        // ---------------- R: rotation, pivot, R's column of step kp ----------------
        const int p = kp & 1;
        const double* hcol = hb + cur * MAXK;  // column kp-1, rows 0..kp
        if (kp >= 2) fill_col(c, a, hb + (cur ^ 1) * MAXK, kp - 2, kp, lane);
        const cplx vk = mk(Vr[IX(kp)], Vi[IX(kp)]);
        const double av = hcol[kp];
        RX_MARK(0);
        const double absv = ghypot(vk.re, vk.im);
        const double r = ghypot(av, absv);
        RX_MARK(1);
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
        // guard 2's bound of max|r_i| and the certification's scale (k_diag_cplx)
        const double rb =
            (robust && live)
                ? ((fabs(cr) + fabs(ci)) * bnd + fabs(sv) * (hmax[kp] + fabs(lre) + fabs(lim))) * DSLACK
                : 0.0;
        const int er = ilogb_pos(rb);
        const double sr = p2(-max(-1000, min(1020, er)));
        RX_MARK(2);
        double tr = 0.0, nvb = 0.0;
        for (int i = pl; i < kp - 1; i += DP) {
          const double hi = hcol[i];
          const cplx v = mk(Vr[IX(i)], Vi[IX(i)]);
          const cplx ri = csub(cmul(ccj, v), cmul(svc, mk(hi, 0.0)));  // R[i, kp]
          RRE(p, i) = ri.re;
          RIM(p, i) = ri.im;
          const double a1 = ri.re * sr, b1 = ri.im * sr;
          const double t1 = a1 * a1 + b1 * b1;
          tr = t1 > tr ? t1 : tr;
          const cplx vn = mk(cr * hi + sv * v.re, ci * hi + sv * v.im);
          const double bv = fabs(vn.re) + fabs(vn.im);
          if (bv > nvb) nvb = bv;
          Vr[IX(i)] = vn.re;
          Vi[IX(i)] = vn.im;
        }
        if (pl == (kp - 1) % DP) {  // the shifted row (diagonal entry h - lambda)
          const int i = kp - 1;
          const double hi = hcol[i];
          const cplx v = mk(Vr[IX(i)], Vi[IX(i)]);
          const cplx ri = csub(cmul(ccj, v), cmul(svc, csub(mk(hi, 0.0), mk(lre, lim))));
          RRE(p, i) = ri.re;
          RIM(p, i) = ri.im;
          const double a1 = ri.re * sr, b1 = ri.im * sr;
          const double t1 = a1 * a1 + b1 * b1;
          tr = t1 > tr ? t1 : tr;
          const double tre = hi - lre, tim = -lim;
          Vr[IX(i)] = (cr * tre - ci * tim) + sv * v.re;
          Vi[IX(i)] = (cr * tim + ci * tre) + sv * v.im;
        }
        RX_MARK(3);
        tr = gmax<DP>(tr);
        bnd = gmax<DP>(nvb);
        if (pl == 0) {
          SC(p, 0) = cr;
          SC(p, 1) = ci;
          SC(p, 2) = sv;
          SC(p, 3) = d.re;
          SC(p, 4) = d.im;
          SC(p, 5) = rb;
          SC(p, 6) = tr;
          SC(p, 7) = (double)er;
          SC(p, 8) = live ? 1.0 : 0.0;
        }
        cp_wait<0>();
        HSRQ_SYNCWARP();
        cur ^= 1;
        RX_MARK(4);
      }
    } else if (kp + 1 <= k - 1) {
      // ---------------- X: the solution chain of step s = kp + 1 ----------------
      const int s = kp + 1;
      const int p = s & 1;
      const cplx d = mk(SC(p, 3), SC(p, 4));
      const double rb = SC(p, 5), tr0 = SC(p, 6);
      const int er = (int)SC(p, 7);
      lv = SC(p, 8) != 0.0;
      RX_MARK(5);
      cplx xk = mk(Xr[IX(s)], Xi[IX(s)]);
      HSRQ_SYNCWARP();  // row s read by every lane before its owner rescales / overwrites it
      double xb = bnd;
      if (robust && lv) {  // guard 1 (robust_trsv_complex :501-508)
        const double adlo = fmax(fabs(d.re), fabs(d.im));
        if (adlo < 1.0 && (fabs(xk.re) + fabs(xk.im)) * DSLACK > adlo * omega) {
          const double ad = cabs_(d), ax = cabs_(xk);
          if (ad < 1.0 && ax > ad * omega) {
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
      RX_MARK(0);
      xk = cdiv(xk, d);
      RX_MARK(1);
      // guard 2 (:510-523): protect_update(max|x_i|, max|r_i|, |x_kp|), i < kp
      bool exact2 = false;
      if (robust && lv)
        exact2 = !protect_update_is_one(xb * DSLACK, rb, (fabs(xk.re) + fabs(xk.im)) * DSLACK, omega);
      if (__any_sync(FULL, exact2)) {
        const int ex = ilogb_pos(xb);
        const double sx = p2(-max(-1000, min(1020, ex)));
        double tx = 0.0;
        for (int i = pl; i < s; i += DP) {
          const double a2 = Xr[IX(i)] * sx, b2 = Xi[IX(i)] * sx;
          const double t2 = a2 * a2 + b2 * b2;
          tx = t2 > tx ? t2 : tx;
        }
        tx = gmax<DP>(tx);
        const double tr = tr0;
        bool full = false;
        int e = 0;
        const double ax = exact2 ? cabs_(xk) : 0.0;
        if (exact2) {
          if (ex > -1000 && ex < 1020 && er > -1000 && er < 1020 && tx >= 0x1p-960 &&
              tr >= 0x1p-960 && tx <= 16.0 && tr <= 16.0) {
            const double qx = sqrt(tx), qr = sqrt(tr);
            const double bl = (qx - qx * 0x1p-47) * p2(ex), bh = (qx + qx * 0x1p-47) * p2(ex);
            const double rl = (qr - qr * 0x1p-47) * p2(er), rh = (qr + qr * 0x1p-47) * p2(er);
            int eh;
            protect_update_e2(bl, rl, bh, rh, ax, omega, e, eh);
            full = e != eh;
          } else {
            full = true;
          }
        }
        if (__any_sync(FULL, full)) {  // exact glibc moduli (rare)
          double rm = 0.0, bm = 0.0;
          for (int i = pl; i < s; i += DP) {
            const double q1 = cabs_(mk(RRE(p, i), RIM(p, i))), q2 = cabs_(mk(Xr[IX(i)], Xi[IX(i)]));
            if (q1 > rm) rm = q1;
            if (q2 > bm) bm = q2;
          }
          rm = gmax<DP>(rm);
          bm = gmax<DP>(bm);
          if (full) e = protect_update_e(bm, rm, ax, omega);
        }
        if (exact2 && e < 0) {
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
      RX_MARK(2);
      if (pl == (s % DP)) {
        Xr[IX(s)] = xk.re;
        Xi[IX(s)] = xk.im;
      }
      double nxb = 0.0;
      for (int i = pl; i < s - 1; i += DP) {
        const cplx ri = mk(RRE(p, i), RIM(p, i));
        const cplx x = csub(mk(Xr[IX(i)], Xi[IX(i)]), cmul(xk, ri));
        const double bx = fabs(x.re) + fabs(x.im);
        if (bx > nxb) nxb = bx;
        Xr[IX(i)] = x.re;
        Xi[IX(i)] = x.im;
      }
      if (pl == (s - 1) % DP) {  // the shifted row
        const int i = s - 1;
        const cplx x = csub(mk(Xr[IX(i)], Xi[IX(i)]), cmul(xk, mk(RRE(p, i), RIM(p, i))));
        Xr[IX(i)] = x.re;
        Xi[IX(i)] = x.im;
      }
      bnd = gmax<DP>(nxb);
      HSRQ_SYNCWARP();
      RX_MARK(3);
    }
    pair_sync(bar);
    RX_MARK(role == 0 ? 5 : 4);
  }
#ifdef HSRQ_STEPPROF
  if (lane == 0 && pair == 0) {
    for (int j = 0; j < 6; j++) atomicAdd(&g_stepprof[role * 6 + j], (unsigned long long)sp_acc[j]);
    if (role == 0) atomicAdd(&g_stepprof[15], 1ULL);
  }
#endif
#undef RX_MARK
  if (role == 0) return;  // the rest is per shift, sequential: X-warp only
  live = lv;

  // j = 0: cross-tile rotation (creduce_diag :449-463) and R[0,0] (:546-550)
  const cplx v0 = mk(Vr[IX(0)], Vi[IX(0)]);
  cplx x0 = mk(Xr[IX(0)], Xi[IX(0)]);
  HSRQ_SYNCWARP();  // row 0 read by every lane before lane 0 rescales / overwrites it
  double c0r = 1.0, c0i = 0.0, s0 = 0.0;
  cplx d = v0;
  if (a.has_left) {
    const double al = c.H[(a.js - 1) * c.ldh + a.js];
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
      c.X[col * c.ldx + a.js + i] = Xr[IX(i)];
      c.X[(col + 1) * c.ldx + a.js + i] = Xi[IX(i)];
    }
  }
  if (live && pl == 0) c.E[(int64_t)a.jt * c.ms + q] += gexp;
  if (a.jt == 0) return;
  diag_cplx_operands<DP>(c, a, q, col, live, pl, grp, k, Xr, Xi, Vr, Vi, c0r, c0i, s0, x0);
#undef IX
#undef RRE
#undef RIM
#undef SC
}
