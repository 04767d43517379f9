// hsrq_tile_update.cuh -- tile-level entry of the panel kernels (included at
// the end of hsrq_kernels.cu): the reference's operator API for one
// off-diagonal tile,
//
//   update_rupdate / cupdate_crupdate   numba_backend.py:198-311, 579-736
//   reduce_offdiag / creduce_offdiag    numba_backend.py:109-125, 467-490
//
// run through the PRODUCTION kernels of the sweep: the panel operands come
// from the diagonal sweep's operand code (diag_real_operands /
// diag_cplx_operands: W_j = c_j prod_{t<j} s_t, P, Z, the step scalars),
// update steps 1-2 from k_scalars, the GEMM A [W | Zs] with the crossover and
// step 3 from k_panel.  The tile is embedded in a synthetic problem whose
// sweep column jt has exactly the caller's tile as its panel:
//
//   shift_active = 1: two tile rows (b_r = m, n = m + k, jt = 1): tile row 0
//     is the super-diagonal tile (the update subtracts lambda rho on its last
//     row, the crossover lambda c0 on it -- reduce_offdiag's shifted form);
//   shift_active = 0: three tile rows (n = 2m + k, jt = 2): tile row 0 is a
//     far tile (no lambda anywhere; reduce_offdiag with lam = 0, as
//     reduce.py:148-156 calls it for such tiles).
//
// H holds the tile at H[0:m, js-1 : js-1+k], X the caller's b (tile row 0)
// and x_below (tile jt), the crossover column jt the caller's r_right, the
// rotation tables the caller's c / s at rows js.., the segment exponents
// alpha (tile jt) and beta (tile row 0).  Results: b updated in place, beta
// <- delta, and r_left (the new crossover column jt-1 of tile row 0).

__global__ void k_tile_place(Ctx c, int m, int k, int b, int cplx, int64_t js,
                             const double* htile, const double* rright, const double* xbelow,
                             const double* bio, const int32_t* aexp, const int32_t* bexp,
                             const double* cre, const double* cim, const double* s) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int w = cplx ? 2 * b : b;  // interleaved columns of the caller's arrays
  // H tile, column t0 of the tile = H column js - 1 + t0
  if (t < (int64_t)m * k) {
    const int i = (int)(t / k), t0 = (int)(t % k);
    const_cast<double*>(c.H)[(js - 1 + t0) * c.ldh + i] = htile[t];
  }
  // b (tile row 0) and r_right into X / Cr; x_below into X rows js..
  if (t < (int64_t)m * w) {
    const int i = (int)(t / w), l = (int)(t % w);
    c.X[(int64_t)l * c.ldx + i] = bio[t];
    c.Cr[(int64_t)l * c.ldx + i] = rright[t];
  }
  if (t < (int64_t)k * w) {
    const int i = (int)(t / w), l = (int)(t % w);
    c.X[(int64_t)l * c.ldx + js + i] = xbelow[t];
  }
  if (t < (int64_t)k * b) {  // rotations of tile jt, row i of shift q
    const int i = (int)(t / b), q = (int)(t % b);
    c.c_re[(int64_t)q * c.ldc + js + i] = cre[t];
    c.c_im[(int64_t)q * c.ldc + js + i] = cplx ? cim[t] : 0.0;
    c.s[(int64_t)q * c.ldc + js + i] = s[t];
  }
  if (t < b) {
    const int jt = (int)(js / c.b_r);
    c.E[(int64_t)jt * c.ms + t] = aexp[t];
    c.E[t] = bexp[t];
  }
}

// XB: max |b| (real) / max(|re| + |im|) (complex) of every tile row, the
// bound k_scalars starts from (the panel epilogue maintains it in a sweep).
__global__ void k_tile_xb(Ctx c) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)c.N * c.ms) return;
  const int tile = (int)(t / c.ms);
  const int64_t q = t % c.ms;
  bool cplx;
  int64_t col;
  col_of_shift(c, q, cplx, col);
  const int64_t r0 = (int64_t)tile * c.b_r, r1 = r0 + c.b_r < c.n ? r0 + c.b_r : c.n;
  double mx = 0.0;
  for (int64_t r = r0; r < r1; r++) {
    const double v = cplx ? fabs(c.X[col * c.ldx + r]) + fabs(c.X[(col + 1) * c.ldx + r])
                          : fabs(c.X[col * c.ldx + r]);
    if (v > mx) mx = v;
  }
  c.XB[t] = mx;
  c.XB[(int64_t)c.N * c.ms + t] = 0.0;
}

// The diagonal sweep's operand code on the caller's x_below and rotations:
// one warp per shift (32 lanes per shift), x in shared memory.
__global__ void __launch_bounds__(128) k_tile_operands(Ctx c, DiagArgs a) {
  __shared__ double sm[4][4 * MAXK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * 4 + warp;
  if (q >= c.ms) return;  // warp-uniform
  double* Xr = sm[warp];
  double* Xi = Xr + MAXK;
  double* Vr = Xi + MAXK;
  double* Vi = Vr + MAXK;
  bool cplx;
  int64_t col;
  col_of_shift(c, q, cplx, col);
  const int k = a.k;
  for (int i = lane; i < k; i += 32) {
    Xr[i] = c.X[col * c.ldx + a.js + i];
    Xi[i] = cplx ? c.X[(col + 1) * c.ldx + a.js + i] : 0.0;
  }
  __syncwarp();
  const double c0r = c.c_re[q * c.ldc + a.rot_off], s0 = c.s[q * c.ldc + a.rot_off];
  if (cplx) {
    const double c0i = c.c_im[q * c.ldc + a.rot_off];
    diag_cplx_operands<32>(c, a, q, col, true, lane, 0, k, Xr, Xi, Vr, Vi, c0r, c0i, s0,
                           mk(Xr[0], Xi[0]));
  } else {
    diag_real_operands<32>(c, a, q, col, true, lane, 0, k, Vr, Xr, c0r, s0, Xr[0]);
  }
}

// b (tile row 0 of X) and r_left (tile row 0 of Cr) back to the caller's
// row-major (m, w) arrays; beta <- delta (E row 0).
__global__ void k_tile_result(Ctx c, int m, int w, double* bio, double* rleft, int32_t* bexp) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < (int64_t)m * w) {
    const int i = (int)(t / w), l = (int)(t % w);
    bio[t] = c.X[(int64_t)l * c.ldx + i];
    if (rleft) rleft[t] = c.Cr[(int64_t)l * c.ldx + i];
  }
  if (t < c.ms) bexp[t] = c.E[t];
}

extern "C" int64_t hsrq_tile_update(int32_t m, int32_t k, int32_t b, int32_t cplx,
                                    const double* htile, const double* rright,
                                    const int32_t* alpha_exp, const double* xbelow,
                                    const double* lam_re, const double* lam_im,
                                    int32_t shift_active, const double* c_re, const double* c_im,
                                    const double* s, int32_t* beta_exp, double* b_io,
                                    double* rleft, int32_t robust, double omega, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (m < 1 || k < 2 || b < 1 || m > MAXK || k > m || (cplx && (!lam_im || !c_im))) {
    snprintf(g_err, sizeof(g_err), "hsrq_tile_update: need 2 <= k <= m <= %d, b >= 1", MAXK);
    return HSRQ_ERR_CONFIG;
  }
  if (const int64_t r = ensure_attrs(); r != 0) return r;
  const int ntiles = shift_active ? 2 : 3;
  const int jt = ntiles - 1;
  const int64_t n = (int64_t)(ntiles - 1) * m + k, js = (int64_t)jt * m;
  const int64_t ldh = n + (n & 1);
  const int64_t mc = cplx ? b : 0, mr = cplx ? 0 : b, ms = b, ncol = cplx ? 2 * b : b;
  const WsLayout L = ws_layout(n, m, mc, mr);
  // device scratch: the solve workspace, H, X, rotation tables, E, shifts, fail
  size_t off = align_up(L.total, 256);
  const size_t oH = off;
  off = align_up(off + sizeof(double) * ldh * n, 256);
  const size_t oX = off;
  off = align_up(off + sizeof(double) * n * ncol, 256);
  const size_t oT = off;
  off = align_up(off + 3 * sizeof(double) * n * ms, 256);
  const size_t oE = off;
  off = align_up(off + sizeof(int32_t) * ntiles * ms, 256);
  const size_t oL = off;
  off = align_up(off + 2 * sizeof(double) * ms, 256);
  const size_t oF = off;
  off = align_up(off + sizeof(int64_t) * ms, 256);
  unsigned char* wsp = nullptr;
  if (!ck(cudaMallocAsync((void**)&wsp, off, stream), "tile scratch")) return HSRQ_ERR_CUDA;
  auto fail = [&](const char* what) {
    cudaFreeAsync(wsp, stream);
    return what ? HSRQ_ERR_CUDA : 0;
  };
  if (!ck(cudaMemsetAsync(wsp, 0, off, stream), "zero")) return fail("zero");
  (void)oL;
  Ctx c;
  memset(&c, 0, sizeof(c));
  c.H = (const double*)(wsp + oH);
  c.ldh = ldh;
  c.n = n;
  c.b_r = m;
  c.N = ntiles;
  c.lam_re = (const double*)(wsp + oL);
  c.lam_im = c.lam_re + ms;
  c.mc = mc;
  c.mr = mr;
  c.ms = ms;
  c.ncol = ncol;
  c.ncol_pad = (ncol + BN - 1) / BN * BN;
  c.X = (double*)(wsp + oX);
  c.ldx = n;
  c.Cr = (double*)(wsp + L.cr);
  c.c_re = (double*)(wsp + oT);
  c.c_im = c.c_re + n * ms;
  c.s = c.c_im + n * ms;
  c.ldc = n;
  c.E = (int32_t*)(wsp + oE);
  c.Bop = (double*)(wsp + L.bop);
  c.SS = (StepScalars*)(wsp + L.ss);
  c.HM0 = (double*)(wsp + L.hm0);
  c.RS = (double*)(wsp + L.rs);
  c.XB = (double*)(wsp + L.xb);
  c.HMK = (double*)(wsp + L.hmk);
  c.fail = (int64_t*)(wsp + oF);
  c.nfail = (unsigned long long*)(wsp + L.nfail);
  c.robust = robust;
  c.mode = 1;
  c.compact = 0;
  c.Rt = (double*)(wsp + L.rt);
  c.omega = robust ? (omega > 0.0 ? omega : (1.7976931348623157e308 / 2.0) / (double)m) : HUGE_VAL;
  c.diag_tl_jt = -1;
  const int w = cplx ? 2 * b : b;
  const int64_t nt = std::max<int64_t>({(int64_t)m * std::max(k, w), (int64_t)k * w, (int64_t)k * b});
  double* lre = const_cast<double*>(c.lam_re);
  if (!ck(cudaMemcpyAsync(lre, lam_re, sizeof(double) * b, cudaMemcpyDeviceToDevice, stream),
          "lam") ||
      (cplx && !ck(cudaMemcpyAsync(lre + ms, lam_im, sizeof(double) * b, cudaMemcpyDeviceToDevice,
                                   stream), "lam")))
    return fail("lam");
  k_tile_place<<<(unsigned)((nt + 255) / 256), 256, 0, stream>>>(
      c, m, k, b, cplx, js, htile, rright, xbelow, b_io, alpha_exp, beta_exp, c_re, c_im, s);
  {
    dim3 gt((unsigned)((n + 255) / 256), (unsigned)(c.N - 1));
    k_tables<<<gt, 256, 0, stream>>>(c);
  }
  k_tile_xb<<<(unsigned)((c.N * ms + 127) / 128), 128, 0, stream>>>(c);
  DiagArgs a;
  memset(&a, 0, sizeof(a));
  a.jt = jt;
  a.js = js;
  a.k = k;
  a.has_left = 1;
  a.q0 = 0;
  a.count = ms;
  a.rot_off = js;
  k_tile_operands<<<(unsigned)((ms + 3) / 4), 128, 0, stream>>>(c, a);
  PanelArgs p;
  p.jt = jt;
  p.js = js;
  p.k = k;
  p.S = std::min(SMAX, std::max(1, BM / m));
  p.t0 = 0;
  p.t1 = jt;
  RowScalars* rsc = (RowScalars*)(wsp + L.rsc);
  k_scalars<<<(unsigned)((jt * ms + 127) / 128), 128, 0, stream>>>(c, p, rsc);
  const size_t panel_smem = sizeof(PanelSmem);
  const bool a16 = (ldh % 2 == 0) && (m % 2 == 0), seg16 = (m % 16) == 0;
  dim3 gp((unsigned)((jt + p.S - 1) / p.S), (unsigned)(c.ncol_pad / BN));
  if (a16 && m == BM && g_panel_fast)
    k_panel<true, true, true><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
  else if (a16 && seg16)
    k_panel<true, true, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
  else if (a16)
    k_panel<true, false, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
  else if (seg16)
    k_panel<false, true, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
  else
    k_panel<false, false, false><<<gp, PANEL_THREADS, panel_smem, stream>>>(c, p, rsc);
  if (!ck(cudaGetLastError(), "tile update launch")) return fail("launch");
  // results: b (tile row 0 of X), beta <- delta (E row 0), r_left (Cr tile row 0)
  k_tile_result<<<(unsigned)(((int64_t)m * w + 255) / 256), 256, 0, stream>>>(c, m, w, b_io, rleft,
                                                                              beta_exp);
  if (!ck(cudaGetLastError(), "tile result")) return fail("result");
  cudaFreeAsync(wsp, stream);
  return 0;
}
