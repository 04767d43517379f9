/*
 * hsrq.h -- C ABI of libhsrq_b200.so, the B200 implementation of the batched
 * shifted-Hessenberg robust RQ solve (H - lambda_j I) x_j = s_j b_j
 * (arXiv 2101.05063) behind the reference hessrq package's inverse-iteration
 * seam.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/hessrq):
 *
 *   hsrq_solve_group   _solve_group, inviter.py:91-106 (tiled_reduce,
 *                      reduce.py:39-171, + robust_tiled_solve(mode="eigvec"),
 *                      backsolve.py:329-347) and, with mode=0 / robust=0,
 *                      the dhsrq3/chsrq3 engine backsolve.py:350-388.
 *                      Returns what SolutionBlock (core.py:251-260) carries:
 *                      x, per-column alpha, segment scales, represented norms.
 *   hsrq_solve_group_host  the same seam with host (numpy) buffers, as
 *                      _solve_group is called (inviter.py:127-133)
 *   hsrq_henry_solve   henry_rq_solve, reference.py:21-60 (kernels
 *                      henry_solve_real / henry_solve_complex,
 *                      numba_backend.py:830-923): Henry's single-sweep
 *                      baseline solver, bit-identical to the reference
 *   hsrq_compact_encode / hsrq_compact_decode
 *                      GivensTable.compact / from_compact (core.py:193-209,
 *                      givens.py:90-198): Stewart's compact rotation codes
 *   hsrq_hessenberg_reduce / hsrq_backmultiply
 *                      householder_hessenberg (testprob.py:146-174) and
 *                      z = Q0 x: the front end
 *   hsrq_protect_update_batch   protect_update, _kernels/numba_backend.py:47-67
 *   hsrq_hypot_batch            libm hypot as bound by numba (every rotation)
 *   hsrq_h_upload / hsrq_pack_download
 *                      the host side of dhsrq3in / chsrq3in / hsrq3in
 *                      (inviter.py:155-254): HessenbergMatrix's copy and
 *                      checks (core.py:60-98) and the result assembly
 *   hsrq_tile_diag              reduce_diag + solve_rsolve (numba_backend.py:
 *                               75-106, 133-195) and creduce_diag +
 *                               csolve_crsolve (:420-464, :554-576) on one
 *                               diagonal tile: the tile-level operator API
 *                               (_kernels/__init__.py) for parity tests.
 *
 * Conventions: every pointer argument is DEVICE memory unless its name ends
 * in _host.  Plain C types only; `stream` is a cudaStream_t passed as void*.
 * All calls are stream-ordered and re-entrant per stream; the library keeps
 * no global state besides cached device attributes.  H is never written.
 *
 * Shift / column layout.  A solve group holds m_cplx complex shifts
 * (Im > 0; the caller conjugates, as chsrq3in does, inviter.py:164-183)
 * followed by m_real real shifts: shift q < m_cplx is complex and owns the
 * two real columns 2q (re) and 2q+1 (im); shift q >= m_cplx is real and owns
 * column 2*m_cplx + (q - m_cplx).  ncol = 2*m_cplx + m_real.  Column-major
 * n x ncol blocks (X, B) use leading dimension ldx / ldb.
 *
 * Scale factors are returned as int32 log2 exponents: the reference's double
 * is ldexp(1, e).  This is bit-identical to the reference wherever
 * e >= -1074 and keeps working where the reference underflows to 0
 * (SURVEY.md §0 finding 6).
 */
#ifndef HSRQ_B200_H
#define HSRQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSRQ_KIND_DEGENERATE 1 /* numba_backend.py:17 */
#define HSRQ_KIND_SINGULAR 2   /* numba_backend.py:18 */

/* Flag or-ed into `mode` of the solve entry points: store the recorded
 * rotations in Stewart's compact form (GivensTable.compact(), core.py:193-209,
 * givens.py:90-198) -- c_re holds the code t of a real shift / t1 of a
 * complex shift, c_im holds t2 of complex shift q < m_cplx (row q), s is
 * not used (may be NULL): 2 instead of 3 reals per complex rotation, 1
 * instead of 2 per real one.  The backtransform decodes the codes. */
#define HSRQ_MODE_COMPACT_ROTATIONS 0x10

/* Error codes (negative returns). */
#define HSRQ_ERR_CONFIG (-1)   /* b_r outside [1, 128], n < 1, bad sizes */
#define HSRQ_ERR_WORKSPACE (-2) /* workspace too small */
#define HSRQ_ERR_CUDA (-3)     /* a CUDA call failed; see hsrq_last_error() */

/* Library version string and the last CUDA error text (thread-local). */
const char* hsrq_version(void);
const char* hsrq_last_error(void);

/* Bytes of device workspace hsrq_solve_group needs. */
size_t hsrq_workspace_bytes(int64_t n, int32_t b_r, int64_t m_cplx, int64_t m_real);

/*
 * Robust tiled RQ solve for one group of shifts (see header comment).
 *
 *  H        n x n column-major, leading dimension ldh (>= n)
 *  lam_re   m_cplx + m_real shift real parts (complex first, then real)
 *  lam_im   imaginary parts (entries for real shifts are ignored)
 *  B        right-hand sides: b_broadcast = 0 -> n x ncol column-major
 *           (ldb); b_broadcast = 1 -> one real n-vector used for every
 *           column (imaginary parts 0), the start vector _iterate repeats
 *           (inviter.py:127-133)
 *  X        out, n x ncol column-major (ldx; this build requires ldx == n,
 *           the in-place crossover block shares X's layout); may alias B
 *           when ldb == ldx
 *  c_re, c_im, s   out, recorded rotations, n x (m_cplx + m_real) column-major
 *           (ldc), row j mixing columns j-1 and j (GivensTable, core.py:168-179);
 *           c_im is written as 0 for real shifts
 *  seg_exp  out, N x (m_cplx + m_real) int32, N = ceil(n / b_r): segment
 *           scale exponents (ScalingMatrix, core.py:234-248), row-major by tile
 *  alpha_exp out, per-shift column scale exponent (alpha_min, or the solve
 *           mode's extra guard, numba_backend.py:326-375)
 *  norms    out, represented 2-norm as the reference's double (may be +inf)
 *  log2norm out, log2 of the represented norm (finite where norms is inf)
 *  fail     out, per shift: 0, or (phase << 56) | (tile << 24) | row of the
 *           first failure (phase 1 = degenerate rotation, 2 = singular factor)
 *  robust   1 = robust_tiled_solve (Omega = DBL_MAX/2/b_r), 0 = tiled_solve
 *  mode     1 = eigvec (normalise), 0 = solve; | HSRQ_MODE_COMPACT_ROTATIONS
 *           for compact rotation storage
 *  ws       workspace of >= hsrq_workspace_bytes(...) bytes
 *
 * Returns the number of failed shifts (>= 0) after synchronising `stream`,
 * or a negative HSRQ_ERR_*.
 */
int64_t hsrq_solve_group(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                         const double* lam_re, const double* lam_im, int64_t m_cplx,
                         int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                         double* X, int64_t ldx, double* c_re, double* c_im, double* s,
                         int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                         double* log2norm, int64_t* fail, int32_t robust, int32_t mode, void* ws,
                         size_t ws_bytes, void* stream);

/* hsrq_solve_group with the caller's overflow budget: omega > 0 is
 * OverflowBudget.omega (overflow.py:31-47; dhsrq3 / chsrq3 budget=,
 * backsolve.py:342-346) in (0, DBL_MAX/2]; omega = 0 means the default
 * DBL_MAX/2/b_r (robust = 0 ignores it: omega = inf). */
int64_t hsrq_solve_group_omega(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                               const double* lam_re, const double* lam_im, int64_t m_cplx,
                               int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                               double* X, int64_t ldx, double* c_re, double* c_im, double* s,
                               int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                               double* log2norm, int64_t* fail, int32_t robust, int32_t mode,
                               double omega, void* ws, size_t ws_bytes, void* stream);

/* Same, but asynchronous: returns 0 once every kernel is enqueued (or a
 * negative error); the failure count is left in the workspace and read with
 * hsrq_failure_count (which synchronises the stream). */
int64_t hsrq_solve_group_async(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                               const double* lam_re, const double* lam_im, int64_t m_cplx,
                               int64_t m_real, const double* B, int64_t ldb,
                               int32_t b_broadcast, double* X, int64_t ldx, double* c_re,
                               double* c_im, double* s, int64_t ldc, int32_t* seg_exp,
                               int32_t* alpha_exp, double* norms, double* log2norm,
                               int64_t* fail, int32_t robust, int32_t mode, void* ws,
                               size_t ws_bytes, void* stream);
int64_t hsrq_failure_count(void* ws, void* stream);

/*
 * CUDA-graph form of one solve group, for callers that repeat a solve of the
 * same shape on the same buffers (new shifts or right-hand sides written into
 * lam_re / lam_im / B between launches): hsrq_graph_capture runs the solve
 * once eagerly, then captures the whole sweep (every kernel, the side-stream
 * forks and joins) into an executable graph returned in *graph_out;
 * hsrq_graph_launch replays it on `stream` (one launch instead of ~12 per
 * tile column -- what matters for small, launch-bound problems); the
 * failure count is read with hsrq_failure_count(ws, stream).  Timing
 * (hsrq_set_timing) must be off.  hsrq_graph_destroy frees the graph.
 */
int64_t hsrq_graph_capture(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                           const double* lam_re, const double* lam_im, int64_t m_cplx,
                           int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                           double* X, int64_t ldx, double* c_re, double* c_im, double* s,
                           int64_t ldc, int32_t* seg_exp, int32_t* alpha_exp, double* norms,
                           double* log2norm, int64_t* fail, int32_t robust, int32_t mode, void* ws,
                           size_t ws_bytes, void* stream, void** graph_out);
int64_t hsrq_graph_launch(void* graph, void* stream);
void hsrq_graph_destroy(void* graph);

/*
 * Host-buffer variant of hsrq_solve_group -- the calling convention of the
 * reference's _solve_group (numpy arrays in, SolutionBlock arrays out), for
 * a ctypes / FFI binding without any device-array library.  Every pointer is
 * HOST memory except dev_ws (device workspace of at least
 * hsrq_host_workspace_bytes(n, b_r, m_cplx, m_real) bytes, reusable across
 * calls).  H is copied to the device in column blocks from right to left on
 * an internal copy stream, overlapped with the sweep (which consumes H in that
 * order); use page-locked (pinned) host buffers for the overlap.  lam_im may
 * be NULL when m_cplx == 0.  B as in hsrq_solve_group (b_broadcast = 1: one
 * n-vector).  Outputs: X (n x ncol, ldx), seg_exp (N x (m_cplx + m_real)),
 * alpha_exp, norms, log2norm, fail -- as hsrq_solve_group; the rotations stay
 * on the device (the reference does not return them from _solve_group).
 * Returns the number of failed shifts after synchronising `stream`, or a
 * negative HSRQ_ERR_*.
 */
size_t hsrq_host_workspace_bytes(int64_t n, int32_t b_r, int64_t m_cplx, int64_t m_real);
int64_t hsrq_solve_group_host(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                              const double* lam_re, const double* lam_im, int64_t m_cplx,
                              int64_t m_real, const double* B, int64_t ldb, int32_t b_broadcast,
                              double* X, int64_t ldx, int32_t* seg_exp, int32_t* alpha_exp,
                              double* norms, double* log2norm, int64_t* fail, int32_t robust,
                              int32_t mode, void* dev_ws, size_t dev_ws_bytes, void* stream);

/*
 * Asynchronous host-buffer solve: the same arguments and results as
 * hsrq_solve_group_host, but the call returns a ticket (>= 0) as soon as
 * everything is enqueued; hsrq_host_wait(ticket) waits for that solve's
 * outputs to be on the host and returns its number of failed shifts.  X and
 * the small outputs travel on their own D2H stream, so a caller that keeps
 * two solves in flight (two device workspaces, two sets of host outputs)
 * downloads solve i while solve i+1 sweeps -- how hsrq3in's w_max groups or
 * a stream of solve groups hide the transfers.  The upload of H starts at
 * once (it does not wait for earlier work on `stream`), so a device
 * workspace may only be passed again after the ticket of its previous solve
 * has been waited.  At most 16 tickets are outstanding per host thread.
 */
int64_t hsrq_solve_group_host_async(const double* H, int64_t ldh, int64_t n, int32_t b_r,
                                    const double* lam_re, const double* lam_im, int64_t m_cplx,
                                    int64_t m_real, const double* B, int64_t ldb,
                                    int32_t b_broadcast, double* X, int64_t ldx, int32_t* seg_exp,
                                    int32_t* alpha_exp, double* norms, double* log2norm,
                                    int64_t* fail, int32_t robust, int32_t mode, void* dev_ws,
                                    size_t dev_ws_bytes, void* stream);
int64_t hsrq_host_wait(int64_t ticket);

/* Guard-path event counters (diagnostics): out_host[32]; reset != 0 zeroes them. */
int64_t hsrq_debug_counters(int64_t* out_host, int32_t reset);
/* Diagnostics build -DHSRQ_STEPPROF only (returns 0 otherwise): per-phase
 * clock64 sums of the complex diagonal sweep's steps ([0..9]) and the number
 * of profiled warps ([15]); out_host holds 16 entries. */
int64_t hsrq_debug_stepprof(int64_t* out_host, int32_t reset);

/* Kernel launches issued by the last solve on this thread (for accounting). */
int64_t hsrq_last_launch_count(void);

/* Per-phase device times (ms), summed over the solves run with timing
 * enabled since the previous call (which this call waits for):
 * out_host[0] = diagonal kernels, [1] = panel GEMM kernels (k_panel), [2] =
 * backtransform, [3] = setup, [4] = guard-scalar kernels (k_scalars).
 * Enable with hsrq_set_timing(1): events around every phase, read back
 * here, so a timed solve is not synchronised by the timing itself.  With
 * the lookahead schedule the diagonal and panel intervals overlap. */
void hsrq_set_timing(int32_t enable);
void hsrq_phase_times(double* out_host);

/* Tuning / test hook for the diagonal-sweep variant (process-wide; the
 * HSRQ_DIAG / HSRQ_DIAG_WSR / HSRQ_DIAG_WS environment variables set the
 * same state).  dp = lanes per shift (0 = automatic), dwr / dwc = warps per
 * CTA of the real / complex sweep; wsr / wsc = warp pairs per CTA of the
 * warp-specialised real / complex sweep (k_diag_real_ws / k_diag_cplx_ws),
 * 0 = off, -1 = automatic.  Every variant computes identical results;
 * unknown combinations fall back to the default kernel.  Returns 0. */
int32_t hsrq_tune_diag(int32_t dp, int32_t dwr, int32_t dwc, int32_t wsr, int32_t wsc);
/* Rotation-ahead warp pairs (k_diag_cplx_rx: the rotation chain one step
 * ahead of the solution chain) for the complex sweep at 16 / 32 lanes per
 * shift: np = 4 / 8 pairs per CTA, 0 = off, -1 = automatic (16-lane pairs,
 * 8 per CTA, where the automatic choice is 32 lanes per shift).  Results
 * are bit-identical either way. */
int32_t hsrq_tune_diag_rx(int32_t np);
/* Panel form for b_r = 128: 1 = 2-CTA clusters of 64-row CTAs (k_panel_cl,
 * default), 0 = one 128-row CTA per tile row (k_panel).  Bit-identical. */
int32_t hsrq_tune_panel(int32_t cluster);

/*
 * Tile-level entry points (parity tests against the reference kernels).
 *
 * hsrq_tile_diag: one diagonal tile, k = rows (<= 128), b shifts.
 *   hdiag   k x (k-1) row-major (the reference's C-order hdiag tile)
 *   hleft   k entries (column left of the tile), used iff has_left
 *   lam_re/lam_im  b shifts (lam_im NULL -> real kernel)
 *   rright  k x b (real) or k x 2b (complex interleaved) row-major crossover
 *   x       k x b / k x 2b row-major, in: right-hand side tile, out: solution
 *   c_re, c_im, s   out, k x b row-major rotations (c_im may be NULL if real)
 *   beta_exp  in/out, b exponents (beta *= gamma)
 *   status    out, b int64 packed status (kind << 42 | row), 0 = ok
 */
int64_t hsrq_tile_diag(int32_t k, int32_t b, const double* hdiag, const double* hleft,
                       int32_t has_left, const double* lam_re, const double* lam_im,
                       const double* rright, double* x, double* c_re, double* c_im, double* s,
                       int32_t* beta_exp, int64_t* status, int32_t robust, double omega,
                       void* stream);

/*
 * hsrq_tile_backtransform: rbacktransform / crbacktransform
 * (numba_backend.py:326-375, :759-822) on b columns of length n with tiles of
 * b_r rows -- the tile-level operator API of the backtransform kernel.
 *   c_re, c_im, s  b x n (row q = shift q's rotations, row i mixing i-1 and i);
 *                  c_im ignored unless cplx
 *   seg_exp        N x b int32 row-major by tile: alpha = 2^seg_exp
 *   x              in/out, column-major n x b (real) or n x 2b (re, im columns)
 *   norms, alpha_exp  out, b entries (the reference's norms_out / alpha_out)
 *   mode           1 = eigvec (normalise), 0 = solve (omega guard)
 */
int64_t hsrq_tile_backtransform(int64_t n, int32_t b_r, int32_t b, int32_t cplx,
                                const double* c_re, const double* c_im, const double* s,
                                const int32_t* seg_exp, double* x, double* norms,
                                int32_t* alpha_exp, int32_t mode, double omega, void* stream);

/*
 * Henry's single-sweep RQ solve (the reference's baseline, henry_rq_solve,
 * reference.py:21-60): (H - lam_l I) x_l = b_l for m shifts, unguarded, in
 * one merged factor-and-substitute sweep per shift, followed by the rotation
 * sweep.  Results are bit-identical to the reference kernels.
 *   H       n x n column-major (ldh)
 *   lam     cplx = 0: m doubles; cplx = 1: m (re, im) pairs (complex128)
 *   X       in: right-hand sides, out: solutions; cplx = 0: n x m doubles,
 *           column-major (ldx); cplx = 1: n x m complex128 column-major
 *           (interleaved re, im; ldx counted in complex elements)
 *   status  optional (may be NULL), per shift: 0 or the packed status
 *           kind << 42 | shift << 21 | row of that shift's failure
 *   ws      workspace of >= hsrq_henry_workspace_bytes(n, m, cplx) bytes
 * Returns, after synchronising `stream`, 0 or the reference's packed status
 * of the first failure in its loop order (row descending, then shift; kind
 * HSRQ_KIND_DEGENERATE / HSRQ_KIND_SINGULAR), or a negative HSRQ_ERR_*.
 */
size_t hsrq_henry_workspace_bytes(int64_t n, int64_t m, int32_t cplx);
int64_t hsrq_henry_solve(const double* H, int64_t ldh, int64_t n, const double* lam, int64_t m,
                         int32_t cplx, double* X, int64_t ldx, int64_t* status, void* ws,
                         size_t ws_bytes, void* stream);

/*
 * Stewart compact rotation codes, elementwise over `count` rotations
 * (compact_encode / compact_decode and the complex pair, givens.py:107-198;
 * GivensTable.compact / from_compact, core.py:193-209), bit-identical to the
 * reference.  Real (cplx = 0): (c_re, s) <-> t1 (c_im, t2 unused).  Complex:
 * (c_re, c_im, s) <-> (t1, t2).
 */
int64_t hsrq_compact_encode(int64_t count, int32_t cplx, const double* c_re, const double* c_im,
                            const double* s, double* t1, double* t2, void* stream);
int64_t hsrq_compact_decode(int64_t count, int32_t cplx, const double* t1, const double* t2,
                            double* c_re, double* c_im, double* s, void* stream);

/*
 * Front end: H = Q^T A Q by Householder reflectors
 * (householder_hessenberg, testprob.py:146-174: same reflectors, sign
 * convention and skip rule -- columns already reduced are left untouched,
 * so a Hessenberg input returns bit for bit with Q = I), blocked as in
 * DGEHRD: panels of 64 reflectors, trailing updates as fp64 GEMMs.
 *   A  in: n x n column-major (lda); out: H (zeros below the subdiagonal)
 *   Q  out: n x n orthogonal (ldq), or NULL to skip accumulating it
 *   ws >= hsrq_hessenberg_workspace_bytes(n) bytes of device memory
 * Synchronises `stream`; returns 0 or a negative HSRQ_ERR_*.
 * hsrq_backmultiply: Z = Q X (eigenvectors of H -> eigenvectors of A,
 * PAPER.md:33-35); ncol real columns (a complex vector is two columns).
 */
size_t hsrq_hessenberg_workspace_bytes(int64_t n);
int64_t hsrq_hessenberg_reduce(double* A, int64_t lda, double* Q, int64_t ldq, int64_t n,
                               void* ws, size_t ws_bytes, void* stream);
int64_t hsrq_backmultiply(const double* Q, int64_t ldq, int64_t n, const double* X, int64_t ldx,
                          int64_t ncol, double* Z, int64_t ldz, void* stream);
const char* hsrq_hessenberg_last_error(void);
/* The front end's fp64 GEMM (csrc/hsrq_blas.cuh, DMMA), exposed for tests:
 * C = alpha op(A) op(B) + beta C, column-major, op = transpose if trans_*.
 * Dispatch: the rank-nb update shape (A B^T, alpha = -1, beta = 1, K <= 64)
 * runs k_dgemm_nt64; operands with 16-byte aligned columns the cp.async
 * pipeline k_dgemm_pipe; anything else the register-prefetch k_dgemm. */
int64_t hsrq_dgemm(int32_t trans_a, int32_t trans_b, int64_t M, int64_t N, int64_t K,
                   double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double beta, double* C, int64_t ldc, void* stream);

/*
 * Host I/O of the drop-in API (csrc/hsrq_hostio.cuh): what hsrq3in /
 * dhsrq3in / chsrq3in (inviter.py:155-254) pay around the solve when called
 * with numpy arrays.  Both stage through a process-wide pinned ring filled /
 * drained by host worker threads; `*_host` pointers are pageable memory.
 *
 * hsrq_h_upload: H from the caller's array (order 1 = column-major /
 *   Fortran, 0 = row-major / C: transposed on the device) into the
 *   column-major device H (ldh >= n).  checks_host[3] receives what
 *   HessenbergMatrix (core.py:60-98) computes on the host: [0] the infinity
 *   norm, bit-identical to np.max(np.sum(np.abs(F-order H), axis=1)) (numpy
 *   sums a Fortran array's rows left to right), [1] the number of nonzeros
 *   below the first subdiagonal (the ConfigError check, core.py:70-73),
 *   [2] the number of zero subdiagonal entries (is_unreduced, core.py:86-91).
 *   `stream` waits for the upload.  Returns 0 or a negative HSRQ_ERR_*.
 *
 * hsrq_pack_download: the solve's columns -> the caller's (n, m) C-order
 *   result (EigvecResult.vectors, inviter.py:53-59): out[i, j] =
 *   X[re_col[j]][i] + 1j * im_sign[j] * X[im_col[j]][i] (cplx_out = 1,
 *   complex128; im_col[j] < 0: real column) or X[re_col[j]][i]
 *   (cplx_out = 0, float64), X column-major n x ncol (ldx).  Column maps are
 *   host arrays of m entries.  Packs row blocks on the device after the work
 *   queued on `stream` and returns once out_host is written.
 */
int64_t hsrq_h_upload(const double* h_host, int32_t order, int64_t n, double* H, int64_t ldh,
                      double* checks_host, void* stream);
/* hsrq_host_prefault: take the first-touch page faults of a fresh host
 * buffer (e.g. the numpy result hsrq_pack_download will fill) on `threads`
 * threads -- meant to run while the device solves.  Returns 0. */
int64_t hsrq_host_prefault(void* ptr, int64_t bytes, int32_t threads);
int64_t hsrq_pack_download(const double* X, int64_t ldx, int64_t n, int64_t m,
                           const int64_t* re_col, const int64_t* im_col, const double* im_sign,
                           int32_t cplx_out, void* out_host, void* stream);

/*
 * hsrq_tile_update: one off-diagonal tile through the sweep's own panel
 * kernels (the diagonal sweep's operand code, k_scalars, k_panel) -- the
 * reference operator API update_rupdate / cupdate_crupdate
 * (numba_backend.py:198-311, 579-736) and reduce_offdiag / creduce_offdiag
 * (:109-125, 467-490) on one tile, for tile-level parity.  Device pointers,
 * row-major like the reference's tiles; b shifts, real or complex
 * (cplx = 1: interleaved re/im columns, 2b wide).
 *   htile      m x k: H[is:ie, js-1:je-1] (column 0 = the column left of tile jt)
 *   rright     m x b / m x 2b: crossover column jt on the tile's rows
 *   alpha_exp  b: log2 alpha (the scale of x_below)
 *   xbelow     k x b / k x 2b: the solved tile jt
 *   lam_re, lam_im   b shifts (lam_im / c_im NULL when real)
 *   shift_active     1: super-diagonal tile (lambda on the last row, for the
 *              update and the crossover); 0: a far tile (no lambda)
 *   c_re, c_im, s    k x b rotations of tile jt
 *   beta_exp   in: log2 beta (scale of b); out: log2 delta
 *   b_io       in/out m x b / m x 2b right-hand side tile
 *   rleft      out (or NULL): the new crossover column jt-1 on the tile's rows
 *   omega      0: DBL_MAX/2/m (OverflowBudget.for_tile_rows(m))
 * Requires 2 <= k <= m <= 128.  Stream-ordered; returns 0 or HSRQ_ERR_*.
 */
int64_t hsrq_tile_update(int32_t m, int32_t k, int32_t b, int32_t cplx, const double* htile,
                         const double* rright, const int32_t* alpha_exp, const double* xbelow,
                         const double* lam_re, const double* lam_im, int32_t shift_active,
                         const double* c_re, const double* c_im, const double* s,
                         int32_t* beta_exp, double* b_io, double* rleft, int32_t robust,
                         double omega, void* stream);

/* Elementwise device evaluations for bit-level parity of the scalar helpers. */
int64_t hsrq_protect_update_batch(const double* bnorm, const double* hnorm, const double* xnorm,
                                  double omega, int64_t count, double* out, void* stream);
/* protect_update at two argument pairs sharing xnorm, evaluated side by side
 * as the complex sweep's guard-2 certification does (protect_update_e2 in
 * csrc/hsrq_device.cuh); each output equals hsrq_protect_update_batch's. */
int64_t hsrq_protect_update_pair_batch(const double* b1, const double* h1, const double* b2,
                                       const double* h2, const double* xnorm, double omega,
                                       int64_t count, double* out1, double* out2, void* stream);
int64_t hsrq_hypot_batch(const double* x, const double* y, int64_t count, double* out,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HSRQ_B200_H */
