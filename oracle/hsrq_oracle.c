/*
 * hsrq_oracle.c -- CPU restatement of the reference hessrq inverse-iteration
 * path, used ONLY as a test checker and as the CPU baseline arm of bench.py.
 *
 * TEST INFRASTRUCTURE.  Nothing in the product package imports, links or
 * calls this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.
 *
 * What it restates (reference = /root/reference/pkg/src/hessrq, "K/" =
 * _kernels/numba_backend.py):
 *   pow2floor            K/numba_backend.py:37-44
 *   protect_update       K/numba_backend.py:47-67
 *   reduce_diag          K/numba_backend.py:75-106
 *   reduce_offdiag       K/numba_backend.py:109-125
 *   solve_rsolve         K/numba_backend.py:133-195
 *   update_rupdate       K/numba_backend.py:198-311   (GEMM via a hook)
 *   backtransform        K/numba_backend.py:314-323
 *   rbacktransform       K/numba_backend.py:326-375
 *   creduce_diag         K/numba_backend.py:420-464
 *   creduce_offdiag      K/numba_backend.py:467-490
 *   robust_trsv_complex  K/numba_backend.py:493-527
 *   _build_complex_r     K/numba_backend.py:530-551
 *   csolve_crsolve       K/numba_backend.py:554-576
 *   cupdate_crupdate     K/numba_backend.py:579-736   (GEMM via a hook)
 *   cbacktransform       K/numba_backend.py:739-756
 *   crbacktransform      K/numba_backend.py:759-822
 *   tiled driver         reduce.py:39-171 (tiled_reduce) and
 *                        backsolve.py:62-313 (_substitute), executed in the
 *                        single-worker program order of scheduler.py:189-219.
 *
 * Arithmetic is kept expression-for-expression (compile with
 * -ffp-contract=off: numba does not contract FMAs, K/numba_backend.py:4-5).
 * Complex arithmetic follows numba's lowering: (a+bi)(c+di) = (ac-bd)+(ad+bc)i
 * with real operands promoted to (x, 0); complex division is CPython's
 * _Py_c_quot; abs(z) = hypot(re, im) (glibc, the libm numba binds).
 *
 * The one deliberate representation change: every power-of-two scale factor
 * (alpha, beta, gamma, delta, xi) is carried as an int exponent e with value
 * ldexp(1, e).  Wherever all exponents stay >= -1074 this is bit-identical to
 * the reference's doubles (every product/ratio of those doubles is exact);
 * below that the reference underflows to 0 and produces NaN (SURVEY.md §0
 * finding 6), while the exponent form keeps going.  The GEMM inside the
 * update kernels goes through `oracle_set_blas`: the Python wrapper can hand
 * it the same Fortran dgemm numba calls (scipy.linalg.cython_blas), which
 * makes the whole driver bit-identical to the reference on the same machine;
 * without it a plain ordered triple loop is used.
 */

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define KIND_DEGENERATE 1
#define KIND_SINGULAR 2
#define EXP_ZERO (-1075) /* exponent of a scale that halved below 2^-1074 */

/* Test hook (oracle_set_stop): end the substitution after tile column jt's
 * updates, without the backtransform, so intermediate sweep states can be
 * compared column by column.  -1 = off. */
static int g_stop_jt = -1;
void oracle_set_stop(int jt) { g_stop_jt = jt; }

/* Test hook (oracle_set_omega): the caller's OverflowBudget.omega for the
 * next solves (dhsrq3 / chsrq3 budget=); 0 = the default DBL_MAX/2/b_r. */
static double g_omega = 0.0;
void oracle_set_omega(double omega) { g_omega = omega; }

static int64_t pack_status(int64_t kind, int64_t shift, int64_t row) {
    return kind * ((int64_t)1 << 42) + (shift << 21) + row;
}

/* ------------------------------------------------------------------ */
/* dgemm hook (Fortran convention, LP64 ints: what numba's np.dot calls) */
/* ------------------------------------------------------------------ */
typedef void (*dgemm_t)(const char*, const char*, const int*, const int*, const int*,
                        const double*, const double*, const int*, const double*,
                        const int*, const double*, double*, const int*);
typedef void (*dgemv_t)(const char*, const int*, const int*, const double*, const double*,
                        const int*, const double*, const int*, const double*, double*,
                        const int*);
typedef double (*ddot_t)(const int*, const double*, const int*, const double*, const int*);
static dgemm_t g_dgemm = NULL;
static dgemv_t g_dgemv = NULL;
static ddot_t g_ddot = NULL;

void oracle_set_blas(void* gemm, void* gemv, void* dot) {
    g_dgemm = (dgemm_t)gemm;
    g_dgemv = (dgemv_t)gemv;
    g_ddot = (ddot_t)dot;
}

/* prod (m x b, C order) = hblock (m x kk, C order) . zblock (kk x b, C order),
 * issued exactly as numba lowers np.dot on C-contiguous 2-d operands
 * (numba/np/linalg.py dot_3_mm): (1,k).(k,1) -> ddot; (m,k).(k,1) -> dgemv('t');
 * (1,k).(k,n) -> dgemv('n'); otherwise dgemm('n','n', b, m, kk, 1, zblock, b,
 * hblock, kk, 0, prod, b). */
static void gemm_hz(int m, int kk, int b, const double* hblock, const double* zblock,
                    double* prod) {
    const double one = 1.0, zero = 0.0;
    const int inc = 1;
    if (g_dgemm && g_dgemv && g_ddot) {
        if (b == 1 && m == 1) {
            prod[0] = g_ddot(&kk, hblock, &inc, zblock, &inc);
        } else if (b == 1) {
            g_dgemv("t", &kk, &m, &one, hblock, &kk, zblock, &inc, &zero, prod, &inc);
        } else if (m == 1) {
            g_dgemv("n", &b, &kk, &one, zblock, &b, hblock, &inc, &zero, prod, &inc);
        } else {
            int lda = b, ldb = kk, ldc = b;
            g_dgemm("n", "n", &b, &m, &kk, &one, zblock, &lda, hblock, &ldb, &zero, prod, &ldc);
        }
        return;
    }
    for (int i = 0; i < m; i++)
        for (int l = 0; l < b; l++) {
            double acc = 0.0;
            for (int j = 0; j < kk; j++) acc += hblock[i * kk + j] * zblock[j * b + l];
            prod[i * b + l] = acc;
        }
}

/* ------------------------------------------------------------------ */
/* scalar helpers                                                       */
/* ------------------------------------------------------------------ */

static inline double p2(int e) { return ldexp(1.0, e); }

/* pow2floor, K/numba_backend.py:37-44; returns the exponent. */
static int pow2floor_e(double x) {
    if (x <= 0.0 || x != x) return -1074;
    if (x == INFINITY) return 0;
    int e;
    frexp(x, &e);
    return e - 1;
}

/* protect_update, K/numba_backend.py:47-67; returns the exponent of xi
 * (0 means xi == 1, EXP_ZERO means xi halved to 0). */
int oracle_protect_update_e(double bnorm, double hnorm, double xnorm, double omega) {
    double cand;
    if (xnorm <= 1.0) {
        if (bnorm + hnorm * xnorm <= omega) return 0;
        cand = (omega * 0.5) / (bnorm * 0.5 + (hnorm * xnorm) * 0.5);
    } else {
        if (bnorm <= omega && hnorm <= (omega - bnorm) / xnorm) return 0;
        double u = bnorm / xnorm;
        cand = ((omega * 0.5) / (u * 0.5 + hnorm * 0.5)) / xnorm;
    }
    if (!(cand > 0.0)) cand = ldexp(1.0, -1074);
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

double oracle_protect_update(double bnorm, double hnorm, double xnorm, double omega) {
    int e = oracle_protect_update_e(bnorm, hnorm, xnorm, omega);
    return e <= EXP_ZERO ? 0.0 : p2(e);
}

double oracle_pow2floor(double x) { return p2(pow2floor_e(x)); }

/* numba complex lowering */
typedef struct { double re, im; } cplx;
static inline cplx C(double re, double im) { cplx z = {re, im}; return z; }
static inline cplx cmul(cplx a, cplx b) {
    double ac = a.re * b.re, bd = a.im * b.im, ad = a.re * b.im, bc = a.im * b.re;
    return C(ac - bd, ad + bc);
}
static inline cplx csub(cplx a, cplx b) { return C(a.re - b.re, a.im - b.im); }
static inline cplx cadd(cplx a, cplx b) { return C(a.re + b.re, a.im + b.im); }
static inline double cabs_(cplx a) { return hypot(a.re, a.im); }
/* CPython _Py_c_quot as lowered by numba (numba/cpython/numbers.py) */
static inline cplx cdiv(cplx a, cplx b) {
    double areal = a.re, aimag = a.im, breal = b.re, bimag = b.im;
    if (fabs(breal) >= fabs(bimag)) {
        if (breal == 0.0) return C(NAN, NAN);
        double ratio = bimag / breal;
        double denom = breal + bimag * ratio;
        return C((areal + aimag * ratio) / denom, (aimag - areal * ratio) / denom);
    } else {
        double ratio = breal / bimag;
        double denom = breal * ratio + bimag;
        return C((areal * ratio + aimag) / denom, (aimag * ratio - areal) / denom);
    }
}

/* ------------------------------------------------------------------ */
/* real tile kernels (arrays C-order, as the reference passes them)     */
/* ------------------------------------------------------------------ */

/* reduce_diag: hdiag k x (k-1), hleft k, rright k x b, c/s out k x b */
int64_t oracle_reduce_diag(int k, int b, const double* hdiag, const double* hleft, int has_left,
                           const double* lam, const double* rright, double* c_out,
                           double* s_out) {
    const int w = k - 1;
    double* v = (double*)malloc(sizeof(double) * (size_t)k * b);
    memcpy(v, rright, sizeof(double) * (size_t)k * b);
    int64_t st = 0;
    for (int kp = k - 1; kp >= 1; kp--) {
        double a = hdiag[kp * w + kp - 1];
        for (int l = 0; l < b; l++) {
            double r = hypot(a, v[kp * b + l]);
            if (r == 0.0) { st = pack_status(KIND_DEGENERATE, l, kp); goto out; }
            c_out[kp * b + l] = v[kp * b + l] / r;
            s_out[kp * b + l] = -a / r;
        }
        for (int i = 0; i < kp - 1; i++) {
            double hi = hdiag[i * w + kp - 1];
            for (int l = 0; l < b; l++)
                v[i * b + l] = c_out[kp * b + l] * hi + s_out[kp * b + l] * v[i * b + l];
        }
        double hd = hdiag[(kp - 1) * w + kp - 1];
        for (int l = 0; l < b; l++)
            v[(kp - 1) * b + l] =
                c_out[kp * b + l] * (hd - lam[l]) + s_out[kp * b + l] * v[(kp - 1) * b + l];
    }
    if (has_left) {
        double a = hleft[0];
        for (int l = 0; l < b; l++) {
            double r = hypot(a, v[l]);
            if (r == 0.0) { st = pack_status(KIND_DEGENERATE, l, 0); goto out; }
            c_out[l] = v[l] / r;
            s_out[l] = -a / r;
        }
    } else {
        for (int l = 0; l < b; l++) { c_out[l] = 1.0; s_out[l] = 0.0; }
    }
out:
    free(v);
    return st;
}

/* reduce_offdiag: htile k x w, c/s w x b, rright k x b, rleft out k x b */
void oracle_reduce_offdiag(int k, int w, int b, const double* htile, const double* lam,
                           const double* c, const double* s, const double* rright,
                           double* rleft) {
    double* v = (double*)malloc(sizeof(double) * (size_t)k * b);
    memcpy(v, rright, sizeof(double) * (size_t)k * b);
    for (int j = w - 1; j >= 1; j--)
        for (int i = 0; i < k; i++) {
            double hi = htile[i * w + j];
            for (int l = 0; l < b; l++) v[i * b + l] = c[j * b + l] * hi + s[j * b + l] * v[i * b + l];
        }
    for (int i = 0; i < k - 1; i++) {
        double hi = htile[i * w];
        for (int l = 0; l < b; l++) rleft[i * b + l] = c[l] * hi + s[l] * v[i * b + l];
    }
    double hk = htile[(k - 1) * w];
    for (int l = 0; l < b; l++)
        rleft[(k - 1) * b + l] = c[l] * (hk - lam[l]) + s[l] * v[(k - 1) * b + l];
    free(v);
}

/* solve_rsolve; beta_e in/out (exponents) */
int64_t oracle_solve_rsolve(int k, int b, const double* hdiag, const double* hleft, int has_left,
                            const double* lam, const double* rright, const double* c,
                            const double* s, double* x, int* beta_e, int robust, double omega) {
    const int w = k - 1;
    double* v = (double*)malloc(sizeof(double) * (size_t)k * b);
    int* ge = (int*)calloc((size_t)b, sizeof(int));
    memcpy(v, rright, sizeof(double) * (size_t)k * b);
    int64_t st = 0;
    for (int kp = k - 1; kp >= 1; kp--) {
        double a = hdiag[kp * w + kp - 1];
        for (int l = 0; l < b; l++) {
            double phi = v[kp * b + l] * c[kp * b + l] - a * s[kp * b + l];
            if (phi == 0.0) { st = pack_status(KIND_SINGULAR, l, kp); goto out; }
            if (robust) {
                double aphi = fabs(phi), ax = fabs(x[kp * b + l]);
                if (aphi < 1.0 && ax > aphi * omega) {
                    int e = pow2floor_e(aphi * omega / ax);
                    double xi = p2(e);
                    for (int i = 0; i < k; i++) x[i * b + l] *= xi;
                    ge[l] += e;
                }
            }
            x[kp * b + l] = x[kp * b + l] / phi;
            if (robust) {
                double xmax = 0.0, vmax = 0.0, hmax = 0.0;
                for (int i = 0; i < kp; i++) {
                    if (fabs(x[i * b + l]) > xmax) xmax = fabs(x[i * b + l]);
                    if (fabs(v[i * b + l]) > vmax) vmax = fabs(v[i * b + l]);
                    if (fabs(hdiag[i * w + kp - 1]) > hmax) hmax = fabs(hdiag[i * w + kp - 1]);
                }
                int e = oracle_protect_update_e(xmax, vmax + hmax + fabs(lam[l]),
                                                fabs(x[kp * b + l]), omega);
                if (e < 0) {
                    double xi = e <= EXP_ZERO ? 0.0 : p2(e);
                    for (int i = 0; i < k; i++) x[i * b + l] *= xi;
                    ge[l] += e;
                }
            }
            double tau1 = s[kp * b + l] * x[kp * b + l];
            double tau2 = c[kp * b + l] * x[kp * b + l];
            for (int i = 0; i < kp - 1; i++) {
                double hi = hdiag[i * w + kp - 1];
                x[i * b + l] = (x[i * b + l] - tau2 * v[i * b + l]) + tau1 * hi;
                v[i * b + l] = c[kp * b + l] * hi + s[kp * b + l] * v[i * b + l];
            }
            double hd = hdiag[(kp - 1) * w + kp - 1];
            x[(kp - 1) * b + l] = (x[(kp - 1) * b + l] - tau2 * v[(kp - 1) * b + l]) + tau1 * (hd - lam[l]);
            v[(kp - 1) * b + l] = c[kp * b + l] * (hd - lam[l]) + s[kp * b + l] * v[(kp - 1) * b + l];
        }
    }
    for (int l = 0; l < b; l++) {
        double v0 = v[l];
        if (has_left) v0 = v0 * c[l] - hleft[0] * s[l];
        if (v0 == 0.0) { st = pack_status(KIND_SINGULAR, l, 0); goto out; }
        if (robust) {
            double av = fabs(v0), ax = fabs(x[l]);
            if (av < 1.0 && ax > av * omega) {
                int e = pow2floor_e(av * omega / ax);
                double xi = p2(e);
                for (int i = 0; i < k; i++) x[i * b + l] *= xi;
                ge[l] += e;
            }
        }
        x[l] = x[l] / v0;
    }
    for (int l = 0; l < b; l++) beta_e[l] += ge[l];
out:
    free(v);
    free(ge);
    return st;
}

/* update_rupdate: htile m x k, rright m x b, alpha_e b, xbelow k x b, c/s k x b,
 * beta_e b in/out, b_io m x b in/out */
void oracle_update_rupdate(int m, int k, int b, const double* htile, const double* rright,
                           const int* alpha_e, const double* xbelow, const double* lam,
                           int shift_active, const double* c, const double* s, int* beta_e,
                           double* b_io, int robust, double omega) {
    int* delta = (int*)malloc(sizeof(int) * b);
    double* fx = (double*)malloc(sizeof(double) * b);
    double* Z = (double*)malloc(sizeof(double) * (size_t)k * b);
    for (int l = 0; l < b; l++) fx[l] = 1.0;
    if (robust) {
        double hmax0 = 0.0;
        for (int i = 0; i < m; i++)
            if (fabs(htile[i * k]) > hmax0) hmax0 = fabs(htile[i * k]);
        for (int l = 0; l < b; l++) {
            int g = alpha_e[l] < beta_e[l] ? alpha_e[l] : beta_e[l];
            double rho_raw = s[l] * xbelow[l];
            double bmax = 0.0;
            for (int i = 0; i < m; i++)
                if (fabs(b_io[i * b + l]) > bmax) bmax = fabs(b_io[i * b + l]);
            int xe = oracle_protect_update_e(p2(g - beta_e[l]) * bmax, hmax0 + fabs(lam[l]),
                                             fabs(rho_raw), omega);
            int d = xe + g;
            delta[l] = d;
            double fb = p2(d - beta_e[l]);
            double fxl = p2(d - alpha_e[l]);
            fx[l] = fxl;
            if (fb != 1.0)
                for (int i = 0; i < m; i++) b_io[i * b + l] *= fb;
            double rho = fxl == 1.0 ? rho_raw : fxl * rho_raw;
            for (int i = 0; i < m; i++) b_io[i * b + l] += rho * htile[i * k];
            if (shift_active) b_io[(m - 1) * b + l] -= lam[l] * rho;
        }
    } else {
        for (int l = 0; l < b; l++) {
            double rho = s[l] * xbelow[l];
            for (int i = 0; i < m; i++) b_io[i * b + l] += rho * htile[i * k];
            if (shift_active) b_io[(m - 1) * b + l] -= lam[l] * rho;
        }
    }
    memcpy(Z, xbelow, sizeof(double) * (size_t)k * b);
    if (robust)
        for (int l = 0; l < b; l++)
            if (fx[l] != 1.0)
                for (int i = 0; i < k; i++) Z[i * b + l] *= fx[l];
    for (int l = 0; l < b; l++) Z[l] = c[l] * Z[l];
    for (int jp = 1; jp < k; jp++)
        for (int l = 0; l < b; l++) {
            double t1 = Z[(jp - 1) * b + l], t2 = Z[jp * b + l];
            Z[(jp - 1) * b + l] = c[jp * b + l] * t1 - s[jp * b + l] * t2;
            Z[jp * b + l] = s[jp * b + l] * t1 + c[jp * b + l] * t2;
        }
    if (robust && k > 1) {
        double rowsum = 0.0;
        for (int i = 0; i < m; i++) {
            double acc = 0.0;
            for (int j = 1; j < k; j++) acc += fabs(htile[i * k + j]);
            if (acc > rowsum) rowsum = acc;
        }
        for (int l = 0; l < b; l++) {
            double bmax = 0.0, zmax = 0.0;
            for (int i = 0; i < m; i++)
                if (fabs(b_io[i * b + l]) > bmax) bmax = fabs(b_io[i * b + l]);
            for (int i = 0; i < k - 1; i++)
                if (fabs(Z[i * b + l]) > zmax) zmax = fabs(Z[i * b + l]);
            int xe = oracle_protect_update_e(bmax, rowsum, zmax, omega);
            if (xe < 0) {
                double xi = xe <= EXP_ZERO ? 0.0 : p2(xe);
                delta[l] += xe;
                for (int i = 0; i < m; i++) b_io[i * b + l] *= xi;
                for (int i = 0; i < k; i++) Z[i * b + l] *= xi;
            }
        }
    }
    if (k > 1) {
        double* hblock = (double*)malloc(sizeof(double) * (size_t)m * (k - 1));
        double* prod = (double*)malloc(sizeof(double) * (size_t)m * b);
        for (int i = 0; i < m; i++)
            for (int j = 1; j < k; j++) hblock[i * (k - 1) + (j - 1)] = htile[i * k + j];
        gemm_hz(m, k - 1, b, hblock, Z, prod);
        for (int i = 0; i < m; i++)
            for (int l = 0; l < b; l++) b_io[i * b + l] -= prod[i * b + l];
        free(hblock);
        free(prod);
    }
    if (robust) {
        for (int l = 0; l < b; l++) {
            double rmax = 0.0, bmax = 0.0;
            for (int i = 0; i < m; i++) {
                if (fabs(rright[i * b + l]) > rmax) rmax = fabs(rright[i * b + l]);
                if (fabs(b_io[i * b + l]) > bmax) bmax = fabs(b_io[i * b + l]);
            }
            int xe = oracle_protect_update_e(bmax, rmax, fabs(Z[(k - 1) * b + l]), omega);
            if (xe < 0) {
                double xi = xe <= EXP_ZERO ? 0.0 : p2(xe);
                delta[l] += xe;
                for (int i = 0; i < m; i++) b_io[i * b + l] *= xi;
                Z[(k - 1) * b + l] *= xi;
            }
            double zk = Z[(k - 1) * b + l];
            for (int i = 0; i < m; i++) b_io[i * b + l] -= rright[i * b + l] * zk;
        }
        for (int l = 0; l < b; l++) beta_e[l] = delta[l];
    } else {
        for (int l = 0; l < b; l++) {
            double zk = Z[(k - 1) * b + l];
            for (int i = 0; i < m; i++) b_io[i * b + l] -= rright[i * b + l] * zk;
        }
    }
    free(delta);
    free(fx);
    free(Z);
}

/* backtransform, K/numba_backend.py:314-323; x n x b */
void oracle_backtransform(int n, int b, const double* c, const double* s, double* x) {
    for (int l = 0; l < b; l++) {
        double t1 = x[l];
        for (int i = 1; i < n; i++) {
            double t2 = x[i * b + l];
            x[(i - 1) * b + l] = c[i * b + l] * t1 - s[i * b + l] * t2;
            t1 = c[i * b + l] * t2 + s[i * b + l] * t1;
        }
        x[(n - 1) * b + l] = t1;
    }
}

/* rbacktransform, K/numba_backend.py:326-375.  alpha_e N x b.  Outputs:
 * norms (reference double, may be inf), log2norm (exact-range log2 of the
 * represented norm), alpha_out_e (exponent of the column scale). */
void oracle_rbacktransform(int n, int b, int N, const double* c, const double* s,
                           const int* alpha_e, const int64_t* tile_ends, double* x, double* norms,
                           double* log2norm, int* alpha_out_e, int mode, double omega) {
    for (int l = 0; l < b; l++) {
        int amin = alpha_e[l];
        for (int t = 1; t < N; t++)
            if (alpha_e[t * b + l] < amin) amin = alpha_e[t * b + l];
        int64_t start = 0;
        for (int t = 0; t < N; t++) {
            int64_t end = tile_ends[t];
            double f = p2(amin - alpha_e[t * b + l]);
            if (f != 1.0)
                for (int64_t i = start; i < end; i++) x[i * b + l] *= f;
            start = end;
        }
        double xmax = 0.0;
        for (int i = 0; i < n; i++)
            if (fabs(x[i * b + l]) > xmax) xmax = fabs(x[i * b + l]);
        if (xmax == 0.0) {
            norms[l] = 0.0;
            log2norm[l] = -INFINITY;
            alpha_out_e[l] = amin;
            continue;
        }
        double tsum = 0.0;
        for (int i = 0; i < n; i++) {
            double q = x[i * b + l] / xmax;
            tsum += q * q;
        }
        double rt = sqrt(tsum);
        norms[l] = ldexp(xmax, -amin) * rt;
        log2norm[l] = log2(xmax) + log2(rt) - (double)amin;
        alpha_out_e[l] = amin;
        if (mode == 1) {
            for (int i = 0; i < n; i++) x[i * b + l] /= xmax;
            for (int i = 0; i < n; i++) x[i * b + l] /= rt;
        } else {
            double q = omega / xmax;
            if (rt > q) {
                int e = pow2floor_e(q / rt);
                double xi = p2(e);
                for (int i = 0; i < n; i++) x[i * b + l] *= xi;
                alpha_out_e[l] = amin + e;
            }
        }
        double t1 = x[l];
        for (int i = 1; i < n; i++) {
            double t2 = x[i * b + l];
            x[(i - 1) * b + l] = c[i * b + l] * t1 - s[i * b + l] * t2;
            t1 = c[i * b + l] * t2 + s[i * b + l] * t1;
        }
        x[(n - 1) * b + l] = t1;
    }
}

/* ------------------------------------------------------------------ */
/* complex tile kernels (interleaved: column 2l = re, 2l+1 = im)        */
/* ------------------------------------------------------------------ */

int64_t oracle_creduce_diag(int k, int b, const double* hdiag, const double* hleft, int has_left,
                            const double* lam_re, const double* lam_im, const double* rright2,
                            double* cre_out, double* cim_out, double* s_out) {
    const int w = k - 1, b2 = 2 * b;
    double* v = (double*)malloc(sizeof(double) * (size_t)k * b2);
    memcpy(v, rright2, sizeof(double) * (size_t)k * b2);
    int64_t st = 0;
    for (int kp = k - 1; kp >= 1; kp--) {
        double a = hdiag[kp * w + kp - 1];
        for (int l = 0; l < b; l++) {
            double absv = hypot(v[kp * b2 + 2 * l], v[kp * b2 + 2 * l + 1]);
            double r = hypot(a, absv);
            if (r == 0.0) { st = pack_status(KIND_DEGENERATE, l, kp); goto out; }
            cre_out[kp * b + l] = v[kp * b2 + 2 * l] / r;
            cim_out[kp * b + l] = v[kp * b2 + 2 * l + 1] / r;
            s_out[kp * b + l] = -a / r;
        }
        for (int i = 0; i < kp - 1; i++) {
            double hi = hdiag[i * w + kp - 1];
            for (int l = 0; l < b; l++) {
                v[i * b2 + 2 * l] = cre_out[kp * b + l] * hi + s_out[kp * b + l] * v[i * b2 + 2 * l];
                v[i * b2 + 2 * l + 1] = cim_out[kp * b + l] * hi + s_out[kp * b + l] * v[i * b2 + 2 * l + 1];
            }
        }
        double hd = hdiag[(kp - 1) * w + kp - 1];
        for (int l = 0; l < b; l++) {
            double tre = hd - lam_re[l], tim = -lam_im[l];
            double cr = cre_out[kp * b + l], ci = cim_out[kp * b + l], sv = s_out[kp * b + l];
            double* vr = &v[(kp - 1) * b2 + 2 * l];
            double nr = (cr * tre - ci * tim) + sv * vr[0];
            double ni = (cr * tim + ci * tre) + sv * vr[1];
            vr[0] = nr;
            vr[1] = ni;
        }
    }
    if (has_left) {
        double a = hleft[0];
        for (int l = 0; l < b; l++) {
            double absv = hypot(v[2 * l], v[2 * l + 1]);
            double r = hypot(a, absv);
            if (r == 0.0) { st = pack_status(KIND_DEGENERATE, l, 0); goto out; }
            cre_out[l] = v[2 * l] / r;
            cim_out[l] = v[2 * l + 1] / r;
            s_out[l] = -a / r;
        }
    } else {
        for (int l = 0; l < b; l++) { cre_out[l] = 1.0; cim_out[l] = 0.0; s_out[l] = 0.0; }
    }
out:
    free(v);
    return st;
}

void oracle_creduce_offdiag(int k, int w, int b, const double* htile, const double* lam_re,
                            const double* lam_im, const double* cre, const double* cim,
                            const double* s, const double* rright2, double* rleft2) {
    const int b2 = 2 * b;
    double* v = (double*)malloc(sizeof(double) * (size_t)k * b2);
    memcpy(v, rright2, sizeof(double) * (size_t)k * b2);
    for (int j = w - 1; j >= 1; j--)
        for (int i = 0; i < k; i++) {
            double hi = htile[i * w + j];
            for (int l = 0; l < b; l++) {
                v[i * b2 + 2 * l] = cre[j * b + l] * hi + s[j * b + l] * v[i * b2 + 2 * l];
                v[i * b2 + 2 * l + 1] = cim[j * b + l] * hi + s[j * b + l] * v[i * b2 + 2 * l + 1];
            }
        }
    for (int i = 0; i < k - 1; i++) {
        double hi = htile[i * w];
        for (int l = 0; l < b; l++) {
            rleft2[i * b2 + 2 * l] = cre[l] * hi + s[l] * v[i * b2 + 2 * l];
            rleft2[i * b2 + 2 * l + 1] = cim[l] * hi + s[l] * v[i * b2 + 2 * l + 1];
        }
    }
    double hk = htile[(k - 1) * w];
    for (int l = 0; l < b; l++) {
        double tre = hk - lam_re[l], tim = -lam_im[l];
        rleft2[(k - 1) * b2 + 2 * l] = (cre[l] * tre - cim[l] * tim) + s[l] * v[(k - 1) * b2 + 2 * l];
        rleft2[(k - 1) * b2 + 2 * l + 1] = (cre[l] * tim + cim[l] * tre) + s[l] * v[(k - 1) * b2 + 2 * l + 1];
    }
    free(v);
}

/* robust_trsv_complex, K/numba_backend.py:493-527; r k x k complex (C order),
 * returns status, *gamma_e = exponent of gamma. */
static int64_t robust_trsv_complex(int k, const cplx* r, cplx* x, int robust, double omega,
                                   int* gamma_e) {
    int ge = 0;
    for (int j = k - 1; j >= 0; j--) {
        cplx d = r[j * k + j];
        if (d.re == 0.0 && d.im == 0.0) { *gamma_e = ge; return pack_status(KIND_SINGULAR, 0, j); }
        if (robust) {
            double ad = cabs_(d), ax = cabs_(x[j]);
            if (ad < 1.0 && ax > ad * omega) {
                int e = pow2floor_e(ad * omega / ax);
                cplx xi = C(p2(e), 0.0);
                for (int i = 0; i < k; i++) x[i] = cmul(x[i], xi);
                ge += e;
            }
        }
        x[j] = cdiv(x[j], d);
        if (j > 0) {
            if (robust) {
                double rmax = 0.0, bmax = 0.0;
                for (int i = 0; i < j; i++) {
                    double q = cabs_(r[i * k + j]);
                    if (q > rmax) rmax = q;
                    q = cabs_(x[i]);
                    if (q > bmax) bmax = q;
                }
                int e = oracle_protect_update_e(bmax, rmax, cabs_(x[j]), omega);
                if (e < 0) {
                    cplx xi = C(e <= EXP_ZERO ? 0.0 : p2(e), 0.0);
                    for (int i = 0; i < k; i++) x[i] = cmul(x[i], xi);
                    ge += e;
                }
            }
            cplx xj = x[j];
            for (int i = 0; i < j; i++) x[i] = csub(x[i], cmul(xj, r[i * k + j]));
        }
    }
    *gamma_e = ge;
    return 0;
}

/* _build_complex_r, K/numba_backend.py:530-551 */
static void build_complex_r(int k, int b, const double* hdiag, const double* hleft, int has_left,
                            cplx lam, const cplx* vcol, const double* cre, const double* cim,
                            const double* s, int l, cplx* r, cplx* v) {
    const int w = k - 1;
    memset(r, 0, sizeof(cplx) * (size_t)k * k);
    memcpy(v, vcol, sizeof(cplx) * (size_t)k);
    for (int kp = k - 1; kp >= 1; kp--) {
        cplx cc = C(cre[kp * b + l], cim[kp * b + l]);
        cplx ccj = C(cre[kp * b + l], -cim[kp * b + l]);
        cplx sv = C(s[kp * b + l], 0.0);
        for (int i = 0; i <= kp; i++) {
            cplx t = C(hdiag[i * w + kp - 1], 0.0);
            if (i == kp - 1) t = csub(t, lam);
            r[i * k + kp] = csub(cmul(ccj, v[i]), cmul(sv, t));
            if (i < kp) v[i] = cadd(cmul(cc, t), cmul(sv, v[i]));
        }
    }
    if (has_left) {
        cplx ccj0 = C(cre[l], -cim[l]);
        r[0] = csub(cmul(ccj0, v[0]), cmul(C(s[l], 0.0), C(hleft[0], 0.0)));
    } else {
        r[0] = v[0];
    }
}

int64_t oracle_csolve_crsolve(int k, int b, const double* hdiag, const double* hleft,
                              int has_left, const double* lam_re, const double* lam_im,
                              const double* rright2, const double* cre, const double* cim,
                              const double* s, double* x2, int* beta_e, int robust,
                              double omega) {
    const int b2 = 2 * b;
    cplx* r = (cplx*)malloc(sizeof(cplx) * (size_t)k * k);
    cplx* v = (cplx*)malloc(sizeof(cplx) * (size_t)k);
    cplx* vcol = (cplx*)malloc(sizeof(cplx) * (size_t)k);
    cplx* xc = (cplx*)malloc(sizeof(cplx) * (size_t)k);
    int64_t st = 0;
    for (int l = 0; l < b; l++) {
        cplx lam = C(lam_re[l], lam_im[l]);
        for (int i = 0; i < k; i++) {
            vcol[i] = C(rright2[i * b2 + 2 * l], rright2[i * b2 + 2 * l + 1]);
            xc[i] = C(x2[i * b2 + 2 * l], x2[i * b2 + 2 * l + 1]);
        }
        build_complex_r(k, b, hdiag, hleft, has_left, lam, vcol, cre, cim, s, l, r, v);
        int ge = 0;
        int64_t status = robust_trsv_complex(k, r, xc, robust, omega, &ge);
        if (status != 0) {
            st = pack_status(KIND_SINGULAR, l, status & ((1 << 21) - 1));
            break;
        }
        for (int i = 0; i < k; i++) {
            x2[i * b2 + 2 * l] = xc[i].re;
            x2[i * b2 + 2 * l + 1] = xc[i].im;
        }
        beta_e[l] += ge;
    }
    free(r);
    free(v);
    free(vcol);
    free(xc);
    return st;
}

void oracle_cupdate_crupdate(int m, int k, int b, const double* htile, const double* rright2,
                             const int* alpha_e, const double* xbelow2, const double* lam_re,
                             const double* lam_im, int shift_active, const double* cre,
                             const double* cim, const double* s, int* beta_e, double* b_io2,
                             int robust, double omega) {
    const int b2 = 2 * b;
    int* delta = (int*)malloc(sizeof(int) * b);
    double* fx = (double*)malloc(sizeof(double) * b);
    double* Z = (double*)malloc(sizeof(double) * (size_t)k * b2);
    for (int l = 0; l < b; l++) fx[l] = 1.0;
    if (robust) {
        double hmax0 = 0.0;
        for (int i = 0; i < m; i++)
            if (fabs(htile[i * k]) > hmax0) hmax0 = fabs(htile[i * k]);
        for (int l = 0; l < b; l++) {
            int g = alpha_e[l] < beta_e[l] ? alpha_e[l] : beta_e[l];
            double rr = s[l] * xbelow2[2 * l];
            double ri = s[l] * xbelow2[2 * l + 1];
            double bmax = 0.0;
            for (int i = 0; i < m; i++) {
                double q = hypot(b_io2[i * b2 + 2 * l], b_io2[i * b2 + 2 * l + 1]);
                if (q > bmax) bmax = q;
            }
            double alam = hypot(lam_re[l], lam_im[l]);
            int xe = oracle_protect_update_e(p2(g - beta_e[l]) * bmax, hmax0 + alam,
                                             hypot(rr, ri), omega);
            int d = xe + g;
            delta[l] = d;
            double fb = p2(d - beta_e[l]);
            double fxl = p2(d - alpha_e[l]);
            fx[l] = fxl;
            if (fb != 1.0)
                for (int i = 0; i < m; i++) {
                    b_io2[i * b2 + 2 * l] *= fb;
                    b_io2[i * b2 + 2 * l + 1] *= fb;
                }
            if (fxl != 1.0) {
                rr = fxl * rr;
                ri = fxl * ri;
            }
            for (int i = 0; i < m; i++) {
                b_io2[i * b2 + 2 * l] += rr * htile[i * k];
                b_io2[i * b2 + 2 * l + 1] += ri * htile[i * k];
            }
            if (shift_active) {
                b_io2[(m - 1) * b2 + 2 * l] -= lam_re[l] * rr - lam_im[l] * ri;
                b_io2[(m - 1) * b2 + 2 * l + 1] -= lam_re[l] * ri + lam_im[l] * rr;
            }
        }
    } else {
        for (int l = 0; l < b; l++) {
            double rr = s[l] * xbelow2[2 * l];
            double ri = s[l] * xbelow2[2 * l + 1];
            for (int i = 0; i < m; i++) {
                b_io2[i * b2 + 2 * l] += rr * htile[i * k];
                b_io2[i * b2 + 2 * l + 1] += ri * htile[i * k];
            }
            if (shift_active) {
                b_io2[(m - 1) * b2 + 2 * l] -= lam_re[l] * rr - lam_im[l] * ri;
                b_io2[(m - 1) * b2 + 2 * l + 1] -= lam_re[l] * ri + lam_im[l] * rr;
            }
        }
    }
    memcpy(Z, xbelow2, sizeof(double) * (size_t)k * b2);
    if (robust)
        for (int l = 0; l < b; l++)
            if (fx[l] != 1.0)
                for (int i = 0; i < k; i++) {
                    Z[i * b2 + 2 * l] *= fx[l];
                    Z[i * b2 + 2 * l + 1] *= fx[l];
                }
    for (int l = 0; l < b; l++) {
        double z0r = Z[2 * l], z0i = Z[2 * l + 1];
        Z[2 * l] = cre[l] * z0r + cim[l] * z0i;
        Z[2 * l + 1] = cre[l] * z0i - cim[l] * z0r;
    }
    for (int jp = 1; jp < k; jp++)
        for (int l = 0; l < b; l++) {
            double cr = cre[jp * b + l], ci = cim[jp * b + l], sv = s[jp * b + l];
            double t1r = Z[(jp - 1) * b2 + 2 * l], t1i = Z[(jp - 1) * b2 + 2 * l + 1];
            double t2r = Z[jp * b2 + 2 * l], t2i = Z[jp * b2 + 2 * l + 1];
            Z[(jp - 1) * b2 + 2 * l] = (cr * t1r - ci * t1i) - sv * t2r;
            Z[(jp - 1) * b2 + 2 * l + 1] = (cr * t1i + ci * t1r) - sv * t2i;
            Z[jp * b2 + 2 * l] = sv * t1r + (cr * t2r + ci * t2i);
            Z[jp * b2 + 2 * l + 1] = sv * t1i + (cr * t2i - ci * t2r);
        }
    if (robust && k > 1) {
        double rowsum = 0.0;
        for (int i = 0; i < m; i++) {
            double acc = 0.0;
            for (int j = 1; j < k; j++) acc += fabs(htile[i * k + j]);
            if (acc > rowsum) rowsum = acc;
        }
        for (int l = 0; l < b; l++) {
            double bmax = 0.0, zmax = 0.0;
            for (int i = 0; i < m; i++) {
                double q = hypot(b_io2[i * b2 + 2 * l], b_io2[i * b2 + 2 * l + 1]);
                if (q > bmax) bmax = q;
            }
            for (int i = 0; i < k - 1; i++) {
                double q = hypot(Z[i * b2 + 2 * l], Z[i * b2 + 2 * l + 1]);
                if (q > zmax) zmax = q;
            }
            int xe = oracle_protect_update_e(bmax, rowsum, zmax, omega);
            if (xe < 0) {
                double xi = xe <= EXP_ZERO ? 0.0 : p2(xe);
                delta[l] += xe;
                for (int i = 0; i < m; i++) {
                    b_io2[i * b2 + 2 * l] *= xi;
                    b_io2[i * b2 + 2 * l + 1] *= xi;
                }
                for (int i = 0; i < k; i++) {
                    Z[i * b2 + 2 * l] *= xi;
                    Z[i * b2 + 2 * l + 1] *= xi;
                }
            }
        }
    }
    if (k > 1) {
        double* hblock = (double*)malloc(sizeof(double) * (size_t)m * (k - 1));
        double* prod = (double*)malloc(sizeof(double) * (size_t)m * b2);
        for (int i = 0; i < m; i++)
            for (int j = 1; j < k; j++) hblock[i * (k - 1) + (j - 1)] = htile[i * k + j];
        gemm_hz(m, k - 1, b2, hblock, Z, prod);
        for (int i = 0; i < m; i++)
            for (int j = 0; j < b2; j++) b_io2[i * b2 + j] -= prod[i * b2 + j];
        free(hblock);
        free(prod);
    }
    if (robust) {
        for (int l = 0; l < b; l++) {
            double rmax = 0.0, bmax = 0.0;
            for (int i = 0; i < m; i++) {
                double q = hypot(rright2[i * b2 + 2 * l], rright2[i * b2 + 2 * l + 1]);
                if (q > rmax) rmax = q;
                q = hypot(b_io2[i * b2 + 2 * l], b_io2[i * b2 + 2 * l + 1]);
                if (q > bmax) bmax = q;
            }
            double zkr = Z[(k - 1) * b2 + 2 * l], zki = Z[(k - 1) * b2 + 2 * l + 1];
            int xe = oracle_protect_update_e(bmax, rmax, hypot(zkr, zki), omega);
            if (xe < 0) {
                double xi = xe <= EXP_ZERO ? 0.0 : p2(xe);
                delta[l] += xe;
                for (int i = 0; i < m; i++) {
                    b_io2[i * b2 + 2 * l] *= xi;
                    b_io2[i * b2 + 2 * l + 1] *= xi;
                }
                zkr *= xi;
                zki *= xi;
            }
            for (int i = 0; i < m; i++) {
                double rre = rright2[i * b2 + 2 * l], rim = rright2[i * b2 + 2 * l + 1];
                b_io2[i * b2 + 2 * l] -= rre * zkr - rim * zki;
                b_io2[i * b2 + 2 * l + 1] -= rre * zki + rim * zkr;
            }
        }
        for (int l = 0; l < b; l++) beta_e[l] = delta[l];
    } else {
        for (int l = 0; l < b; l++) {
            double zkr = Z[(k - 1) * b2 + 2 * l], zki = Z[(k - 1) * b2 + 2 * l + 1];
            for (int i = 0; i < m; i++) {
                double rre = rright2[i * b2 + 2 * l], rim = rright2[i * b2 + 2 * l + 1];
                b_io2[i * b2 + 2 * l] -= rre * zkr - rim * zki;
                b_io2[i * b2 + 2 * l + 1] -= rre * zki + rim * zkr;
            }
        }
    }
    free(delta);
    free(fx);
    free(Z);
}

void oracle_cbacktransform(int n, int b, const double* cre, const double* cim, const double* s,
                           double* x2) {
    const int b2 = 2 * b;
    for (int l = 0; l < b; l++) {
        double t1r = x2[2 * l], t1i = x2[2 * l + 1];
        for (int i = 1; i < n; i++) {
            double cr = cre[i * b + l], ci = cim[i * b + l], sv = s[i * b + l];
            double t2r = x2[i * b2 + 2 * l], t2i = x2[i * b2 + 2 * l + 1];
            x2[(i - 1) * b2 + 2 * l] = (cr * t1r - ci * t1i) - sv * t2r;
            x2[(i - 1) * b2 + 2 * l + 1] = (cr * t1i + ci * t1r) - sv * t2i;
            double nr = sv * t1r + (cr * t2r + ci * t2i);
            double ni = sv * t1i + (cr * t2i - ci * t2r);
            t1r = nr;
            t1i = ni;
        }
        x2[(n - 1) * b2 + 2 * l] = t1r;
        x2[(n - 1) * b2 + 2 * l + 1] = t1i;
    }
}

void oracle_crbacktransform(int n, int b, int N, const double* cre, const double* cim,
                            const double* s, const int* alpha_e, const int64_t* tile_ends,
                            double* x2, double* norms, double* log2norm, int* alpha_out_e,
                            int mode, double omega) {
    const int b2 = 2 * b;
    for (int l = 0; l < b; l++) {
        int amin = alpha_e[l];
        for (int t = 1; t < N; t++)
            if (alpha_e[t * b + l] < amin) amin = alpha_e[t * b + l];
        int64_t start = 0;
        for (int t = 0; t < N; t++) {
            int64_t end = tile_ends[t];
            double f = p2(amin - alpha_e[t * b + l]);
            if (f != 1.0)
                for (int64_t i = start; i < end; i++) {
                    x2[i * b2 + 2 * l] *= f;
                    x2[i * b2 + 2 * l + 1] *= f;
                }
            start = end;
        }
        double xmax = 0.0;
        for (int i = 0; i < n; i++) {
            double q = hypot(x2[i * b2 + 2 * l], x2[i * b2 + 2 * l + 1]);
            if (q > xmax) xmax = q;
        }
        if (xmax == 0.0) {
            norms[l] = 0.0;
            log2norm[l] = -INFINITY;
            alpha_out_e[l] = amin;
            continue;
        }
        double tsum = 0.0;
        for (int i = 0; i < n; i++) {
            double qr = x2[i * b2 + 2 * l] / xmax, qi = x2[i * b2 + 2 * l + 1] / xmax;
            tsum += qr * qr + qi * qi;
        }
        double rt = sqrt(tsum);
        norms[l] = ldexp(xmax, -amin) * rt;
        log2norm[l] = log2(xmax) + log2(rt) - (double)amin;
        alpha_out_e[l] = amin;
        if (mode == 1) {
            for (int i = 0; i < n; i++) {
                x2[i * b2 + 2 * l] /= xmax;
                x2[i * b2 + 2 * l + 1] /= xmax;
            }
            for (int i = 0; i < n; i++) {
                x2[i * b2 + 2 * l] /= rt;
                x2[i * b2 + 2 * l + 1] /= rt;
            }
        } else {
            double q = omega / xmax;
            if (rt > q) {
                int e = pow2floor_e(q / rt);
                double xi = p2(e);
                for (int i = 0; i < n; i++) {
                    x2[i * b2 + 2 * l] *= xi;
                    x2[i * b2 + 2 * l + 1] *= xi;
                }
                alpha_out_e[l] = amin + e;
            }
        }
        double t1r = x2[2 * l], t1i = x2[2 * l + 1];
        for (int i = 1; i < n; i++) {
            double cr = cre[i * b + l], ci = cim[i * b + l], sv = s[i * b + l];
            double t2r = x2[i * b2 + 2 * l], t2i = x2[i * b2 + 2 * l + 1];
            x2[(i - 1) * b2 + 2 * l] = (cr * t1r - ci * t1i) - sv * t2r;
            x2[(i - 1) * b2 + 2 * l + 1] = (cr * t1i + ci * t1r) - sv * t2i;
            double nr = sv * t1r + (cr * t2r + ci * t2i);
            double ni = sv * t1i + (cr * t2i - ci * t2r);
            t1r = nr;
            t1i = ni;
        }
        x2[(n - 1) * b2 + 2 * l] = t1r;
        x2[(n - 1) * b2 + 2 * l + 1] = t1i;
    }
}

/* ------------------------------------------------------------------ */
/* tiled driver: one batch of b shifts (reduce.py:39-171 + backsolve.py:62-313) */
/* ------------------------------------------------------------------ */

/* copy H[r0:r1, c0:c1] (H column-major, ld n) into a C-order buffer */
static void take_tile(const double* H, int64_t n, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                      double* out) {
    int64_t w = c1 - c0;
    for (int64_t i = r0; i < r1; i++)
        for (int64_t j = c0; j < c1; j++) out[(i - r0) * w + (j - c0)] = H[j * n + i];
}

/* Runs one batch.  ncol = b (real) or 2b (complex, interleaved).
 * X: n x ncol (C order) holds B on entry and the solution on exit.
 * c_re/c_im/s: n x b (C order) out.  alpha_e: N x b out (segment exponents).
 * Returns 0, or a packed status with *phase = 1 (reduce: degenerate) / 2 (solve:
 * singular) and *tile = tile column. */
static int64_t solve_batch(const double* H, int64_t n, int b_r, int cplx_, int b,
                           const double* lam_re, const double* lam_im, double* X, double* c_re,
                           double* c_im, double* s_arr, int* alpha_e, double* norms,
                           double* log2norm, int* alpha_col_e, int robust, int mode, int* phase,
                           int* tile) {
    const int N = (int)((n + b_r - 1) / b_r);
    const int ncol = cplx_ ? 2 * b : b;
    /* OverflowBudget.for_grid (overflow.py:41-47), or the caller's budget
     * (backsolve.py:342-346) set with oracle_set_omega */
    const double omega = robust ? (g_omega > 0.0 ? g_omega : (1.7976931348623157e308 / 2.0) / (double)b_r)
                                : INFINITY;
    int64_t* ends = (int64_t*)malloc(sizeof(int64_t) * N);
    for (int t = 0; t < N; t++) ends[t] = (int64_t)(t + 1) * b_r < n ? (int64_t)(t + 1) * b_r : n;
    double* cross = (double*)malloc(sizeof(double) * (size_t)n * N * ncol); /* (n, N, ncol) */
#define CR(i, t) (cross + ((size_t)(i) * N + (t)) * ncol)
    double* zeros = (double*)calloc((size_t)b, sizeof(double));
    double* hbuf = (double*)malloc(sizeof(double) * (size_t)b_r * b_r);
    double* hleft = (double*)malloc(sizeof(double) * (size_t)b_r);
    double* tA = (double*)malloc(sizeof(double) * (size_t)b_r * ncol);
    double* tB = (double*)malloc(sizeof(double) * (size_t)b_r * ncol);
    double* tC = (double*)malloc(sizeof(double) * (size_t)b_r * b);
    double* tCi = (double*)malloc(sizeof(double) * (size_t)b_r * b);
    double* tS = (double*)malloc(sizeof(double) * (size_t)b_r * b);
    int64_t st = 0;
    *phase = 0;
    *tile = -1;

    /* crossover init, reduce.py:66-69 / 77-78 */
    for (int64_t i = 0; i < n; i++) {
        double* row = CR(i, N - 1);
        for (int l = 0; l < b; l++) {
            if (cplx_) {
                row[2 * l] = H[(n - 1) * n + i];
                row[2 * l + 1] = 0.0;
            } else {
                row[l] = H[(n - 1) * n + i];
            }
        }
    }
    for (int l = 0; l < b; l++) {
        if (cplx_) {
            CR(n - 1, N - 1)[2 * l] -= lam_re[l];
            CR(n - 1, N - 1)[2 * l + 1] -= lam_im[l];
        } else {
            CR(n - 1, N - 1)[l] -= lam_re[l];
        }
    }

    /* ---- reduction, tile columns right to left ---- */
    for (int jt = N - 1; jt >= 0; jt--) {
        int64_t js = (int64_t)jt * b_r, je = ends[jt];
        int k = (int)(je - js);
        take_tile(H, n, js, je, js, je - 1, hbuf);
        int has_left = jt > 0;
        for (int i = 0; i < k; i++) hleft[i] = has_left ? H[(js - 1) * n + js + i] : 0.0;
        for (int i = 0; i < k; i++) memcpy(tA + (size_t)i * ncol, CR(js + i, jt), sizeof(double) * ncol);
        int64_t r;
        if (cplx_)
            r = oracle_creduce_diag(k, b, hbuf, hleft, has_left, lam_re, lam_im, tA, tC, tCi, tS);
        else
            r = oracle_reduce_diag(k, b, hbuf, hleft, has_left, lam_re, tA, tC, tS);
        if (r) { st = r; *phase = 1; *tile = jt; goto out; }
        memcpy(c_re + js * b, tC, sizeof(double) * (size_t)k * b);
        if (cplx_) memcpy(c_im + js * b, tCi, sizeof(double) * (size_t)k * b);
        memcpy(s_arr + js * b, tS, sizeof(double) * (size_t)k * b);
        for (int it = jt - 1; it >= 0; it--) {
            int64_t is = (int64_t)it * b_r, ie = ends[it];
            int kk = (int)(ie - is), w = k;
            int shifted = it == jt - 1;
            take_tile(H, n, is, ie, js - 1, je - 1, hbuf);
            for (int i = 0; i < kk; i++) memcpy(tA + (size_t)i * ncol, CR(is + i, jt), sizeof(double) * ncol);
            if (cplx_)
                oracle_creduce_offdiag(kk, w, b, hbuf, shifted ? lam_re : zeros,
                                       shifted ? lam_im : zeros, c_re + js * b, c_im + js * b,
                                       s_arr + js * b, tA, tB);
            else
                oracle_reduce_offdiag(kk, w, b, hbuf, shifted ? lam_re : zeros, c_re + js * b,
                                      s_arr + js * b, tA, tB);
            for (int i = 0; i < kk; i++) memcpy(CR(is + i, jt - 1), tB + (size_t)i * ncol, sizeof(double) * ncol);
        }
    }

    /* ---- substitution (backsolve.py:62-313) ---- */
    for (size_t q = 0; q < (size_t)N * b; q++) alpha_e[q] = 0;
    int stopped = 0;
    for (int jt = N - 1; jt >= 0; jt--) {
        int64_t js = (int64_t)jt * b_r, je = ends[jt];
        int k = (int)(je - js);
        take_tile(H, n, js, je, js, je - 1, hbuf);
        int has_left = jt > 0;
        for (int i = 0; i < k; i++) hleft[i] = has_left ? H[(js - 1) * n + js + i] : 0.0;
        for (int i = 0; i < k; i++) memcpy(tA + (size_t)i * ncol, CR(js + i, jt), sizeof(double) * ncol);
        int64_t r;
        if (cplx_)
            r = oracle_csolve_crsolve(k, b, hbuf, hleft, has_left, lam_re, lam_im, tA, c_re + js * b,
                                      c_im + js * b, s_arr + js * b, X + js * ncol,
                                      alpha_e + (size_t)jt * b, robust, omega);
        else
            r = oracle_solve_rsolve(k, b, hbuf, hleft, has_left, lam_re, tA, c_re + js * b,
                                    s_arr + js * b, X + js * ncol, alpha_e + (size_t)jt * b,
                                    robust, omega);
        if (r) { st = r; *phase = 2; *tile = jt; goto out; }
        if (jt == 0) break;
        for (int it = jt - 1; it >= 0; it--) {
            int64_t is = (int64_t)it * b_r, ie = ends[it];
            int mm = (int)(ie - is);
            int shifted = it == jt - 1;
            take_tile(H, n, is, ie, js - 1, je - 1, hbuf);
            for (int i = 0; i < mm; i++) memcpy(tA + (size_t)i * ncol, CR(is + i, jt), sizeof(double) * ncol);
            if (cplx_)
                oracle_cupdate_crupdate(mm, k, b, hbuf, tA, alpha_e + (size_t)jt * b, X + js * ncol,
                                        shifted ? lam_re : zeros, shifted ? lam_im : zeros, shifted,
                                        c_re + js * b, c_im + js * b, s_arr + js * b,
                                        alpha_e + (size_t)it * b, X + is * ncol, robust, omega);
            else
                oracle_update_rupdate(mm, k, b, hbuf, tA, alpha_e + (size_t)jt * b, X + js * ncol,
                                      shifted ? lam_re : zeros, shifted, c_re + js * b,
                                      s_arr + js * b, alpha_e + (size_t)it * b, X + is * ncol,
                                      robust, omega);
        }
        if (jt == g_stop_jt) {  /* test hook: the state after column jt's updates */
            stopped = 1;
            break;
        }
    }
    if (stopped) {
        for (int l = 0; l < b; l++) {
            norms[l] = NAN;
            log2norm[l] = NAN;
            alpha_col_e[l] = 0;
        }
    } else if (robust) {
        if (cplx_)
            oracle_crbacktransform((int)n, b, N, c_re, c_im, s_arr, alpha_e, ends, X, norms,
                                   log2norm, alpha_col_e, mode, omega);
        else
            oracle_rbacktransform((int)n, b, N, c_re, s_arr, alpha_e, ends, X, norms, log2norm,
                                  alpha_col_e, mode, omega);
    } else {
        if (cplx_)
            oracle_cbacktransform((int)n, b, c_re, c_im, s_arr, X);
        else
            oracle_backtransform((int)n, b, c_re, s_arr, X);
        for (int l = 0; l < b; l++) {
            norms[l] = NAN;
            log2norm[l] = NAN;
            alpha_col_e[l] = 0;
        }
    }
out:
#undef CR
    free(ends);
    free(cross);
    free(zeros);
    free(hbuf);
    free(hleft);
    free(tA);
    free(tB);
    free(tC);
    free(tCi);
    free(tS);
    return st;
}

typedef struct {
    const double* H;
    int64_t n;
    int b_r, b_c, cplx_;
    int64_t m;
    int N, ncols_all, M;
    const double *lam_re, *lam_im, *B;
    double *X, *c_re, *c_im, *s;
    int *seg_alpha_e, *alpha_col_e;
    double *norms, *log2norm;
    int robust, mode;
    int64_t* bst;
    int *bphase, *btile;
    int next;
    pthread_mutex_t lock;
} batch_job;

/* one batch of the reference's ShiftBatch (core.py:132-158) */
static void run_one_batch(batch_job* j, int bi) {
    const int64_t n = j->n, m = j->m;
    const int N = j->N, cplx_ = j->cplx_, ncols_all = j->ncols_all;
    int ls = bi * j->b_c, le = ls + j->b_c < m ? ls + j->b_c : (int)m;
    int b = le - ls, nc = cplx_ ? 2 * b : b;
    double* Xb = (double*)malloc(sizeof(double) * (size_t)n * nc);
    double* cb = (double*)malloc(sizeof(double) * (size_t)n * b);
    double* cib = cplx_ ? (double*)malloc(sizeof(double) * (size_t)n * b) : NULL;
    double* sb = (double*)malloc(sizeof(double) * (size_t)n * b);
    int* ab = (int*)malloc(sizeof(int) * (size_t)N * b);
    double* nb = (double*)malloc(sizeof(double) * b);
    double* lb = (double*)malloc(sizeof(double) * b);
    int* acb = (int*)malloc(sizeof(int) * b);
    int co = cplx_ ? 2 * ls : ls;
    for (int64_t i = 0; i < n; i++) memcpy(Xb + i * nc, j->B + i * ncols_all + co, sizeof(double) * nc);
    j->bst[bi] = solve_batch(j->H, n, j->b_r, cplx_, b, j->lam_re + ls, cplx_ ? j->lam_im + ls : NULL,
                             Xb, cb, cib, sb, ab, nb, lb, acb, j->robust, j->mode, &j->bphase[bi],
                             &j->btile[bi]);
    if (!j->bst[bi]) {
        for (int64_t i = 0; i < n; i++) {
            memcpy(j->X + i * ncols_all + co, Xb + i * nc, sizeof(double) * nc);
            if (j->c_re) memcpy(j->c_re + i * m + ls, cb + i * b, sizeof(double) * b);
            if (j->c_im && cplx_) memcpy(j->c_im + i * m + ls, cib + i * b, sizeof(double) * b);
            if (j->s) memcpy(j->s + i * m + ls, sb + i * b, sizeof(double) * b);
        }
        for (int t = 0; t < N; t++)
            if (j->seg_alpha_e)
                memcpy(j->seg_alpha_e + (size_t)t * m + ls, ab + (size_t)t * b, sizeof(int) * b);
        for (int l = 0; l < b; l++) {
            if (j->alpha_col_e) j->alpha_col_e[ls + l] = acb[l];
            if (j->norms) j->norms[ls + l] = nb[l];
            if (j->log2norm) j->log2norm[ls + l] = lb[l];
        }
    }
    free(Xb); free(cb); free(cib); free(sb); free(ab); free(nb); free(lb); free(acb);
}

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    for (;;) {
        pthread_mutex_lock(&j->lock);
        int bi = j->next++;
        pthread_mutex_unlock(&j->lock);
        if (bi >= j->M) break;
        run_one_batch(j, bi);
    }
    return NULL;
}

/*
 * oracle_hsrq_solve -- dhsrq3/chsrq3 (backsolve.py:350-388) and the
 * _solve_group seam (inviter.py:91-106, mode=1 eigvec).
 *
 * H: n x n column-major.  lam_re/lam_im: m shifts (lam_im NULL for real).
 * B/X: n x ncols C-order (ncols = m real, 2m complex interleaved); B may
 * alias X.  Outputs (any may be NULL): c_re, c_im, s (n x m C order),
 * seg_alpha_e (N x m), alpha_col_e (m), norms (m), log2norm (m).
 * Batches of b_c shifts are independent; nthreads > 1 runs them in parallel.
 * Returns 0 or the packed status of the first failure in the reference's
 * single-worker order (all reductions precede all solves, batches in order);
 * err[0] = phase (1 degenerate / 2 singular), err[1] = tile column,
 * err[2] = global shift index, err[3] = local row.
 */
int64_t oracle_hsrq_solve(const double* H, int64_t n, int b_r, int b_c, int cplx_, int64_t m,
                          const double* lam_re, const double* lam_im, const double* B, double* X,
                          double* c_re, double* c_im, double* s, int* seg_alpha_e,
                          int* alpha_col_e, double* norms, double* log2norm, int robust, int mode,
                          int nthreads, int64_t* err) {
    const int N = (int)((n + b_r - 1) / b_r);
    const int ncols_all = cplx_ ? 2 * (int)m : (int)m;
    if (b_c > m) b_c = (int)m;
    const int M = (int)((m + b_c - 1) / b_c);
    int64_t* bst = (int64_t*)calloc((size_t)M, sizeof(int64_t));
    int* bphase = (int*)calloc((size_t)M, sizeof(int));
    int* btile = (int*)calloc((size_t)M, sizeof(int));
    if (nthreads < 1) nthreads = 1;
    if (nthreads > M) nthreads = M;
    batch_job job = {H, n, b_r, b_c, cplx_, m, N, ncols_all, M, lam_re, lam_im, B, X, c_re, c_im, s,
                     seg_alpha_e, alpha_col_e, norms, log2norm, robust, mode, bst, bphase, btile, 0};
    pthread_mutex_init(&job.lock, NULL);
    if (nthreads == 1) {
        batch_worker(&job);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
        for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, batch_worker, &job);
        for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
        free(th);
    }
    pthread_mutex_destroy(&job.lock);
    int64_t st = 0;
    for (int pass = 1; pass <= 2 && !st; pass++)
        for (int bi = 0; bi < M; bi++)
            if (bst[bi] && bphase[bi] == pass) {
                st = bst[bi];
                if (err) {
                    err[0] = pass;
                    err[1] = btile[bi];
                    err[2] = (int64_t)bi * b_c + ((st >> 21) & ((1 << 21) - 1));
                    err[3] = st & ((1 << 21) - 1);
                }
                break;
            }
    free(bst);
    free(bphase);
    free(btile);
    return st;
}

/* ------------------------------------------------------------------ */
/* Henry's single-sweep RQ solve (the reference's baseline solver)      */
/* ------------------------------------------------------------------ */

/*
 * oracle_henry_solve_real -- henry_solve_real, K/numba_backend.py:830-873,
 * behind henry_rq_solve (reference.py:21-60).  H n x n column-major; lam b
 * shifts; x in/out C-order (n, b).  Loop order kept: kp descending, shifts
 * inside, so the returned packed status is the reference's first failure.
 * Ends with the unguarded backtransform (K/numba_backend.py:314-323).
 */
int64_t oracle_henry_solve_real(const double* H, int64_t n, int b, const double* lam, double* x) {
#define HH(i, j) H[(int64_t)(j) * n + (i)]
    double* v = (double*)malloc(sizeof(double) * (size_t)n * b);
    double* cc = (double*)malloc(sizeof(double) * (size_t)n * b);
    double* cs = (double*)malloc(sizeof(double) * (size_t)n * b);
    int64_t st = 0;
    for (int64_t i = 0; i < n; i++)
        for (int l = 0; l < b; l++) v[i * b + l] = HH(i, n - 1);
    for (int l = 0; l < b; l++) v[(n - 1) * b + l] -= lam[l];
    for (int l = 0; l < b; l++) {
        cc[l] = 1.0;
        cs[l] = 0.0;
    }
    for (int64_t kp = n - 1; kp > 0 && !st; kp--) {
        const double a = HH(kp, kp - 1);
        for (int l = 0; l < b; l++) {
            const double vk = v[kp * b + l];
            const double r = hypot(a, vk);
            if (r == 0.0) { st = pack_status(KIND_DEGENERATE, l, kp); break; }
            const double c = vk / r, s = -a / r;
            cc[kp * b + l] = c;
            cs[kp * b + l] = s;
            const double phi = vk * c - a * s;
            if (phi == 0.0) { st = pack_status(KIND_SINGULAR, l, kp); break; }
            x[kp * b + l] /= phi;
            const double tau1 = s * x[kp * b + l], tau2 = c * x[kp * b + l];
            for (int64_t i = 0; i < kp - 1; i++) {
                const double hi = HH(i, kp - 1);
                x[i * b + l] = (x[i * b + l] - tau2 * v[i * b + l]) + tau1 * hi;
                v[i * b + l] = c * hi + s * v[i * b + l];
            }
            const double hd = HH(kp - 1, kp - 1);
            x[(kp - 1) * b + l] = (x[(kp - 1) * b + l] - tau2 * v[(kp - 1) * b + l]) +
                                  tau1 * (hd - lam[l]);
            v[(kp - 1) * b + l] = c * (hd - lam[l]) + s * v[(kp - 1) * b + l];
        }
    }
    if (!st) {
        for (int l = 0; l < b; l++) {
            if (v[l] == 0.0) { st = pack_status(KIND_SINGULAR, l, 0); break; }
            x[l] /= v[l];
        }
    }
    if (!st) oracle_backtransform((int)n, b, cc, cs, x);
    free(v);
    free(cc);
    free(cs);
    return st;
}

/*
 * oracle_henry_solve_complex -- henry_solve_complex, K/numba_backend.py:876-923.
 * lam: b complex shifts interleaved (re, im); x in/out C-order (n, b) complex
 * (interleaved doubles, numpy complex128 layout).  numba lowers real*complex
 * and complex/real by promoting the real to (r, 0).
 */
int64_t oracle_henry_solve_complex(const double* H, int64_t n, int b, const double* lam2,
                                   double* x2) {
    cplx* v = (cplx*)malloc(sizeof(cplx) * (size_t)n * b);
    cplx* cc = (cplx*)malloc(sizeof(cplx) * (size_t)n * b);
    double* cs = (double*)malloc(sizeof(double) * (size_t)n * b);
    cplx* x = (cplx*)x2;
    const cplx* lam = (const cplx*)lam2;
    int64_t st = 0;
    for (int64_t i = 0; i < n; i++)
        for (int l = 0; l < b; l++) v[i * b + l] = C(HH(i, n - 1), 0.0);
    for (int l = 0; l < b; l++) v[(n - 1) * b + l] = csub(v[(n - 1) * b + l], lam[l]);
    for (int l = 0; l < b; l++) {
        cc[l] = C(1.0, 0.0);
        cs[l] = 0.0;
    }
    for (int64_t kp = n - 1; kp > 0 && !st; kp--) {
        const double a = HH(kp, kp - 1);
        for (int l = 0; l < b; l++) {
            const cplx vk = v[kp * b + l];
            const double r = hypot(a, cabs_(vk));
            if (r == 0.0) { st = pack_status(KIND_DEGENERATE, l, kp); break; }
            const cplx c = cdiv(vk, C(r, 0.0));
            const double s = -a / r;
            cc[kp * b + l] = c;
            cs[kp * b + l] = s;
            const cplx cj = C(c.re, -c.im);
            const cplx phi = csub(cmul(cj, vk), C(a * s, 0.0));
            if (phi.re == 0.0 && phi.im == 0.0) { st = pack_status(KIND_SINGULAR, l, kp); break; }
            x[kp * b + l] = cdiv(x[kp * b + l], phi);
            const cplx tau1 = cmul(C(s, 0.0), x[kp * b + l]);
            const cplx tau2 = cmul(cj, x[kp * b + l]);
            for (int64_t i = 0; i < kp - 1; i++) {
                const cplx hi = C(HH(i, kp - 1), 0.0);
                x[i * b + l] = cadd(csub(x[i * b + l], cmul(tau2, v[i * b + l])), cmul(tau1, hi));
                v[i * b + l] = cadd(cmul(c, hi), cmul(C(s, 0.0), v[i * b + l]));
            }
            const cplx hdl = csub(C(HH(kp - 1, kp - 1), 0.0), lam[l]);
            x[(kp - 1) * b + l] =
                cadd(csub(x[(kp - 1) * b + l], cmul(tau2, v[(kp - 1) * b + l])), cmul(tau1, hdl));
            v[(kp - 1) * b + l] = cadd(cmul(c, hdl), cmul(C(s, 0.0), v[(kp - 1) * b + l]));
        }
    }
    for (int l = 0; l < b && !st; l++) {
        if (v[l].re == 0.0 && v[l].im == 0.0) { st = pack_status(KIND_SINGULAR, l, 0); break; }
        x[l] = cdiv(x[l], v[l]);
        cplx t1 = x[l];
        for (int64_t i = 1; i < n; i++) {
            const cplx t2 = x[i * b + l];
            const cplx ci = cc[i * b + l];
            const cplx si = C(cs[i * b + l], 0.0);
            x[(i - 1) * b + l] = csub(cmul(ci, t1), cmul(si, t2));
            t1 = cadd(cmul(si, t1), cmul(C(ci.re, -ci.im), t2));
        }
        x[(n - 1) * b + l] = t1;
    }
    free(v);
    free(cc);
    free(cs);
    return st;
#undef HH
}

/* ------------------------------------------------------------------ */
/* Stewart compact rotation codes, givens.py:90-198                    */
/* ------------------------------------------------------------------ */

static double compact_encode1(double c, double s) { /* compact_encode, givens.py:107-113 */
    if (fabs(s) <= fabs(c)) {
        const double base = c >= 0.0 ? 0.0 : 2.0;
        return s != 0.0 ? copysign(fabs(s) + base, s) : base;
    }
    const double base = s >= 0.0 ? 4.0 : 6.0;
    return c != 0.0 ? copysign(fabs(c) + base, c) : base;
}

static double max0(double u) { return u > 0.0 ? u : 0.0; } /* Python max(0.0, u) */

static void compact_decode1(double t, double* c, double* s) { /* givens.py:116-131 */
    const double at = fabs(t);
    if (at <= 1.0) {
        *s = t;
        *c = sqrt(max0(1.0 - *s * *s));
    } else if (at <= 3.0) {
        *s = at != 2.0 ? copysign(at - 2.0, t) : 0.0;
        *c = -sqrt(max0(1.0 - *s * *s));
    } else if (at <= 5.0) {
        *c = at != 4.0 ? copysign(at - 4.0, t) : 0.0;
        *s = sqrt(max0(1.0 - *c * *c));
    } else {
        *c = at != 6.0 ? copysign(at - 6.0, t) : 0.0;
        *s = -sqrt(max0(1.0 - *c * *c));
    }
}

/* compact_encode_table(_complex) / compact_decode_table(_complex), elementwise. */
void oracle_compact_encode(int64_t count, int cplx, const double* c_re, const double* c_im,
                           const double* s, double* t1, double* t2) {
    for (int64_t i = 0; i < count; i++) {
        if (!cplx) {
            t1[i] = compact_encode1(c_re[i], s[i]);
            continue;
        }
        const double ac = hypot(c_re[i], c_im[i]); /* abs(complex) */
        t1[i] = compact_encode1(ac, s[i]);
        t2[i] = ac == 0.0 ? compact_encode1(1.0, 0.0) : compact_encode1(c_re[i] / ac, c_im[i] / ac);
    }
}

void oracle_compact_decode(int64_t count, int cplx, const double* t1, const double* t2,
                           double* c_re, double* c_im, double* s) {
    for (int64_t i = 0; i < count; i++) {
        if (!cplx) {
            compact_decode1(t1[i], &c_re[i], &s[i]);
            continue;
        }
        double ac, dc, ds;
        compact_decode1(t1[i], &ac, &s[i]);
        compact_decode1(t2[i], &dc, &ds);
        c_re[i] = ac * dc;
        c_im[i] = ac * ds;
    }
}

/* ------------------------------------------------------------------ */
/* Front end: householder_hessenberg, testprob.py:146-174 (unblocked)  */
/* ------------------------------------------------------------------ */

/* a: n x n column-major, overwritten by H; q: n x n column-major out (Q, with
 * Q^T A Q = H).  Per column j: x = a[j+1:, j]; skipped when x[1:].x[1:] == 0;
 * alpha = -sign(x0) hypot(x0, sqrt(tail)); v = (x - alpha e1)/||.||; the
 * two-sided update with P = I - 2 v v^T and Q <- Q P. */
void oracle_householder_hessenberg(int64_t n, double* a, double* q) {
#define A_(i, j) a[(int64_t)(j) * n + (i)]
#define Q_(i, j) q[(int64_t)(j) * n + (i)]
    for (int64_t j = 0; j < n; j++)
        for (int64_t i = 0; i < n; i++) Q_(i, j) = i == j ? 1.0 : 0.0;
    double* v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j + 2 < n; j++) {
        const int64_t m = n - j - 1;
        double tail = 0.0;
        for (int64_t r = 1; r < m; r++) tail += A_(j + 1 + r, j) * A_(j + 1 + r, j);
        if (tail == 0.0) continue;
        const double x0 = A_(j + 1, j);
        const double nrm = hypot(x0, sqrt(tail));
        const double alpha = x0 >= 0.0 ? -nrm : nrm;
        double mx = 0.0, ss = 0.0;
        for (int64_t r = 0; r < m; r++) {
            v[r] = r == 0 ? x0 - alpha : A_(j + 1 + r, j);
            if (fabs(v[r]) > mx) mx = fabs(v[r]);
        }
        for (int64_t r = 0; r < m; r++) ss += (v[r] / mx) * (v[r] / mx);
        const double vn = mx * sqrt(ss);
        for (int64_t r = 0; r < m; r++) v[r] /= vn;
        /* left: a[j+1:, j:] -= 2 v (v^T a[j+1:, j:]) */
        for (int64_t c = j; c < n; c++) {
            double d = 0.0;
            for (int64_t r = 0; r < m; r++) d += v[r] * A_(j + 1 + r, c);
            for (int64_t r = 0; r < m; r++) A_(j + 1 + r, c) -= 2.0 * v[r] * d;
        }
        /* right: a[:, j+1:] -= 2 (a[:, j+1:] v) v^T ; q likewise */
        for (int pass = 0; pass < 2; pass++) {
            double* M = pass ? q : a;
            for (int64_t i = 0; i < n; i++) {
                double d = 0.0;
                for (int64_t r = 0; r < m; r++) d += M[(j + 1 + r) * n + i] * v[r];
                w[i] = d;
            }
            for (int64_t r = 0; r < m; r++)
                for (int64_t i = 0; i < n; i++) M[(j + 1 + r) * n + i] -= 2.0 * w[i] * v[r];
        }
        A_(j + 1, j) = alpha;
        for (int64_t r = j + 2; r < n; r++) A_(r, j) = 0.0;
    }
    free(v);
    free(w);
#undef A_
#undef Q_
}
