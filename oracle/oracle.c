/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for arXiv 2111.14317.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2111_14317_b200/csrc) and
 * never includes or calls it.
 *
 * What it computes (each function cites the passage it follows; "P:n" is a line of
 * /root/reference/PAPER.md, "S:n" a line of SPEC.md):
 *
 *   orc_evaluate      H, dH/dx, dH/dt of the polyhedral homotopy, Eq. (1) P:117-126,
 *                     by the DEFINITION: every monomial by repeated complex
 *                     multiplication (exponentiation by squaring), every derivative
 *                     by symbolic term-wise differentiation.  No log, no exp, no GEMM
 *                     (BASELINE.json north_star).  Also returns the
 *                     absolute term sums used by the parity metric (R9).
 *   orc_evaluate_x    the same algorithm on an extended-range type (mantissa, int64
 *                     binary exponent) for inputs whose monomials leave double range
 *                     (SURVEY O2).
 *   orc_lu_solve      Gaussian elimination with partial pivoting (route 1).
 *   orc_dirs_qr       the paper's route: Householder QR of J^T, null space = conjugate
 *                     of the last two columns of Q, row-reduce the trailing 2x2 to I
 *                     (Alg. 3).
 *   orc_euler_newton  affine Euler direction (Davidenko) and Newton
 *                     direction: Jx dE = -dH/dt, Jx dN = -H.
 *   orc_pc_step       the paper's simplified Euler-Newton step: one Euler
 *                     prediction in tau (t = e^tau, Eq. (2)) followed by K
 *                     Newton iterations.
 *   orc_track         adaptive predictor-corrector tracking tau0 -> 0 (SURVEY §8(c) O4,
 *                     step control = DESIGN.md reading R14).
 *   orc_track_x       the same tracker with extended-range state for start points far outside
 *                     double range (polyhedral start points at large |tau0|).
 *   orc_proj_*        the projective formulation and its directions (P:237-252,
 *                     P:277-291): evaluation of the homogenised system, the bordered
 *                     [dH^/dy; y^*] 2-RHS solve, the step and the tracker in homogeneous
 *                     coordinates.
 *
 * All complex numbers are interleaved (re, im) doubles.  Arithmetic is plain C
 * double in a fixed order; OpenMP only distributes independent points/paths.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

enum {
    ORC_PT_OK = 0,
    ORC_PT_ZERO_COORD = 1,
    ORC_PT_NONFINITE = 2,
    ORC_PT_SINGULAR = 4,
    ORC_PT_STEP_UNDERFLOW = 8,
    ORC_PT_MAX_STEPS = 16,
    ORC_PT_DIVERGED = 32,
};

/* ------------------------------------------------------------------ */
/* complex helpers written out (no reliance on C Annex G semantics)    */
/* ------------------------------------------------------------------ */
static inline cplx mk(double re, double im) { return CMPLX(re, im); }

static inline cplx cmul(cplx a, cplx b)
{
    double ar = creal(a), ai = cimag(a), br = creal(b), bi = cimag(b);
    return mk(ar * br - ai * bi, ar * bi + ai * br);
}

/* Smith's algorithm for a / b. */
static inline cplx cdiv(cplx a, cplx b)
{
    double ar = creal(a), ai = cimag(a), br = creal(b), bi = cimag(b);
    if (fabs(br) >= fabs(bi)) {
        double r = bi / br, d = br + bi * r;
        return mk((ar + ai * r) / d, (ai - ar * r) / d);
    } else {
        double r = br / bi, d = br * r + bi;
        return mk((ar * r + ai) / d, (ai * r - ar) / d);
    }
}

static inline double cabs1(cplx a) { return fabs(creal(a)) + fabs(cimag(a)); }

static inline cplx load(const double *p) { return mk(p[0], p[1]); }
static inline void store(double *p, cplx v) { p[0] = creal(v); p[1] = cimag(v); }

/* b^e for integer e >= 0 by exponentiation by squaring. */
static cplx cpow_nat(cplx b, int64_t e)
{
    cplx r = mk(1.0, 0.0);
    while (e > 0) {
        if (e & 1) r = cmul(r, b);
        e >>= 1;
        if (e) b = cmul(b, b);
    }
    return r;
}

static double rpow_nat(double b, int64_t e)
{
    double r = 1.0;
    while (e > 0) {
        if (e & 1) r *= b;
        e >>= 1;
        if (e) b *= b;
    }
    return r;
}

/* x^a for an integer (Laurent) exponent: negative powers multiply r = 1/x. */
static cplx cpow_int(cplx x, cplx r, int64_t a)
{
    return a >= 0 ? cpow_nat(x, a) : cpow_nat(r, -a);
}

/* ------------------------------------------------------------------ */
/* the system: per-equation term segments of Eq. (1)       */
/* ------------------------------------------------------------------ */
typedef struct {
    int n;                 /* equations                                  */
    const int64_t *off;    /* [n+1] terms of eq k are [off[k], off[k+1]) */
    const int32_t *a;      /* [M][nv] integer exponents a                */
    const double *c;       /* [M][2] coefficients c_{k,a}                */
    const int64_t *w;      /* [M] integer liftings omega_k(a) >= 0       */
    int nv;                /* variables: n (affine) or n + 1 (projective) */
} orc_sys;

/*
 * Evaluate one point:
 *   h_k        = sum_a c x^a t^w
 *   dh_k/dx_j  = sum_{a_j != 0} c a_j x^{a - e_j} t^w          (symbolic)
 *   dh_k/dt    = sum_{w >= 1}   c w   x^a t^{w-1}
 * S* are the absolute term sums sum |term| of each entry (parity metric scale).
 * Returns a status bit set.
 */
static int eval_point(const orc_sys *s, const double *xp, double t,
                      double *H, double *Jx, double *Jt,
                      double *SH, double *SJx, double *SJt)
{
    const int n = s->n, nv = s->nv;
    cplx x[65], r[65];
    int st = ORC_PT_OK;
    for (int j = 0; j < nv; ++j) {
        x[j] = load(xp + 2 * j);
        if (creal(x[j]) == 0.0 && cimag(x[j]) == 0.0) st |= ORC_PT_ZERO_COORD;
        if (!isfinite(creal(x[j])) || !isfinite(cimag(x[j]))) st |= ORC_PT_NONFINITE;
        r[j] = cdiv(mk(1.0, 0.0), x[j]);
    }
    for (int k = 0; k < n; ++k) {
        cplx h = 0, ht = 0, hx[65];
        double sh = 0, sht = 0, shx[65];
        for (int j = 0; j < nv; ++j) { hx[j] = 0; shx[j] = 0; }
        for (int64_t i = s->off[k]; i < s->off[k + 1]; ++i) {
            const int32_t *a = s->a + i * nv;
            const cplx c = load(s->c + 2 * i);
            const int64_t w = s->w[i];
            /* the term itself: c * prod_j x_j^{a_j} * t^w */
            cplx T = c;
            for (int j = 0; j < nv; ++j)
                if (a[j] != 0) T = cmul(T, cpow_int(x[j], r[j], a[j]));
            T = cmul(T, mk(rpow_nat(t, w), 0.0));
            h += T;
            sh += cabs(T);
            /* d/dx_j: c * a_j * prod_l x_l^{a_l - [l==j]} * t^w, from scratch */
            for (int j = 0; j < nv; ++j) {
                if (a[j] == 0) continue;
                cplx D = cmul(c, mk((double)a[j], 0.0));
                for (int l = 0; l < nv; ++l) {
                    int64_t e = a[l] - (l == j ? 1 : 0);
                    if (e != 0) D = cmul(D, cpow_int(x[l], r[l], e));
                }
                D = cmul(D, mk(rpow_nat(t, w), 0.0));
                hx[j] += D;
                shx[j] += cabs(D);
            }
            /* d/dt: c * w * x^a * t^{w-1} */
            if (w >= 1) {
                cplx D = cmul(c, mk((double)w, 0.0));
                for (int j = 0; j < nv; ++j)
                    if (a[j] != 0) D = cmul(D, cpow_int(x[j], r[j], a[j]));
                D = cmul(D, mk(rpow_nat(t, w - 1), 0.0));
                ht += D;
                sht += cabs(D);
            }
        }
        if (H) store(H + 2 * k, h);
        if (Jt) store(Jt + 2 * k, ht);
        if (SH) SH[k] = sh;
        if (SJt) SJt[k] = sht;
        for (int j = 0; j < nv; ++j) {
            if (Jx) store(Jx + 2 * (k * nv + j), hx[j]);
            if (SJx) SJx[k * nv + j] = shx[j];
        }
    }
    return st;
}

int orc_evaluate(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                 int64_t p, const double *x, const double *t,
                 double *H, double *Jx, double *Jt, double *SH, double *SJx, double *SJt,
                 uint8_t *status)
{
    if (n < 1 || n > 64) return -1;
    orc_sys s = {n, off, a, c, w, n};
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < p; ++q) {
        int st = eval_point(&s, x + 2 * n * q, t[q],
                            H ? H + 2 * n * q : 0, Jx ? Jx + 2 * n * n * q : 0,
                            Jt ? Jt + 2 * n * q : 0, SH ? SH + n * q : 0,
                            SJx ? SJx + n * n * q : 0, SJt ? SJt + n * q : 0);
        if (status) status[q] = (uint8_t)st;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* extended range: value = m * 2^e                         */
/* ------------------------------------------------------------------ */
typedef struct { cplx m; int64_t e; } xc;

static xc xnorm(cplx m, int64_t e)
{
    double big = fmax(fabs(creal(m)), fabs(cimag(m)));
    xc r;
    if (big == 0.0 || !isfinite(big)) { r.m = m; r.e = big == 0.0 ? 0 : e; return r; }
    int s;
    frexp(big, &s);
    r.m = mk(ldexp(creal(m), -s), ldexp(cimag(m), -s));
    r.e = e + s;
    return r;
}

static xc xmul(xc a, xc b) { return xnorm(cmul(a.m, b.m), a.e + b.e); }

static xc xadd(xc a, xc b)
{
    if (creal(b.m) == 0.0 && cimag(b.m) == 0.0) return a;
    if (creal(a.m) == 0.0 && cimag(a.m) == 0.0) return b;
    if (a.e < b.e) { xc t = a; a = b; b = t; }
    int64_t d = b.e - a.e; /* <= 0 */
    if (d < -1200) return a;
    cplx bm = mk(ldexp(creal(b.m), (int)d), ldexp(cimag(b.m), (int)d));
    return xnorm(a.m + bm, a.e);
}

static xc xpow_nat(xc b, int64_t e)
{
    xc r = {mk(1.0, 0.0), 0};
    r = xnorm(r.m, 0);
    while (e > 0) {
        if (e & 1) r = xmul(r, b);
        e >>= 1;
        if (e) b = xmul(b, b);
    }
    return r;
}

static xc xinv(xc a)
{
    /* 1/(m 2^e) = (1/m) 2^-e */
    return xnorm(cdiv(mk(1.0, 0.0), a.m), -a.e);
}

static double xabs_log2(xc a) /* log2 |a|, for the scale sums */
{
    double m = cabs(a.m);
    return m == 0.0 ? -INFINITY : log2(m) + (double)a.e;
}

/*
 * Extended-range evaluation of one point (the same definition as eval_point):
 * x[j], t as xc values; outputs H[k], Jx[k*n+j], Jt[k] and the absolute term sums (xc).
 */
static xc xexp_real(double tau);

/* wr (optional): real per-term liftings omega' (cell-shifted, pht_track_cells); then the t-powers
 * are e^{tau omega'} (Eq. (2)) and Jt receives dh/dtau = sum omega' T instead of dh/dt. */
static void eval_point_x_w(const orc_sys *s, const xc *x, xc t, double tau, const double *wr, xc *H, xc *Jx,
                           xc *Jt, xc *SH, xc *SJx, xc *SJt)
{
    const int n = s->n;
    xc r[64];
    for (int j = 0; j < n; ++j) r[j] = xinv(x[j]);
    for (int k = 0; k < n; ++k) {
        xc h = {0, 0}, ht = {0, 0}, hx[64];
        xc sh = {0, 0}, sht = {0, 0}, shx[64];
        for (int j = 0; j < n; ++j) { hx[j].m = 0; hx[j].e = 0; shx[j].m = 0; shx[j].e = 0; }
        for (int64_t i = s->off[k]; i < s->off[k + 1]; ++i) {
            const int32_t *ai = s->a + i * n;
            xc cc = xnorm(load(s->c + 2 * i), 0);
            xc tw = wr ? xexp_real(tau * wr[i]) : xpow_nat(t, s->w[i]);
            xc T = cc;
            for (int j = 0; j < n; ++j)
                if (ai[j] != 0) T = xmul(T, ai[j] > 0 ? xpow_nat(x[j], ai[j]) : xpow_nat(r[j], -ai[j]));
            T = xmul(T, tw);
            h = xadd(h, T);
            sh = xadd(sh, xnorm(mk(cabs(T.m), 0), T.e));
            for (int j = 0; j < n; ++j) {
                if (ai[j] == 0) continue;
                xc D = xmul(cc, xnorm(mk((double)ai[j], 0), 0));
                for (int l = 0; l < n; ++l) {
                    int64_t e = ai[l] - (l == j ? 1 : 0);
                    if (e != 0) D = xmul(D, e > 0 ? xpow_nat(x[l], e) : xpow_nat(r[l], -e));
                }
                D = xmul(D, tw);
                hx[j] = xadd(hx[j], D);
                shx[j] = xadd(shx[j], xnorm(mk(cabs(D.m), 0), D.e));
            }
            if (wr) { /* d/dtau of c x^a e^{tau omega'} = omega' T */
                xc D = xmul(T, xnorm(mk(wr[i], 0), 0));
                ht = xadd(ht, D);
                sht = xadd(sht, xnorm(mk(cabs(D.m), 0), D.e));
            } else if (s->w[i] >= 1) {
                xc D = xmul(cc, xnorm(mk((double)s->w[i], 0), 0));
                for (int j = 0; j < n; ++j)
                    if (ai[j] != 0) D = xmul(D, ai[j] > 0 ? xpow_nat(x[j], ai[j]) : xpow_nat(r[j], -ai[j]));
                D = xmul(D, xpow_nat(t, s->w[i] - 1));
                ht = xadd(ht, D);
                sht = xadd(sht, xnorm(mk(cabs(D.m), 0), D.e));
            }
        }
        H[k] = h;
        Jt[k] = ht;
        if (SH) SH[k] = sh;
        if (SJt) SJt[k] = sht;
        for (int j = 0; j < n; ++j) {
            Jx[k * n + j] = hx[j];
            if (SJx) SJx[k * n + j] = shx[j];
        }
    }
}

static void eval_point_x(const orc_sys *s, const xc *x, xc t, xc *H, xc *Jx, xc *Jt, xc *SH, xc *SJx, xc *SJt)
{
    eval_point_x_w(s, x, t, 0.0, 0, H, Jx, Jt, SH, SJx, SJt);
}

/* x_j = xm_j * 2^{xe_j}, t = tm * 2^{te}; outputs as (mantissa, exponent) pairs and the
 * log2 of the absolute term sums (LSH etc.) for the parity metric. */
int orc_evaluate_x(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                   int64_t p, const double *xm, const int64_t *xe, const double *tm,
                   const int64_t *te, double *Hm, int64_t *He, double *Jxm, int64_t *Jxe,
                   double *Jtm, int64_t *Jte, double *LSH, double *LSJx, double *LSJt)
{
    if (n < 1 || n > 64) return -1;
    orc_sys s = {n, off, a, c, w, n};
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t q = 0; q < p; ++q) {
        xc x[64], H[64], Jx[64 * 64], Jt[64], SH[64], SJx[64 * 64], SJt[64];
        for (int j = 0; j < n; ++j) x[j] = xnorm(load(xm + 2 * (q * n + j)), xe[q * n + j]);
        xc t = xnorm(mk(tm[q], 0.0), te[q]);
        eval_point_x(&s, x, t, H, Jx, Jt, SH, SJx, SJt);
        for (int k = 0; k < n; ++k) {
            int64_t o = q * n + k;
            store(Hm + 2 * o, H[k].m); He[o] = H[k].e;
            store(Jtm + 2 * o, Jt[k].m); Jte[o] = Jt[k].e;
            LSH[o] = xabs_log2(SH[k]);
            LSJt[o] = xabs_log2(SJt[k]);
            for (int j = 0; j < n; ++j) {
                int64_t oo = o * n + j;
                store(Jxm + 2 * oo, Jx[k * n + j].m); Jxe[oo] = Jx[k * n + j].e;
                LSJx[oo] = xabs_log2(SJx[k * n + j]);
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* route 1: Gaussian elimination with partial pivoting     */
/* ------------------------------------------------------------------ */
/*
 * Solve A X = B, A n x n row-major complex, B n x nrhs row-major complex.
 * Pivot: max |Re|+|Im| in the column, lowest row index on ties (ledger R12).
 * Singular when the pivot |u_kk| <= 1e-14 * (largest |entry| of that row in the original A),
 * or a pivot is non-finite (ledger R13: row-relative, so the flag is invariant under the row
 * scaling of S:316).
 * Returns 0, or ORC_PT_SINGULAR.
 */
int orc_lu_solve(int n, int nrhs, const double *Ain, const double *Bin, double *Xout)
{
    cplx A[64 * 64], B[64 * 4];
    double rmax[64];
    if (n < 1 || n > 64 || nrhs < 1 || nrhs > 4) return -1;
    for (int i = 0; i < n; ++i) {
        rmax[i] = 0.0;
        for (int j = 0; j < n; ++j) {
            A[i * n + j] = load(Ain + 2 * (i * n + j));
            double v = cabs1(A[i * n + j]);
            if (!(v <= rmax[i])) rmax[i] = v; /* NaN propagates */
        }
    }
    for (int i = 0; i < n * nrhs; ++i) B[i] = load(Bin + 2 * i);
    for (int k = 0; k < n; ++k) {
        int piv = k;
        double best = cabs1(A[k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (cabs1(A[i * n + k]) > best) { best = cabs1(A[i * n + k]); piv = i; }
        if (!isfinite(best) || !isfinite(rmax[piv]) || !(best > 1e-14 * rmax[piv])) return ORC_PT_SINGULAR;
        if (piv != k) {
            for (int j = 0; j < n; ++j) { cplx tmp = A[k * n + j]; A[k * n + j] = A[piv * n + j]; A[piv * n + j] = tmp; }
            for (int j = 0; j < nrhs; ++j) { cplx tmp = B[k * nrhs + j]; B[k * nrhs + j] = B[piv * nrhs + j]; B[piv * nrhs + j] = tmp; }
            double tr = rmax[k]; rmax[k] = rmax[piv]; rmax[piv] = tr;
        }
        for (int i = k + 1; i < n; ++i) {
            cplx l = cdiv(A[i * n + k], A[k * n + k]);
            for (int j = k + 1; j < n; ++j) A[i * n + j] -= cmul(l, A[k * n + j]);
            for (int j = 0; j < nrhs; ++j) B[i * nrhs + j] -= cmul(l, B[k * nrhs + j]);
            A[i * n + k] = 0;
        }
    }
    for (int r = 0; r < nrhs; ++r) {
        for (int i = n - 1; i >= 0; --i) {
            cplx s = B[i * nrhs + r];
            for (int j = i + 1; j < n; ++j) s -= cmul(A[i * n + j], load(Xout + 2 * (j * nrhs + r)));
            store(Xout + 2 * (i * nrhs + r), cdiv(s, A[i * n + i]));
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* route 2: the paper's QR null space (Alg. 3)    */
/* ------------------------------------------------------------------ */
/*
 * J is n x (n+2) row-major ([Jx | Jt | H] in the affine form).  Factor
 * J^T = Q [R; 0] with Householder reflections (Q (n+2)x(n+2) unitary).  The null space of
 * J is spanned by conj(Q[:, n]) and conj(Q[:, n+1]).  Stack them as the rows
 * of V (2 x (n+2)) and row-reduce so that the trailing 2x2 block is I (Alg. 3 line
 * P:844); the leading n entries of the two rows are then dE and dN:
 *   J [dE; 1; 0] = 0  and  J [dN; 0; 1] = 0.
 * Returns 0 or ORC_PT_SINGULAR (trailing block singular).
 */
int orc_dirs_qr(int n, const double *J, double *dE, double *dN)
{
    const int m = n + 2;
    cplx A[66 * 66], Q[66 * 66];
    if (n < 1 || n > 64) return -1;
    /* A = J^T (m x n) */
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) A[i * n + j] = load(J + 2 * (j * m + i));
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) Q[i * m + j] = (i == j) ? 1.0 : 0.0;
    for (int k = 0; k < n; ++k) {
        double nrm2 = 0.0;
        for (int i = k; i < m; ++i) nrm2 += creal(A[i * n + k]) * creal(A[i * n + k]) + cimag(A[i * n + k]) * cimag(A[i * n + k]);
        double nrm = sqrt(nrm2);
        if (nrm == 0.0) continue;
        cplx x0 = A[k * n + k];
        double ax0 = cabs(x0);
        cplx phase = ax0 > 0 ? x0 / ax0 : 1.0;
        cplx alpha = -phase * nrm;
        cplx v[66];
        for (int i = 0; i < m; ++i) v[i] = 0;
        for (int i = k; i < m; ++i) v[i] = A[i * n + k];
        v[k] -= alpha;
        double vv = 0.0;
        for (int i = k; i < m; ++i) vv += creal(v[i]) * creal(v[i]) + cimag(v[i]) * cimag(v[i]);
        if (vv == 0.0) continue;
        /* A <- (I - 2 v v^* / v^* v) A */
        for (int j = 0; j < n; ++j) {
            cplx s = 0;
            for (int i = k; i < m; ++i) s += conj(v[i]) * A[i * n + j];
            s *= 2.0 / vv;
            for (int i = k; i < m; ++i) A[i * n + j] -= v[i] * s;
        }
        /* Q <- Q (I - 2 v v^* / v^* v) */
        for (int i = 0; i < m; ++i) {
            cplx s = 0;
            for (int l = k; l < m; ++l) s += Q[i * m + l] * v[l];
            s *= 2.0 / vv;
            for (int l = k; l < m; ++l) Q[i * m + l] -= s * conj(v[l]);
        }
    }
    /* V rows = conj of the last two columns of Q */
    cplx V[2][66];
    for (int i = 0; i < m; ++i) { V[0][i] = conj(Q[i * m + n]); V[1][i] = conj(Q[i * m + n + 1]); }
    /* trailing 2x2 block T = V[:, n:n+2]; V <- T^{-1} V */
    cplx a = V[0][n], b = V[0][n + 1], c = V[1][n], d = V[1][n + 1];
    cplx det = cmul(a, d) - cmul(b, c);
    if (cabs(det) == 0.0 || !isfinite(cabs(det))) return ORC_PT_SINGULAR;
    cplx ia = cdiv(d, det), ib = cdiv(-b, det), ic = cdiv(-c, det), id = cdiv(a, det);
    for (int i = 0; i < n; ++i) {
        cplx e = cmul(ia, V[0][i]) + cmul(ib, V[1][i]);
        cplx f = cmul(ic, V[0][i]) + cmul(id, V[1][i]);
        store(dE + 2 * i, e);
        store(dN + 2 * i, f);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* directions and steps                        */
/* ------------------------------------------------------------------ */
/*
 * Solve at one point: dE = dx/dt with Jx dE = -dH/dt, dN with Jx dN = -H.
 * The system is solved in logarithmic coordinates: Jz = Jx diag(x) = dH/dz (the
 * chain rule of the diag(e^{-z}) rescale), Jz delta = -rhs, dx = x (.) delta.  This is
 * the same solution; it keeps the row-relative singular test (reading R13) independent of the
 * scale of the coordinates, which for polyhedral start points spans many orders of magnitude.
 */
static int solve_point(const orc_sys *s, const double *xp, double t, double *dE, double *dN)
{
    const int n = s->n;
    double H[128], Jx[64 * 64 * 2], Jt[128], B[64 * 2 * 2], X[64 * 2 * 2];
    int st = eval_point(s, xp, t, H, Jx, Jt, 0, 0, 0);
    if (st) return st;
    for (int k = 0; k < n; ++k) {
        for (int j = 0; j < n; ++j) /* Jz[k][j] = Jx[k][j] * x_j */
            store(Jx + 2 * (k * n + j), cmul(load(Jx + 2 * (k * n + j)), load(xp + 2 * j)));
        B[2 * (k * 2 + 0) + 0] = -Jt[2 * k];
        B[2 * (k * 2 + 0) + 1] = -Jt[2 * k + 1];
        B[2 * (k * 2 + 1) + 0] = -H[2 * k];
        B[2 * (k * 2 + 1) + 1] = -H[2 * k + 1];
    }
    st = orc_lu_solve(n, 2, Jx, B, X);
    if (st) return st;
    for (int k = 0; k < n; ++k) {
        const cplx xk = load(xp + 2 * k);
        if (dE) store(dE + 2 * k, cmul(xk, load(X + 2 * (k * 2))));
        if (dN) store(dN + 2 * k, cmul(xk, load(X + 2 * (k * 2 + 1))));
    }
    for (int k = 0; k < 2 * n; ++k)
        if ((dE && !isfinite(dE[k])) || (dN && !isfinite(dN[k]))) return ORC_PT_NONFINITE;
    return 0;
}

int orc_euler_newton(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                     int64_t p, const double *x, const double *t, double *dE, double *dN,
                     uint8_t *status)
{
    if (n < 1 || n > 64) return -1;
    orc_sys s = {n, off, a, c, w, n};
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < p; ++q)
        status[q] = (uint8_t)solve_point(&s, x + 2 * n * q, t[q], dE + 2 * n * q, dN + 2 * n * q);
    return 0;
}

static double vnorm(int n, const double *v)
{
    double s = 0.0;
    for (int i = 0; i < 2 * n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/*
 * The paper's simplified Euler-Newton step, in tau (t = e^tau, Eq. (2)):
 *   (dE,_) = solve(x, tau);   x~ = x + h * t * dE;  tau~ = tau + h      (Euler, dx/dtau = t dx/dt)
 *   repeat K times: (_,dN) = solve(x~, tau~);  x~ = x~ + dN              (Newton)
 * x, tau updated in place; dn_norm[q] = ||dN|| of the last Newton iteration.
 */
int orc_pc_step(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                int64_t p, double *x, double *tau, const double *dtau, int K, uint8_t *status,
                double *dn_norm)
{
    if (n < 1 || n > 64) return -1;
    orc_sys s = {n, off, a, c, w, n};
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < p; ++q) {
        double *xq = x + 2 * n * q, dE[128] = {0}, dN[128] = {0}, xt[128];
        double h = dtau[q];
        int st = solve_point(&s, xq, exp(tau[q]), dE, 0);
        double t = exp(tau[q]);
        for (int i = 0; i < 2 * n; ++i) xt[i] = xq[i] + h * t * dE[i];
        double tt = tau[q] + h;
        double nrm = 0.0;
        for (int it = 0; it < K; ++it) {
            st |= solve_point(&s, xt, exp(tt), 0, dN);
            for (int i = 0; i < 2 * n; ++i) xt[i] += dN[i];
            nrm = vnorm(n, dN);
        }
        memcpy(xq, xt, sizeof(double) * 2 * n);
        tau[q] = tt;
        status[q] = (uint8_t)st;
        if (dn_norm) dn_norm[q] = nrm;
    }
    return 0;
}

/* max_j |d_j| / |x_j|: componentwise relative size of a correction (reading R14). */
static double relmax(int n, const double *d, const double *x)
{
    double r = 0.0;
    for (int j = 0; j < n; ++j) {
        double ax = hypot(x[2 * j], x[2 * j + 1]);
        double ad = hypot(d[2 * j], d[2 * j + 1]);
        double q = ad / ax;
        if (!(q <= r)) r = q; /* NaN propagates */
    }
    return r;
}

/*
 * Adaptive tracking tau0 -> 0 (step control = DESIGN.md reading R14: the
 * corrector converges when max_j |dN_j|/|x_j| <= newton_tol, a scale-invariant test because
 * polyhedral start points span many orders of magnitude).
 * opt[] = {dtau_init, dtau_min, dtau_max, newton_tol, shrink, grow, final_tol, inf_norm, pred_tol}
 * iopt[] = {K (max corrector iters), grow_after, max_steps, final_iters, pred_log, reuse_tangent}
 * pred_log: the Euler predictor in the log chart, x exp(h dz/dtau), instead of x + h dx/dtau.
 * reuse_tangent: the last corrector solve's Euler direction (relative, dz/dtau at that iterate)
 * predicts the next step (P:659-667 consolidation), one solve fewer per accepted step.
 * stats[q] = {accepted steps, rejected steps, evaluations (solves), final Newton iters}.
 */
int orc_track(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
              int64_t p, double *x, double *tau, const double *opt, const int32_t *iopt,
              uint8_t *status, int64_t *stats)
{
    if (n < 1 || n > 64) return -1;
    orc_sys s = {n, off, a, c, w, n};
    const double dtau_init = opt[0], dtau_min = opt[1], dtau_max = opt[2], newton_tol = opt[3];
    const double shrink = opt[4], grow = opt[5], final_tol = opt[6], inf_norm = opt[7];
    const double pred_tol = opt[8]; /* step control (reading R14), <= 0: grow_after rule */
    const int K = iopt[0], grow_after = iopt[1], max_steps = iopt[2], final_iters = iopt[3];
    if (final_iters < 1) return -1; /* as pht_track: at least one refinement iteration */
    const int pred_log = iopt[4], reuse = iopt[5];
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < p; ++q) {
        double *xq = x + 2 * n * q, dE[128], dN[128], xt[128], dEn[128], rel[128];
        double tq = tau[q], dt = dtau_init;
        int64_t steps = 0, rejects = 0, evals = 0, fin = 0;
        int succ = 0, st = 0;
        double nd1 = -1.0; /* first corrector update of the current step */
        if (!isfinite(tq)) {
            status[q] = ORC_PT_NONFINITE;
            for (int u = 0; u < 4; ++u) stats[4 * q + u] = 0;
            continue;
        }
        int tok = 0; /* dE holds the Euler direction of the current accepted point */
        while (tq < 0.0) {
            if (steps == max_steps) { st = ORC_PT_MAX_STEPS; break; }
            double h = fmin(dt, -tq);
            /* after a rejection the predictor restarts from the same point: its Euler direction is
             * the one already computed (the same evaluation; not repeated) */
            int s1 = 0;
            if (!tok) {
                s1 = solve_point(&s, xq, exp(tq), dE, 0);
                ++evals;
                tok = !s1;
            }
            int ok = 0;
            double tt = tq + h;
            if (!s1) {
                double t = exp(tq), prev = INFINITY;
                nd1 = -1.0;
                if (pred_log) { /* Euler in the log chart: x exp(h dz/dtau), dz/dtau = t dE / x */
                    for (int j = 0; j < n; ++j) {
                        cplx xv = load(xq + 2 * j);
                        cplx dz = cdiv(cmul(mk(t, 0.0), load(dE + 2 * j)), xv);
                        store(xt + 2 * j, cmul(xv, cexp(h * dz)));
                    }
                } else {
                    for (int i = 0; i < 2 * n; ++i) xt[i] = xq[i] + h * t * dE[i];
                }
                for (int it = 1; it <= K; ++it) {
                    s1 = solve_point(&s, xt, exp(tt), reuse ? dEn : 0, dN);
                    ++evals;
                    if (s1) break;
                    if (reuse) /* dz/dtau / t at this iterate (relative direction) */
                        for (int j = 0; j < n; ++j) store(rel + 2 * j, cdiv(load(dEn + 2 * j), load(xt + 2 * j)));
                    double nd = relmax(n, dN, xt);
                    for (int i = 0; i < 2 * n; ++i) xt[i] += dN[i];
                    if (it == 1) nd1 = nd;
                    /* converged: the update, or the update times the observed contraction
                     * (quadratic-convergence estimate of the remaining error) <= newton_tol */
                    if (nd <= newton_tol || (it >= 2 && nd * (nd / prev) <= newton_tol)) { ok = 1; break; }
                    if (it >= 2 && nd > 0.5 * prev) break;
                    prev = nd;
                }
            }
            if (ok) {
                memcpy(xq, xt, sizeof(double) * 2 * n);
                tok = 0;
                if (reuse && tt < 0.0) { /* the iterate's relative direction, at the accepted point */
                    for (int j = 0; j < n; ++j) store(dE + 2 * j, cmul(load(rel + 2 * j), load(xq + 2 * j)));
                    tok = 1;
                }
                tq = tt;
                ++steps;
                if (pred_tol > 0.0) { /* next step from the Euler predictor's error e1 = O(dt^2) */
                    const double f = nd1 > 0.0 ? fmin(fmax(sqrt(pred_tol / nd1), shrink), grow) : grow;
                    dt = fmin(f * dt, dtau_max);
                } else if (++succ == grow_after) {
                    dt = fmin(grow * dt, dtau_max);
                    succ = 0;
                }
            } else {
                ++rejects;
                dt *= shrink;
                succ = 0;
                if (dt < dtau_min) { st = (s1 & ORC_PT_SINGULAR) ? ORC_PT_SINGULAR : ORC_PT_STEP_UNDERFLOW; break; }
            }
        }
        if (st == 0) {
            /* refine at t = 1: up to final_iters Newton iterations until ||dN|| <= final_tol
             * (SURVEY §8(c) O4 / ledger A24; componentwise relative norm, reading R14) */
            int conv = 0;
            for (int it = 1; it <= final_iters; ++it) {
                int s1 = solve_point(&s, xq, 1.0, 0, dN);
                ++evals; ++fin;
                if (s1) break;
                const double nd = relmax(n, dN, xq);
                for (int i = 0; i < 2 * n; ++i) xq[i] += dN[i];
                if (nd <= final_tol) { conv = 1; break; }
            }
            double xinf = 0.0;
            for (int j = 0; j < n; ++j) xinf = fmax(xinf, cabs(load(xq + 2 * j)));
            st = (conv && xinf <= inf_norm) ? ORC_PT_OK : ORC_PT_DIVERGED;
        }
        tau[q] = tq;
        status[q] = (uint8_t)st;
        stats[4 * q + 0] = steps;
        stats[4 * q + 1] = rejects;
        stats[4 * q + 2] = evals;
        stats[4 * q + 3] = fin;
    }
    return 0;
}


/* t = e^tau as an extended-range value (Eq. (2)): t = 2^e * exp(tau - e ln 2). */
static xc xexp_real(double tau)
{
    const double L2 = 0.69314718055994530942;
    double e = floor(tau / L2);
    return xnorm(mk(exp(tau - e * L2), 0.0), (int64_t)e);
}

/* Extended-range direction solve at (x, tau): rows [D_z h_k | t dh_k/dt | h_k] with
 * D_z h = Jx diag(x), each row divided by its largest binary exponent (row
 * scaling leaves the solution unchanged), then LU in double:
 * D_z H delta_E = -dH/dtau, D_z H delta_N = -H (dx = x (.) delta). */
static int solve_point_x(const orc_sys *s, const xc *x, double tau, const double *wr, double *dEr, double *dNr)
{
    const int n = s->n;
    xc H[64], Jx[64 * 64], Jt[64];
    xc t = xexp_real(tau);
    for (int j = 0; j < n; ++j)
        if (creal(x[j].m) == 0.0 && cimag(x[j].m) == 0.0) return ORC_PT_ZERO_COORD;
    eval_point_x_w(s, x, t, tau, wr, H, Jx, Jt, 0, 0, 0);
    double A[64 * 64 * 2], B[64 * 2 * 2], X[64 * 2 * 2];
    for (int k = 0; k < n; ++k) {
        xc row[66];
        for (int j = 0; j < n; ++j) row[j] = xmul(Jx[k * n + j], x[j]);
        row[n] = wr ? Jt[k] : xmul(Jt[k], t); /* dh/dtau */
        row[n + 1] = H[k];
        int64_t emax = INT64_MIN;
        for (int j = 0; j < n + 2; ++j)
            if ((creal(row[j].m) != 0.0 || cimag(row[j].m) != 0.0) && row[j].e > emax) emax = row[j].e;
        if (emax == INT64_MIN) emax = 0;
        for (int j = 0; j < n + 2; ++j) {
            int64_t d = row[j].e - emax;
            cplx v = d < -1100 ? mk(0.0, 0.0) : mk(ldexp(creal(row[j].m), (int)d), ldexp(cimag(row[j].m), (int)d));
            if (!isfinite(creal(v)) || !isfinite(cimag(v))) return ORC_PT_NONFINITE;
            if (j < n) store(A + 2 * (k * n + j), v);
            else if (j == n) store(B + 2 * (k * 2 + 0), -v);
            else store(B + 2 * (k * 2 + 1), -v);
        }
    }
    int st = orc_lu_solve(n, 2, A, B, X);
    if (st) return st;
    for (int k = 0; k < n; ++k) {
        if (dEr) { dEr[2 * k] = X[2 * (k * 2)]; dEr[2 * k + 1] = X[2 * (k * 2) + 1]; }
        if (dNr) { dNr[2 * k] = X[2 * (k * 2 + 1)]; dNr[2 * k + 1] = X[2 * (k * 2 + 1) + 1]; }
    }
    for (int k = 0; k < 2 * n; ++k)
        if ((dEr && !isfinite(dEr[k])) || (dNr && !isfinite(dNr[k]))) return ORC_PT_NONFINITE;
    return 0;
}

static double relmax_d(int n, const double *d)
{
    double r = 0.0;
    for (int j = 0; j < n; ++j) {
        double q = hypot(d[2 * j], d[2 * j + 1]);
        if (!(q <= r)) r = q;
    }
    return r;
}

/* x (.) (1 + h delta) in extended range */
static void xupdate(int n, xc *x, const double *delta, double h)
{
    for (int j = 0; j < n; ++j)
        x[j] = xmul(x[j], xnorm(mk(1.0 + h * delta[2 * j], h * delta[2 * j + 1]), 0));
}

/*
 * orc_track with extended-range state (SURVEY O2/O4 for the large-lifting start points): the
 * same control flow, step control and statuses as orc_track; x = xm 2^xe in/out.
 * cellw/path_cell (optional): track in cell coordinates with the cell-shifted liftings
 * omega' = cellw[path_cell[q]][i] (include/pht.h pht_track_cells); t^omega' = e^{tau omega'}.
 */
int orc_track_x(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                int64_t p, double *xm, int64_t *xe, double *tau, const double *opt, const int32_t *iopt,
                uint8_t *status, int64_t *stats, const double *cellw, const int32_t *path_cell)
{
    if (n < 1 || n > 64) return -1;
    orc_sys s = {n, off, a, c, w, n};
    const double dtau_init = opt[0], dtau_min = opt[1], dtau_max = opt[2], newton_tol = opt[3];
    const double shrink = opt[4], grow = opt[5], final_tol = opt[6], inf_norm = opt[7];
    const double pred_tol = opt[8]; /* step control (reading R14), <= 0: grow_after rule */
    const int K = iopt[0], grow_after = iopt[1], max_steps = iopt[2], final_iters = iopt[3];
    if (final_iters < 1) return -1; /* as pht_track: at least one refinement iteration */
    const int pred_log = iopt[4];
    /* predictor 1: cubic Hermite extrapolation in the log chart through the previous and the
     * current accepted point and their Euler directions, log chart only */
    const int hermite = pred_log && iopt[5] == 1;
    const int reuse = iopt[6] && !hermite; /* reuse_tangent (see orc_track) */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < p; ++q) {
        xc xq[64], xt[64];
        double dE[128], dN[128], dEn[128];
        /* continuous log coordinates of the current, trial and previous accepted points (the
         * Hermite predictor needs differences of z without branch jumps) */
        cplx zq[64], zt[64], zp[64], ep[64];
        int has_prev = 0;
        double tp = 0.0;
        const double *wr = cellw ? cellw + (size_t)path_cell[q] * off[n] : 0;
        for (int j = 0; j < n; ++j) {
            xq[j] = xnorm(load(xm + 2 * (q * n + j)), xe[q * n + j]);
            zq[j] = clog(xq[j].m) + (double)xq[j].e * 0.69314718055994530942;
        }
        double tq = tau[q], dt = dtau_init;
        int64_t steps = 0, rejects = 0, evals = 0, fin = 0;
        int succ = 0, st = 0;
        double nd1 = -1.0; /* first corrector update of the current step */
        if (!isfinite(tq)) {
            status[q] = ORC_PT_NONFINITE;
            for (int u = 0; u < 4; ++u) stats[4 * q + u] = 0;
            continue;
        }
        int tok = 0; /* dE holds the Euler direction of the current accepted point (as orc_track) */
        while (tq < 0.0) {
            if (steps == max_steps) { st = ORC_PT_MAX_STEPS; break; }
            double h = fmin(dt, -tq);
            int s1 = 0;
            if (!tok || hermite) { /* (the Hermite predictor keeps the round-1 evaluation count) */
                s1 = solve_point_x(&s, xq, tq, wr, dE, 0);
                ++evals;
                tok = !s1;
            }
            int ok = 0;
            double tt = tq + h;
            if (!s1) {
                double prev = INFINITY;
                nd1 = -1.0;
                for (int j = 0; j < n; ++j) xt[j] = xq[j];
                if (hermite && has_prev) {
                    /* p(s) on [tp, tq], s = (tau - tp) / D, evaluated at s = 1 + h / D:
                     * z~ = h00 z_p + h10 D e_p + h01 z_q + h11 D e_q */
                    const double D = tq - tp, sv = 1.0 + h / D, s2 = sv * sv, s3 = s2 * sv;
                    const double h00 = 2 * s3 - 3 * s2 + 1, h10 = s3 - 2 * s2 + sv, h01 = -2 * s3 + 3 * s2,
                                 h11 = s3 - s2;
                    for (int j = 0; j < n; ++j) {
                        const cplx eq = load(dE + 2 * j);
                        zt[j] = h00 * zp[j] + h10 * D * ep[j] + h01 * zq[j] + h11 * D * eq;
                        xt[j] = xmul(xt[j], xnorm(cexp(zt[j] - zq[j]), 0));
                    }
                } else if (pred_log) { /* Euler in the log chart: x exp(h delta_E) */
                    for (int j = 0; j < n; ++j) {
                        xt[j] = xmul(xt[j], xnorm(cexp(h * load(dE + 2 * j)), 0));
                        zt[j] = zq[j] + h * load(dE + 2 * j);
                    }
                } else {
                    xupdate(n, xt, dE, h);
                }
                for (int it = 1; it <= K; ++it) {
                    s1 = solve_point_x(&s, xt, tt, wr, reuse ? dEn : 0, dN);
                    ++evals;
                    if (s1) break;
                    double nd = relmax_d(n, dN);
                    xupdate(n, xt, dN, 1.0);
                    if (pred_log)
                        for (int j = 0; j < n; ++j) zt[j] += clog(1.0 + load(dN + 2 * j));
                    if (it == 1) nd1 = nd;
                    /* converged: the update, or the update times the observed contraction
                     * (quadratic-convergence estimate of the remaining error) <= newton_tol */
                    if (nd <= newton_tol || (it >= 2 && nd * (nd / prev) <= newton_tol)) { ok = 1; break; }
                    if (it >= 2 && nd > 0.5 * prev) break;
                    prev = nd;
                }
            }
            if (ok) {
                if (hermite)
                    for (int j = 0; j < n; ++j) { zp[j] = zq[j]; ep[j] = load(dE + 2 * j); }
                has_prev = 1;
                tp = tq;
                tok = 0;
                if (reuse && tt < 0.0) { /* delta_E of the last corrector iterate (relative) */
                    memcpy(dE, dEn, sizeof(double) * 2 * n);
                    tok = 1;
                }
                for (int j = 0; j < n; ++j) { xq[j] = xt[j]; zq[j] = zt[j]; }
                tq = tt;
                ++steps;
                if (pred_tol > 0.0) { /* next step from the Euler predictor's error e1 = O(dt^2) */
                    const double f = nd1 > 0.0 ? fmin(fmax(sqrt(pred_tol / nd1), shrink), grow) : grow;
                    dt = fmin(f * dt, dtau_max);
                } else if (++succ == grow_after) {
                    dt = fmin(grow * dt, dtau_max);
                    succ = 0;
                }
            } else {
                ++rejects;
                dt *= shrink;
                succ = 0;
                if (dt < dtau_min) { st = (s1 & ORC_PT_SINGULAR) ? ORC_PT_SINGULAR : ORC_PT_STEP_UNDERFLOW; break; }
            }
        }
        if (st == 0) {
            int conv = 0; /* final refinement to final_tol: as orc_track (ledger A24) */
            for (int it = 1; it <= final_iters; ++it) {
                int s1 = solve_point_x(&s, xq, 0.0, wr, 0, dN);
                ++evals; ++fin;
                if (s1) break;
                const double nd = relmax_d(n, dN);
                xupdate(n, xq, dN, 1.0);
                if (nd <= final_tol) { conv = 1; break; }
            }
            double lmax = -INFINITY;
            for (int j = 0; j < n; ++j) lmax = fmax(lmax, xabs_log2(xq[j]));
            st = (conv && lmax <= log2(inf_norm)) ? ORC_PT_OK : ORC_PT_DIVERGED;
        }
        for (int j = 0; j < n; ++j) { store(xm + 2 * (q * n + j), xq[j].m); xe[q * n + j] = xq[j].e; }
        tau[q] = tq;
        status[q] = (uint8_t)st;
        stats[4 * q + 0] = steps;
        stats[4 * q + 1] = rejects;
        stats[4 * q + 2] = evals;
        stats[4 * q + 3] = fin;
    }
    return 0;
}

#ifdef _OPENMP
#include <omp.h>
#endif
/* Thread count used by the parallel-for loops (timing only; results do not depend on it). */
/* ------------------------------------------------------------------ */
/* projective formulation (Eq. (3)) and its directions      */
/* (P:237-252): y in C^{n+1}, homogenising coordinate LAST  */
/* (SURVEY A8), a^ = (a, deg(f_k) - 1^T a) with deg(f_k) = max 1^T a.   */
/* ------------------------------------------------------------------ */

/* a^ for every term: int32 [M][n+1] (caller frees). */
static int32_t *homogenize(int n, const int64_t *off, const int32_t *a)
{
    const int64_t M = off[n];
    int32_t *ah = (int32_t *)malloc(sizeof(int32_t) * (size_t)(M > 0 ? M : 1) * (n + 1));
    if (!ah) return 0;
    for (int k = 0; k < n; ++k) {
        int64_t deg = INT64_MIN;
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            int64_t d = 0;
            for (int j = 0; j < n; ++j) d += a[i * n + j];
            if (d > deg) deg = d;
        }
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            int64_t d = 0;
            for (int j = 0; j < n; ++j) {
                ah[i * (n + 1) + j] = a[i * n + j];
                d += a[i * n + j];
            }
            ah[i * (n + 1) + n] = (int32_t)(deg - d);
        }
    }
    return ah;
}

/* H^, dH^/dy (n x (n+1)), dH^/dt at homogeneous points y (Eq. (3)). */
int orc_proj_evaluate(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                      int64_t p, const double *y, const double *t, double *H, double *Jy, double *Jt,
                      double *SH, double *SJy, double *SJt, uint8_t *status)
{
    if (n < 1 || n > 63) return -1;
    int32_t *ah = homogenize(n, off, a);
    if (!ah) return -2;
    orc_sys s = {n, off, ah, c, w, n + 1};
    const int m = n + 1;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < p; ++q) {
        int st = eval_point(&s, y + 2 * m * q, t[q], H ? H + 2 * n * q : 0, Jy ? Jy + 2 * n * m * q : 0,
                            Jt ? Jt + 2 * n * q : 0, SH ? SH + n * q : 0, SJy ? SJy + n * m * q : 0,
                            SJt ? SJt + n * q : 0);
        if (status) status[q] = (uint8_t)st;
    }
    free(ah);
    return 0;
}

/*
 * Projective Euler and Newton directions: one LU solve with two
 * right-hand sides of the bordered (n+1) x (n+1) system
 *     [ dH^/dy ] [E N] = - [ dH^/dtau  H^ ]        dH^/dtau = t dH^/dt  (tau = log t)
 *     [  y^*   ]           [    0       0 ]
 * y^* = row of conjugated coordinates.  E = dy/dtau, N = the projective Newton direction.
 */
static int proj_solve_point(const orc_sys *s, const double *yp, double t, double *E, double *N)
{
    const int n = s->n, m = n + 1;
    double H[128], Jy[64 * 65 * 2], Jt[128], A[65 * 65 * 2], B[65 * 2 * 2], X[65 * 2 * 2];
    int st = eval_point(s, yp, t, H, Jy, Jt, 0, 0, 0);
    if (st) return st;
    for (int k = 0; k < n; ++k) {
        for (int j = 0; j < m; ++j) store(A + 2 * (k * m + j), load(Jy + 2 * (k * m + j)));
        store(B + 2 * (k * 2 + 0), mk(-t * Jt[2 * k], -t * Jt[2 * k + 1]));
        store(B + 2 * (k * 2 + 1), mk(-H[2 * k], -H[2 * k + 1]));
    }
    for (int j = 0; j < m; ++j) store(A + 2 * (n * m + j), conj(load(yp + 2 * j)));
    store(B + 2 * (n * 2 + 0), mk(0.0, 0.0));
    store(B + 2 * (n * 2 + 1), mk(0.0, 0.0));
    st = orc_lu_solve(m, 2, A, B, X);
    if (st) return st;
    for (int j = 0; j < m; ++j) {
        if (E) store(E + 2 * j, load(X + 2 * (j * 2)));
        if (N) store(N + 2 * j, load(X + 2 * (j * 2 + 1)));
    }
    for (int k = 0; k < 2 * m; ++k)
        if ((E && !isfinite(E[k])) || (N && !isfinite(N[k]))) return ORC_PT_NONFINITE;
    return 0;
}

int orc_proj_euler_newton(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                          int64_t p, const double *y, const double *t, double *E, double *N, uint8_t *status)
{
    if (n < 1 || n > 63) return -1;
    int32_t *ah = homogenize(n, off, a);
    if (!ah) return -2;
    orc_sys s = {n, off, ah, c, w, n + 1};
    const int m = n + 1;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < p; ++q)
        status[q] = (uint8_t)proj_solve_point(&s, y + 2 * m * q, t[q], E + 2 * m * q, N + 2 * m * q);
    free(ah);
    return 0;
}

/* y <- y / ||y|| (points of P^n are kept on the unit sphere, reading R29) */
static void proj_normalize(int m, double *y)
{
    double s2 = 0.0;
    for (int i = 0; i < 2 * m; ++i) s2 += y[i] * y[i];
    const double f = 1.0 / sqrt(s2);
    for (int i = 0; i < 2 * m; ++i) y[i] *= f;
}

/*
 * The Euler-Newton step in homogeneous coordinates: y~ = y + h E; tau~ = tau + h;
 * K times y~ += N(y~, tau~); y is renormalised to ||y|| = 1 after every update (reading R29).
 * dn_norm = ||N|| of the last Newton iteration (relative to ||y|| = 1).
 */
int orc_proj_pc_step(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                     int64_t p, double *y, double *tau, const double *dtau, int K, uint8_t *status,
                     double *dn_norm)
{
    if (n < 1 || n > 63) return -1;
    int32_t *ah = homogenize(n, off, a);
    if (!ah) return -2;
    orc_sys s = {n, off, ah, c, w, n + 1};
    const int m = n + 1;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < p; ++q) {
        double *yq = y + 2 * m * q, E[130] = {0}, N[130] = {0}, yt[130];
        const double h = dtau[q];
        int st = proj_solve_point(&s, yq, exp(tau[q]), E, 0);
        for (int i = 0; i < 2 * m; ++i) yt[i] = yq[i] + h * E[i];
        proj_normalize(m, yt);
        const double tt = tau[q] + h;
        double nrm = 0.0;
        for (int it = 0; it < K; ++it) {
            st |= proj_solve_point(&s, yt, exp(tt), 0, N);
            for (int i = 0; i < 2 * m; ++i) yt[i] += N[i];
            nrm = vnorm(m, N);
            proj_normalize(m, yt);
        }
        memcpy(yq, yt, sizeof(double) * 2 * m);
        tau[q] = tt;
        status[q] = (uint8_t)st;
        if (dn_norm) dn_norm[q] = nrm;
    }
    free(ah);
    return 0;
}

/*
 * Adaptive tracking in homogeneous coordinates: orc_track's control flow (reading R14) with
 * the projective directions, y renormalised after every update, norm-relative corrector tests
 * (||dy|| / ||y|| <= newton_tol; componentwise tests are meaningless for coordinates going to
 * 0 at infinity), and the endpoint classified finite iff |y_n| >= ||y|| / inf_norm (the affine
 * point y_{0..n-1} / y_n has norm <= inf_norm), else DIVERGED: a solution at infinity.
 * Affine Euler predictor only (pred_log is ignored).
 */
int orc_proj_track(int n, const int64_t *off, const int32_t *a, const double *c, const int64_t *w,
                   int64_t p, double *y, double *tau, const double *opt, const int32_t *iopt,
                   uint8_t *status, int64_t *stats)
{
    if (n < 1 || n > 63) return -1;
    int32_t *ah = homogenize(n, off, a);
    if (!ah) return -2;
    orc_sys s = {n, off, ah, c, w, n + 1};
    const int m = n + 1;
    const double dtau_init = opt[0], dtau_min = opt[1], dtau_max = opt[2], newton_tol = opt[3];
    const double shrink = opt[4], grow = opt[5], final_tol = opt[6], inf_norm = opt[7];
    const double pred_tol = opt[8]; /* step control (reading R14), <= 0: grow_after rule */
    const int K = iopt[0], grow_after = iopt[1], max_steps = iopt[2], final_iters = iopt[3];
    if (final_iters < 1) return -1; /* as pht_track: at least one refinement iteration */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < p; ++q) {
        double *yq = y + 2 * m * q, E[130], N[130], yt[130];
        double tq = tau[q], dt = dtau_init;
        int64_t steps = 0, rejects = 0, evals = 0, fin = 0;
        int succ = 0, st = 0;
        double nd1 = -1.0; /* first corrector update of the current step */
        if (!isfinite(tq)) {
            status[q] = ORC_PT_NONFINITE;
            for (int u = 0; u < 4; ++u) stats[4 * q + u] = 0;
            continue;
        }
        proj_normalize(m, yq);
        while (tq < 0.0) {
            if (steps == max_steps) { st = ORC_PT_MAX_STEPS; break; }
            double h = fmin(dt, -tq);
            int s1 = proj_solve_point(&s, yq, exp(tq), E, 0);
            ++evals;
            int ok = 0;
            double tt = tq + h;
            if (!s1) {
                double prev = INFINITY;
                nd1 = -1.0;
                for (int i = 0; i < 2 * m; ++i) yt[i] = yq[i] + h * E[i];
                proj_normalize(m, yt);
                for (int it = 1; it <= K; ++it) {
                    s1 = proj_solve_point(&s, yt, exp(tt), 0, N);
                    ++evals;
                    if (s1) break;
                    double nd = vnorm(m, N); /* ||y~|| = 1 */
                    for (int i = 0; i < 2 * m; ++i) yt[i] += N[i];
                    proj_normalize(m, yt);
                    if (it == 1) nd1 = nd;
                    /* converged: the update, or the update times the observed contraction
                     * (quadratic-convergence estimate of the remaining error) <= newton_tol */
                    if (nd <= newton_tol || (it >= 2 && nd * (nd / prev) <= newton_tol)) { ok = 1; break; }
                    if (it >= 2 && nd > 0.5 * prev) break;
                    prev = nd;
                }
            }
            if (ok) {
                memcpy(yq, yt, sizeof(double) * 2 * m);
                tq = tt;
                ++steps;
                if (pred_tol > 0.0) { /* next step from the Euler predictor's error e1 = O(dt^2) */
                    const double f = nd1 > 0.0 ? fmin(fmax(sqrt(pred_tol / nd1), shrink), grow) : grow;
                    dt = fmin(f * dt, dtau_max);
                } else if (++succ == grow_after) {
                    dt = fmin(grow * dt, dtau_max);
                    succ = 0;
                }
            } else {
                ++rejects;
                dt *= shrink;
                succ = 0;
                if (dt < dtau_min) { st = (s1 & ORC_PT_SINGULAR) ? ORC_PT_SINGULAR : ORC_PT_STEP_UNDERFLOW; break; }
            }
        }
        if (st == 0) {
            int conv = 0, solved = 1;
            double nd = INFINITY;
            for (int it = 1; it <= final_iters; ++it) {
                int s1 = proj_solve_point(&s, yq, 1.0, 0, N);
                ++evals; ++fin;
                if (s1) { solved = 0; break; }
                nd = vnorm(m, N);
                for (int i = 0; i < 2 * m; ++i) yq[i] += N[i];
                proj_normalize(m, yq);
                if (nd <= final_tol) { conv = 1; break; }
            }
            if (!conv && solved && nd <= newton_tol) conv = 1;
            const double yn = hypot(yq[2 * n], yq[2 * n + 1]);
            st = (conv && yn * inf_norm >= 1.0) ? ORC_PT_OK : ORC_PT_DIVERGED;
        }
        tau[q] = tq;
        status[q] = (uint8_t)st;
        stats[4 * q + 0] = steps;
        stats[4 * q + 1] = rejects;
        stats[4 * q + 2] = evals;
        stats[4 * q + 3] = fin;
    }
    free(ah);
    return 0;
}

int orc_set_threads(int nt)
{
#ifdef _OPENMP
    if (nt > 0) omp_set_num_threads(nt);
    return omp_get_max_threads();
#else
    (void)nt;
    return 1;
#endif
}

int orc_version(void) { return 1; }
