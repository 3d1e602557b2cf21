// pht_kernels.cuh — sm_100a kernels for the polyhedral-homotopy hot path (arXiv 2111.14317).
//
// Two templated kernels cover the entry points of include/pht.h: k_phte<N, MODE> (evaluation,
// persistent) and k_pht<N, MODE> (directions / Euler-Newton step, evaluation + solve).
// Mapping: a CTA owns a tile of Geo<N>::PTS points and runs two layouts.
//  * "W" (evaluation): thread (k, q) = (equation k, point q) computes ROW k of the extended
//    Jacobian of point q, [ dh_k/dz_1 .. dh_k/dz_N | dh_k/dtau | h_k ] (P:525-542,
//    "e^{z A} B_k^T"), in registers.  A warp holds one equation for 32 points, so every read of
//    the term table is a warp-uniform broadcast.
//  * "L" (direction solve): rows go through shared memory so that each warp owns whole points
//    (lane = (point, row)); Gauss-Jordan with partial pivoting on [G | G_tau | h] for both
//    right-hand sides (§6 P:656-731 consolidated as in BASELINE.json north_star) then needs
//    only warp-level synchronisation (redux.sync argmax, __syncwarp pivot-row broadcast).
//
// Stages:
//   a1  log split   rho = log|x_j|, vartheta = arg x_j, tau = log t
//   a2  exponents   phi = sum_j a_j rho_j + omega tau + log|c|,
//                   theta = sum_j a_j vartheta_j + arg c
//   a3  exp*cis     w = exp(phi - e ln2) (cos theta + i sin theta), e = row exponent
//                   (range handling for large liftings, ledger R7)
//   a4  contraction h += w, dh/dz_j += a_j w, dh/dtau += omega w
//       epilogue    dh/dx_j = dh/dz_j / x_j (diag(e^{-z}) P:554-555), dh/dt = dh/dtau / t
//   a5  solve       G delta = -[dh/dtau | h],  dx = x (.) delta
//   a6  step        Euler prediction + K Newton iterations
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstddef>
#else
// run-time compilation (pht_jit.cu, NVRTC): no host headers
typedef unsigned char uint8_t;
typedef long long int64_t;
#ifndef INFINITY
#define INFINITY __longlong_as_double(0x7ff0000000000000ll)
#endif
#endif

namespace pht {

enum Mode : int { MODE_EVAL_X = 0, MODE_EVAL_Z = 1, MODE_DIRS = 2, MODE_STEP = 3 };

enum : int { PT_ZERO_COORD = 1, PT_NONFINITE = 2, PT_SINGULAR = 4, PT_FLOOR = 64 };

// Kernel families (include/pht.h pht_system_set_kernels): AUTO = the measured-best family per
// entry point; the others force one family wherever it implements the entry point.
enum : int { FAM_AUTO = 0, FAM_TILE = 1, FAM_WARP = 2, FAM_DENSE = 3, FAM_SPECIALIZED = 4 };

enum : int { SOLVER_LU = 0, SOLVER_QR = 1 };

// Term record stride in doubles: a_0..a_{n-1}, omega, log|c|, arg c, padded to even.
__host__ __device__ constexpr int rec_stride(int n) { return (n + 3 + 1) & ~1; }

struct DevSys {
    const double2 *rec;    // [M][rec_stride(n)/2] term records (a0 packer, pht_capi.cu)
    const int *off;        // [n+1] equation segments
    const double *exptab;  // [256] 2^(j/256)
    const double2 *cistab; // [256] (cos, sin)(2 pi j / 256)
    int n;
    int proj; // projective system: N = n_eq + 1 homogeneous coordinates, row N-1 = y^*
    int mt;   // most terms of one equation (k_stepw's shared-memory record table)
    const double2 *logtab; // [128] (1/c_j rounded, -log of it), c_j = 1 + (j + 1/2)/128 (log_split_t)
    const double *atantab; // [65] atan(k/64)
};

struct Args {
    int64_t P;
    const double2 *xin;  // x (EVAL_X, DIRS) or z (EVAL_Z)
    const double *tin;   // t (EVAL_X, DIRS) or tau (EVAL_Z)
    double2 *H, *J, *Jt; // evaluate outputs
    int *rexp;           // row_exp2 or nullptr (unscaled)
    uint8_t *status;
    double2 *dE, *dN;    // directions
    double2 *xio;        // STEP: x in/out
    double *tauio;       // STEP: tau in/out
    const double *dtau;  // STEP
    double *dnnorm;      // STEP
    int K;               // STEP: Newton iterations
    int solver;          // DIRS/STEP: SOLVER_LU (Gauss-Jordan, lsolve) or SOLVER_QR (qsolve)
};

// Tracker options (include/pht.h pht_track_opts) and arguments.
struct TrackOpts {
    double dtau_init, dtau_min, dtau_max, newton_tol, shrink, grow, final_tol, inf_norm;
    int K, grow_after, max_steps, final_iters;
    int log_state; // state arrays hold z = log x instead of x
    int pred_log;  // Euler predictor in the log chart: z + h dz/dtau (x exp(h dz/dtau))
    double pred_tol; // step control from the first corrector update (<= 0: grow_after rule)
    int predictor;   // 1: cubic Hermite extrapolation in the log chart (pred_log), else Euler
    int reuse_tangent; // the last corrector iterate's Euler direction predicts the next step
};
struct TrackArgs {
    int64_t P;
    double2 *x;          // [P][N] start points in, endpoints out
    double *tau;         // [P] tau0 in, final tau out
    uint8_t *status;     // [P]
    long long *stats;    // [P][4] accepted steps, rejected steps, evaluations, final iterations
    unsigned long long *queue; // path counter (zeroed by the host)
    const double *cellw;       // optional [ncells][M] cell-shifted liftings (pht_track_cells)
    const int *path_cell;      // [P] cell of each path
    int ncells, M;
    int solver; // SOLVER_LU / SOLVER_QR
    TrackOpts o;
};

// ---- constants (Cody-Waite splits computed with 80-digit arithmetic) ----
__device__ constexpr double SHIFT = 0x1.8p52;               // round-to-integer shifter
__device__ constexpr double INV_LN2 = 0x1.71547652b82fep+0;
__device__ constexpr double LN2_HI = 0x1.62e42fee00000p-1;   // 21 trailing zero bits
__device__ constexpr double LN2_LO = 0x1.a39ef35793c76p-33;
__device__ constexpr double K256_LN2 = 0x1.71547652b82fep+8; // 256 / ln 2
__device__ constexpr double LN2_256_HI = 0x1.62e42fee00000p-9;
__device__ constexpr double LN2_256_LO = 0x1.a39ef35793c76p-41;
__device__ constexpr double K256_2PI = 0x1.45f306dc9c883p+5; // 256 / (2 pi)
__device__ constexpr double C1 = 0x1.921fb54400000p-6;       // 2 pi / 256 in three parts
__device__ constexpr double C2 = 0x1.0b4611a600000p-40;
__device__ constexpr double C3 = 0x1.3198a2e037073p-75;
__device__ constexpr double INV_2PI = 0x1.45f306dc9c883p-3;
__device__ constexpr double TWO_PI_HI = 0x1.921fb54400000p+2;
__device__ constexpr double TWO_PI_LO = 0x1.0b4611a626331p-32;

// exp / cis tables in shared memory.  Default: 256 entries (2^(j/256), cis(2 pi j/256)), one copy;
// the data-dependent lookups of a warp cause bank conflicts (ncu: ~60% excess wavefronts on these
// two loads).  PHT_TAB64=1: 64 entries replicated per bank (16 copies of 2^(j/64), 8 copies of
// cis(2 pi j/64), copy = lane mod 16 / mod 8: conflict free) at one more polynomial term per
// function -- measured 3% slower on the step (profiles/r01_tables.txt), so off.
#ifndef PHT_TAB64
#define PHT_TAB64 0
#endif
#if PHT_TAB64
constexpr int TAB_E = 64 * 16, TAB_C = 64 * 8;
#else
constexpr int TAB_E = 256, TAB_C = 256;
#endif

// Polynomial / reduction constants as a __constant__ table: the compiler then feeds them to DFMA
// as constant-bank operands instead of materialising each 64-bit immediate with two UMOVs.
#if PHT_TAB64
__constant__ double KC[20] = {
    0x1.71547652b82fep+6,  // 0 64/ln2
    0x1.62e42fee00000p-7,  // 1 ln2/64 hi
    0x1.a39ef35793c76p-39, // 2 ln2/64 lo
    1.0 / 24.0,            // 3
    1.0 / 6.0,             // 4
    0x1.45f306dc9c883p+3,  // 5 64/(2pi)
    0x1.921fb54400000p-4,  // 6 2pi/64 in three parts
    0x1.0b4611a600000p-38, // 7
    0x1.3198a2e037073p-73, // 8
    1.0 / 120.0,           // 9
    -1.0 / 6.0,            // 10
    -1.0 / 720.0,          // 11
    0x1.62e42fee00000p-1,  // 12 ln2 hi
    0x1.a39ef35793c76p-33, // 13 ln2 lo
    0x1.71547652b82fep+0,  // 14 1/ln2
    0.0,                   // 15
    -1.0 / 5040.0,         // 16
    1.0 / 40320.0,         // 17
    1.0 / 120.0,           // 18
    0.0};
#else
__constant__ double KC[16] = {
    0x1.71547652b82fep+8,  // 0 256/ln2
    0x1.62e42fee00000p-9,  // 1 ln2/256 hi
    0x1.a39ef35793c76p-41, // 2 ln2/256 lo
    1.0 / 24.0,            // 3
    1.0 / 6.0,             // 4
    0x1.45f306dc9c883p+5,  // 5 256/(2pi)
    0x1.921fb54400000p-6,  // 6 C1
    0x1.0b4611a600000p-40, // 7 C2
    0x1.3198a2e037073p-75, // 8 C3
    1.0 / 120.0,           // 9
    -1.0 / 6.0,            // 10
    -1.0 / 720.0,          // 11
    0x1.62e42fee00000p-1,  // 12 ln2 hi
    0x1.a39ef35793c76p-33, // 13 ln2 lo
    0x1.71547652b82fep+0,  // 14 1/ln2
    0.0};
#endif

__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
// Row maxima of non-negative values through their bit patterns: for x >= 0 the IEEE order is the
// unsigned order of the patterns, and every pattern >= DBITS_INF is inf or NaN (of either sign).
// 4 integer instructions per 64-bit max instead of fmax's ~8 (NaN handling).
constexpr unsigned long long DBITS_INF = 0x7ff0000000000000ull;
__device__ __forceinline__ unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }
// 2^e for a normal power of two (-1022 <= e <= 1023) from its exponent bits; 0 outside (callers
// take scalbn there).  Multiplying by it rounds once, like scalbn.
__device__ __forceinline__ double pow2i(int e) { return __hiloint2double((e + 1023) << 20, 0); }
// v * 2^e (the unscaled outputs of a row with binary row exponent e): one DMUL per part
template <int C>
__device__ __forceinline__ void scale_row2(double2 (&row)[C], int e)
{
    if (e == 0) return;
    if (e >= -1022 && e <= 1023) {
        const double f = pow2i(e);
#pragma unroll
        for (int c = 0; c < C; ++c) row[c] = make_double2(row[c].x * f, row[c].y * f);
    } else {
#pragma unroll
        for (int c = 0; c < C; ++c) row[c] = make_double2(scalbn(row[c].x, e), scalbn(row[c].y, e));
    }
}
// 1/d for a normal d: MUFU.RCP64H seed (~20 bits) + two Newton steps (<= 1 ulp, no slow path).
__device__ __forceinline__ double rcp_nr(double d)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a - l * b
__device__ __forceinline__ double2 cfms(double2 a, double2 l, double2 b)
{
    return make_double2(fma(-l.x, b.x, fma(l.y, b.y, a.x)), fma(-l.x, b.y, fma(-l.y, b.x, a.y)));
}
// 1 / b, scaled like Smith's algorithm (no overflow for |b| in range)
__device__ __forceinline__ double2 crecip(double2 b)
{
    if (fabs(b.x) >= fabs(b.y)) {
        double r = b.y / b.x, d = 1.0 / fma(b.y, r, b.x);
        return make_double2(d, -r * d);
    } else {
        double r = b.x / b.y, d = 1.0 / fma(b.x, r, b.y);
        return make_double2(r * d, -d);
    }
}

// exp / cis tables -> shared memory (layout: see PHT_TAB64); S holds the 256-entry tables
__device__ __forceinline__ void load_tables(const DevSys &S, double *et, double2 *ct, int tid, int nt)
{
#if PHT_TAB64
    for (int i = tid; i < TAB_E; i += nt) et[i] = __ldg(S.exptab + ((i >> 4) << 2));
    for (int i = tid; i < TAB_C; i += nt) ct[i] = __ldg(S.cistab + ((i >> 3) << 2));
#else
    for (int i = tid; i < 256; i += nt) {
        et[i] = __ldg(S.exptab + i);
        ct[i] = __ldg(S.cistab + i);
    }
#endif
}

// a1: rho = log|x|, vartheta = arg x (principal branch, ledger R15), 1/x.
__device__ __forceinline__ void log_split(double2 x, double &rho, double &th, double2 &inv, int &st)
{
    const double ax = fabs(x.x), ay = fabs(x.y);
    if (!(isfinite(x.x) && isfinite(x.y))) {
        st |= PT_NONFINITE;
        rho = 0.0; th = 0.0; inv = make_double2(1.0, 0.0);
        return;
    }
    const double m = fmax(ax, ay);
    if (m == 0.0) {
        st |= PT_ZERO_COORD;
        rho = 0.0; th = 0.0; inv = make_double2(1.0, 0.0);
        return;
    }
    if (m > 0x1p-500 && m < 0x1p+500) {
        const double s = fma(x.x, x.x, x.y * x.y);
        rho = 0.5 * log(s);
        const double is = 1.0 / s;
        inv = make_double2(x.x * is, -x.y * is);
    } else {
        const double mn = fmin(ax, ay) / m;
        rho = log(m) + 0.5 * log1p(mn * mn);
        inv = crecip(x);
    }
    th = atan2(x.y, x.x);
}

// a1 with table-driven log and atan2 (about half the FP64 work of libdevice log + atan2; error
// <= ~1 ulp of max(|log|, 1) and ~1.1 ulp of pi): log s = e ln2 + log c_j + log1p(r)
// with s = 2^e m, c_j the midpoint of m's 1/128 interval, r = m / c_j - 1 (|r| <= 2^-8, degree-7
// series); atan(t) for t = min/max in [0, 1] as atan(k/64) + atan((t - t_k) / (1 + t t_k))
// (|u| <= 2^-7, degree-7 series), then the octant.  Extreme magnitudes take log_split.
// log s for a normal s (2^-1022 < s < 2^1024), table-driven (see log_split_t)
__device__ __forceinline__ double log_t(double s, const double2 *logtab)
{
    const long long bits = __double_as_longlong(s);
    const int j = (int)(bits >> 45) & 127;
    const double mm = __longlong_as_double((bits & 0x000fffffffffffffll) | 0x3ff0000000000000ll);
    const double2 tj = __ldg(logtab + j);
    const double r = fma(mm, tj.x, -1.0);
    double q = fma(r, 1.0 / 7.0, -1.0 / 6.0);
    q = fma(q, r, 0.2);
    q = fma(q, r, -0.25);
    q = fma(q, r, 1.0 / 3.0);
    q = fma(q, r, -0.5);
    const double ef = (double)((int)(bits >> 52) - 1023);
    return fma(ef, KC[12], tj.y + fma(ef, KC[13], fma(q * r, r, r)));
}
// atan2(y, x) for finite (x, y) not both 0 with max(|x|, |y|) normal, table-driven (see log_split_t);
// m = max(|x|, |y|)
__device__ __forceinline__ double atan2_t(double y, double x, double m, const double *atantab)
{
    const double ax = fabs(x), ay = fabs(y);
    const bool swap = ay > ax;
    const double t = (swap ? ax : ay) * rcp_nr(m);
    const double kd = rint(t * 64.0);
    const double tk = kd * (1.0 / 64.0);
    const double u = (t - tk) * rcp_nr(fma(t, tk, 1.0));
    const double u2 = u * u;
    double w = fma(u2, -1.0 / 7.0, 0.2);
    w = fma(w, u2, -1.0 / 3.0);
    const double at = __ldg(atantab + (int)kd) + fma(w * u2, u, u);
    double a = swap ? (0x1.921fb54442d18p+0 - at) + 0x1.1a62633145c07p-54 : at; // pi/2 - at
    a = (x < 0.0) ? (0x1.921fb54442d18p+1 - a) + 0x1.1a62633145c07p-53 : a;    // pi - a
    return (y < 0.0) ? -a : a;
}

__device__ __forceinline__ void log_split_t(double2 x, double &rho, double &th, double2 &inv, int &st,
                                            const double2 *logtab, const double *atantab)
{
    const double m = fmax(fabs(x.x), fabs(x.y));
    if (!(m > 0x1p-500 && m < 0x1p+500)) { // zero, non-finite or extreme: the general routine
        log_split(x, rho, th, inv, st);
        return;
    }
    const double s = fma(x.x, x.x, x.y * x.y);
    rho = 0.5 * log_t(s, logtab);
    const double is = rcp_nr(s);
    inv = make_double2(x.x * is, -x.y * is);
    th = atan2_t(x.y, x.x, m, atantab);
}

// a3: w = exp(y) * (cos th + i sin th), y <= ~0.35 by construction of the row exponent.
// Table-driven: 2^(j/256) and cis(2 pi j/256) in shared memory, degree-4/5/6 polynomials on
// the reduced arguments (|r| <= ln2/512, |s| <= pi/256); error <= ~4 ulp.
// PHT_TAB64=1: 64-entry bank-replicated tables, degree 5/7/8 (|r| <= ln2/128, |s| <= pi/64).
template <bool TL = false>
__device__ __forceinline__ double2 expcis(double y, double th, const double *etab, const double2 *ctab,
                                          double th_lo = 0.0)
{
    // terms more than e^-2000 below the row scale flush to 0; clamping first keeps y*256/ln2
    // inside the 32-bit integer extracted from the shifter (|y| up to ~10^8 occurs for large
    // cell-shifted liftings)
    y = (y < -2000.0) ? -2000.0 : y; // (a select: cheaper than fmax, and NaN propagates)
#if PHT_TAB64
    unsigned lane;
    asm("mov.u32 %0, %%laneid;" : "=r"(lane));
    // |r| <= ln2/128: e^r to r^5 (truncation 3.5e-17); |s| <= pi/64: sin to s^7, cos to s^8
    const double kf = fma(y, KC[0], SHIFT);
    const int ki = __double2loint(kf);
    const double kd = kf - SHIFT;
    double r = fma(kd, -KC[1], y);
    r = fma(kd, -KC[2], r);
    const double p = fma(fma(fma(fma(fma(r, KC[18], KC[3]), r, KC[4]), r, 0.5), r, 1.0), r, 1.0);
    double mag = etab[((ki & 63) << 4) | (lane & 15)] * p;
    const int m = ki >> 6;
    const unsigned hi = (unsigned)__double2hiint(mag) + ((unsigned)m << 20);
    mag = (m < -1000) ? 0.0 : __hiloint2double((int)hi, __double2loint(mag));

    const double qf = fma(th, KC[5], SHIFT);
    const int qi = __double2loint(qf);
    const double qd = qf - SHIFT;
    double s = fma(qd, -KC[6], th);
    s = fma(qd, -KC[7], s);
    s = fma(qd, -KC[8], s);
    const double s2 = s * s;
    const double sn = fma(s * s2, fma(s2, fma(s2, KC[16], KC[9]), KC[10]), s);
    const double cs = fma(s2, fma(s2, fma(s2, fma(s2, KC[17], KC[11]), KC[3]), -0.5), 1.0);
    const double2 T = ctab[((qi & 63) << 3) | (lane & 7)];
#else
    const double kf = fma(y, KC[0], SHIFT);
    const int ki = __double2loint(kf);
    const double kd = kf - SHIFT;
    double r = fma(kd, -KC[1], y);
    r = fma(kd, -KC[2], r);
    const double p = fma(fma(fma(fma(r, KC[3], KC[4]), r, 0.5), r, 1.0), r, 1.0);
    double mag = etab[ki & 255] * p;
    const int m = ki >> 8;
    const unsigned hi = (unsigned)__double2hiint(mag) + ((unsigned)m << 20);
    mag = (m < -1000) ? 0.0 : __hiloint2double((int)hi, __double2loint(mag));

    const double qf = fma(TL ? th + th_lo : th, KC[5], SHIFT);
    const int qi = __double2loint(qf);
    const double qd = qf - SHIFT;
    double s = fma(qd, -KC[6], th); // exact for the compensated th (TL): th is a multiple of 2^-20
    s = fma(qd, -KC[7], s);
    s = fma(qd, -KC[8], s);
    if (TL) s += th_lo;
    const double s2 = s * s;
    const double sn = fma(s * s2, fma(s2, KC[9], KC[10]), s);
    const double cs = fma(s2, fma(s2, fma(s2, KC[11], KC[3]), -0.5), 1.0);
    const double2 T = ctab[qi & 255];
#endif
    const double cr = fma(T.x, cs, -T.y * sn);
    const double ci = fma(T.y, cs, T.x * sn);
    return make_double2(mag * cr, mag * ci);
}

#ifndef PHT_RT_SMEM
#define PHT_RT_SMEM(n) ((n) <= 12)
#endif
#ifndef PHT_PAIR
#define PHT_PAIR(n) ((n) <= 8)
#endif
#ifndef PHT_STEPW_UNROLL
#define PHT_STEPW_UNROLL 1 // unroll factor of k_stepw's single-term row loop (experiments)
#endif
constexpr int kStepwUnroll = PHT_STEPW_UNROLL; // (#pragma unroll does not expand macros)


// ---- tile geometry --------------------------------------------------------------------
// W layout (evaluation): WL point lanes per equation, thread (k, q) = (tid / WL, tid % WL).
// L layout (solve): PPW points per warp, lane = (point, row).  PTS is chosen so that the L
// groups exactly fill the CTA's warps (no second round), and CTAs stay small (<= 8 warps) so
// that two co-resident CTAs overlap each other's load / barrier phases.
template <int N>
struct GeoS {
    static constexpr int WL = N <= 5 ? 32 : (N <= 16 ? 16 : 8);
    static constexpr int NTW = N * WL;                 // W-layout threads
    static constexpr int NWARP = (NTW + 31) / 32;
    static constexpr int NT = NWARP * 32;              // threads per CTA (whole warps for the L layout)
    static constexpr int PPW = 32 / N;                 // L layout: points per warp
    static constexpr int GMAX = WL / PPW < NWARP ? WL / PPW : NWARP;
    static constexpr int PTS = PPW * (GMAX > 0 ? GMAX : 1) <= WL ? PPW * (GMAX > 0 ? GMAX : 1) : WL;
    static constexpr int NGRP = (PTS + PPW - 1) / PPW; // L-layout point groups (<= NWARP)
    static constexpr int RW = N + 2;                   // row width (complex)
    static constexpr int MS = (N * RW) | 1;            // matrix slot stride: odd => conflict-free
    static constexpr int KS = (N + 3) & ~3;            // pivot-key slot per point (16 B aligned)
    // co-resident CTAs per SM: aim at 16 warps (4 per SMSP -> 128 registers per thread)
#ifdef PHT_GEOS_MINB
    static constexpr int MINB = N <= 12 ? PHT_GEOS_MINB : 1; // experiments
#else
    static constexpr int MINB = N <= 12 ? (PHT_RT_SMEM(N) ? (16 / NWARP > 1 ? 16 / NWARP : 1) : 2) : 1;
#endif
};

// Geometry of the system-specialised kernels (pht_jit.cu): the generated row code is
// straight-line per equation, so a warp must hold ONE equation for 32 points (W lanes = points,
// warp = equation); the L-layout solve then covers PPW * N points per pass.
#ifndef PHT_JIT_WARPS_PER_SM
#define PHT_JIT_WARPS_PER_SM 20
#endif
template <int N>
struct GeoJ {
    static constexpr int WL = 32;
    static constexpr int NTW = N * WL;
    static constexpr int NWARP = N;
    static constexpr int NT = NWARP * 32;
    static constexpr int PPW = 32 / N;
    static constexpr int PTS = PPW * N < 32 ? PPW * N : 32;
    static constexpr int NGRP = (PTS + PPW - 1) / PPW;
    static constexpr int RW = N + 2;
    static constexpr int MS = (N * RW) | 1;
    static constexpr int KS = (N + 3) & ~3;
    static constexpr int MINB = PHT_JIT_WARPS_PER_SM / N > 1 ? (PHT_JIT_WARPS_PER_SM / N < 8 ? PHT_JIT_WARPS_PER_SM / N : 8) : 1;
};

#ifdef PHT_JIT
template <int N>
using Geo = GeoJ<N>;
#else
template <int N>
using Geo = GeoS<N>;
#endif

template <int N>
struct Smem {
    // [variable][point] tiles use a row stride of WL + 1 (odd in 16-byte units): accesses with
    // consecutive threads on consecutive variables of a point are then bank-conflict free.
    static constexpr int WL = Geo<N>::WL + 1;
    double exptab[TAB_E];
    double2 cistab[TAB_C];
    double2 rt[N][WL];    // (rho, vartheta) per variable
    double2 xs[N][WL];    // x (or z) of the tile
    double2 inv[N][WL];   // 1/x (EVAL_X); staging of dE (DIRS)
    double2 out2[N][WL];  // staging of dN (DIRS)
    double dn2[N][WL];
    double tau[Geo<N>::WL];
    double tinv[Geo<N>::WL];
    int st[Geo<N>::WL];
    alignas(16) unsigned keys[Geo<N>::NWARP][Geo<N>::PPW * Geo<N>::KS]; // pivot keys (L layout)
    alignas(16) double2 mat[Geo<N>::PTS * Geo<N>::MS]; // [q][row][col]: solve tile / staged output
};

// Term record -> registers: a_0..a_{N-1}, omega, log|c|, arg c (pht_capi.cu packer).
template <int N>
__device__ __forceinline__ void load_rec(const double2 *r, double (&a)[rec_stride(N)])
{
#pragma unroll
    for (int u = 0; u < rec_stride(N) / 2; ++u) {
        const double2 v = __ldg(r + u);
        a[2 * u] = v.x;
        a[2 * u + 1] = v.y;
    }
}

// (rho, vartheta) of one point: in registers, or read from the shared tile per term
// (PHT_RT_SMEM: 4N fewer registers -> more resident warps; broadcast-free LDS.128 per variable).
template <int N, bool SMEM>
struct PointLog;
template <int N>
struct PointLog<N, false> {
    double rho[N], th[N];
    template <int WL>
    __device__ __forceinline__ void load(const double2 (*rt)[WL], int q)
    {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double2 v = rt[j][q];
            rho[j] = v.x;
            th[j] = v.y;
        }
    }
    __device__ __forceinline__ double2 get(int j) const { return make_double2(rho[j], th[j]); }
};
// PHT_RT_VOL (experiments): 1 = every term re-reads (rho, vartheta) from shared memory (volatile
// loads the compiler cannot hoist out of the term loop: 4N fewer live registers); 2 = only rho
// re-read, vartheta hoisted
#ifndef PHT_RT_VOL
#define PHT_RT_VOL 0
#endif
template <int N>
struct PointLog<N, true> {
    const double2 *base;
    int stride;
    template <int WL>
    __device__ __forceinline__ void load(const double2 (*rt)[WL], int q)
    {
        base = &rt[0][q];
        stride = WL;
    }
    __device__ __forceinline__ double2 get(int j) const
    {
#if PHT_RT_VOL == 1
        double2 v;
        const unsigned a = (unsigned)__cvta_generic_to_shared(base + j * stride);
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
        return v;
#elif PHT_RT_VOL == 2
        double r;
        const unsigned a = (unsigned)__cvta_generic_to_shared(base + j * stride);
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(a));
        return make_double2(r, base[j * stride].y);
#else
        return base[j * stride];
#endif
    }
};

// phi = omega tau + log|c| + sum_j a_j rho_j and theta = arg c + sum_j a_j vartheta_j, each with
// two interleaved partial sums (ILP).
template <int N, class PL>
__device__ __forceinline__ void phi_theta(const double (&a)[rec_stride(N)], const PL &pl, double tau,
                                          double &phi, double &theta)
{
    double p0 = fma(a[N], tau, a[N + 1]), p1 = 0.0, t0 = a[N + 2], t1 = 0.0;
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        const double2 v = pl.get(j);
        p0 = fma(a[j], v.x, p0);
        t0 = fma(a[j], v.y, t0);
        if (j + 1 < N) {
            const double2 u = pl.get(j + 1);
            p1 = fma(a[j + 1], u.x, p1);
            t1 = fma(a[j + 1], u.y, t1);
        }
    }
    phi = p0 + p1;
    theta = t0 + t1;
}

template <int N, class PL>
__device__ __forceinline__ double phi_of(const double (&a)[rec_stride(N)], const PL &pl, double tau)
{
    double p0 = fma(a[N], tau, a[N + 1]), p1 = 0.0;
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        p0 = fma(a[j], pl.get(j).x, p0);
        if (j + 1 < N) p1 = fma(a[j + 1], pl.get(j + 1).x, p1);
    }
    return p0 + p1;
}

// Compensated stage 2 for the tracker's final refinement (reading R30): each log
// coordinate is split exactly as v = v_hi + v_lo with v_hi a multiple of 2^-20 (|v| < 2^30), so
// sum_j a_j v_hi_j is exact (|a_j| <= 1024) and the rounding of the dot product moves to the small
// part: phi = phi_hi + phi_lo, theta = th_hi + th_lo with an absolute error ~u instead of u |phi|.
__device__ __forceinline__ double split_hi(double v)
{
    const double C = 0x1.8p+32; // 1.5 * 2^32: rounds |v| < 2^30 to a multiple of 2^-20
    const double h = (v + C) - C;
    return (fabs(v) < 0x1p30) ? h : v;
}
template <int N, class PL>
__device__ __forceinline__ void phi_theta_c(const double (&a)[rec_stride(N)], const PL &pl, double tau, double &ph,
                                            double &pl_, double &th, double &tl)
{
    double p0 = 0.0, p1 = fma(a[N], tau, a[N + 1]), t0 = 0.0, t1 = a[N + 2];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const double2 v = pl.get(j);
        const double rh = split_hi(v.x), vh = split_hi(v.y);
        p0 = fma(a[j], rh, p0);          // exact
        p1 = fma(a[j], v.x - rh, p1);    // v.x - rh exact
        t0 = fma(a[j], vh, t0);
        t1 = fma(a[j], v.y - vh, t1);
    }
    ph = p0;
    pl_ = p1;
    th = t0;
    tl = t1;
}

// Row accumulator with an online binary row exponent e (ledger R7): the row holds
// sum_i w_i 2^-e; a term more than e^512 above the current scale rescales the row exactly.
template <int N>
struct RowAcc {
    double2 g[N], gt, h;
    double ed; // row exponent; y = phi - ed ln2 with ln2 = LN2_HI + LN2_LO (ed LN2_HI exact)

    __device__ __forceinline__ void init(double phi0)
    {
#pragma unroll
        for (int j = 0; j < N; ++j) g[j] = make_double2(0.0, 0.0);
        gt = h = make_double2(0.0, 0.0);
        set_exp(rint(phi0 * KC[14]));
    }
    __device__ __forceinline__ void set_exp(double e) { ed = e; }
    __device__ __forceinline__ double reduced(double phi) const { return fma(-ed, KC[13], fma(-ed, KC[12], phi)); }
    // the same for phi = ph + pl (compensated stage 2): ph - e LN2_HI is exact
    __device__ __forceinline__ double reduced2(double ph, double pl) const
    {
        return fma(-ed, KC[12], ph) + fma(-ed, KC[13], pl);
    }
    __device__ __forceinline__ double reduce(double phi)
    {
        double y = reduced(phi);
        if (__builtin_expect(y > 512.0, 0)) { // rare: rescale everything to the new leading term (exact power of two)
            const double e2 = rint(phi * KC[14]);
            // the shift d = ed - e2 lies in [-2000, -738]: applied as two factors 2^d1 2^d2 (each >=
            // 2^-1000, normal), because the accumulators hold up to ~2^745 and a single 2^d would
            // underflow to 0 for d < -1074 although the rescaled entries are representable
            const int d = (int)fmax(ed - e2, -2000.0), d1 = d / 2, d2 = d - d1;
            const double f1 = scalbn(1.0, d1), f2 = scalbn(1.0, d2);
#pragma unroll
            for (int j = 0; j < N; ++j) g[j] = make_double2(g[j].x * f1 * f2, g[j].y * f1 * f2);
            gt = make_double2(gt.x * f1 * f2, gt.y * f1 * f2);
            h = make_double2(h.x * f1 * f2, h.y * f1 * f2);
            set_exp(e2);
            y = reduced(phi);
        }
        return y;
    }
    __device__ __forceinline__ void add(const double (&a)[rec_stride(N)], double2 w)
    {
        h.x += w.x;
        h.y += w.y;
        gt.x = fma(a[N], w.x, gt.x);
        gt.y = fma(a[N], w.y, gt.y);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            g[j].x = fma(a[j], w.x, g[j].x);
            g[j].y = fma(a[j], w.y, g[j].y);
        }
    }
};

#ifdef PHT_JIT
// system-specialised rows: defined by the generated source (pht_jit.cu) after this header.
// jit_row_core: row k of the point whose (rho, vartheta) column is rt[j * ST].
template <int N>
__device__ void jit_row_core(int k, const double2 *rt, int ST, double tau, const double *etab, const double2 *ctab,
                             double2 (&row)[N + 2], int &e, const double *wq);
template <int N>
__device__ void jit_row(const DevSys &S, const Smem<N> &sm, int k, int q, double2 (&row)[N + 2], int &e,
                        const double *wq);
#endif

// a2-a4 for row k of point q: row = [G_1..G_N | G_tau | h] scaled by 2^-e.
// Terms are processed two at a time (independent dependency chains for the FP64 pipe).
// wq (optional): per-point lifting table (cell-shifted liftings omega', pht_track_cells); the
// term's omega is replaced by wq[i] (global term index i).
template <int N, bool COMP = false>
__device__ __forceinline__ void eval_row(const DevSys &S, const Smem<N> &sm, int k, int q,
                                         double2 (&row)[N + 2], int &e, const double *wq = nullptr)
{
    if (S.proj && k == N - 1) {
        // the bordering row y^* of the projective directions in log
        // coordinates: y^* (y (.) delta) = sum_j |y_j|^2 delta_j; no dH/dtau, no H entry
#pragma unroll
        for (int j = 0; j < N; ++j) row[j] = make_double2(exp(2.0 * sm.rt[j][q].x), 0.0);
        row[N] = make_double2(0.0, 0.0);
        row[N + 1] = make_double2(0.0, 0.0);
        e = 0;
        return;
    }
#ifdef PHT_JIT
    jit_row<N>(S, sm, k, q, row, e, wq);
    return;
#endif
    constexpr int RS = rec_stride(N);
    PointLog<N, (bool)PHT_RT_SMEM(N)> pl;
    pl.template load<Smem<N>::WL>(sm.rt, q);
    const double tau = sm.tau[q];
    const int i0 = __ldg(S.off + k), i1 = __ldg(S.off + k + 1);
    const double2 *rec = S.rec + (size_t)i0 * (RS / 2);
    const int m = i1 - i0;

    const double *wk = wq ? wq + i0 : nullptr;
    RowAcc<N> acc;
    {
        double a[RS];
        load_rec<N>(rec, a);
        if (wk) a[N] = __ldg(wk);
        acc.init(phi_of<N>(a, pl, tau));
    }
    int i = 0;
    if (COMP) { // compensated stage 2 for the tracker's final refinement (reading R30)
        for (; i < m; ++i) {
            double a[RS];
            load_rec<N>(rec + (size_t)i * (RS / 2), a);
            if (wk) a[N] = __ldg(wk + i);
            double ph, pl_, th, tl;
            phi_theta_c<N>(a, pl, tau, ph, pl_, th, tl);
            acc.reduce(ph + pl_);
            acc.add(a, expcis<true>(acc.reduced2(ph, pl_), th, sm.exptab, sm.cistab, tl));
        }
    }
    // two terms per iteration only while the register budget allows it (ILP vs spills)
    for (; PHT_PAIR(N) && i + 1 < m; i += 2) {
        double a[RS], b[RS];
        load_rec<N>(rec + (size_t)i * (RS / 2), a);
        load_rec<N>(rec + (size_t)(i + 1) * (RS / 2), b);
        if (wk) {
            a[N] = __ldg(wk + i);
            b[N] = __ldg(wk + i + 1);
        }
        double pa, pb, ta, tb;
        phi_theta<N>(a, pl, tau, pa, ta);
        phi_theta<N>(b, pl, tau, pb, tb);
        // both rescale checks first: a rescale triggered by b must also apply to a's term
        acc.reduce(pa);
        acc.reduce(pb);
        const double ya = acc.reduced(pa), yb = acc.reduced(pb);
        const double2 wa = expcis(ya, ta, sm.exptab, sm.cistab);
        const double2 wb = expcis(yb, tb, sm.exptab, sm.cistab);
        acc.add(a, wa);
        acc.add(b, wb);
    }
    for (; i < m; ++i) {
        double a[RS];
        load_rec<N>(rec + (size_t)i * (RS / 2), a);
        if (wk) a[N] = __ldg(wk + i);
        double pa, ta;
        phi_theta<N>(a, pl, tau, pa, ta);
        const double ya = acc.reduce(pa);
        acc.add(a, expcis(ya, ta, sm.exptab, sm.cistab));
    }
#pragma unroll
    for (int j = 0; j < N; ++j) row[j] = acc.g[j];
    row[N] = acc.gt;
    row[N + 1] = acc.h;
    e = (int)acc.ed;
}

// a1 for the whole tile: (rho, vartheta) from xs (x in EVAL_X/DIRS/STEP, z in EVAL_Z).
template <int N, int MODE>
__device__ __forceinline__ void stage1(Smem<N> &sm, int tid)
{
    if (tid >= N * Geo<N>::PTS) return;
    const int q = tid / N, j = tid % N;
    const double2 v = sm.xs[j][q];
    double rho, th;
    int st = 0;
    if (MODE == MODE_EVAL_Z) {
        if (!(isfinite(v.x) && isfinite(v.y))) { st |= PT_NONFINITE; rho = 0.0; th = 0.0; }
        else {
            rho = v.x;
            const double kq = rint(v.y * INV_2PI); // wrap Im z into [-pi, pi] (integer a)
            th = fma(-kq, TWO_PI_LO, fma(-kq, TWO_PI_HI, v.y));
        }
    } else {
        double2 inv;
        log_split(v, rho, th, inv, st);
        if (MODE == MODE_EVAL_X) sm.inv[j][q] = inv;
    }
    sm.rt[j][q] = make_double2(rho, th);
    if (st) atomicOr(&sm.st[q], st);
}

// W -> shared: normalise the row by an exact power of two (rows are scale-free for the solve,
// S:316) and store it into the point's matrix slot.
template <int N>
__device__ __forceinline__ void normalize_row(double2 (&row)[N + 2])
{
    // the exponent of max_j |row_j|_1 is in the high words: one integer max per entry
    unsigned hmax = 0u;
#pragma unroll
    for (int j = 0; j < N; ++j) hmax = max(hmax, (unsigned)__double2hiint(cabs1(row[j])));
    const int ef = (int)(hmax >> 20); // biased exponent (>= 0x7ff: inf/NaN)
    if (ef >= 1 && ef <= 2045) {
        const double f = __hiloint2double((2046 - ef) << 20, 0); // 2^-ilogb(rmax), exact
#pragma unroll
        for (int c = 0; c < N + 2; ++c) row[c] = make_double2(row[c].x * f, row[c].y * f);
    } else if (ef == 0 || ef == 2046) { // subnormal or [2^1023, inf) maximum (rare): general path
        double rmax = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) rmax = fmax(rmax, cabs1(row[j]));
        if (rmax > 0.0 && isfinite(rmax)) {
            const double f = scalbn(1.0, -ilogb(rmax));
#pragma unroll
            for (int c = 0; c < N + 2; ++c) row[c] = make_double2(row[c].x * f, row[c].y * f);
        }
    }
}

template <int N>
__device__ __forceinline__ void store_row(Smem<N> &sm, int k, int q, double2 (&row)[N + 2])
{
    normalize_row<N>(row);
    double2 *dst = sm.mat + q * Geo<N>::MS + k * Geo<N>::RW;
#pragma unroll
    for (int c = 0; c < N + 2; ++c) dst[c] = row[c];
}

// a5 in the L layout: lane (seg, i) of a warp holds row i of point q = g*PPW + seg.
// Gauss-Jordan with partial pivoting (max |Re|+|Im| of the column among unused rows, lowest
// row on ties — ledger R12; the comparison key keeps the top 15 mantissa bits).  The keys go
// through shared memory (one STS, ceil(N/4) LDS.128, integer max); the pivot lane publishes its
// row; elimination is branch-free (multiplier 0 on the pivot lane).  On return the lane whose row
// pivoted column `col` holds dE = -row[N]/u, dN = -row[N+1]/u for variable col:
// G [dE | dN] = -[G_tau | h].
// The elimination on rows held in registers: lane (seg0 = lane / N, i) holds row i of its point;
// prow: the point's pivot-row buffer (N + 2 entries, shared memory), kseg: its pivot keys (PPW > 4).
// Pivot-row broadcast: PHT_W_SHFL = 1 moves the pivot row lane-to-lane with shuffles (4 SHFL per
// complex entry, no shared-memory store/load and no __syncwarp per pivot); 0 publishes it through
// the point's shared buffer prow.  IMAJ: lane order of the caller, index-major (lane = i * PPW +
// seg, warp-per-group kernels) or point-major (lane = seg * N + i, tile kernels).
#ifndef PHT_W_SHFL
#define PHT_W_SHFL 0
#endif
__device__ __forceinline__ double2 shfl2(double2 v, int src)
{
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

template <int N, int PPW, int KS, bool IMAJ = false, int LPR = 1, bool SHFL = (bool)PHT_W_SHFL, bool DB = false>
__device__ __forceinline__ void lsolve_regs(double2 (&a)[N + 2], double2 *prow, unsigned *kseg, int seg0, int seg,
                                            int i, bool act, int &col, double2 &dE, double2 &dN, bool &singular,
                                            bool prim = true)
{
    constexpr int RW = N + 2;
    unsigned long long rbits = 0ull;
#pragma unroll
    for (int j = 0; j < N; ++j) rbits = max(rbits, dbits(cabs1(a[j])));
    // singular threshold of this row (ledger R13); a non-finite entry makes the point singular
    const double thr = 1e-14 * __longlong_as_double((long long)rbits);
    __syncwarp();
    bool used = false;
    col = 0;
    singular = rbits >= DBITS_INF;
    double2 myrcp = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < N; ++j) {
        // 1/|a_j|^2 on every lane (its latency overlaps the pivot search).  For an accepted pivot,
        // thr < |a_j|_1 < 2^510 keeps |a_j|^2 normal, so the Newton reciprocal is exact to 1 ulp.
        const double crd = rcp_nr(fma(a[j].x, a[j].x, a[j].y * a[j].y));
        const double2 crcp = make_double2(a[j].x * crd, -a[j].y * crd);
        unsigned key = 0u;
        if (!used) key = ((unsigned)__double2hiint(cabs1(a[j])) & ~63u) | (unsigned)(32 - i);
        unsigned kmax = 0u;
        if (PPW <= 4) {
            // one full-warp redux per point segment (uniform datapath, no divergence)
#pragma unroll
            for (int sg = 0; sg < PPW; ++sg) {
                const unsigned m = __reduce_max_sync(0xffffffffu, (seg0 == sg) ? key : 0u);
                kmax = (seg == sg) ? m : kmax;
            }
        } else {
            if (act && prim) kseg[i] = key;
            __syncwarp();
#pragma unroll
            for (int u = 0; u < KS; u += 4) {
                const uint4 v = *reinterpret_cast<const uint4 *>(kseg + u);
                kmax = max(kmax, (u + 0 < N) ? v.x : 0u);
                kmax = max(kmax, (u + 1 < N) ? v.y : 0u);
                kmax = max(kmax, (u + 2 < N) ? v.z : 0u);
                kmax = max(kmax, (u + 3 < N) ? v.w : 0u);
            }
        }
        const int r = 32 - (int)(kmax & 63u);
        const bool me = (i == r);
        if (me) {
            used = true;
            col = j;
        }
        if (SHFL) {
        const int src = IMAJ ? (r * PPW + seg) * LPR : seg * N + r; // a lane holding this point's pivot row
        const double2 rcp = shfl2(crcp, src);
        {
            const double pa = cabs1(a[j]);
            singular = singular || (me && !(pa > thr && pa < 0x1p510));
            myrcp = me ? crcp : myrcp;
        }
        double2 l = cmul(a[j], rcp);
        l = me ? make_double2(0.0, 0.0) : l;
#pragma unroll
        for (int c = j + 1; c < RW; ++c) a[c] = cfms(a[c], l, shfl2(a[c], src));
        a[j] = me ? a[j] : make_double2(0.0, 0.0);
        if (PPW > 4) __syncwarp(); // kseg is rewritten by the next pivot search
        } else {
        // DB: pivots alternate between two row buffers, so the barrier after the
        // elimination goes (pivot j + 1's publish barrier orders pivot j's reads before pivot
        // j + 2's writes); the caller then provides 2 (RW | 1) entries per point
        double2 *pr = prow + (DB ? (j & 1) * (RW | 1) : 0);
        if (me && act && prim) {
            // the pivot row with the pivot replaced by its reciprocal (computed before the
            // argmax by every lane for its own candidate: the reciprocal's latency overlaps the
            // pivot search instead of following the row broadcast)
            pr[j] = crcp;
#pragma unroll
            for (int c = j + 1; c < RW; ++c) pr[c] = a[c];
        }
        __syncwarp();
        const double2 rcp = pr[j];
        {
            // branch-free: pivot at or below the threshold, or too large for a normal |a_j|^2
            const double pa = cabs1(a[j]);
            singular = singular || (me && !(pa > thr && pa < 0x1p510));
        }
        // branch-free elimination: the pivot lane uses multiplier 0 and keeps its row; column j of
        // the other rows is not read again, so it is not zeroed (measured: predicating the
        // elimination on !me instead of the multiplier select is 2% slower -- divergence)
        double2 l = cmul(a[j], rcp);
        l = me ? make_double2(0.0, 0.0) : l;
#pragma unroll
        for (int c = j + 1; c < RW; ++c) a[c] = cfms(a[c], l, pr[c]);
        if (!DB) __syncwarp();
        }
    }
    if (!SHFL) {
        // prow[c] (c < N) still holds the reciprocal of column c's pivot (later steps only write
        // prow[j'..] with j' > c): the lane's own pivot reciprocal without a select per pivot
        myrcp = prow[(DB ? (col & 1) * (RW | 1) : 0) + col]; // (written by this lane)
        __syncwarp(); // the caller may reuse prow
    }
    const double2 e = cmul(a[N], myrcp), n = cmul(a[N + 1], myrcp);
    dE = make_double2(-e.x, -e.y);
    dN = make_double2(-n.x, -n.y);
}

// a5 in the L layout of the tile kernels: the rows come from the point's matrix slot
template <int N>
__device__ __forceinline__ void lsolve(Smem<N> &sm, int lane, int w, int g, int &col, double2 &dE,
                                       double2 &dN, bool &singular, bool &act, int &q)
{
    constexpr int RW = Geo<N>::RW, MS = Geo<N>::MS, PPW = Geo<N>::PPW, KS = Geo<N>::KS;
    const int seg0 = lane / N;
    const bool inseg = seg0 < PPW;
    const int seg = inseg ? seg0 : 0, i = inseg ? lane - seg0 * N : 0;
    q = g * PPW + seg;
    act = inseg && (q < Geo<N>::PTS);
    // lanes without a point of their own read their group's first point (same warp: no cross-warp
    // access to another group's slot; compute-sanitizer racecheck)
    const int qc = (q < Geo<N>::PTS) ? q : g * PPW;
    double2 *slot = sm.mat + qc * MS;
    unsigned *kseg = &sm.keys[w][seg * KS];
    double2 a[RW];
#pragma unroll
    for (int c = 0; c < RW; ++c) a[c] = slot[i * RW + c];
    __syncwarp(); // every row is in registers before the slot doubles as the pivot-row buffer
    lsolve_regs<N, PPW, KS>(a, slot, kseg, seg0, seg, i, act, col, dE, dN, singular);
}

// y <- y / ||y|| for the point q of a [variable][point] tile (projective systems, reading R29)
template <int N, int WLP>
__device__ __forceinline__ void proj_normalize(double2 (*v)[WLP], int q)
{
    double s2 = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s2 = fma(v[j][q].x, v[j][q].x, fma(v[j][q].y, v[j][q].y, s2));
    const double f = (s2 > 0.0 && isfinite(s2)) ? rsqrt(s2) : 1.0;
#pragma unroll
    for (int j = 0; j < N; ++j) v[j][q] = make_double2(v[j][q].x * f, v[j][q].y * f);
}

// a5, QR route (the paper's mechanism P:708-726, Alg. 3).
// Column layout: lane (seg, c) of a warp holds COLUMN c of [G | G_tau | h] of point
// q = g*PPQ + seg (PPQ = 32 / (N+2) points per warp).  Householder reflections from the left
// (no pivoting: backward stable for any Jx) reduce G to R and carry the two right-hand-side
// columns along (lanes N, N+1 end with Q^H G_tau, Q^H h); a row-oriented back substitution
// R [dE | dN] = -Q^H [G_tau | h] then leaves dE_c, dN_c on lane c.  The reflector of step k is
// built by lane k from its column and published through the point's matrix slot.  Singular
// (reading R26): |R_kk| <= 1e-14 ||G||_F or non-finite.  inv/out2 of the point serve as the
// broadcast buffer of the back substitution.
template <int N>
__device__ __forceinline__ void qsolve(Smem<N> &sm, int lane, int g, int &col, double2 &dE, double2 &dN,
                                       bool &singular, bool &act, int &q)
{
    constexpr int RW = Geo<N>::RW, MS = Geo<N>::MS, PPQ = 32 / RW;
    const int seg0 = lane / RW;
    const bool inseg = seg0 < PPQ;
    const int seg = inseg ? seg0 : 0, c = inseg ? lane - seg0 * RW : 0;
    q = g * PPQ + seg;
    const bool live = inseg && (q < Geo<N>::PTS);
    act = live && (c < N);
    const int qc = live ? q : g * PPQ; // (see lsolve: same-warp slot for lanes without a point)
    double2 *slot = sm.mat + qc * MS;
    double *scr = reinterpret_cast<double *>(slot);
    double2 a[N];
#pragma unroll
    for (int r = 0; r < N; ++r) a[r] = slot[r * RW + c];
    double n2 = 0.0;
#pragma unroll
    for (int r = 0; r < N; ++r) n2 = fma(a[r].x, a[r].x, fma(a[r].y, a[r].y, n2));
    __syncwarp();
    if (live && c < N) scr[c] = n2;
    __syncwarp();
    double fro2 = 0.0;
#pragma unroll
    for (int u = 0; u < N; ++u) fro2 += scr[u];
    __syncwarp();
    const double thr = 1e-14 * sqrt(fro2);
    singular = !isfinite(thr);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        // reflector from column k (every lane evaluates it for its own column; lane k publishes)
        double s2 = 0.0;
#pragma unroll
        for (int r = k; r < N; ++r) s2 = fma(a[r].x, a[r].x, fma(a[r].y, a[r].y, s2));
        const double nrm = sqrt(s2), ax0 = sqrt(fma(a[k].x, a[k].x, a[k].y * a[k].y));
        const double2 ph = (ax0 > 0.0) ? make_double2(a[k].x / ax0, a[k].y / ax0) : make_double2(1.0, 0.0);
        const double2 alpha = make_double2(-ph.x * nrm, -ph.y * nrm);
        if (live && c == k) {
            const double den = nrm * (nrm + ax0);
            scr[2 * N] = (den > 0.0) ? 1.0 / den : 0.0; // beta = 2 / v^H v (after v in slot[0..N-1])
            slot[k] = make_double2(ph.x * (ax0 + nrm), ph.y * (ax0 + nrm)); // v_k = x0 - alpha
#pragma unroll
            for (int r = k + 1; r < N; ++r) slot[r] = a[r];
            singular = singular || !(nrm > thr);
        }
        __syncwarp();
        const double beta = scr[2 * N];
        double2 sdot = make_double2(0.0, 0.0);
#pragma unroll
        for (int r = k; r < N; ++r) {
            const double2 v = slot[r];
            sdot.x = fma(v.x, a[r].x, fma(v.y, a[r].y, sdot.x));
            sdot.y = fma(v.x, a[r].y, fma(-v.y, a[r].x, sdot.y));
        }
        const double2 t = make_double2(beta * sdot.x, beta * sdot.y);
        const bool upd = c > k;
#pragma unroll
        for (int r = k; r < N; ++r) {
            const double2 v = slot[r];
            const double2 nv = make_double2(a[r].x - (t.x * v.x - t.y * v.y), a[r].y - (t.x * v.y + t.y * v.x));
            a[r] = upd ? nv : a[r];
        }
        if (c == k) {
            a[k] = alpha;
#pragma unroll
            for (int r = k + 1; r < N; ++r) a[r] = make_double2(0.0, 0.0);
        }
        __syncwarp();
    }
    // R and Q^H [G_tau | h] back into the slot ([row][col]), then rows on lanes c < N
    if (live) {
#pragma unroll
        for (int r = 0; r < N; ++r) slot[r * RW + c] = a[r];
    }
    __syncwarp();
    const int i = (c < N) ? c : 0;
    double2 b1 = slot[i * RW + N], b2 = slot[i * RW + N + 1];
    b1 = make_double2(-b1.x, -b1.y);
    b2 = make_double2(-b2.x, -b2.y);
    const double2 rii = slot[i * RW + i];
    const double rd = 1.0 / fma(rii.x, rii.x, rii.y * rii.y);
    const double2 rinv = make_double2(rii.x * rd, -rii.y * rd);
    double2 d1 = make_double2(0.0, 0.0), d2 = d1;
#pragma unroll
    for (int j = N - 1; j >= 0; --j) {
        if (c == j) {
            d1 = cmul(b1, rinv);
            d2 = cmul(b2, rinv);
            if (live) {
                sm.inv[j][qc] = d1;
                sm.out2[j][qc] = d2;
            }
        }
        __syncwarp();
        if (c < j) {
            const double2 e1 = sm.inv[j][qc], e2 = sm.out2[j][qc], rij = slot[c * RW + j];
            b1 = cfms(b1, rij, e1);
            b2 = cfms(b2, rij, e2);
        }
    }
    __syncwarp();
    col = i;
    dE = d1;
    dN = d2;
}

// Evaluation modes (pht_evaluate, pht_evaluate_log): one tile of the persistent kernel k_phte.
template <int N, int MODE>
__device__ __forceinline__ void eval_tile(const DevSys &S, const Args &A, Smem<N> &sm, const int64_t base)
{
    using G = Geo<N>;
    constexpr int PTS = G::PTS, WL = G::WL;
    const int tid = threadIdx.x;
    const int k = tid / WL, q = tid % WL;           // W layout
    const int64_t gq = base + q;
    const bool valid = (k < N) && (q < PTS) && (gq < A.P);

    // load the tile's points, coalesced: flat element tid = (point tid/N, variable tid%N)
    const double2 *xsrc = A.xin;
    if (tid < N * PTS) {
        const int qq = tid / N, j = tid % N;
        double2 v = make_double2(MODE == MODE_EVAL_Z ? 0.0 : 1.0, 0.0);
        if (base + qq < A.P) v = xsrc[(base * N) + tid];
        sm.xs[j][qq] = v;
    }
    if (tid < WL) {
        sm.st[tid] = 0;
        const int64_t g = base + tid;
        const bool in = (tid < PTS) && (g < A.P);
        double tv = (MODE == MODE_EVAL_Z) ? 0.0 : 1.0;
        if (in) tv = A.tin[g];
        if (MODE == MODE_EVAL_Z) {
            sm.tau[tid] = tv;
            if (!isfinite(tv)) { sm.st[tid] |= PT_NONFINITE; sm.tau[tid] = 0.0; }
        } else {
            if (!(tv > 0.0) || !isfinite(tv)) { sm.st[tid] |= PT_NONFINITE; tv = 1.0; }
            sm.tau[tid] = log(tv);
            sm.tinv[tid] = 1.0 / tv;
        }
        if (tid >= PTS) { // unused W lanes evaluate a harmless dummy point
            for (int j = 0; j < N; ++j) sm.xs[j][tid] = make_double2(MODE == MODE_EVAL_Z ? 0.0 : 1.0, 0.0);
        }
    }
    __syncthreads();
    {
        stage1<N, MODE>(sm, tid);
        if (tid < WL && tid >= PTS)
            for (int j = 0; j < N; ++j) sm.rt[j][tid] = make_double2(0.0, 0.0);
        __syncthreads();
        double2 row[N + 2];
        int e = 0;
        const bool wthr = k < N; // W-layout thread (the CTA is padded to whole warps)
        if (wthr) eval_row<N>(S, sm, k, q, row, e);
        const bool scaled = A.rexp != nullptr;
        bool fin = true;
        if (MODE == MODE_EVAL_X) {
            const double ti = sm.tinv[q];
            row[N] = make_double2(row[N].x * ti, row[N].y * ti);
#pragma unroll
            for (int j = 0; j < N; ++j) row[j] = cmul(row[j], sm.inv[j][q]);
        }
        if (!scaled) scale_row2<N + 2>(row, e);
#pragma unroll
        for (int c = 0; c < N + 2; ++c) fin = fin && isfinite(row[c].x) && isfinite(row[c].y);
        if (wthr && !fin && q < PTS) atomicOr(&sm.st[q], PT_NONFINITE);
        if (wthr && scaled && valid) A.rexp[gq * N + k] = e;
        // stage the tile's rows in shared memory: [q][k][0..N-1 | Jt | H], then copy each output
        // array's contiguous block with coalesced 16-byte stores
        if (wthr && q < PTS) {
            double2 *dst = sm.mat + q * Geo<N>::MS + k * Geo<N>::RW;
#pragma unroll
            for (int c = 0; c < N + 2; ++c) dst[c] = row[c];
        }
        __syncthreads();
        const int64_t npts = (A.P - base < PTS) ? (A.P - base) : PTS;
        if (A.J) {
            double2 *dstJ = A.J + base * N * N;
            for (int u = tid; u < npts * N * N; u += G::NT) {
                const int qq = u / (N * N), r = u - qq * N * N, kk = r / N, j = r - kk * N;
                dstJ[u] = sm.mat[qq * Geo<N>::MS + kk * Geo<N>::RW + j];
            }
        }
        for (int u = tid; u < npts * N; u += G::NT) {
            const int qq = u / N, kk = u - qq * N;
            const double2 *src = sm.mat + qq * Geo<N>::MS + kk * Geo<N>::RW;
            if (A.Jt) A.Jt[base * N + u] = src[N];
            if (A.H) A.H[base * N + u] = src[N + 1];
        }
        if (tid < PTS && base + tid < A.P && A.status) A.status[base + tid] = (uint8_t)sm.st[tid];
    }
}

// Persistent evaluation kernel: the grid (SMs x resident CTAs, at most one CTA per tile) walks
// the tiles and loads the exp/cis tables once per CTA (cyclic-10 evaluation 0.52 -> 0.60 G
// points/s with the power-of-two epilogue).  The fused DIRS/STEP kernel k_pht keeps one tile per
// CTA: a tile loop there costs live registers and spills (measured 524 -> 490 M evals/s).
template <int N, int MODE>
__global__ void __launch_bounds__(Geo<N>::NT, Geo<N>::MINB) k_phte(const DevSys S, const Args A)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<N> &sm = *reinterpret_cast<Smem<N> *>(smem_raw);
    load_tables(S, sm.exptab, sm.cistab, threadIdx.x, Geo<N>::NT);
    const int64_t tiles = (A.P + Geo<N>::PTS - 1) / Geo<N>::PTS;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        eval_tile<N, MODE>(S, A, sm, t * Geo<N>::PTS);
        __syncthreads(); // the tile's shared-memory readers are done before the next tile's loads
    }
}

// DIRS and STEP (pht_euler_newton, pht_pc_step): evaluation + two-RHS solve, one tile per CTA.
template <int N, int MODE>
__global__ void __launch_bounds__(Geo<N>::NT, Geo<N>::MINB) k_pht(const DevSys S, const Args A)
{
    static_assert(MODE == MODE_DIRS || MODE == MODE_STEP, "evaluation modes run k_phte");
    using G = Geo<N>;
    constexpr int PTS = G::PTS, WL = G::WL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<N> &sm = *reinterpret_cast<Smem<N> *>(smem_raw);
    const int tid = threadIdx.x;
    const int k = tid / WL, q = tid % WL;           // W layout
    const int lane = tid & 31, warp = tid >> 5;      // L layout
    load_tables(S, sm.exptab, sm.cistab, tid, G::NT);
    const int64_t base = (int64_t)blockIdx.x * PTS;

    // load the tile's points, coalesced: flat element tid = (point tid/N, variable tid%N)
    const double2 *xsrc = (MODE == MODE_STEP) ? A.xio : A.xin;
    if (tid < N * PTS) {
        const int qq = tid / N, j = tid % N;
        double2 v = make_double2(MODE == MODE_EVAL_Z ? 0.0 : 1.0, 0.0);
        if (base + qq < A.P) v = xsrc[(base * N) + tid];
        sm.xs[j][qq] = v;
    }
    if (tid < WL) {
        sm.st[tid] = 0;
        const int64_t g = base + tid;
        const bool in = (tid < PTS) && (g < A.P);
        double tv = (MODE == MODE_EVAL_Z || MODE == MODE_STEP) ? 0.0 : 1.0;
        if (in) tv = (MODE == MODE_STEP) ? A.tauio[g] : A.tin[g];
        if (MODE == MODE_EVAL_Z || MODE == MODE_STEP) {
            sm.tau[tid] = tv;
            if (!isfinite(tv)) { sm.st[tid] |= PT_NONFINITE; sm.tau[tid] = 0.0; }
        } else {
            if (!(tv > 0.0) || !isfinite(tv)) { sm.st[tid] |= PT_NONFINITE; tv = 1.0; }
            sm.tau[tid] = log(tv);
            sm.tinv[tid] = 1.0 / tv;
        }
        if (tid >= PTS) { // unused W lanes evaluate a harmless dummy point
            for (int j = 0; j < N; ++j) sm.xs[j][tid] = make_double2(MODE == MODE_EVAL_Z ? 0.0 : 1.0, 0.0);
        }
    }
    __syncthreads();

    // DIRS and STEP: evaluation (W) -> shared-memory tile -> warp-level solve (L).
    const int iters = (MODE == MODE_STEP) ? A.K + 1 : 1;
    // affine step: the apply phase below also computes (rho, vartheta) of each updated coordinate,
    // so stage 1 (and its barrier) runs only once; projective points are renormalised after the
    // apply phase, so they take the stage-1 pass every iteration
    const bool fused_log = (MODE == MODE_STEP) && !S.proj;
    for (int it = 0; it < iters; ++it) {
        if (it == 0 || !fused_log) {
            stage1<N, MODE>(sm, tid);
            if (tid < WL && tid >= PTS)
                for (int j = 0; j < N; ++j) sm.rt[j][tid] = make_double2(0.0, 0.0);
            __syncthreads();
        }
        {
            if (k < N) {
                double2 row[N + 2];
                int e;
                eval_row<N>(S, sm, k, q, row, e);
                if (q < PTS) store_row<N>(sm, k, q, row);
            }
        }
        __syncthreads();
        // tau~ = tau + dtau for the Newton evaluations; the solve does not read tau, and the
        // barrier after it orders this before the next evaluation
        if (MODE == MODE_STEP && it == 0 && tid < PTS)
            sm.tau[tid] += (base + tid < A.P) ? A.dtau[base + tid] : 0.0;
        auto apply = [&](int col, int qq, double2 dE, double2 dN, bool sing) {
            if (sing) atomicOr(&sm.st[qq], PT_SINGULAR);
            const double2 xv = sm.xs[col][qq];
            if (MODE == MODE_DIRS) {
                // dx/dt = x (.) delta_E / t, dN_x = x (.) delta_N (Jx = G diag(1/x), Jt = G_tau/t)
                const double2 de = cmul(xv, dE), dn = cmul(xv, dN);
                const double ti = sm.tinv[qq];
                sm.inv[col][qq] = make_double2(de.x * ti, de.y * ti);
                sm.out2[col][qq] = dn;
            } else {
                double2 xn;
                if (it == 0) {
                    // Euler: dx/dtau = x (.) delta_E  ->  x~ = x + h x delta_E
                    const double h = (base + qq < A.P) ? A.dtau[base + qq] : 0.0;
                    const double2 d = cmul(xv, dE);
                    xn = make_double2(fma(h, d.x, xv.x), fma(h, d.y, xv.y));
                } else {
                    // Newton: x~ = x~ + x~ (.) delta_N
                    const double2 d = cmul(xv, dN);
                    xn = make_double2(xv.x + d.x, xv.y + d.y);
                    sm.dn2[col][qq] = fma(d.x, d.x, d.y * d.y);
                }
                sm.xs[col][qq] = xn;
                if (fused_log && it + 1 < iters) { // stage 1 of the next evaluation, for this coordinate
                    double rho, th;
                    double2 iv;
                    int st = 0;
                    log_split_t(xn, rho, th, iv, st, S.logtab, S.atantab);
                    sm.rt[col][qq] = make_double2(rho, th);
                    if (st) atomicOr(&sm.st[qq], st);
                }
            }
        };
        if (A.solver == SOLVER_QR) {
            constexpr int NGQ = (PTS + 32 / (N + 2) - 1) / (32 / (N + 2));
            for (int g = warp; g < NGQ; g += G::NWARP) {
                int col, qq;
                double2 dE, dN;
                bool sing, act;
                qsolve<N>(sm, lane, g, col, dE, dN, sing, act, qq);
                if (act) apply(col, qq, dE, dN, sing);
            }
        } else {
            for (int g = warp; g < G::NGRP; g += G::NWARP) {
                int col, qq;
                double2 dE, dN;
                bool sing, act;
                lsolve<N>(sm, lane, warp, g, col, dE, dN, sing, act, qq);
                if (act) apply(col, qq, dE, dN, sing);
            }
        }
        __syncthreads();
        if (MODE == MODE_STEP && S.proj) { // points of P^n stay on ||y|| = 1 (reading R29)
            if (tid < PTS) proj_normalize<N>(sm.xs, tid);
            __syncthreads();
        }
    }

    if (MODE == MODE_DIRS) {
        if (tid < N * PTS) {
            const int qq = tid / N, j = tid % N;
            if (base + qq < A.P) {
                if (A.dE) A.dE[base * N + tid] = sm.inv[j][qq];
                if (A.dN) A.dN[base * N + tid] = sm.out2[j][qq];
            }
        }
        if (tid < PTS && base + tid < A.P && A.status) A.status[base + tid] = (uint8_t)sm.st[tid];
        return;
    }
    // MODE_STEP epilogue
    if (tid < N * PTS) {
        const int qq = tid / N;
        if (base + qq < A.P) A.xio[base * N + tid] = sm.xs[tid % N][qq];
    }
    if (tid < PTS && base + tid < A.P) {
        A.tauio[base + tid] = sm.tau[tid];
        if (A.status) A.status[base + tid] = (uint8_t)sm.st[tid];
        if (A.dnnorm) {
            double s2 = 0.0;
            for (int j = 0; j < N; ++j) s2 += sm.dn2[j][tid];
            A.dnnorm[base + tid] = A.K > 0 ? sqrt(s2) : 0.0;
        }
    }
}


// ---------------------------------------------------------------------------------------
#ifndef PHT_STEPW_PAIR
#define PHT_STEPW_PAIR(n) PHT_PAIR(n) // two terms per iteration in k_stepw's row loop
#endif
#ifndef PHT_STEPW_RTREG
#define PHT_STEPW_RTREG 0 // experiments: (rho, vartheta) in registers in k_stepw's row loop
#endif
// Warp-per-group Euler-Newton step (pht_pc_step, LU, affine).  One warp owns a
// group of PPW = 32/N points and keeps ONE lane mapping through every stage: lane (q, i) = (point
// q of the group, index i).  It loads x_i, runs stage 1 for variable i, evaluates ROW i of the
// point's extended Jacobian (stage 2-4, equation i) into registers, and that row is the row the
// lane holds in the Gauss-Jordan solve -- no shared-memory matrix tile, no staging of rows, no
// CTA barriers (warps of a CTA only share the exp/cis tables and the term records, loaded once:
// the kernel is persistent).  The records sit in shared memory term-major, R[t][k], so the lanes
// of one step of the term loop read neighbouring records.
template <int N>
struct GeoW {
    static constexpr int PPW = 32 / N; // points per warp
#ifndef PHT_STEPW_WARPS
#define PHT_STEPW_WARPS 4
#endif
#ifndef PHT_STEPW_MINB
#define PHT_STEPW_MINB 4
#endif
    static constexpr int WARPS = PHT_STEPW_WARPS;
    static constexpr int NT = WARPS * 32;
    static constexpr int RW = N + 2;
    static constexpr int KS = (N + 3) & ~3;
    static constexpr int MINB = PHT_STEPW_MINB; // tracker: 4 CTAs x 4 warps per SM at <= 128 registers
    // the step kernel: one 16-warp CTA per SM (+2.7% on cyclic-10 over 2 x 8: one copy of the tables
    // and records per SM); the tracker uses 4-warp CTAs, which spread few paths over more SMs
    // (katsura-10, 990 paths: 5.5 ms with 4-warp CTAs, 5.9 with 8, 7.5 with 16)
#ifndef PHT_STEPW_SWARPS
#define PHT_STEPW_SWARPS 16
#endif
    static constexpr int SWARPS = PHT_STEPW_SWARPS;
    static constexpr int SNT = SWARPS * 32;
    static constexpr int SMINB = 1;
};

template <int N>
struct SmemW {
    double exptab[TAB_E];
    double2 cistab[TAB_C];
    struct Warp {
        double2 rt[N][GeoW<N>::PPW];                // (rho, vartheta) of the group's points
        double2 xs[N][GeoW<N>::PPW];                // x of the group's points
        double2 prow[GeoW<N>::PPW][GeoW<N>::RW | 1]; // pivot-row buffer per point (odd stride)
        alignas(16) unsigned keys[GeoW<N>::PPW * GeoW<N>::KS];
        double dn2[N][GeoW<N>::PPW];
        double tau[GeoW<N>::PPW];
        double tinv[GeoW<N>::PPW];
        int st[GeoW<N>::PPW];
    } w[GeoW<N>::SWARPS];
    int mk[N]; // terms per equation
    // followed by the records R[MT][N][rec_stride(N) / 2] (double2)
};

// Term records of the warp-per-group kernels in shared memory.  PHT_W_REC16 = 1: compact records
// of 3 x 16 B per term (n <= 12): the exponents as int16 (exact: |a| <= PHT_MAX_EXP = 1024) in the
// first 24 bytes, then omega, log|c|, arg c as doubles; a term costs 3 LDS.128 instead of
// rec_stride(n) / 2 (7 at n = 10) and each exponent one I2F.F64.S16.  0: the packer's double records.
// Measured (cyclic-10 step, ncu): shared-memory wavefronts -18%, time -0.6% (the step kernel is
// latency-bound at 16 warps per SM, not shared-pipe-bound); noon-10 tracking 34.4 -> 32.7 ms.
#ifndef PHT_W_REC16
#define PHT_W_REC16 1
#endif
template <int N, bool WIDE = false>
struct RecW {
    // compact layout (the kernels run for n <= 12); WIDE: the packer's doubles.  The point-per-lane
    // evaluation k_evalw reads every record as a warp broadcast (one address per LDS.128, 2 cycles),
    // so the 7 wide loads cost less than 3 compact loads + N int16 -> double conversions on the FP64
    // pipe per lane (measured cyclic-10 1.11 -> 1.18, noon-10 1.02 -> 1.09 G points/s); the lane-per-
    // row kernels read N different records per load, where the compact records win
    static constexpr bool C16 = !WIDE && PHT_W_REC16 && N <= 12;
    static constexpr int U = C16 ? 3 : rec_stride(N) / 2;  // 16-byte units per term
};

// one record, packer layout (rec_stride(N) doubles from global memory) -> shared-memory layout
template <int N, bool WIDE = false>
__device__ __forceinline__ void pack_rec_w(const double2 *src, double2 *dst)
{
    if (RecW<N, WIDE>::C16) {
        unsigned e[6] = {0u, 0u, 0u, 0u, 0u, 0u};
        for (int j = 0; j < N && j < 12; ++j) {
            const double2 v = __ldg(src + j / 2);
            const int a = (int)((j & 1) ? v.y : v.x);
            e[j >> 1] |= ((unsigned)a & 0xffffu) << (16 * (j & 1));
        }
        const double w = ((N & 1) ? __ldg(src + N / 2).y : __ldg(src + N / 2).x);
        const double lc = ((N + 1) & 1) ? __ldg(src + (N + 1) / 2).y : __ldg(src + (N + 1) / 2).x;
        const double ac = ((N + 2) & 1) ? __ldg(src + (N + 2) / 2).y : __ldg(src + (N + 2) / 2).x;
        uint4 *d = reinterpret_cast<uint4 *>(dst);
        d[0] = make_uint4(e[0], e[1], e[2], e[3]);
        d[1] = make_uint4(e[4], e[5], (unsigned)__double2loint(w), (unsigned)__double2hiint(w));
        d[2] = make_uint4((unsigned)__double2loint(lc), (unsigned)__double2hiint(lc), (unsigned)__double2loint(ac),
                          (unsigned)__double2hiint(ac));
    } else {
        for (int u = 0; u < rec_stride(N) / 2; ++u) dst[u] = __ldg(src + u);
    }
}

// compact record (3 x 16 B, RecW<N>::C16) -> doubles
template <int N>
__device__ __forceinline__ void unpack_rec16(const uint4 &u0, const uint4 &u1, const uint4 &u2, double (&a)[rec_stride(N)])
{
    const unsigned e[6] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y};
#pragma unroll
    for (int j = 0; j < N && j < 12; ++j) a[j] = (double)(short)(e[j >> 1] >> (16 * (j & 1))); // I2F.F64.S16
    a[N] = __hiloint2double((int)u1.w, (int)u1.z);
    a[N + 1] = __hiloint2double((int)u2.y, (int)u2.x);
    a[N + 2] = __hiloint2double((int)u2.w, (int)u2.z);
}

template <int N, bool WIDE = false>
__device__ __forceinline__ void load_rec_s(const double2 *r, double (&a)[rec_stride(N)])
{
    if (RecW<N, WIDE>::C16) {
        const uint4 *u = reinterpret_cast<const uint4 *>(r);
        unpack_rec16<N>(u[0], u[1], u[2], a);
    } else {
#pragma unroll
        for (int u = 0; u < rec_stride(N) / 2; ++u) {
            const double2 v = r[u];
            a[2 * u] = v.x;
            a[2 * u + 1] = v.y;
        }
    }
}

// stages 2-4 for row k of group point q (records from shared memory, term-major)
template <int N>
__device__ __forceinline__ void eval_row_w(const SmemW<N> &sm, const double2 *R, const typename SmemW<N>::Warp &W,
                                           int k, int q, double2 (&row)[N + 2], int &e)
{
    constexpr int RS = rec_stride(N), PPW = GeoW<N>::PPW;
#if PHT_STEPW_RTREG
    PointLog<N, false> pl; // (rho, vartheta) of the point in registers for the whole row
    pl.template load<PPW>(W.rt, q);
#else
    PointLog<N, true> pl;
    pl.base = &W.rt[0][q];
    pl.stride = PPW;
#endif
    const double tau = W.tau[q];
    const int m = sm.mk[k];
    const double2 *rec = R + (size_t)k * RecW<N>::U;
    constexpr size_t TS = (size_t)N * RecW<N>::U; // record stride between terms of one equation
    RowAcc<N> acc;
    {
        double a[RS];
        load_rec_s<N>(rec, a);
        acc.init(phi_of<N>(a, pl, tau));
    }
    int i = 0;
    for (; PHT_STEPW_PAIR(N) && i + 1 < m; i += 2) {
        double a[RS], b[RS];
        load_rec_s<N>(rec + (size_t)i * TS, a);
        load_rec_s<N>(rec + (size_t)(i + 1) * TS, b);
        double pa, pb, ta, tb;
        phi_theta<N>(a, pl, tau, pa, ta);
        phi_theta<N>(b, pl, tau, pb, tb);
        acc.reduce(pa);
        acc.reduce(pb);
        const double ya = acc.reduced(pa), yb = acc.reduced(pb);
        const double2 wa = expcis(ya, ta, sm.exptab, sm.cistab);
        const double2 wb = expcis(yb, tb, sm.exptab, sm.cistab);
        acc.add(a, wa);
        acc.add(b, wb);
    }
#pragma unroll kStepwUnroll
    for (; i < m; ++i) {
        double a[RS];
        load_rec_s<N>(rec + (size_t)i * TS, a);
        double pa, ta;
        phi_theta<N>(a, pl, tau, pa, ta);
        const double ya = acc.reduce(pa);
        acc.add(a, expcis(ya, ta, sm.exptab, sm.cistab));
    }
#pragma unroll
    for (int j = 0; j < N; ++j) row[j] = acc.g[j];
    row[N] = acc.gt;
    row[N + 1] = acc.h;
    e = (int)acc.ed;
}

// MODE_STEP: the Euler-Newton step in place; MODE_DIRS: the directions dE = dx/dt, dN at (x, t)
// (pht_euler_newton) -- one evaluation and solve, dE and dN staged in the x and (rho, vartheta)
// tiles (each lane overwrites only its own variable col, which no other lane reads any more).
template <int N, int MODE>
__global__ void __launch_bounds__(GeoW<N>::SNT, GeoW<N>::SMINB) k_stepw(const DevSys S, const Args A, int MT)
{
    static_assert(MODE == MODE_DIRS || MODE == MODE_STEP || MODE == MODE_EVAL_X, "k_stepw: modes");
    constexpr bool DIRS = MODE == MODE_DIRS, EVAL = MODE == MODE_EVAL_X;
    using G = GeoW<N>;
    constexpr int RS = rec_stride(N), PPW = G::PPW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemW<N> &sm = *reinterpret_cast<SmemW<N> *>(smem_raw);
    double2 *R = reinterpret_cast<double2 *>(smem_raw + ((sizeof(SmemW<N>) + 15) & ~(size_t)15));
    const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    load_tables(S, sm.exptab, sm.cistab, tid, G::SNT);
    for (int idx = tid; idx < MT * N; idx += G::SNT) { // records, term-major (only t < m_k is read)
        const int kk = idx % N, t = idx / N;
        const int i0 = __ldg(S.off + kk), m = __ldg(S.off + kk + 1) - i0;
        if (t < m) pack_rec_w<N>(S.rec + (size_t)(i0 + t) * (RS / 2), R + (size_t)idx * RecW<N>::U);
    }
    if (tid < N) sm.mk[tid] = __ldg(S.off + tid + 1) - __ldg(S.off + tid);
    __syncthreads();
    typename SmemW<N>::Warp &W = sm.w[wi];
    // lane = i * PPW + q (index-major): the PPW lanes of one index read the same term record
    // (a broadcast), so a record load touches N distinct 16-byte chunks, not N per point
    const bool inseg = lane < N * PPW;
    const int q = inseg ? lane % PPW : 0, i = inseg ? lane / PPW : 0; // point of the group, index
    const int seg0 = inseg ? q : PPW;                                 // segment (PPW: no point)
    const int64_t groups = (A.P + PPW - 1) / PPW;
    for (int64_t grp = (int64_t)blockIdx.x * G::SWARPS + wi; grp < groups; grp += (int64_t)gridDim.x * G::SWARPS) {
        const int64_t base = grp * PPW, gp = base + q;
        const bool act = inseg && gp < A.P;
        double2 xv = make_double2(1.0, 0.0); // lanes of points past P carry a harmless dummy
        if (act) xv = (DIRS || EVAL) ? A.xin[gp * N + i] : A.xio[gp * N + i];
        if (lane < PPW) {
            int st = 0;
            if (DIRS || EVAL) { // t > 0 in, tau = log t
                double tv = (base + lane < A.P) ? A.tin[base + lane] : 1.0;
                if (!(tv > 0.0) || !isfinite(tv)) { st = PT_NONFINITE; tv = 1.0; }
                W.tau[lane] = log(tv);
                W.tinv[lane] = 1.0 / tv;
            } else {
                double tv = (base + lane < A.P) ? A.tauio[base + lane] : 0.0;
                if (!isfinite(tv)) { st = PT_NONFINITE; tv = 0.0; }
                W.tau[lane] = tv;
            }
            W.st[lane] = st;
        }
        __syncwarp();
        {
            double rho, th;
            double2 iv;
            int st = 0;
            log_split_t(xv, rho, th, iv, st, S.logtab, S.atantab); // a1 for variable i
            if (inseg) {
                W.rt[i][q] = make_double2(rho, th);
                W.xs[i][q] = EVAL ? iv : xv; // evaluation: 1/x_i for the diag(1/x) epilogue
                W.dn2[i][q] = 0.0;
            }
            if (st && act) atomicOr(&W.st[q], st);
        }
        __syncwarp();
        const int iters = DIRS ? 1 : A.K + 1;
        for (int it = 0; it < iters; ++it) {
            double2 a[N + 2];
            int e;
            eval_row_w<N>(sm, R, W, i, q, a, e); // row i of point q: [dh_i/dz | dh_i/dtau | h_i] 2^-e
            if (EVAL) { // pht_evaluate: Jx_ij = G_ij / x_j, Jt = G_tau / t, H = h, row i
                const double ti = W.tinv[q];
                a[N] = make_double2(a[N].x * ti, a[N].y * ti);
#pragma unroll
                for (int j = 0; j < N; ++j) a[j] = cmul(a[j], W.xs[j][q]);
                const bool scaled = A.rexp != nullptr;
                if (!scaled) scale_row2<N + 2>(a, e);
                bool fin = true;
#pragma unroll
                for (int c = 0; c < N + 2; ++c) fin = fin && isfinite(a[c].x) && isfinite(a[c].y);
                if (act) {
                    if (!fin) atomicOr(&W.st[q], PT_NONFINITE);
                    const int64_t r = gp * N + i;
                    if (A.J) {
#pragma unroll
                        for (int j = 0; j < N; ++j) A.J[r * N + j] = a[j];
                    }
                    if (A.Jt) A.Jt[r] = a[N];
                    if (A.H) A.H[r] = a[N + 1];
                    if (scaled) A.rexp[r] = e;
                }
                break;
            }
            normalize_row<N>(a);
            __syncwarp(); // every lane has read tau and (rho, vartheta)
            if (!DIRS && it == 0 && lane < PPW && base + lane < A.P) W.tau[lane] += A.dtau[base + lane];
            int col;
            double2 dE, dN;
            bool sing;
            lsolve_regs<N, PPW, G::KS, true>(a, &W.prow[q][0], &W.keys[q * G::KS], seg0, q, i, act, col, dE, dN, sing);
            if (act && DIRS) { // dx/dt = x (.) delta_E / t, dN_x = x (.) delta_N (Jx = G diag(1/x))
                if (sing) atomicOr(&W.st[q], PT_SINGULAR);
                const double2 xo = W.xs[col][q];
                const double2 de = cmul(xo, dE), dn = cmul(xo, dN);
                const double ti = W.tinv[q];
                W.xs[col][q] = make_double2(de.x * ti, de.y * ti);
                W.rt[col][q] = dn;
            } else if (act) { // the lane whose row pivoted column col updates variable col
                if (sing) atomicOr(&W.st[q], PT_SINGULAR);
                const double2 xo = W.xs[col][q];
                double2 xn;
                if (it == 0) { // Euler: x~ = x + h x (.) delta_E
                    const double h = A.dtau[gp];
                    const double2 d = cmul(xo, dE);
                    xn = make_double2(fma(h, d.x, xo.x), fma(h, d.y, xo.y));
                } else {       // Newton: x~ = x~ + x~ (.) delta_N
                    const double2 d = cmul(xo, dN);
                    xn = make_double2(xo.x + d.x, xo.y + d.y);
                    W.dn2[col][q] = fma(d.x, d.x, d.y * d.y);
                }
                W.xs[col][q] = xn;
                if (it < A.K) { // stage 1 of the next evaluation, for this coordinate
                    double rho, th;
                    double2 iv;
                    int st = 0;
                    log_split_t(xn, rho, th, iv, st, S.logtab, S.atantab);
                    W.rt[col][q] = make_double2(rho, th);
                    if (st) atomicOr(&W.st[q], st);
                }
            }
            __syncwarp();
        }
        if (EVAL) {
            __syncwarp();
            if (lane < PPW && base + lane < A.P && A.status) A.status[base + lane] = (uint8_t)W.st[lane];
            __syncwarp();
            continue;
        }
        if (DIRS) {
            if (act && A.dE) A.dE[gp * N + i] = W.xs[i][q];
            if (act && A.dN) A.dN[gp * N + i] = W.rt[i][q];
            if (lane < PPW && base + lane < A.P && A.status) A.status[base + lane] = (uint8_t)W.st[lane];
            __syncwarp();
            continue;
        }
        if (act) A.xio[gp * N + i] = W.xs[i][q];
        if (lane < PPW && base + lane < A.P) {
            A.tauio[base + lane] = W.tau[lane];
            if (A.status) A.status[base + lane] = (uint8_t)W.st[lane];
            if (A.dnnorm) {
                double s2 = 0.0;
                for (int j = 0; j < N; ++j) s2 += W.dn2[j][lane];
                A.dnnorm[base + lane] = A.K > 0 ? sqrt(s2) : 0.0;
            }
        }
        __syncwarp();
    }
}

#ifdef PHT_JIT
// ---------------------------------------------------------------------------------------
// Specialised evaluation, one point per thread (pht_evaluate / pht_evaluate_log after
// pht_system_specialize).  No solve follows, so no per-point matrix tile is needed: each thread
// runs stage 1 for its point, then the generated rows of all equations in sequence and writes
// every row straight out.  All warps walk the same equation stream (instruction-cache
// friendly, unlike the warp-per-equation layout the fused kernels need).
#ifndef PHT_EVALP_T
#define PHT_EVALP_T 128
#endif
template <int N>
struct SmemE {
    double exptab[TAB_E];
    double2 cistab[TAB_C];
    double2 rt[N][PHT_EVALP_T + 1];  // (rho, vartheta) columns, one per thread
    double2 inv[N][PHT_EVALP_T + 1]; // 1/x (EVAL_X epilogue): off the registers live across the rows
};

template <int N, int MODE>
__global__ void __launch_bounds__(PHT_EVALP_T, 4) k_evalp(const DevSys S, const Args A)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemE<N> &sm = *reinterpret_cast<SmemE<N> *>(smem_raw);
    const int tid = threadIdx.x;
    load_tables(S, sm.exptab, sm.cistab, tid, PHT_EVALP_T);
    const int64_t q = (int64_t)blockIdx.x * PHT_EVALP_T + tid;
    const bool live = q < A.P;
    int st = 0;
    double tau = 0.0, tinv = 1.0;
    {
        double tv = live ? A.tin[q] : (MODE == MODE_EVAL_Z ? 0.0 : 1.0);
        if (MODE == MODE_EVAL_Z) {
            if (!isfinite(tv)) { st |= PT_NONFINITE; tv = 0.0; }
            tau = tv;
        } else {
            if (!(tv > 0.0) || !isfinite(tv)) { st |= PT_NONFINITE; tv = 1.0; }
            tau = log(tv);
            tinv = 1.0 / tv;
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double2 v = live ? A.xin[q * N + j] : make_double2(MODE == MODE_EVAL_Z ? 0.0 : 1.0, 0.0);
            double rho, th;
            if (MODE == MODE_EVAL_Z) {
                if (!(isfinite(v.x) && isfinite(v.y))) { st |= PT_NONFINITE; rho = 0.0; th = 0.0; }
                else {
                    rho = v.x;
                    const double kq = rint(v.y * INV_2PI);
                    th = fma(-kq, TWO_PI_LO, fma(-kq, TWO_PI_HI, v.y));
                }
            } else {
                double2 iv;
                log_split_t(v, rho, th, iv, st, S.logtab, S.atantab);
                sm.inv[j][tid] = iv;
            }
            sm.rt[j][tid] = make_double2(rho, th);
        }
    }
    __syncthreads(); // the tables (each rt column is private to its thread)
    const bool scaled = A.rexp != nullptr;
    for (int k = 0; k < N; ++k) {
        double2 row[N + 2];
        int e = 0;
        if (S.proj && k == N - 1) { // bordering row y^* (see eval_row)
#pragma unroll
            for (int j = 0; j < N; ++j) row[j] = make_double2(exp(2.0 * sm.rt[j][tid].x), 0.0);
            row[N] = make_double2(0.0, 0.0);
            row[N + 1] = make_double2(0.0, 0.0);
        } else {
            jit_row_core<N>(k, &sm.rt[0][tid], PHT_EVALP_T + 1, tau, sm.exptab, sm.cistab, row, e, nullptr);
        }
        if (MODE == MODE_EVAL_X) {
            row[N] = make_double2(row[N].x * tinv, row[N].y * tinv);
#pragma unroll
            for (int j = 0; j < N; ++j) row[j] = cmul(row[j], sm.inv[j][tid]);
        }
        if (!scaled) scale_row2<N + 2>(row, e);
        bool fin = true;
#pragma unroll
        for (int c = 0; c < N + 2; ++c) fin = fin && isfinite(row[c].x) && isfinite(row[c].y);
        if (!fin) st |= PT_NONFINITE;
        if (live) {
            if (A.J) {
#pragma unroll
                for (int j = 0; j < N; ++j) A.J[(q * N + k) * N + j] = row[j];
            }
            if (A.Jt) A.Jt[q * N + k] = row[N];
            if (A.H) A.H[q * N + k] = row[N + 1];
            if (scaled) A.rexp[q * N + k] = e;
        }
    }
    if (live && A.status) A.status[q] = (uint8_t)st;
}
#endif

// ---------------------------------------------------------------------------------------
// a6: persistent device tracker (SURVEY §8(a) a6, step control = DESIGN.md reading R14).
// Every CTA slot runs one path as a state machine; every loop iteration performs one
// evaluation + two-RHS solve for all slots at their current query point:
//   PREDICT  query (x, tau):    x~ = x + h dx/dtau, tau~ = tau + h, h = min(dtau, -tau)
//   CORRECT  query (x~, tau~):  x~ += dN; converged -> accept, contraction/K exhausted -> reject
//   FINAL    query (x, 0):      x += dN until ||dN|| <= final_tol ||x|| (<= final_iters)
// Finished slots write their path back and take the next index from a global atomic queue.
enum : int { PH_IDLE = 0, PH_PREDICT = 1, PH_CORRECT = 2, PH_FINAL = 3 };

template <int N>
struct TrackSmem {
    Smem<N> s;
    double2 xa[N][Geo<N>::WL + 1];   // accepted point (padded rows: see Smem)
    double2 xt[N][Geo<N>::WL + 1];   // trial point
    double2 dd[N][Geo<N>::WL + 1];   // direction of this iteration (delta_E or delta_N, log coords)
    double2 zp[N][Geo<N>::WL + 1];   // Hermite predictor: previous accepted point (log chart) ...
    double2 ep[N][Geo<N>::WL + 1];   // ... and its Euler direction dz/dtau
    double2 ec[N][Geo<N>::WL + 1];   // Euler direction at the current accepted point
    double2 ecn[N][Geo<N>::WL + 1];  // reuse_tangent: Euler direction at the latest corrector iterate
    double nd2[N][Geo<N>::WL + 1];   // |dx_j / x_j|^2 of this iteration
    double tau_a[Geo<N>::WL], tau_t[Geo<N>::WL], dt[Geo<N>::WL], prev[Geo<N>::WL], nd1[Geo<N>::WL], tau_p[Geo<N>::WL];
    int has_prev[Geo<N>::WL];
    int tok[Geo<N>::WL];    // the Euler direction of the accepted point is in ec (its evaluation succeeded)
    int repred[Geo<N>::WL]; // next iteration: form the trial point from ec without an evaluation
    long long path[Geo<N>::WL], steps[Geo<N>::WL], rej[Geo<N>::WL], evals[Geo<N>::WL], fin[Geo<N>::WL];
    int phase[Geo<N>::WL], it[Geo<N>::WL], succ[Geo<N>::WL], cell[Geo<N>::WL];
    int acc[Geo<N>::WL];         // this iteration: 1 accept x~ -> x
    long long done_path[Geo<N>::WL]; // path finished this iteration (-1 none)
    int refill[Geo<N>::WL];      // 1: load a new path into the slot
    int active;
};

template <int N, class TT>
__device__ __forceinline__ void trk_pop(TT &T, const TrackArgs &A, int q)
{
    unsigned long long idx = atomicAdd(A.queue, 1ull);
    while ((long long)idx < A.P && !isfinite(A.tau[idx])) { // unusable start: report and skip
        A.status[idx] = (uint8_t)PT_NONFINITE;
        if (A.stats)
            for (int u = 0; u < 4; ++u) A.stats[4 * idx + u] = 0;
        idx = atomicAdd(A.queue, 1ull);
    }
    while ((long long)idx < A.P && A.cellw &&
           (A.path_cell[idx] < 0 || A.path_cell[idx] >= A.ncells)) { // bad cell id: report and skip
        A.status[idx] = (uint8_t)PT_NONFINITE;
        if (A.stats)
            for (int u = 0; u < 4; ++u) A.stats[4 * idx + u] = 0;
        idx = atomicAdd(A.queue, 1ull);
    }
    if ((long long)idx < A.P) {
        T.path[q] = (long long)idx;
        T.cell[q] = A.cellw ? A.path_cell[idx] : 0;
        T.refill[q] = 1;
        const double t0 = A.tau[idx];
        T.tau_a[q] = t0;
        T.dt[q] = A.o.dtau_init;
        T.steps[q] = T.rej[q] = T.evals[q] = T.fin[q] = 0;
        T.succ[q] = 0;
        T.it[q] = 0;
        T.has_prev[q] = 0;
        T.tok[q] = 0;
        T.repred[q] = 0;
        T.phase[q] = (t0 < 0.0) ? PH_PREDICT : PH_FINAL;
    } else {
        T.path[q] = -1;
        T.refill[q] = 0;
        T.phase[q] = PH_IDLE;
    }
}

template <int N, class TT>
__device__ __forceinline__ void trk_finish(TT &T, const TrackArgs &A, int q, int status)
{
    const long long pth = T.path[q];
    A.status[pth] = (uint8_t)status;
    A.tau[pth] = T.tau_a[q];
    if (A.stats) {
        A.stats[4 * pth + 0] = T.steps[q];
        A.stats[4 * pth + 1] = T.rej[q];
        A.stats[4 * pth + 2] = T.evals[q];
        A.stats[4 * pth + 3] = T.fin[q];
    }
    T.done_path[q] = pth;
}

// z <- z + log(1 + u): the affine update x <- x (1 + u) in logarithmic coordinates
__device__ __forceinline__ double2 zlog1p_add(double2 z, double2 u)
{
    const double re = 0.5 * log1p(fma(u.x, 2.0 + u.x, u.y * u.y));
    const double im = atan2(u.y, 1.0 + u.x);
    return make_double2(z.x + re, z.y + im);
}
// the same with the table-driven log / atan2 (log_split_t): log|1 + u|^2 = log(s_hi) + log1p(s_lo /
// s_hi) with s_hi + s_lo = 1 + v exactly (Fast2Sum, v = 2 Re u + |u|^2 > -1, |v| <= 1 taken here),
// the second term to first order (|s_lo / s_hi| <= u); libdevice outside 1/4 < |1 + u| < 4 or for
// non-finite u
__device__ __forceinline__ double2 zlog1p_add_t(double2 z, double2 u, const double2 *logtab, const double *atantab)
{
    const double v = fma(u.x, 2.0 + u.x, u.y * u.y);
    const double wx = 1.0 + u.x, m = fmax(fabs(wx), fabs(u.y));
    if (!(fabs(v) <= 1.0 && m > 0.25 && m < 4.0)) return zlog1p_add(z, u);
    const double sh = 1.0 + v, sl = (1.0 - sh) + v;
    const double re = 0.5 * fma(sl, rcp_nr(sh), log_t(sh, logtab));
    const double im = atan2_t(u.y, wx, m, atantab);
    return make_double2(z.x + re, z.y + im);
}

// Euler predictor in the log chart: z + h delta (log state) or x exp(h delta) (x state)
template <bool LOGS>
__device__ __forceinline__ double2 trk_predict_log(double2 v, double2 delta, double h)
{
    if (LOGS) return make_double2(fma(h, delta.x, v.x), fma(h, delta.y, v.y));
    double sn, cs;
    sincos(h * delta.y, &sn, &cs);
    const double m = exp(h * delta.x);
    return cmul(v, make_double2(m * cs, m * sn));
}

template <int N, bool LOGS>
__device__ __forceinline__ double2 trk_update(double2 v, double2 delta, double h, const DevSys &S)
{
    if (LOGS) return zlog1p_add_t(v, make_double2(h * delta.x, h * delta.y), S.logtab, S.atantab);
    const double2 d = cmul(v, delta);
    return make_double2(fma(h, d.x, v.x), fma(h, d.y, v.y));
}

// (4) of the tracker: the per-slot decisions of one iteration (the oracle's control flow, oracle.c
// orc_track); T: the tile tracker's TrackSmem or the warp tracker's per-warp state (same fields).
template <int N, bool LOGS, class TT>
__device__ __forceinline__ void trk_decide(TT &T, const TrackArgs &A, const DevSys &S, int qq, int bad)
{
    const TrackOpts &o = A.o;
    const int ph = T.phase[qq];
    T.evals[qq] += 1;
    int finish = -1; // status when the path ends this iteration
    bool reject = false;
    if (ph == PH_PREDICT) {
        if (bad) reject = true;
        else {
            T.tau_t[qq] = T.tau_a[qq] + fmin(T.dt[qq], -T.tau_a[qq]);
            T.phase[qq] = PH_CORRECT;
            T.it[qq] = 1;
            T.prev[qq] = INFINITY;
            T.tok[qq] = 1; // this evaluation's Euler direction (at the accepted point) is in ec
        }
    } else if (ph == PH_CORRECT) {
        if (bad) reject = true;
        else {
            double nd = 0.0; // max_j |dx_j| / |x_j| (componentwise relative, reading R14)
            for (int j = 0; j < N; ++j) nd = S.proj ? nd + T.nd2[j][qq] : fmax(nd, T.nd2[j][qq]);
            nd = sqrt(nd);      // projective: ||dy|| (||y|| = 1, reading R29)
            if (T.it[qq] == 1) T.nd1[qq] = nd;
            // converged: the update, or the update times the observed contraction (the
            // quadratic-convergence estimate of the remaining error), <= newton_tol (R14)
            if (nd <= o.newton_tol || (T.it[qq] >= 2 && nd * (nd / T.prev[qq]) <= o.newton_tol)) {
                T.acc[qq] = 1;
                T.tok[qq] = 0; // the accepted point moves: its Euler direction is not known yet
                T.tau_p[qq] = T.tau_a[qq];
                T.has_prev[qq] = 1;
                T.tau_a[qq] = T.tau_t[qq];
                T.steps[qq] += 1;
                if (o.pred_tol > 0.0) { // next step from the Euler predictor's error, O(dtau^2)
                    const double e1 = T.nd1[qq];
                    const double f = (e1 > 0.0) ? fmin(fmax(sqrt(o.pred_tol / e1), o.shrink), o.grow) : o.grow;
                    T.dt[qq] = fmin(f * T.dt[qq], o.dtau_max);
                } else if (++T.succ[qq] == o.grow_after) {
                    T.dt[qq] = fmin(o.grow * T.dt[qq], o.dtau_max);
                    T.succ[qq] = 0;
                }
                T.phase[qq] = (T.tau_a[qq] < 0.0) ? PH_PREDICT : PH_FINAL;
                if (T.phase[qq] == PH_PREDICT && T.steps[qq] == o.max_steps) finish = 16; // MAX_STEPS
                else if (T.phase[qq] == PH_PREDICT && o.reuse_tangent && o.predictor != 1 && !S.proj) {
                    // reuse_tangent: the consolidated solve of the last corrector iteration gave the
                    // Euler direction at that iterate; it predicts the next step
                    T.tok[qq] = 1;
                    T.tau_t[qq] = T.tau_a[qq] + fmin(T.dt[qq], -T.tau_a[qq]);
                    T.phase[qq] = PH_CORRECT;
                    T.it[qq] = 1;
                    T.prev[qq] = INFINITY;
                    T.repred[qq] = 2;
                }
            } else if ((T.it[qq] >= 2 && nd > 0.5 * T.prev[qq]) || T.it[qq] >= o.K) {
                reject = true;
            } else {
                T.prev[qq] = nd;
                T.it[qq] += 1;
            }
        }
    } else { // FINAL
        T.fin[qq] += 1;
        if (bad) finish = 32;
        else {
            double nd = 0.0, xinf = 0.0; // xinf: max |x_j| (or max Re z_j in log state)
            for (int j = 0; j < N; ++j) {
                nd = S.proj ? nd + T.nd2[j][qq] : fmax(nd, T.nd2[j][qq]);
                const double2 v = T.xa[j][qq];
                xinf = fmax(xinf, LOGS ? v.x : sqrt(fma(v.x, v.x, v.y * v.y)));
            }
            const double2 yn = T.xa[N - 1][qq]; // projective: finite iff |y_n| >= 1 / inf_norm
            const bool finite = S.proj ? (sqrt(fma(yn.x, yn.x, yn.y * yn.y)) * o.inf_norm >= 1.0)
                                       : (LOGS ? (xinf <= log(o.inf_norm)) : (xinf <= o.inf_norm));
            if (sqrt(nd) <= o.final_tol) finish = finite ? 0 : 32;
            else if (T.fin[qq] >= o.final_iters) // not refined to final_tol (ledger A24): DIVERGED,
                // or FLOOR when the corrections reached newton_tol -- a finite endpoint at the log/exp
                // evaluation's accuracy floor (reading R30), reported apart from OK
                finish = (sqrt(nd) <= o.newton_tol && finite) ? PT_FLOOR : 32;
        }
    }
    if (reject) {
        T.rej[qq] += 1;
        T.dt[qq] *= o.shrink;
        T.succ[qq] = 0;
        if (T.dt[qq] < o.dtau_min) finish = (bad & PT_SINGULAR) ? PT_SINGULAR : 8; // STEP_UNDERFLOW
        else {
            T.phase[qq] = PH_PREDICT;
            if (T.steps[qq] == o.max_steps) finish = 16;
            else if (ph == PH_CORRECT && T.tok[qq] && o.predictor != 1 && !S.proj) {
                // re-prediction from the same accepted point: its Euler direction is the cached one
                // (bitwise the evaluation the PREDICT phase would repeat), so the trial point is
                // formed without an evaluation and the next evaluation is the first correction
                T.tau_t[qq] = T.tau_a[qq] + fmin(T.dt[qq], -T.tau_a[qq]);
                T.phase[qq] = PH_CORRECT;
                T.it[qq] = 1;
                T.prev[qq] = INFINITY;
                T.repred[qq] = 1;
            }
        }
    }
    if (finish >= 0) {
        trk_finish<N>(T, A, qq, finish);
        trk_pop<N>(T, A, qq);
    }
}

template <int N, bool LOGS>
__global__ void __launch_bounds__(Geo<N>::NT, Geo<N>::MINB) k_track(const DevSys S, const TrackArgs A)
{
    using G = Geo<N>;
    constexpr int PTS = G::PTS, WL = G::WL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrackSmem<N> &T = *reinterpret_cast<TrackSmem<N> *>(smem_raw);
    Smem<N> &sm = T.s;
    const int tid = threadIdx.x;
    const int k = tid / WL, q = tid % WL;
    const int lane = tid & 31, warp = tid >> 5;
    const TrackOpts &o = A.o;
    load_tables(S, sm.exptab, sm.cistab, tid, G::NT);
    if (tid < WL) {
        T.done_path[tid] = -1;
        T.cell[tid] = 0;
        if (tid < PTS) trk_pop<N>(T, A, tid);
        else { T.path[tid] = -1; T.refill[tid] = 0; T.phase[tid] = PH_IDLE; }
        T.acc[tid] = 0;
    }
    __syncthreads();
    for (;;) {
        // (1) write back finished paths, accept trial points, load new paths, select the query
        if (tid < N * PTS) {
            const int qq = tid / N, j = tid % N;
            if (T.acc[qq]) {
                if (o.predictor == 1) { // Hermite history: the point being replaced and its direction
                    T.zp[j][qq] = T.xa[j][qq];
                    T.ep[j][qq] = T.ec[j][qq];
                }
                T.xa[j][qq] = T.xt[j][qq];
            }
            if (T.done_path[qq] >= 0) A.x[T.done_path[qq] * N + j] = T.xa[j][qq];
            if (T.refill[qq]) T.xa[j][qq] = A.x[T.path[qq] * N + j];
            if (T.repred[qq]) { // re-prediction from the cached Euler direction (trk_decide)
                if (T.repred[qq] == 2) T.ec[j][qq] = T.ecn[j][qq]; // reuse_tangent: the iterate's
                const double h = fmin(T.dt[qq], -T.tau_a[qq]);
                T.xt[j][qq] = o.pred_log ? trk_predict_log<LOGS>(T.xa[j][qq], T.ec[j][qq], h)
                                         : trk_update<N, LOGS>(T.xa[j][qq], T.ec[j][qq], h, S);
            }
            const int ph = T.phase[qq];
            sm.xs[j][qq] = (ph == PH_CORRECT) ? T.xt[j][qq]
                                              : (ph == PH_IDLE ? make_double2(LOGS ? 0.0 : 1.0, 0.0) : T.xa[j][qq]);
        }
        __syncthreads();
        if (tid < WL) {
            if (S.proj && tid < PTS && T.refill[tid]) { // new projective path: onto ||y|| = 1
                proj_normalize<N>(T.xa, tid);
                for (int j = 0; j < N; ++j) sm.xs[j][tid] = T.xa[j][tid];
            }
            T.done_path[tid] = -1;
            T.acc[tid] = 0;
            T.refill[tid] = 0;
            if (tid < PTS) T.repred[tid] = 0;
            sm.st[tid] = 0;
            const int ph = (tid < PTS) ? T.phase[tid] : PH_IDLE;
            sm.tau[tid] = (ph == PH_CORRECT) ? T.tau_t[tid] : ((ph == PH_PREDICT) ? T.tau_a[tid] : 0.0);
            if (tid >= PTS)
                for (int j = 0; j < N; ++j) sm.xs[j][tid] = make_double2(LOGS ? 0.0 : 1.0, 0.0);
        }
        if (tid == 0) T.active = 0;
        __syncthreads();
        // (2) evaluation + solve at the query points (same code as pht_pc_step / evaluate_log)
        stage1<N, LOGS ? MODE_EVAL_Z : MODE_STEP>(sm, tid);
        if (tid < WL && tid >= PTS)
            for (int j = 0; j < N; ++j) sm.rt[j][tid] = make_double2(0.0, 0.0);
        // any slot in the final refinement: the compensated stage 2 (R30) for the rows of those
        // slots only (per point: a path's arithmetic never depends on the other slots' phases)
        const int comp = __syncthreads_or(tid < PTS && T.phase[tid] == PH_FINAL);
        if (k < N) {
            double2 row[N + 2];
            int e;
            const double *wq = A.cellw ? A.cellw + (size_t)T.cell[q] * A.M : nullptr;
#ifdef PHT_JIT
            eval_row<N>(S, sm, k, q, row, e, wq); // generated rows: no compensated variant (FLOOR possible)
            (void)comp;
#else
            if (comp && q < PTS && T.phase[q] == PH_FINAL) eval_row<N, true>(S, sm, k, q, row, e, wq);
            else eval_row<N>(S, sm, k, q, row, e, wq);
#endif
            if (q < PTS) store_row<N>(sm, k, q, row);
        }
        __syncthreads();
        if (A.solver == SOLVER_QR) {
            constexpr int NGQ = (PTS + 32 / (N + 2) - 1) / (32 / (N + 2));
            for (int g = warp; g < NGQ; g += G::NWARP) {
                int col, qq;
                double2 dE, dN;
                bool sing, act;
                qsolve<N>(sm, lane, g, col, dE, dN, sing, act, qq);
                if (act) {
                    if (sing) atomicOr(&sm.st[qq], PT_SINGULAR);
                    T.dd[col][qq] = (T.phase[qq] == PH_PREDICT) ? dE : dN;
                    if (o.reuse_tangent && T.phase[qq] == PH_CORRECT) T.ecn[col][qq] = dE;
                }
            }
        } else {
            for (int g = warp; g < G::NGRP; g += G::NWARP) {
                int col, qq;
                double2 dE, dN;
                bool sing, act;
                lsolve<N>(sm, lane, warp, g, col, dE, dN, sing, act, qq);
                if (act) {
                    if (sing) atomicOr(&sm.st[qq], PT_SINGULAR);
                    T.dd[col][qq] = (T.phase[qq] == PH_PREDICT) ? dE : dN;
                    if (o.reuse_tangent && T.phase[qq] == PH_CORRECT) T.ecn[col][qq] = dE;
                }
            }
        }
        __syncthreads();
        // (3) element-parallel updates
        if (tid < N * PTS) {
            const int qq = tid / N, j = tid % N;
            const int ph = T.phase[qq];
            if (sm.st[qq] == 0 && ph != PH_IDLE) {
                const double2 dl = T.dd[j][qq];
                if (ph == PH_PREDICT) {
                    const double h = fmin(T.dt[qq], -T.tau_a[qq]);
                    if (LOGS && o.pred_log && o.predictor == 1 && T.has_prev[qq]) {
                        // cubic Hermite through (tau_p, z_p, e_p), (tau_a, z_a, delta_E) at s = 1 + h/D
                        const double D = T.tau_a[qq] - T.tau_p[qq], sv = 1.0 + h / D, s2 = sv * sv, s3 = s2 * sv;
                        const double h00 = 2 * s3 - 3 * s2 + 1, h10 = s3 - 2 * s2 + sv, h01 = -2 * s3 + 3 * s2,
                                     h11 = s3 - s2;
                        const double2 zp = T.zp[j][qq], ep = T.ep[j][qq], za = T.xa[j][qq];
                        T.xt[j][qq] = make_double2(h00 * zp.x + h10 * D * ep.x + h01 * za.x + h11 * D * dl.x,
                                                   h00 * zp.y + h10 * D * ep.y + h01 * za.y + h11 * D * dl.y);
                    } else {
                        T.xt[j][qq] = o.pred_log ? trk_predict_log<LOGS>(T.xa[j][qq], dl, h)
                                                 : trk_update<N, LOGS>(T.xa[j][qq], dl, h, S);
                    }
                    T.ec[j][qq] = dl;
                } else if (ph == PH_CORRECT) {
                    const double2 v = T.xt[j][qq];
                    T.xt[j][qq] = trk_update<N, LOGS>(v, dl, 1.0, S);
                    // |dx_j / x_j|^2 (reading R14); projective: |dy_j|^2 with ||y|| = 1 (R29)
                    const double r2 = fma(dl.x, dl.x, dl.y * dl.y);
                    T.nd2[j][qq] = S.proj ? r2 * fma(v.x, v.x, v.y * v.y) : r2;
                } else { // FINAL
                    const double2 v = T.xa[j][qq];
                    T.xa[j][qq] = trk_update<N, LOGS>(v, dl, 1.0, S);
                    const double r2 = fma(dl.x, dl.x, dl.y * dl.y);
                    T.nd2[j][qq] = S.proj ? r2 * fma(v.x, v.x, v.y * v.y) : r2;
                }
            }
        }
        __syncthreads();
        if (S.proj) { // updated points back onto ||y|| = 1 (x state only, reading R29)
            if (tid < PTS && sm.st[tid] == 0 && T.phase[tid] != PH_IDLE)
                proj_normalize<N>(T.phase[tid] == PH_FINAL ? T.xa : T.xt, tid);
            __syncthreads();
        }
        // (4) per-slot decisions (the oracle's control flow, oracle.c orc_track)
        if (tid < PTS && T.phase[tid] != PH_IDLE) {
            trk_decide<N, LOGS>(T, A, S, tid, sm.st[tid]);
            if (T.phase[tid] != PH_IDLE) atomicAdd(&T.active, 1);
        }
        __syncthreads();
        if (T.active == 0) {
            // flush the last finished paths
            if (tid < N * PTS) {
                const int qq = tid / N, j = tid % N;
                if (T.acc[qq]) T.xa[j][qq] = T.xt[j][qq]; // accepted in the last iteration (MAX_STEPS)
                if (T.done_path[qq] >= 0) A.x[T.done_path[qq] * N + j] = T.xa[j][qq];
            }
            break;
        }
    }
}

// ---------------------------------------------------------------------------------------
// Warp-per-group tracker (n <= 12, LU, affine/log/cell state, Euler predictor): the k_stepw
// lane mapping (lane = i * PPW + q) with the tracker's state machine per warp -- each warp runs
// PPW path slots on its own (no CTA barriers); the warps of a CTA share the exp/cis tables and the
// term records (shared memory, loaded once).  Same control flow as k_track (trk_decide).
// LPR = lanes per row: with few paths the tracker is latency-bound (one warp per SMSP), so each
// row's term loop is split over LPR lanes (terms t = h, h + LPR, ...) whose partial rows are
// combined with shuffles; the duplicated rows then run the same solve (bitwise identical).
#ifndef PHT_TRACKW_LOWOCC_MINB
#define PHT_TRACKW_LOWOCC_MINB 4 // resident 4-warp CTAs per SM the LPR > 1 (few-path) tracker is built for
#endif
#ifndef PHT_TRACKW_LOWOCC_SHFL
#define PHT_TRACKW_LOWOCC_SHFL 0 // measured: katsura-10 4.3 ms with shuffles vs 3.8 through shared memory
#endif
#ifndef PHT_TRACKW_LOWOCC_DB
#define PHT_TRACKW_LOWOCC_DB 1 // LPR > 1: double-buffered pivot row, one warp barrier less per pivot (katsura-10 -3%)
#endif
#ifndef PHT_TRACKW_LOWOCC_PAIR
#define PHT_TRACKW_LOWOCC_PAIR 0 // LPR > 1: two terms per iteration (ILP) for n <= 12
#endif
template <int N, int LPR>
struct GeoTW {
    static constexpr int PPW = (N * LPR <= 32) ? 32 / (N * LPR) : 1; // paths (slots) per warp
    static constexpr int MINB = LPR > 1 ? PHT_TRACKW_LOWOCC_MINB : GeoW<N>::MINB;
    static constexpr bool PAIR = LPR > 1 ? (PHT_TRACKW_LOWOCC_PAIR && N <= 12) : PHT_PAIR(N);
    // pivot-row broadcast by shuffles in the latency-bound few-path tracker (no shared round trip
    // and no __syncwarp per pivot), through shared memory in the throughput kernels
    static constexpr bool SHFL = LPR > 1 ? (bool)PHT_TRACKW_LOWOCC_SHFL : (bool)PHT_W_SHFL;
    // double-buffered pivot row in the latency-bound few-path tracker
    static constexpr bool DB = LPR > 1 && PHT_TRACKW_LOWOCC_DB;
    // the shuffle broadcast finds the pivot row's lane as (r PPW + q) LPR: not the balanced layout
    static_assert(!(SHFL && LPR == 3), "balanced lanes (LPR = 3) broadcast the pivot row through shared memory");
};

template <int N, int LPR = 1>
struct TrackW {
    static constexpr int PPW = GeoTW<N, LPR>::PPW;
    double2 rt[N][PPW];                 // (rho, vartheta) of the query points
    double2 xa[N][PPW], xt[N][PPW];     // accepted and trial points
    double2 dd[N][PPW];                 // direction of this iteration
    double2 ec[N][PPW];                 // Euler direction at the accepted point (re-prediction)
    double2 ecn[N][PPW];                // reuse_tangent: Euler direction at the latest corrector iterate
    double nd2[N][PPW];
    double2 prow[PPW][(1 + GeoTW<N, LPR>::DB) * (GeoW<N>::RW | 1)];
    alignas(16) unsigned keys[PPW * GeoW<N>::KS];
    double tau[PPW];                    // query tau
    double tau_a[PPW], tau_t[PPW], dt[PPW], prev[PPW], nd1[PPW], tau_p[PPW];
    long long path[PPW], steps[PPW], rej[PPW], evals[PPW], fin[PPW], done_path[PPW];
    int phase[PPW], it[PPW], succ[PPW], cell[PPW], acc[PPW], refill[PPW], has_prev[PPW], st[PPW];
    int tok[PPW], repred[PPW];          // (see TrackSmem)
};

template <int N, int LPR = 1>
struct SmemTW {
    double exptab[TAB_E];
    double2 cistab[TAB_C];
    TrackW<N, LPR> w[GeoW<N>::WARPS];
    int mk[N], off[N + 1];
    // followed by the records R[MT][N][RecW<N>::U] (16-byte units)
};

// row k of group point q for the tracker: records from shared memory; cell mode replaces each
// term's omega by the path's shifted lifting wq[global term index].  Lane h of the LPR lanes of
// the row takes the terms h, h + LPR, ...; the partial rows (each with its own binary row
// exponent) are aligned to the larger exponent and summed across the LPR lanes (shfl_xor).
// COMP: compensated stage 2 (phi_theta_c) for the final refinement at t = 1 (reading R30).
#ifndef PHT_TRACKW_RTREG
#define PHT_TRACKW_RTREG 0 // experiments: (rho, vartheta) held in registers through the row loop
#endif
// LPR = 3 is the balanced mode (trackw_lanes): row k owns gk = 2 or 3 consecutive lanes from lane
// gbase, lane h of them takes the terms h, h + gk, ...
template <int N, int LPR, bool COMP = false>
__device__ __forceinline__ void eval_row_tw(const SmemTW<N, LPR> &sm, const double2 *R, const TrackW<N, LPR> &W,
                                            int k, int q, int h, const double *wq, double2 (&row)[N + 2], int &e,
                                            unsigned mask = 0xffffffffu, // lanes executing this call (LPR shuffles)
                                            int gk = LPR, int gbase = 0)
{
    constexpr int RS = rec_stride(N), PPW = GeoTW<N, LPR>::PPW;
    const int step = (LPR == 3) ? gk : LPR; // term stride of this lane
#if PHT_TRACKW_RTREG
    PointLog<N, false> pl; // (rho, vartheta) of the slot's point in registers for the whole row
    pl.template load<PPW>(W.rt, q);
#else
    PointLog<N, true> pl;
    pl.base = &W.rt[0][q];
    pl.stride = PPW;
#endif
    const double tau = W.tau[q];
    const int m = sm.mk[k];
    const double2 *rec = R + (size_t)k * RecW<N>::U;
    constexpr size_t TS = (size_t)N * RecW<N>::U;
    const double *wk = wq ? wq + sm.off[k] : nullptr;
    RowAcc<N> acc;
    if (h < m) {
        double a[RS];
        load_rec_s<N>(rec + (size_t)h * TS, a);
        if (wk) a[N] = __ldg(wk + h);
        acc.init(phi_of<N>(a, pl, tau));
    } else { // no term on this lane: an empty partial row far below any real one
        acc.init(0.0);
        acc.set_exp(-1e6);
    }
    int i = h;
    if (COMP) {
        for (; i < m; i += step) {
            double a[RS];
            load_rec_s<N>(rec + (size_t)i * TS, a);
            if (wk) a[N] = __ldg(wk + i);
            double ph, pl_, th, tl;
            phi_theta_c<N>(a, pl, tau, ph, pl_, th, tl);
            acc.reduce(ph + pl_);
            acc.add(a, expcis<true>(acc.reduced2(ph, pl_), th, sm.exptab, sm.cistab, tl));
        }
    }
    for (; GeoTW<N, LPR>::PAIR && i + step < m; i += 2 * step) {
        double a[RS], b[RS];
        load_rec_s<N>(rec + (size_t)i * TS, a);
        load_rec_s<N>(rec + (size_t)(i + step) * TS, b);
        if (wk) {
            a[N] = __ldg(wk + i);
            b[N] = __ldg(wk + i + step);
        }
        double pa, pb, ta, tb;
        phi_theta<N>(a, pl, tau, pa, ta);
        phi_theta<N>(b, pl, tau, pb, tb);
        acc.reduce(pa);
        acc.reduce(pb);
        const double ya = acc.reduced(pa), yb = acc.reduced(pb);
        const double2 wa = expcis(ya, ta, sm.exptab, sm.cistab);
        const double2 wb = expcis(yb, tb, sm.exptab, sm.cistab);
        acc.add(a, wa);
        acc.add(b, wb);
    }
    for (; i < m; i += step) {
        double a[RS];
        load_rec_s<N>(rec + (size_t)i * TS, a);
        if (wk) a[N] = __ldg(wk + i);
        double pa, ta;
        phi_theta<N>(a, pl, tau, pa, ta);
        const double ya = acc.reduce(pa);
        acc.add(a, expcis(ya, ta, sm.exptab, sm.cistab));
    }
#pragma unroll
    for (int j = 0; j < N; ++j) row[j] = acc.g[j];
    row[N] = acc.gt;
    row[N + 1] = acc.h;
    double ed = acc.ed;
    if constexpr (LPR == 3) {
        // balanced mode: every lane of the group forms the same sum in the same order (lane
        // gbase + 0, + 1, + 2), each partial row first aligned to the group's largest exponent
        const int s1 = gbase + 1, s2 = gbase + (gk == 3 ? 2 : 1);
        const double e0 = __shfl_sync(mask, ed, gbase), e1 = __shfl_sync(mask, ed, s1),
                     e2 = __shfl_sync(mask, ed, s2);
        const double em = fmax(fmax(e0, e1), e2);
        const int d = (int)fmax(ed - em, -2000.0), d1 = d / 2;
        const double f1 = scalbn(1.0, d1), f2 = scalbn(1.0, d - d1);
#pragma unroll
        for (int c = 0; c < N + 2; ++c) {
            const double2 v = make_double2(row[c].x * f1 * f2, row[c].y * f1 * f2);
            const double x0 = __shfl_sync(mask, v.x, gbase), y0 = __shfl_sync(mask, v.y, gbase);
            const double x1 = __shfl_sync(mask, v.x, s1), y1 = __shfl_sync(mask, v.y, s1);
            const double x2 = __shfl_sync(mask, v.x, s2), y2 = __shfl_sync(mask, v.y, s2);
            row[c] = gk == 3 ? make_double2((x0 + x1) + x2, (y0 + y1) + y2) : make_double2(x0 + x1, y0 + y1);
        }
        e = (int)em;
    } else {
#pragma unroll
    for (int off = 1; off < LPR; off <<= 1) {
        // align to the larger row exponent (two normal power-of-two factors, see RowAcc::reduce),
        // then add the partner's partial row
        const double eo = __shfl_xor_sync(mask, ed, off), em = fmax(ed, eo);
        const int d = (int)fmax(ed - em, -2000.0), d1 = d / 2;
        const double f1 = scalbn(1.0, d1), f2 = scalbn(1.0, d - d1);
#pragma unroll
        for (int c = 0; c < N + 2; ++c) {
            const double2 v = make_double2(row[c].x * f1 * f2, row[c].y * f1 * f2);
            row[c] = make_double2(v.x + __shfl_xor_sync(mask, v.x, off),
                                  v.y + __shfl_xor_sync(mask, v.y, off));
        }
        ed = em;
    }
    e = (int)ed;
    }
}

// PROJ: projective systems (x state, LPR = 1): the bordering row and the unit-sphere renormalisation,
// compiled in only where used (the checks cost the affine kernels ~8% when present at run time)
template <int N, bool LOGS, int LPR, bool PROJ = false>
__global__ void __launch_bounds__(GeoW<N>::NT, (GeoTW<N, LPR>::MINB)) k_trackw(const DevSys S, const TrackArgs A, int MT)
{
    using G = GeoW<N>;
    constexpr int RS = rec_stride(N), PPW = GeoTW<N, LPR>::PPW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemTW<N, LPR> &sm = *reinterpret_cast<SmemTW<N, LPR> *>(smem_raw);
    double2 *R = reinterpret_cast<double2 *>(smem_raw + ((sizeof(SmemTW<N, LPR>) + 15) & ~(size_t)15));
    const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    const TrackOpts &o = A.o;
    load_tables(S, sm.exptab, sm.cistab, tid, G::NT);
    // a projective system has N - 1 polynomial rows; row N - 1 is the bordering row y^* (no terms)
    const int NE = PROJ ? N - 1 : N;
    for (int idx = tid; idx < MT * N; idx += G::NT) { // records, term-major (only t < m_k is read)
        const int kk = idx % N, t = idx / N;
        if (kk >= NE) continue;
        const int i0 = __ldg(S.off + kk), m = __ldg(S.off + kk + 1) - i0;
        if (t < m) pack_rec_w<N>(S.rec + (size_t)(i0 + t) * (RS / 2), R + (size_t)idx * RecW<N>::U);
    }
    if (tid < N) sm.mk[tid] = tid < NE ? __ldg(S.off + tid + 1) - __ldg(S.off + tid) : 0;
    if (tid <= N) sm.off[tid] = __ldg(S.off + (tid < NE ? tid : NE));
    TrackW<N, LPR> &W = sm.w[wi];
    // lane = (i * PPW + q) * LPR + h: row / variable i of slot q, term share h of that row;
    // balanced mode (LPR = 3, one slot): row i owns gi = 3 lanes if it is among the 32 - 2N rows
    // with the most terms, else 2 (ties: lower index first), the rows' groups in index order
    int gi = LPR, gbase = 0, ibal = 0, hbal = 0, used = N * PPW * LPR;
    if (LPR == 3) {
        int mk_[N];
#pragma unroll
        for (int j = 0; j < N; ++j) mk_[j] = __ldg(S.off + j + 1) - __ldg(S.off + j);
        const int n3 = min(N, 32 - 2 * N);
        int b = 0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            int rank = 0;
#pragma unroll
            for (int l = 0; l < N; ++l) rank += (mk_[l] > mk_[j] || (mk_[l] == mk_[j] && l < j)) ? 1 : 0;
            const int g = rank < n3 ? 3 : 2;
            if (lane >= b && lane < b + g) {
                ibal = j;
                hbal = lane - b;
                gi = g;
                gbase = b;
            }
            b += g;
        }
        used = b;
    }
    const bool inseg = lane < used;
    const int gl = LPR == 3 ? ibal : lane / LPR, h = LPR == 3 ? hbal : lane % LPR;
    const int q = inseg ? gl % PPW : 0, i = inseg ? gl / PPW : 0;
    const int seg0 = inseg ? q : PPW;
    const bool prim = inseg && h == 0; // the lane that owns row / variable i of slot q
    if (lane < PPW) {
        W.done_path[lane] = -1;
        W.cell[lane] = 0;
        W.acc[lane] = 0;
        trk_pop<N>(W, A, lane);
    }
    __syncthreads(); // tables and records
    for (;;) {
        // (1) write back finished paths, accept trial points, load new paths; the query point
        double2 xv = make_double2(LOGS ? 0.0 : 1.0, 0.0);
        if (prim) {
            if (W.acc[q]) W.xa[i][q] = W.xt[i][q];
            if (W.done_path[q] >= 0) A.x[W.done_path[q] * N + i] = W.xa[i][q];
            if (W.refill[q]) W.xa[i][q] = A.x[W.path[q] * N + i];
            if (W.repred[q]) { // re-prediction from the cached Euler direction (trk_decide)
                if (W.repred[q] == 2) W.ec[i][q] = W.ecn[i][q]; // reuse_tangent: the iterate's
                const double hh = fmin(W.dt[q], -W.tau_a[q]);
                W.xt[i][q] = o.pred_log ? trk_predict_log<LOGS>(W.xa[i][q], W.ec[i][q], hh)
                                        : trk_update<N, LOGS>(W.xa[i][q], W.ec[i][q], hh, S);
            }
            const int ph = W.phase[q];
            if (ph == PH_CORRECT) xv = W.xt[i][q];
            else if (ph != PH_IDLE) xv = W.xa[i][q];
        }
        __syncwarp();
        if (PROJ) { // a new projective path goes onto ||y|| = 1 first (reading R29)
            if (lane < PPW && W.refill[lane]) proj_normalize<N>(W.xa, lane);
            __syncwarp();
            if (prim && W.phase[q] != PH_CORRECT && W.phase[q] != PH_IDLE) xv = W.xa[i][q];
        }
        if (lane < PPW) {
            W.done_path[lane] = -1;
            W.acc[lane] = 0;
            W.refill[lane] = 0;
            W.repred[lane] = 0;
            W.st[lane] = 0;
            const int ph = W.phase[lane];
            W.tau[lane] = (ph == PH_CORRECT) ? W.tau_t[lane] : ((ph == PH_PREDICT) ? W.tau_a[lane] : 0.0);
        }
        __syncwarp();
        // (2) stage 1 for variable i, row i, solve (lane (i, q) ends with variable col)
        if (prim) {
            double rho, th;
            int st = 0;
            if (LOGS) {
                if (!(isfinite(xv.x) && isfinite(xv.y))) { st = PT_NONFINITE; rho = 0.0; th = 0.0; }
                else {
                    rho = xv.x;
                    const double kq = rint(xv.y * INV_2PI); // wrap Im z into [-pi, pi] (integer a)
                    th = fma(-kq, TWO_PI_LO, fma(-kq, TWO_PI_HI, xv.y));
                }
            } else {
                double2 iv;
                log_split_t(xv, rho, th, iv, st, S.logtab, S.atantab);
            }
            W.rt[i][q] = make_double2(rho, th);
            if (st) atomicOr(&W.st[q], st);
        }
        __syncwarp();
        {
            double2 a[N + 2];
            int e;
            const double *wq = A.cellw ? A.cellw + (size_t)W.cell[q] * A.M : nullptr;
            // the final refinement at t = 1 evaluates with the compensated stage 2 (reading R30),
            // chosen per slot: a slot's arithmetic never depends on the phases of the other slots
            // of its warp (a warp-uniform choice made the endpoints of paths that shared a warp with
            // a finishing path differ in the last bits from run to run).  A mixed warp runs the two
            // variants one after the other (a few % of the iterations); the LPR lanes of a row
            // belong to one slot, so their shuffles stay inside one branch.
            const bool fin = W.phase[q] == PH_FINAL;
            const unsigned bal = __ballot_sync(0xffffffffu, fin);
            if (bal == 0u)
                eval_row_tw<N, LPR, false>(sm, R, W, i, q, h, wq, a, e, 0xffffffffu, gi, gbase);
            else if (bal == 0xffffffffu)
                eval_row_tw<N, LPR, true>(sm, R, W, i, q, h, wq, a, e, 0xffffffffu, gi, gbase);
            else if (fin)
                eval_row_tw<N, LPR, true>(sm, R, W, i, q, h, wq, a, e, bal, gi, gbase);
            else
                eval_row_tw<N, LPR, false>(sm, R, W, i, q, h, wq, a, e, ~bal, gi, gbase);
            __syncwarp();
            if (PROJ && i == N - 1) { // bordering row y^* (P:237-252): y^* (y (.) delta) = sum |y_j|^2 delta_j
#pragma unroll
                for (int j = 0; j < N; ++j) a[j] = make_double2(exp(2.0 * W.rt[j][q].x), 0.0);
                a[N] = a[N + 1] = make_double2(0.0, 0.0);
                e = 0;
            }
            normalize_row<N>(a);
            int col;
            double2 dE, dN;
            bool sing;
            lsolve_regs<N, PPW, G::KS, true, LPR, GeoTW<N, LPR>::SHFL, GeoTW<N, LPR>::DB>(a, &W.prow[q][0], &W.keys[q * G::KS], seg0, q,
                                                                        i, inseg, col, dE, dN, sing, prim);
            if (prim) {
                if (sing) atomicOr(&W.st[q], PT_SINGULAR);
                W.dd[col][q] = (W.phase[q] == PH_PREDICT) ? dE : dN;
                if (o.reuse_tangent && W.phase[q] == PH_CORRECT) W.ecn[col][q] = dE;
            }
        }
        __syncwarp();
        // (3) element-parallel updates (lane (i, q): variable i of slot q)
        if (prim) {
            const int ph = W.phase[q];
            if (W.st[q] == 0 && ph != PH_IDLE) {
                const double2 dl = W.dd[i][q];
                if (ph == PH_PREDICT) {
                    const double hh = fmin(W.dt[q], -W.tau_a[q]);
                    W.ec[i][q] = dl; // cached for a re-prediction after a rejection
                    W.xt[i][q] = o.pred_log ? trk_predict_log<LOGS>(W.xa[i][q], dl, hh)
                                            : trk_update<N, LOGS>(W.xa[i][q], dl, hh, S);
                } else if (ph == PH_CORRECT) {
                    const double2 v = W.xt[i][q];
                    W.xt[i][q] = trk_update<N, LOGS>(v, dl, 1.0, S);
                    // |dx_i / x_i|^2 (reading R14); projective: |dy_i|^2 with ||y|| = 1 (R29)
                    const double r2 = fma(dl.x, dl.x, dl.y * dl.y);
                    W.nd2[i][q] = PROJ ? r2 * fma(v.x, v.x, v.y * v.y) : r2;
                } else { // FINAL
                    const double2 v = W.xa[i][q];
                    W.xa[i][q] = trk_update<N, LOGS>(v, dl, 1.0, S);
                    const double r2 = fma(dl.x, dl.x, dl.y * dl.y);
                    W.nd2[i][q] = PROJ ? r2 * fma(v.x, v.x, v.y * v.y) : r2;
                }
            }
        }
        __syncwarp();
        if (PROJ) { // updated points back onto ||y|| = 1 (x state only, reading R29)
            if (lane < PPW && W.st[lane] == 0 && W.phase[lane] != PH_IDLE)
                proj_normalize<N>(W.phase[lane] == PH_FINAL ? W.xa : W.xt, lane);
            __syncwarp();
        }
        // (4) per-slot decisions
        if (lane < PPW && W.phase[lane] != PH_IDLE) trk_decide<N, LOGS>(W, A, S, lane, W.st[lane]);
        __syncwarp();
        const bool busy = __any_sync(0xffffffffu, lane < PPW && W.phase[lane] != PH_IDLE);
        if (!busy) {
            if (prim && W.acc[q]) W.xa[i][q] = W.xt[i][q]; // accepted in the last iteration (MAX_STEPS)
            if (prim && W.done_path[q] >= 0) A.x[W.done_path[q] * N + i] = W.xa[i][q];
            break;
        }
    }
}

#ifndef __CUDACC_RTC__
// k_trackw: n <= 12, LU, affine or projective systems, Euler predictor; PHT_TRACKW=0 selects k_track.
template <int N>
bool trackw_eligible(const DevSys &S, const TrackArgs &A)
{
    return N <= 12 && A.solver == SOLVER_LU && A.o.predictor != 1 && S.mt > 0; // projective: LPR = 1
}

template <int N, bool LOGS, int LPR, bool PROJ = false>
cudaError_t launch_trackw_l(const DevSys &S, const TrackArgs &A, cudaStream_t stream, int sms)
{
    constexpr int PPW = GeoTW<N, LPR>::PPW;
    const size_t sb = ((sizeof(SmemTW<N, LPR>) + 15) & ~(size_t)15) + (size_t)S.mt * N * RecW<N>::U * 16;
    if (sb > 200 * 1024) return cudaErrorNotSupported;
    static std::atomic<int64_t> conf_sb[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if ((int64_t)sb > conf_sb[dev & 63].load()) {
        cudaError_t e = cudaFuncSetAttribute(k_trackw<N, LOGS, LPR, PROJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        if (e != cudaSuccess) return e;
        conf_sb[dev & 63].store((int64_t)sb);
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trackw<N, LOGS, LPR, PROJ>, GeoW<N>::NT, sb);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)sms * per_sm;
    const int64_t need = (A.P + (int64_t)PPW * GeoW<N>::WARPS - 1) / ((int64_t)PPW * GeoW<N>::WARPS);
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    k_trackw<N, LOGS, LPR, PROJ><<<dim3((unsigned)grid), dim3(GeoW<N>::NT), sb, stream>>>(S, A, S.mt);
    return cudaGetLastError();
}

// Lanes per row of k_trackw: when every path gets its own slot in one wave with LPR = 2 (or 4)
// lanes per row, the per-iteration latency of the row loop (the time to the last path at small
// path counts, katsura-10: 990 paths) shrinks; otherwise one lane per row (throughput).
#ifndef PHT_TRACKW_BALANCED
#define PHT_TRACKW_BALANCED 1 // few paths and n >= 9: 2-3 lanes per row over the whole warp (LPR = 3)
#endif
#ifndef PHT_TRACKW_LPR
#define PHT_TRACKW_LPR 0 // 0: automatic; 1, 2, 3 (balanced), 4: forced (experiments)
#endif
template <int N, bool LOGS>
cudaError_t launch_trackw_t(const DevSys &S, const TrackArgs &A, cudaStream_t stream, int sms)
{
    // warps resident per SM of the LPR > 1 kernels (their register budget: GeoTW::MINB)
    const int64_t slots_per_sm = (int64_t)GeoW<N>::WARPS * GeoTW<N, 2>::MINB;
    if (S.proj) { // projective systems (x state only): one lane per row
        if constexpr (!LOGS) return launch_trackw_l<N, false, 1, true>(S, A, stream, sms);
        return cudaErrorNotSupported;
    }
    int lpr = PHT_TRACKW_LPR;
    if (lpr == 0) {
        lpr = 1;
        if (N * 4 <= 32 && (A.P + GeoTW<N, 4>::PPW - 1) / GeoTW<N, 4>::PPW <= sms * slots_per_sm) lpr = 4;
        else if (N * 2 <= 32 && (A.P + GeoTW<N, 2>::PPW - 1) / GeoTW<N, 2>::PPW <= sms * slots_per_sm) lpr = 2;
    }
    if (lpr == 4 && N * 4 <= 32) return launch_trackw_l<N, LOGS, (N * 4 <= 32 ? 4 : 1)>(S, A, stream, sms);
    // n >= 9 (no LPR = 4): the balanced mode gives every row 2 or 3 lanes of the warp (katsura-10,
    // n = 11: 10 rows x 3 + 1 x 2 = 32 lanes, at most 4 terms per lane instead of 6)
    if ((lpr == 3 || (lpr == 2 && PHT_TRACKW_BALANCED)) && N * 2 <= 32 && N * 4 > 32)
        return launch_trackw_l<N, LOGS, (N * 2 <= 32 ? 3 : 1)>(S, A, stream, sms);
    if (lpr >= 2 && N * 2 <= 32) return launch_trackw_l<N, LOGS, (N * 2 <= 32 ? 2 : 1)>(S, A, stream, sms);
    return launch_trackw_l<N, LOGS, 1>(S, A, stream, sms);
}

template <int N, bool LOGS>
cudaError_t launch_track_t(const DevSys &S, const TrackArgs &A, cudaStream_t stream, int sms)
{
    const size_t sb = sizeof(TrackSmem<N>);
    static std::atomic<unsigned long long> configured{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(configured.load() & bit)) {
        cudaError_t e = cudaFuncSetAttribute(k_track<N, LOGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit);
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_track<N, LOGS>, Geo<N>::NT, sb);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)sms * per_sm;
    const int64_t need = (A.P + Geo<N>::PTS - 1) / Geo<N>::PTS;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    k_track<N, LOGS><<<dim3((unsigned)grid), dim3(Geo<N>::NT), sb, stream>>>(S, A);
    return cudaGetLastError();
}

// family: FAM_TILE forces k_track; otherwise k_trackw where eligible (FAM_AUTO, FAM_WARP)
template <int N>
cudaError_t launch_track(const DevSys &S, const TrackArgs &A, cudaStream_t stream, int sms, int family)
{
    if (family != FAM_TILE && trackw_eligible<N>(S, A)) {
        const cudaError_t e = A.o.log_state ? launch_trackw_t<N, true>(S, A, stream, sms)
                                            : launch_trackw_t<N, false>(S, A, stream, sms);
        if (e != cudaErrorNotSupported) return e;
    }
    return A.o.log_state ? launch_track_t<N, true>(S, A, stream, sms) : launch_track_t<N, false>(S, A, stream, sms);
}

template <int N, int MODE>
size_t smem_bytes()
{
    return sizeof(Smem<N>);
}

template <int N, int MODE>
cudaError_t launch_mode(const DevSys &S, const Args &A, cudaStream_t stream)
{
    constexpr int PTS = Geo<N>::PTS;
    const int64_t tiles = (A.P + PTS - 1) / PTS;
    if (tiles == 0) return cudaSuccess;
    const size_t sb = smem_bytes<N, MODE>();
    static std::atomic<unsigned long long> configured{0}; // one bit per device
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(configured.load() & bit)) {
        cudaError_t e = cudaFuncSetAttribute(k_pht<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit);
    }
    k_pht<N, MODE><<<dim3((unsigned)tiles), dim3(Geo<N>::NT), sb, stream>>>(S, A);
    return cudaGetLastError();
}

// Grid of a persistent kernel: SMs x resident CTAs per SM.
inline int64_t persistent_grid(const void *kernel, int threads, size_t smem)
{
    int dev = 0, sms = 1, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    return (int64_t)(sms > 0 ? sms : 1) * (per_sm > 0 ? per_sm : 1);
}

template <int N, int MODE>
cudaError_t launch_eval_mode(const DevSys &S, const Args &A, cudaStream_t stream)
{
    constexpr int PTS = Geo<N>::PTS;
    const int64_t tiles = (A.P + PTS - 1) / PTS;
    if (tiles == 0) return cudaSuccess;
    const size_t sb = smem_bytes<N, MODE>();
    static std::atomic<int64_t> full_grid[64]; // per device: SMs x resident CTAs (0: not yet configured)
    int dev = 0;
    cudaGetDevice(&dev);
    int64_t fg = full_grid[dev & 63].load();
    if (fg == 0) {
        cudaError_t e = cudaFuncSetAttribute(k_phte<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        if (e != cudaSuccess) return e;
        fg = persistent_grid(reinterpret_cast<const void *>(k_phte<N, MODE>), Geo<N>::NT, sb);
        full_grid[dev & 63].store(fg);
    }
    k_phte<N, MODE><<<dim3((unsigned)(tiles < fg ? tiles : fg)), dim3(Geo<N>::NT), sb, stream>>>(S, A);
    return cudaGetLastError();
}

// k_stepw: affine systems, LU solver, n <= 12 (the tile kernel keeps (rho, vartheta) in registers
// from n = 13 on and is faster there: cyclic-14 174 vs 154 M evals/s), records in shared memory
// (max_terms = MT per equation); PHT_STEPW=0 selects the tile kernel k_pht (experiments).
template <int N>
bool stepw_eligible(const DevSys &S, const Args &A)
{
    return N <= 12 && !S.proj && A.solver == SOLVER_LU && S.mt > 0;
}

// pht_evaluate through k_stepw<N, EVAL_X>: affine systems, n <= 12 (cyclic-5 2.44 -> 3.24, cyclic-10
// 0.59 -> 0.73 G points/s over the tile kernel k_phte)
template <int N>
bool stepw_eval_eligible(const DevSys &S)
{
    return N <= 12 && !S.proj && S.mt > 0;
}

template <int N, int MODE>
cudaError_t launch_stepw(const DevSys &S, const Args &A, cudaStream_t stream)
{
    constexpr int PPW = GeoW<N>::PPW;
    const int64_t groups = (A.P + PPW - 1) / PPW;
    if (groups == 0) return cudaSuccess;
    const size_t sb = ((sizeof(SmemW<N>) + 15) & ~(size_t)15) + (size_t)S.mt * N * RecW<N>::U * 16;
    if (sb > 200 * 1024) return cudaErrorNotSupported;
    // per device: the largest shared-memory size configured so far and the grid for the last size
    static std::atomic<int64_t> conf_sb[64], last_sb[64], last_fg[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if ((int64_t)sb > conf_sb[dev & 63].load()) {
        cudaError_t e = cudaFuncSetAttribute(k_stepw<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        if (e != cudaSuccess) return e;
        conf_sb[dev & 63].store((int64_t)sb);
    }
    int64_t fg = (last_sb[dev & 63].load() == (int64_t)sb) ? last_fg[dev & 63].load() : 0;
    if (fg == 0) {
        fg = persistent_grid(reinterpret_cast<const void *>(k_stepw<N, MODE>), GeoW<N>::SNT, sb);
        last_fg[dev & 63].store(fg);
        last_sb[dev & 63].store((int64_t)sb);
    }
    const int64_t need = (groups + GeoW<N>::SWARPS - 1) / GeoW<N>::SWARPS;
    k_stepw<N, MODE><<<dim3((unsigned)(need < fg ? need : fg)), dim3(GeoW<N>::SNT), sb, stream>>>(S, A, S.mt);
    return cudaGetLastError();
}

// Host-side launcher for one n (instantiated per n in inst_n*.cu).  family: FAM_TILE forces the
// tile kernels (k_phte, k_pht); otherwise the warp-per-group kernel k_stepw where eligible.
template <int N>
cudaError_t launch(int mode, const DevSys &S, const Args &A, cudaStream_t stream, int family)
{
    const bool tile = family == FAM_TILE;
    switch (mode) {
    case MODE_EVAL_X: {
        cudaError_t e = cudaErrorNotSupported;
        if (!tile && stepw_eval_eligible<N>(S)) e = launch_stepw<N, MODE_EVAL_X>(S, A, stream);
        return e == cudaErrorNotSupported ? launch_eval_mode<N, MODE_EVAL_X>(S, A, stream) : e;
    }
    case MODE_EVAL_Z: return launch_eval_mode<N, MODE_EVAL_Z>(S, A, stream);
    case MODE_DIRS: {
        cudaError_t e = cudaErrorNotSupported;
        if (!tile && stepw_eligible<N>(S, A)) e = launch_stepw<N, MODE_DIRS>(S, A, stream);
        return e == cudaErrorNotSupported ? launch_mode<N, MODE_DIRS>(S, A, stream) : e;
    }
    case MODE_STEP: {
        cudaError_t e = cudaErrorNotSupported;
        if (!tile && stepw_eligible<N>(S, A)) e = launch_stepw<N, MODE_STEP>(S, A, stream);
        return e == cudaErrorNotSupported ? launch_mode<N, MODE_STEP>(S, A, stream) : e;
    }
    default: return cudaErrorInvalidValue;
    }
}
#endif // !__CUDACC_RTC__

} // namespace pht
