// pht_kernels.cuh — sm_100a kernels for the polyhedral-homotopy hot path (arXiv 2111.14317).
//
// One templated kernel, k_pht<N, PTS, MODE>, covers the four entry points of include/pht.h.
// Mapping: a CTA owns a tile of PTS points; thread (k, q) = (equation k,
// point q of the tile) computes ROW k of the extended Jacobian of point q
//     [ dh_k/dz_1 .. dh_k/dz_N | dh_k/dtau | h_k ]        ("e^{z A} B_k^T")
// in registers.  With PTS = 32 a warp holds one equation for 32 points, so every read of the
// term table is a warp-uniform broadcast.  The rows of one point then stay in the registers
// of N threads for the direction solve (Gauss-Jordan with partial pivoting, two right-hand
// sides — §6 P:656-731 consolidated as in BASELINE.json north_star).
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

#include <cuda_runtime.h>
#include <stdint.h>

namespace pht {

enum Mode : int { MODE_EVAL_X = 0, MODE_EVAL_Z = 1, MODE_DIRS = 2, MODE_STEP = 3 };

enum : int { PT_ZERO_COORD = 1, PT_NONFINITE = 2, PT_SINGULAR = 4 };

// Points per CTA tile for a given n (register budget: 65536 / (N * PTS) per thread).
#ifndef PHT_PTS_SMALLN
#define PHT_PTS_SMALLN 32
#endif
__host__ __device__ constexpr int pts_for(int n) { return n <= 12 ? PHT_PTS_SMALLN : 16; }
// Term record stride in doubles: a_0..a_{n-1}, omega, log|c|, arg c, padded to even.
__host__ __device__ constexpr int rec_stride(int n) { return (n + 3 + 1) & ~1; }

struct DevSys {
    const double2 *rec;    // [M][rec_stride(n)/2] term records (a0 packer, pht_capi.cu)
    const int *off;        // [n+1] equation segments
    const double *exptab;  // [256] 2^(j/256)
    const double2 *cistab; // [256] (cos, sin)(2 pi j / 256)
    int n;
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

__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
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

// a3: w = exp(y) * (cos th + i sin th), y <= ~0.35 by construction of the row exponent.
// Table-driven: 2^(j/256) and cis(2 pi j/256) in shared memory, degree-4/5/6 polynomials on
// the reduced arguments (|r| <= ln2/512, |s| <= pi/256); error <= ~4 ulp.
__device__ __forceinline__ double2 expcis(double y, double th, const double *etab, const double2 *ctab)
{
    const double kf = fma(y, K256_LN2, SHIFT);
    const int ki = __double2loint(kf);
    const double kd = kf - SHIFT;
    double r = fma(kd, -LN2_256_HI, y);
    r = fma(kd, -LN2_256_LO, r);
    const double p = fma(fma(fma(fma(r, 1.0 / 24.0, 1.0 / 6.0), r, 0.5), r, 1.0), r, 1.0);
    double mag = etab[ki & 255] * p;
    const int m = ki >> 8;
    const unsigned hi = (unsigned)__double2hiint(mag) + ((unsigned)m << 20);
    mag = (m < -1000) ? 0.0 : __hiloint2double((int)hi, __double2loint(mag));

    const double qf = fma(th, K256_2PI, SHIFT);
    const int qi = __double2loint(qf);
    const double qd = qf - SHIFT;
    double s = fma(qd, -C1, th);
    s = fma(qd, -C2, s);
    s = fma(qd, -C3, s);
    const double s2 = s * s;
    const double sn = fma(s * s2, fma(s2, 1.0 / 120.0, -1.0 / 6.0), s);
    const double cs = fma(s2, fma(s2, fma(s2, -1.0 / 720.0, 1.0 / 24.0), -0.5), 1.0);
    const double2 T = ctab[qi & 255];
    const double cr = fma(T.x, cs, -T.y * sn);
    const double ci = fma(T.y, cs, T.x * sn);
    return make_double2(mag * cr, mag * ci);
}

template <int N, int PTS>
struct Smem {
    double exptab[256];
    double2 cistab[256];
    double2 rt[N][PTS];   // (rho, vartheta) per variable; reused for dN staging in DIRS
    double2 xs[N][PTS];   // x (or z) of the tile
    double2 inv[N][PTS];  // 1/x (EVAL_X); reused for dE staging in DIRS
    double tau[PTS];
    double tinv[PTS];
    int st[PTS];
    double cand[N][PTS];  // pivot candidates
    double2 prow[N + 2][PTS];
    double2 pinv[PTS];
    double dn2[N][PTS];
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

// phi = omega tau + log|c| + sum_j a_j rho_j  with two interleaved partial sums (ILP).
template <int N>
__device__ __forceinline__ double phi_of(const double (&a)[rec_stride(N)], const double (&rho)[N], double tau)
{
    double p0 = fma(a[N], tau, a[N + 1]), p1 = 0.0;
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        p0 = fma(a[j], rho[j], p0);
        if (j + 1 < N) p1 = fma(a[j + 1], rho[j + 1], p1);
    }
    return p0 + p1;
}

template <int N>
__device__ __forceinline__ double theta_of(const double (&a)[rec_stride(N)], const double (&th)[N])
{
    double p0 = a[N + 2], p1 = 0.0;
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        p0 = fma(a[j], th[j], p0);
        if (j + 1 < N) p1 = fma(a[j + 1], th[j + 1], p1);
    }
    return p0 + p1;
}

template <int N>
__device__ __forceinline__ void accumulate(const double (&a)[rec_stride(N)], double2 w, double2 (&g)[N],
                                           double2 &gt, double2 &h)
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

// a2-a4 for row k of point q: row = [G_1..G_N | G_tau | h] scaled by 2^-e.
// Terms are processed two at a time (independent dependency chains for the FP64 pipe).
template <int N, int PTS>
__device__ __forceinline__ void eval_row(const DevSys &S, const Smem<N, PTS> &sm, int k, int q,
                                         double2 (&row)[N + 2], int &e)
{
    constexpr int RS = rec_stride(N);
    double rho[N], th[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const double2 v = sm.rt[j][q];
        rho[j] = v.x;
        th[j] = v.y;
    }
    const double tau = sm.tau[q];
    const int i0 = __ldg(S.off + k), i1 = __ldg(S.off + k + 1);
    const double2 *rec = S.rec + (size_t)i0 * (RS / 2);
    const int m = i1 - i0;

    // pass 1: row scale s = max_i (phi_i + log|c_i|)  (ledger R7)
    double s0 = -INFINITY, s1 = -INFINITY;
    int i = 0;
    for (; i + 1 < m; i += 2) {
        double a[RS], b[RS];
        load_rec<N>(rec + (size_t)i * (RS / 2), a);
        load_rec<N>(rec + (size_t)(i + 1) * (RS / 2), b);
        s0 = fmax(s0, phi_of<N>(a, rho, tau));
        s1 = fmax(s1, phi_of<N>(b, rho, tau));
    }
    if (i < m) {
        double a[RS];
        load_rec<N>(rec + (size_t)i * (RS / 2), a);
        s0 = fmax(s0, phi_of<N>(a, rho, tau));
    }
    const double smax = fmax(s0, s1);
    const double ed = isfinite(smax) ? rint(smax * INV_LN2) : 0.0;
    e = (int)ed;
    const double eh = ed * LN2_HI, el = ed * LN2_LO;

    // pass 2: w_i = exp(phi_i - e ln2) cis(theta_i) and the contractions
    double2 g[N], gt = make_double2(0.0, 0.0), h = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < N; ++j) g[j] = make_double2(0.0, 0.0);
    i = 0;
    for (; i + 1 < m; i += 2) {
        double a[RS], b[RS];
        load_rec<N>(rec + (size_t)i * (RS / 2), a);
        load_rec<N>(rec + (size_t)(i + 1) * (RS / 2), b);
        const double ya = (phi_of<N>(a, rho, tau) - eh) - el;
        const double yb = (phi_of<N>(b, rho, tau) - eh) - el;
        const double ta = theta_of<N>(a, th), tb = theta_of<N>(b, th);
        const double2 wa = expcis(ya, ta, sm.exptab, sm.cistab);
        const double2 wb = expcis(yb, tb, sm.exptab, sm.cistab);
        accumulate<N>(a, wa, g, gt, h);
        accumulate<N>(b, wb, g, gt, h);
    }
    if (i < m) {
        double a[RS];
        load_rec<N>(rec + (size_t)i * (RS / 2), a);
        const double ya = (phi_of<N>(a, rho, tau) - eh) - el;
        const double2 wa = expcis(ya, theta_of<N>(a, th), sm.exptab, sm.cistab);
        accumulate<N>(a, wa, g, gt, h);
    }
#pragma unroll
    for (int j = 0; j < N; ++j) row[j] = g[j];
    row[N] = gt;
    row[N + 1] = h;
}

// a5: Gauss-Jordan elimination with partial pivoting across the N row-threads of each point.
// Pivot = max |Re|+|Im| of the column among rows not yet used, lowest row on ties (ledger R12).
// On return the thread whose row was the pivot of column `col` holds
//   dE = -row[N] / row[col],  dN = -row[N+1] / row[col]   (G [dE|dN] = -[G_tau | h]).
template <int N, int PTS>
__device__ __forceinline__ void gj_solve(Smem<N, PTS> &sm, int k, int q, double2 (&a)[N + 2],
                                         int &col, double2 &dE, double2 &dN, bool &singular)
{
    double rmax = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) rmax = fmax(rmax, cabs1(a[j]));
    col = -1;
    singular = false;
    double2 myinv = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double cand = -1.0;
        if (col < 0) {
            cand = cabs1(a[j]);
            if (cand != cand) cand = INFINITY;
        }
        sm.cand[k][q] = cand;
        __syncthreads();
        int r = 0;
        double best = sm.cand[0][q];
#pragma unroll
        for (int kk = 1; kk < N; ++kk) {
            const double v = sm.cand[kk][q];
            if (v > best) { best = v; r = kk; }
        }
        if (k == r) {
            col = j;
            const double pv = cabs1(a[j]);
            if (!(pv > 1e-14 * rmax) || !isfinite(pv) || !isfinite(rmax)) singular = true;
            myinv = crecip(a[j]);
            sm.pinv[q] = myinv;
#pragma unroll
            for (int c = j + 1; c < N + 2; ++c) sm.prow[c][q] = a[c];
        }
        __syncthreads();
        if (k != r) {
            const double2 l = cmul(a[j], sm.pinv[q]);
#pragma unroll
            for (int c = j + 1; c < N + 2; ++c) a[c] = cfms(a[c], l, sm.prow[c][q]);
            a[j] = make_double2(0.0, 0.0);
        }
    }
    const double2 e = cmul(a[N], myinv), n = cmul(a[N + 1], myinv);
    dE = make_double2(-e.x, -e.y);
    dN = make_double2(-n.x, -n.y);
}

// a1 for the whole tile: (rho, vartheta) from xs (x in EVAL_X/DIRS/STEP, z in EVAL_Z).
template <int N, int PTS, int MODE>
__device__ __forceinline__ void stage1(Smem<N, PTS> &sm, int tid)
{
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

template <int N, int PTS, int MODE>
__global__ void __launch_bounds__(N *PTS, (N * PTS <= 192) ? 2 : 1) k_pht(const DevSys S, const Args A)
{
    __shared__ Smem<N, PTS> sm;
    const int tid = threadIdx.x;
    const int k = tid / PTS, q = tid % PTS;
    for (int i = tid; i < 256; i += N * PTS) {
        sm.exptab[i] = __ldg(S.exptab + i);
        sm.cistab[i] = __ldg(S.cistab + i);
    }
    const int64_t base = (int64_t)blockIdx.x * PTS;
    const int64_t gq = base + q;
    const bool valid = gq < A.P;

    // load the tile's points, coalesced: flat element tid = (point tid/N, variable tid%N)
    const double2 *xsrc = (MODE == MODE_STEP) ? A.xio : A.xin;
    {
        const int qq = tid / N, j = tid % N;
        double2 v = make_double2(MODE == MODE_EVAL_Z ? 0.0 : 1.0, 0.0);
        if (base + qq < A.P) v = xsrc[(base * N) + tid];
        sm.xs[j][qq] = v;
    }
    if (tid < PTS) {
        sm.st[tid] = 0;
        const int64_t g = base + tid;
        double tv = (MODE == MODE_EVAL_Z || MODE == MODE_STEP) ? 0.0 : 1.0;
        if (g < A.P) tv = (MODE == MODE_STEP) ? A.tauio[g] : A.tin[g];
        if (MODE == MODE_EVAL_Z || MODE == MODE_STEP) {
            sm.tau[tid] = tv;
            if (!isfinite(tv)) sm.st[tid] |= PT_NONFINITE;
        } else {
            if (!(tv > 0.0) || !isfinite(tv)) { sm.st[tid] |= PT_NONFINITE; tv = 1.0; }
            sm.tau[tid] = log(tv);
            sm.tinv[tid] = 1.0 / tv;
        }
    }
    __syncthreads();

    if (MODE == MODE_EVAL_X || MODE == MODE_EVAL_Z) {
        stage1<N, PTS, MODE>(sm, tid);
        __syncthreads();
        double2 row[N + 2];
        int e;
        eval_row<N, PTS>(S, sm, k, q, row, e);
        const bool scaled = A.rexp != nullptr;
        bool fin = true;
        if (MODE == MODE_EVAL_X) {
            const double ti = sm.tinv[q];
            row[N] = make_double2(row[N].x * ti, row[N].y * ti);
#pragma unroll
            for (int j = 0; j < N; ++j) row[j] = cmul(row[j], sm.inv[j][q]);
        }
        if (!scaled && e != 0) {
#pragma unroll
            for (int c = 0; c < N + 2; ++c) row[c] = make_double2(scalbn(row[c].x, e), scalbn(row[c].y, e));
        }
#pragma unroll
        for (int c = 0; c < N + 2; ++c) fin = fin && isfinite(row[c].x) && isfinite(row[c].y);
        if (!fin) atomicOr(&sm.st[q], PT_NONFINITE);
        if (valid) {
            const int64_t o = gq * N + k;
            if (A.H) A.H[o] = row[N + 1];
            if (A.Jt) A.Jt[o] = row[N];
            if (A.J) {
                double2 *dst = A.J + o * N;
#pragma unroll
                for (int j = 0; j < N; ++j) dst[j] = row[j];
            }
            if (scaled) A.rexp[o] = e;
        }
        __syncthreads();
        if (tid < PTS && base + tid < A.P && A.status) A.status[base + tid] = (uint8_t)sm.st[tid];
        return;
    }

    if (MODE == MODE_DIRS) {
        stage1<N, PTS, MODE>(sm, tid);
        __syncthreads();
        double2 row[N + 2];
        int e, col;
        double2 dE, dN;
        bool sing;
        eval_row<N, PTS>(S, sm, k, q, row, e);
        gj_solve<N, PTS>(sm, k, q, row, col, dE, dN, sing);
        if (sing) atomicOr(&sm.st[q], PT_SINGULAR);
        // dx/dt = x (.) delta_E / t,  dN_x = x (.) delta_N  (Jx = G diag(1/x), Jt = G_tau / t)
        const double2 xv = sm.xs[col][q];
        const double2 de = cmul(xv, dE), dn = cmul(xv, dN);
        const double ti = sm.tinv[q];
        sm.inv[col][q] = make_double2(de.x * ti, de.y * ti);
        sm.rt[col][q] = dn;
        __syncthreads();
        {
            const int qq = tid / N, j = tid % N;
            if (base + qq < A.P) {
                if (A.dE) A.dE[base * N + tid] = sm.inv[j][qq];
                if (A.dN) A.dN[base * N + tid] = sm.rt[j][qq];
            }
        }
        if (tid < PTS && base + tid < A.P && A.status) {
            int st = sm.st[tid];
            A.status[base + tid] = (uint8_t)st;
        }
        return;
    }

    // MODE_STEP: x~ = x + h dx/dtau ; tau~ = tau + h ; K x { x~ += dN(x~, tau~) }
    {
        double h = 0.0;
        if (valid) h = A.dtau[gq];
        for (int it = 0; it <= A.K; ++it) {
            stage1<N, PTS, MODE>(sm, tid);
            __syncthreads();
            double2 row[N + 2];
            int e, col;
            double2 dE, dN;
            bool sing;
            eval_row<N, PTS>(S, sm, k, q, row, e);
            gj_solve<N, PTS>(sm, k, q, row, col, dE, dN, sing);
            if (sing) atomicOr(&sm.st[q], PT_SINGULAR);
            const double2 xv = sm.xs[col][q];
            if (it == 0) {
                // dx/dtau = x (.) delta_E  ->  x~ = x + h x delta_E
                const double2 d = cmul(xv, dE);
                sm.xs[col][q] = make_double2(fma(h, d.x, xv.x), fma(h, d.y, xv.y));
            } else {
                const double2 d = cmul(xv, dN);
                sm.xs[col][q] = make_double2(xv.x + d.x, xv.y + d.y);
                sm.dn2[col][q] = fma(d.x, d.x, d.y * d.y);
            }
            __syncthreads();
            if (it == 0 && tid < PTS) sm.tau[tid] += (base + tid < A.P) ? A.dtau[base + tid] : 0.0;
            // (the next iteration's stage1 is preceded by this barrier)
            __syncthreads();
        }
        {
            const int qq = tid / N;
            if (base + qq < A.P) A.xio[base * N + tid] = sm.xs[tid % N][qq];
        }
        if (tid < PTS && base + tid < A.P) {
            A.tauio[base + tid] = sm.tau[tid];
            if (A.status) A.status[base + tid] = (uint8_t)sm.st[tid];
            if (A.dnnorm) {
                double s = 0.0;
                for (int j = 0; j < N; ++j) s += sm.dn2[j][tid];
                A.dnnorm[base + tid] = A.K > 0 ? sqrt(s) : 0.0;
            }
        }
    }
}

// Host-side launcher for one n (instantiated per n in inst_n*.cu).
template <int N>
cudaError_t launch(int mode, const DevSys &S, const Args &A, cudaStream_t stream)
{
    constexpr int PTS = pts_for(N);
    const int64_t tiles = (A.P + PTS - 1) / PTS;
    if (tiles == 0) return cudaSuccess;
    const dim3 grid((unsigned)tiles), block(N * PTS);
    switch (mode) {
    case MODE_EVAL_X: k_pht<N, PTS, MODE_EVAL_X><<<grid, block, 0, stream>>>(S, A); break;
    case MODE_EVAL_Z: k_pht<N, PTS, MODE_EVAL_Z><<<grid, block, 0, stream>>>(S, A); break;
    case MODE_DIRS: k_pht<N, PTS, MODE_DIRS><<<grid, block, 0, stream>>>(S, A); break;
    case MODE_STEP: k_pht<N, PTS, MODE_STEP><<<grid, block, 0, stream>>>(S, A); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

} // namespace pht
