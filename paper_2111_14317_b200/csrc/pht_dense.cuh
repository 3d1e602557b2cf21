// pht_dense.cuh — FP64 tensor-core (DMMA) evaluation for genuinely dense systems.
//
// BASELINE.json north_star: stage 2 "forms the monomial exponents as dense products of the
// stacked integer exponent/lifting matrix [A; omega] against the log-point matrix ... FP64
// tensor-core DMMA tiles only where the contraction is genuinely dense" (config C4: random dense
// Laurent n=20, 50 terms per equation).  sm_100a has no f64 tcgen05 kind; FP64 tensor work is
// mma.sync.m8n8k4.f64 (SASS DMMA), measured at 37.1 TFLOP/s on B200 (profiles/r01_microbench).
//
// Per warp: NMT M-tiles of 8 points.  The terms of all equations are streamed in n-tiles of 8
// slots (a tile may end one equation and start the next: segments A = [0, sb), B = [sb, 8)):
//   stage 2  Phi(8 pts x 8 terms)   = [rho | tau | 1 | 0]   (8 x KP) . B_phi(KP x 8)   (DMMA)
//            Theta(8 pts x 8 terms) = [theta | 0 | 1 | 0] (8 x KP) . B_th (KP x 8)    (DMMA)
//            with B_phi rows = (a_i, omega_i, log|c_i|), B_th rows = (a_i, 0, arg c_i)
//   stage 3  w = exp(phi - e ln2) cis(theta) on the accumulator fragments; e = per-point online
//            row exponent (quad shuffles; exact power-of-two rescale of the accumulators, R7)
//   stage 4  [G_1..G_N | G_tau | h](8 x CT*8) += W(8 x 4) . B4(4 x 8) per 4-term k-step, real
//            and imaginary parts of W as separate A operands; B4 rows = (a_i, omega_i, 1)
//            ("e^{z A} B_k^T").  W moves from accumulator to operand layout with
//            quad shuffles.
// B operands are pre-swizzled on the host into fragment order: one coalesced 256-byte load per
// (tile, k-step) per warp, reused for all NMT M-tiles.
// Fragment layouts of mma.m8n8k4 f64 (lane = 4*g + r): A(8x4): A[g][r]; B(4x8): B[r][g];
// C(8x8): C[g][2r], C[g][2r+1].
#pragma once

#include "pht_kernels.cuh"

namespace pht {

struct DenseSys {
    const double *b2phi;   // [ntiles][KS][32]
    const double *b2th;    // [ntiles][KS][32]
    const double *b4;      // [2*ntiles][CT][32]
    const int *tinfo;      // [2n] per equation: ts | te << 16, sb | done << 8 | endB << 9 (build_dense)
    int ntiles;            // n-tiles of 8 slots of the packed term stream
    int chunk;             // most n-tiles one equation processes: size of its staged B operands
};

// doubles of one n-tile's B operands staged in shared memory: b2phi, b2th (KS x 32) and
// b4 (2 x CT x 32); an equation's staged range holds at most D.chunk tiles
template <int N>
__host__ __device__ constexpr int dense_eq_doubles_per_tile()
{
    return ((N + 2 + 3) / 4) * 32 * 2 + ((N + 2 + 7) / 8) * 32 * 2;
}

// 16-byte asynchronous global -> shared copies (LDGSTS), all threads of the CTA
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K)); }

#ifndef PHT_DENSE_MINB
#define PHT_DENSE_MINB 3 // resident CTAs per SM k_dense is compiled for (register budget)
#endif
template <int N>
struct DGeo {
    static constexpr int KP = (N + 2 + 3) & ~3; // stage-2 K (vars + tau/const) padded to 4
    static constexpr int KS = KP / 4;          // stage-2 k-steps
    static constexpr int CT = (N + 2 + 7) / 8; // stage-4 column tiles of 8
#ifndef PHT_DENSE_NMT
#define PHT_DENSE_NMT 1
#endif
    // measured (profiles/r01_dense_tuning.txt): n <= 15: 8 warps share a double-buffered staged B
    // (prefetch of equation k+1 during k); n >= 16 (32 KB of B per equation): 4 warps, one buffer
    // (shared memory then still allows 3 CTAs per SM)
#ifdef PHT_DENSE_WARPS
    static constexpr int WARPS = PHT_DENSE_WARPS;
#else
    static constexpr int WARPS = N >= 16 ? 4 : 8;
#endif
#ifdef PHT_DENSE_NBUF
    static constexpr int NBUF = PHT_DENSE_NBUF;
#else
    static constexpr int NBUF = N >= 16 ? 1 : 2;
#endif
    static constexpr int NMT = PHT_DENSE_NMT;     // M-tiles (8 points) per warp
    static constexpr int PTS = WARPS * NMT * 8; // points per CTA
};

// monotone 32-bit integer key of a double's high word (NaN above +inf) and its inverse (low word 0)
__device__ __forceinline__ int dkey_hi(double v)
{
    const int h = __double2hiint(v);
    return h ^ ((h >> 31) & 0x7fffffff);
}
__device__ __forceinline__ double dkey_hi_inv(int k) { return __hiloint2double(k ^ ((k >> 31) & 0x7fffffff), 0); }

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int N>
struct DenseSmem {
    double exptab[TAB_E];
    double2 cistab[TAB_C];
    double ap[DGeo<N>::PTS][DGeo<N>::KP + 1]; // A operand rows for phi: rho_j, tau, 1
    double at[DGeo<N>::PTS][DGeo<N>::KP + 1]; // A operand rows for theta: theta_j, 0, 1
    double2 inv[DGeo<N>::PTS][N + 1];         // 1/x (EVAL_X)
    double tinv[DGeo<N>::PTS];
    int st[DGeo<N>::PTS];
};

template <int N, int MODE>
__global__ void __launch_bounds__(DGeo<N>::WARPS * 32, PHT_DENSE_MINB) k_dense(const DevSys S, const DenseSys D, const Args A)
{
    using G = DGeo<N>;
    constexpr int KP = G::KP, KS = G::KS, CT = G::CT, NMT = G::NMT, PTS = G::PTS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DenseSmem<N> &sm = *reinterpret_cast<DenseSmem<N> *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, r = lane & 3; // fragment coordinates
    load_tables(S, sm.exptab, sm.cistab, tid, G::WARPS * 32);
    const int64_t base = (int64_t)blockIdx.x * PTS;
    for (int q = tid; q < PTS; q += G::WARPS * 32) sm.st[q] = 0;
    __syncthreads();
    // stage 1: log split of every (point, variable) of the tile, plus tau
    for (int e = tid; e < PTS * N; e += G::WARPS * 32) {
        const int q = e / N, j = e - q * N;
        double rho = 0.0, th = 0.0;
        int st = 0;
        if (base + q < A.P) {
            const double2 v = A.xin[(base + q) * N + j];
            if (MODE == MODE_EVAL_Z) {
                if (!(isfinite(v.x) && isfinite(v.y))) st |= PT_NONFINITE;
                else {
                    rho = v.x;
                    const double kq = rint(v.y * INV_2PI);
                    th = fma(-kq, TWO_PI_LO, fma(-kq, TWO_PI_HI, v.y));
                }
            } else {
                double2 inv;
                log_split_t(v, rho, th, inv, st, S.logtab, S.atantab);
                sm.inv[q][j] = inv;
            }
        }
        sm.ap[q][j] = rho;
        sm.at[q][j] = th;
        if (st) atomicOr(&sm.st[q], st);
    }
    for (int q = tid; q < PTS; q += G::WARPS * 32) {
        double tau = 0.0;
        int st = 0;
        sm.tinv[q] = 1.0;
        if (base + q < A.P) {
            const double tv = A.tin[base + q];
            if (MODE == MODE_EVAL_Z) {
                tau = tv;
                if (!isfinite(tv)) { st |= PT_NONFINITE; tau = 0.0; }
            } else {
                if (!(tv > 0.0) || !isfinite(tv)) st |= PT_NONFINITE;
                else { tau = log(tv); sm.tinv[q] = 1.0 / tv; }
            }
        }
        for (int c = N; c < KP; ++c) {
            sm.ap[q][c] = (c == N) ? tau : (c == N + 1 ? 1.0 : 0.0);
            sm.at[q][c] = (c == N + 1) ? 1.0 : 0.0;
        }
        if (st) atomicOr(&sm.st[q], st);
    }
    __syncthreads();
    // A fragments (constant over equations): thread holds A[point 8m+g][col 4kk+r]
    double aP[NMT][KS], aT[NMT][KS];
#pragma unroll
    for (int m = 0; m < NMT; ++m) {
        const int q = (warp * NMT + m) * 8 + g;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            aP[m][kk] = sm.ap[q][4 * kk + r];
            aT[m][kk] = sm.at[q][4 * kk + r];
        }
    }
    const bool scaled = A.rexp != nullptr;
    // B operands of equation k are staged in shared memory (double-buffered, cp.async): the
    // warps of the CTA share them instead of each streaming them from L2 (ncu: long-scoreboard
    // stalls on the B loads were the first limiter)
    double *bbuf = reinterpret_cast<double *>(smem_raw + ((sizeof(DenseSmem<N>) + 15) & ~(size_t)15));
    const int EQB = D.chunk * dense_eq_doubles_per_tile<N>();
    // equation k processes the n-tiles [ts, te) of the packed stream: the tiles that start with
    // its terms, plus (when it ends inside a tile where equation k + 1 starts) that boundary tile
    // (build_dense: einfo[2k] = ts | te << 16, einfo[2k + 1] = sb | done << 8 | endB << 9)
    auto stage = [&](int k, int buf) {
        const int rg = __ldg(D.tinfo + 2 * k), t0 = rg & 0xffff, nt = (rg >> 16) - t0;
        double *dst = bbuf + (size_t)buf * EQB;
        const int n2 = nt * KS * 32, n4 = 2 * nt * CT * 32; // doubles per segment (multiples of 32)
        const double *s0 = D.b2phi + (size_t)t0 * KS * 32, *s1 = D.b2th + (size_t)t0 * KS * 32,
                     *s2 = D.b4 + (size_t)t0 * 2 * CT * 32;
        for (int u = tid; u < n2 / 2; u += G::WARPS * 32) {
            cp_async16(dst + 2 * u, s0 + 2 * u);
            cp_async16(dst + n2 + 2 * u, s1 + 2 * u);
        }
        for (int u = tid; u < n4 / 2; u += G::WARPS * 32) cp_async16(dst + 2 * n2 + 2 * u, s2 + 2 * u);
    };
    constexpr int NB = G::NBUF;
    if (NB == 2) {
        stage(0, 0);
        cp_async_commit();
    }
    // stage-4 accumulators [m][ct][re/im][2] of the current equation (carried into the next one
    // when it starts inside a boundary tile)
    double acc[NMT][CT][2][2];
    double ed[NMT], eh[NMT], el[NMT]; // per-point row exponent of the current equation (row g)
#pragma unroll
    for (int m = 0; m < NMT; ++m) {
        ed[m] = -1e300;
#pragma unroll
        for (int ct = 0; ct < CT; ++ct)
            acc[m][ct][0][0] = acc[m][ct][0][1] = acc[m][ct][1][0] = acc[m][ct][1][1] = 0.0;
    }
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
        const int rg = __ldg(D.tinfo + 2 * k), fl = __ldg(D.tinfo + 2 * k + 1);
        const int ts = rg & 0xffff, te = rg >> 16, sb = fl & 0xff;
        const bool done = (fl >> 8) & 1, endB = (fl >> 9) & 1;
        if (NB == 2) {
            if (k + 1 < N) stage(k + 1, (k + 1) & 1);
            cp_async_commit();
            cp_async_wait<1>(); // equation k's tiles have landed (this thread's copies)
        } else {
            stage(k, 0);
            cp_async_commit();
            cp_async_wait<0>();
        }
        __syncthreads(); // ... and everyone else's
        if (!done) {
        const double *bk = bbuf + (size_t)(NB == 2 ? (k & 1) : 0) * EQB;
        const int n2k = (te - ts) * KS * 32;
        const bool bnd = sb < 8;           // the last tile is a boundary tile
        const int tf = bnd ? te - 1 : te;  // tiles [ts, tf) hold equation k only
        // stage 2 of tile nt: phi and theta for its 8 slots
        auto stage2 = [&](int nt, double (&ph)[NMT][2], double (&th)[NMT][2]) {
#pragma unroll
            for (int m = 0; m < NMT; ++m) ph[m][0] = ph[m][1] = th[m][0] = th[m][1] = 0.0;
            const double *bp = bk + ((size_t)(nt - ts) * KS) * 32 + lane;
            const double *bt = bp + n2k;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                const double vp = bp[kk * 32], vt = bt[kk * 32];
#pragma unroll
                for (int m = 0; m < NMT; ++m) {
                    dmma(ph[m][0], ph[m][1], aP[m][kk], vp);
                    dmma(th[m][0], th[m][1], aT[m][kk], vt);
                }
            }
        };
        // online row exponent of the current equation from a quad maximum key (row g is shared
        // by the quad): the first tile sets it, a term more than e^512 above rescales exactly
        auto row_exp = [&](int m, int kx) {
            kx = max(kx, __shfl_xor_sync(0xffffffffu, kx, 1));
            kx = max(kx, __shfl_xor_sync(0xffffffffu, kx, 2));
            const double mx = dkey_hi_inv(kx);
            if (ed[m] == -1e300) {
                ed[m] = isfinite(mx) ? rint(mx * KC[14]) : 0.0;
                eh[m] = ed[m] * KC[12];
                el[m] = ed[m] * KC[13];
            } else if ((mx - eh[m]) - el[m] > 512.0) {
                const double e2 = rint(mx * KC[14]);
                // two normal factors (see RowAcc::reduce): one 2^d underflows for d < -1074
                const int d = (int)fmax(ed[m] - e2, -2000.0), d1 = d / 2;
                const double f1 = scalbn(1.0, d1), f2 = scalbn(1.0, d - d1);
#pragma unroll
                for (int ct = 0; ct < CT; ++ct)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        acc[m][ct][u][0] = acc[m][ct][u][0] * f1 * f2;
                        acc[m][ct][u][1] = acc[m][ct][u][1] * f1 * f2;
                    }
                ed[m] = e2;
                eh[m] = e2 * KC[12];
                el[m] = e2 * KC[13];
            }
        };
        // stage 4, k-step h of tile nt: A operand W[row g][slot 4h + r] from the quad, zero
        // outside the slot range [lo, hi)
        auto stage4 = [&](int nt, int h, const double (&wr)[NMT][2], const double (&wi)[NMT][2], int lo, int hi,
                          bool masked) {
            const int jt = 4 * h + r;                // slot of this lane's A element
            const int src = (lane & ~3) | (jt >> 1); // quad lane holding it
            const bool keep = !masked || (jt >= lo && jt < hi);
            const double *b4 = bk + 2 * n2k + ((size_t)(2 * (nt - ts) + h) * CT) * 32 + lane;
            double bv[CT];
#pragma unroll
            for (int ct = 0; ct < CT; ++ct) bv[ct] = b4[ct * 32];
#pragma unroll
            for (int m = 0; m < NMT; ++m) {
                const double r0 = __shfl_sync(0xffffffffu, wr[m][0], src);
                const double r1 = __shfl_sync(0xffffffffu, wr[m][1], src);
                const double i0 = __shfl_sync(0xffffffffu, wi[m][0], src);
                const double i1 = __shfl_sync(0xffffffffu, wi[m][1], src);
                const double ar = keep ? ((jt & 1) ? r1 : r0) : 0.0, ai = keep ? ((jt & 1) ? i1 : i0) : 0.0;
#pragma unroll
                for (int ct = 0; ct < CT; ++ct) {
                    dmma(acc[m][ct][0][0], acc[m][ct][0][1], ar, bv[ct]);
                    dmma(acc[m][ct][1][0], acc[m][ct][1][1], ai, bv[ct]);
                }
            }
        };
        for (int nt = ts; nt < tf; ++nt) { // tiles of equation k only (the common case)
            double ph[NMT][2], th[NMT][2];
            stage2(nt, ph, th);
            // stage 3: row exponent (row maximum on the integer pipe: the high words of the
            // doubles as a monotone integer key; measured: the FP64 DSETP.MAX chain was the
            // hottest stall of the kernel, on the datapath DMMA shares) and exp*cis
            double wr[NMT][2], wi[NMT][2];
#pragma unroll
            for (int m = 0; m < NMT; ++m) {
                row_exp(m, max(dkey_hi(ph[m][0]), dkey_hi(ph[m][1])));
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const double2 w = expcis((ph[m][u] - eh[m]) - el[m], th[m][u], sm.exptab, sm.cistab);
                    wr[m][u] = w.x;
                    wi[m][u] = w.y;
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) stage4(nt, h, wr, wi, 0, 8, false);
        }
        // the boundary tile: slots [0, sb) end equation k, [sb, 8) start equation k + 1 (its own
        // exponent from its own maximum); W of the boundary tile kept across equation k's epilogue
        double wr[NMT][2], wi[NMT][2], edB[NMT];
        if (bnd) {
            double ph[NMT][2], th[NMT][2];
            stage2(te - 1, ph, th);
            const bool inA0 = 2 * r < sb, inA1 = 2 * r + 1 < sb;
            constexpr int KMIN = (int)0x80000000;
#pragma unroll
            for (int m = 0; m < NMT; ++m) {
                const int k0 = dkey_hi(ph[m][0]), k1 = dkey_hi(ph[m][1]);
                row_exp(m, max(inA0 ? k0 : KMIN, inA1 ? k1 : KMIN));
                int kb = max(inA0 ? KMIN : k0, inA1 ? KMIN : k1);
                kb = max(kb, __shfl_xor_sync(0xffffffffu, kb, 1));
                kb = max(kb, __shfl_xor_sync(0xffffffffu, kb, 2));
                const double mb = dkey_hi_inv(kb);
                edB[m] = isfinite(mb) ? rint(mb * KC[14]) : 0.0;
                const double bh = edB[m] * KC[12], bl = edB[m] * KC[13];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const bool ia = u ? inA1 : inA0;
                    const double2 w = expcis((ph[m][u] - (ia ? eh[m] : bh)) - (ia ? el[m] : bl), th[m][u],
                                             sm.exptab, sm.cistab);
                    wr[m][u] = w.x;
                    wi[m][u] = w.y;
                }
            }
        }
        // segment 0: the rest of equation k (the boundary tile's A slots), then its row;
        // segment 1 (boundary tiles): equation k + 1's first slots, and its row if it ends here
#pragma unroll 1
        for (int sg = 0; sg < (bnd ? 2 : 1); ++sg) {
            if (bnd) {
                const int lo = sg ? sb : 0, hi = sg ? 8 : sb;
                for (int h = lo >> 2; h < ((hi + 3) >> 2); ++h) stage4(te - 1, h, wr, wi, lo, hi, true);
            }
            if (sg == 1 && !endB) break;
            // epilogue for equation kr: this thread holds columns 8ct + 2r + {0,1} of point row g
            const int kr = k + sg;
#pragma unroll
            for (int m = 0; m < NMT; ++m) {
                const int q = (warp * NMT + m) * 8 + g;
                const int64_t gq = base + q;
                const int e = (int)ed[m];
                bool fin = true;
#pragma unroll
                for (int ct = 0; ct < CT; ++ct)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int cc = 8 * ct + 2 * r + u;
                        if (cc >= N + 2) continue;
                        double2 v = make_double2(acc[m][ct][0][u], acc[m][ct][1][u]);
                        acc[m][ct][0][u] = acc[m][ct][1][u] = 0.0;
                        if (MODE == MODE_EVAL_X) {
                            if (cc < N) v = cmul(v, sm.inv[q][cc]);
                            else if (cc == N) v = make_double2(v.x * sm.tinv[q], v.y * sm.tinv[q]);
                        }
                        if (!scaled && e != 0) {
                            if (e >= -1022 && e <= 1023) v = make_double2(v.x * pow2i(e), v.y * pow2i(e));
                            else v = make_double2(scalbn(v.x, e), scalbn(v.y, e));
                        }
                        fin = fin && isfinite(v.x) && isfinite(v.y);
                        if (gq < A.P) {
                            if (cc < N) { if (A.J) A.J[(gq * N + kr) * N + cc] = v; }
                            else if (cc == N) { if (A.Jt) A.Jt[gq * N + kr] = v; }
                            else if (A.H) A.H[gq * N + kr] = v;
                        }
                    }
                if (!fin) atomicOr(&sm.st[q], PT_NONFINITE);
                if (scaled && r == 0 && gq < A.P) A.rexp[gq * N + kr] = e;
                // the next equation: the boundary tile's B exponent, else fresh
                ed[m] = (sg == 0 && bnd) ? edB[m] : -1e300;
                eh[m] = ed[m] * KC[12];
                el[m] = ed[m] * KC[13];
            }
        }
        }
        __syncthreads(); // buffer (k & 1) is refilled by the prefetch of equation k + 2
    }
    __syncthreads();
    for (int q = tid; q < PTS; q += G::WARPS * 32)
        if (base + q < A.P && A.status) A.status[base + q] = (uint8_t)sm.st[q];
}

template <int N, int MODE>
cudaError_t launch_dense_mode(const DevSys &S, const DenseSys &D, const Args &A, cudaStream_t stream)
{
    constexpr int PTS = DGeo<N>::PTS;
    const int64_t tiles = (A.P + PTS - 1) / PTS;
    if (tiles == 0) return cudaSuccess;
    const size_t sb = ((sizeof(DenseSmem<N>) + 15) & ~(size_t)15) +
                      (size_t)DGeo<N>::NBUF * D.chunk * dense_eq_doubles_per_tile<N>() * sizeof(double);
    // the staged B tiles make the size system dependent: set the attribute to the largest seen
    static std::atomic<size_t> configured_sb[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured_sb[dev & 63].load() < sb) {
        cudaError_t e = cudaFuncSetAttribute(k_dense<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        if (e != cudaSuccess) return e;
        configured_sb[dev & 63].store(sb);
    }
    k_dense<N, MODE><<<dim3((unsigned)tiles), dim3(DGeo<N>::WARPS * 32), sb, stream>>>(S, D, A);
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_dense(int mode, const DevSys &S, const DenseSys &D, const Args &A, cudaStream_t stream)
{
    if (mode == MODE_EVAL_X) return launch_dense_mode<N, MODE_EVAL_X>(S, D, A, stream);
    if (mode == MODE_EVAL_Z) return launch_dense_mode<N, MODE_EVAL_Z>(S, D, A, stream);
    return cudaErrorInvalidValue;
}

} // namespace pht
