// pht_evalw.cuh — point-per-lane batched evaluation (pht_evaluate / pht_evaluate_log, n <= 12).
//
// The standalone evaluation writes H, Jx, Jt to HBM (2,089 B per point at n = 10)
// and needs no direction solve, so the lane mapping of the fused step kernel (lane = (point,
// equation), 3 points per warp, a different term record per lane) is not required.  Here a warp
// owns 32 points, one per lane, and walks the N equations in order (the paper's Alg. 2 row by row,
// P:788-805):
//   * stage 1 once per point: (rho_j, vartheta_j) stay in registers for all N rows;
//   * every lane of the warp reads the SAME term record (the equation is warp-uniform), so a record
//     load is a shared-memory broadcast (2 cycles per LDS.128 instead of 4, 3 loads per term) and
//     serves 32 points instead of 3;
//   * stages 2-4 per row as in the other kernels (RowAcc, expcis: P:453-556), Jx = G diag(1/x)
//      with 1/x_j kept in shared memory;
//   * output: the row of equation k for the warp's 32 points is staged in shared memory and written
//     by ONE TMA tensor store per output array (cp.async.bulk.tensor: Jx viewed as [P][N][2N]
//     doubles, box {2N, 1, 32}; Jt, H as [P][N][2], box {2, 1, 32}), asynchronously while the warp
//     evaluates the next row; the TMA unit clips the ragged tail.  Without tensor maps (unaligned
//     pointers) the rows are stored from registers.
#pragma once

#include "pht_kernels.cuh"

#ifndef __CUDACC_RTC__
#include <cuda.h> // CUtensorMap
#endif

namespace pht {

#ifndef __CUDACC_RTC__
// TMA tensor maps of the three row outputs of one pht_evaluate call (host-encoded per call)
struct EvalMaps {
    CUtensorMap J, T, H;
    int tma; // 1: store through the maps; 0: direct stores
};

#ifndef PHT_EVALW_WARPS
#define PHT_EVALW_WARPS 12
#endif
#ifndef PHT_EVALW_TMA
#define PHT_EVALW_TMA 1 // 0: direct stores from registers (experiments)
#endif
#ifndef PHT_EVALW_PAIR
#define PHT_EVALW_PAIR 0 // two terms per iteration in k_evalw's row loop (experiments)
#endif
#ifndef PHT_EVALW_MINB
#define PHT_EVALW_MINB 1
#endif
template <int N>
struct GeoEW {
    static constexpr int WARPS = PHT_EVALW_WARPS;
    static constexpr int NT = WARPS * 32;
    static constexpr int MINB = PHT_EVALW_MINB; // one 12-warp CTA per SM, <= 168 registers (measured
    // cyclic-10 1.06 G points/s; 8 x 2 warps with spills 0.81, 10 x 1 0.88, 14 x 1 0.83, 8 x 1 0.87)
};

template <int N>
struct SmemEW {
    double exptab[TAB_E];
    double2 cistab[TAB_C];
    int mk[N];
    struct alignas(128) Warp {
        double sj[32][2 * N]; // staged Jx (Jz) rows of one equation, point-major (the TMA box layout)
        alignas(16) double st[32][2];
        alignas(16) double sh[32][2];
        double2 inv[N][33]; // 1/x_j of the warp's points (EVAL_X), padded against bank conflicts
    } w[GeoEW<N>::WARPS];
    // followed by the records R[MT][N][RecW<N, WIDE>::U] (16-byte units, the packer's doubles), 16-byte aligned
};

__device__ __forceinline__ void tma_store3(const CUtensorMap *map, const void *smem, int c0, int c1, int c2)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                 :
                 : "l"(map), "r"(s), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

// WIDE: term records as the packer's doubles (RecW); compact int16 records when those do not fit
template <int N, int MODE, bool WIDE = true>
__global__ void __launch_bounds__(GeoEW<N>::NT, GeoEW<N>::MINB)
    k_evalw(const DevSys S, const Args A, int MT, const __grid_constant__ EvalMaps M)
{
    static_assert(MODE == MODE_EVAL_X || MODE == MODE_EVAL_Z, "k_evalw: evaluation modes");
    constexpr bool XM = MODE == MODE_EVAL_X;
    constexpr int RS = rec_stride(N);
    extern __shared__ __align__(128) unsigned char smem_ew[]; // (TMA sources: 128-byte aligned rows)
    SmemEW<N> &sm = *reinterpret_cast<SmemEW<N> *>(smem_ew);
    double2 *R = reinterpret_cast<double2 *>(smem_ew + ((sizeof(SmemEW<N>) + 15) & ~(size_t)15));
    const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    load_tables(S, sm.exptab, sm.cistab, tid, GeoEW<N>::NT);
    for (int idx = tid; idx < MT * N; idx += GeoEW<N>::NT) { // records, equation-major per term slot
        const int kk = idx % N, t = idx / N;
        const int i0 = __ldg(S.off + kk), m = __ldg(S.off + kk + 1) - i0;
        if (t < m) pack_rec_w<N, WIDE>(S.rec + (size_t)(i0 + t) * (RS / 2), R + (size_t)idx * RecW<N, WIDE>::U);
    }
    if (tid < N) sm.mk[tid] = __ldg(S.off + tid + 1) - __ldg(S.off + tid);
    __syncthreads();
    typename SmemEW<N>::Warp &W = sm.w[wi];
    constexpr size_t TS = (size_t)N * RecW<N, WIDE>::U; // record stride between terms of one equation
    const int64_t groups = (A.P + 31) / 32;
    bool pending = false; // a TMA store of this warp's staging may still read it
    for (int64_t grp = (int64_t)blockIdx.x * GeoEW<N>::WARPS + wi; grp < groups;
         grp += (int64_t)gridDim.x * GeoEW<N>::WARPS) {
        const int64_t p = grp * 32 + lane;
        const bool act = p < A.P;
        // stage 1 for this lane's point (a1): (rho, vartheta) in registers
        PointLog<N, false> pl;
        int st = 0;
        double tau, tinv = 1.0;
        {
            double tv = XM ? 1.0 : 0.0;
            if (act) tv = A.tin[p];
            if (XM) {
                if (!(tv > 0.0) || !isfinite(tv)) { st |= PT_NONFINITE; tv = 1.0; }
                tau = log(tv);
                tinv = 1.0 / tv;
            } else {
                if (!isfinite(tv)) { st |= PT_NONFINITE; tv = 0.0; }
                tau = tv;
            }
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double2 v = make_double2(XM ? 1.0 : 0.0, 0.0);
            if (act) v = A.xin[p * N + j];
            if (XM) {
                double2 iv;
                log_split_t(v, pl.rho[j], pl.th[j], iv, st, S.logtab, S.atantab);
                W.inv[j][lane] = iv;
            } else if (!(isfinite(v.x) && isfinite(v.y))) {
                st |= PT_NONFINITE;
                pl.rho[j] = 0.0;
                pl.th[j] = 0.0;
            } else {
                pl.rho[j] = v.x;
                const double kq = rint(v.y * INV_2PI); // wrap Im z into [-pi, pi] (integer a)
                pl.th[j] = fma(-kq, TWO_PI_LO, fma(-kq, TWO_PI_HI, v.y));
            }
        }
        for (int k = 0; k < N; ++k) {
            // a2-a4 for row k of this lane's point: every lane reads the same records (broadcast)
            const int m = sm.mk[k];
            const double2 *rec = R + (size_t)k * RecW<N, WIDE>::U;
            RowAcc<N> acc;
            {
                double a[RS];
                load_rec_s<N, WIDE>(rec, a);
                acc.init(phi_of<N>(a, pl, tau));
            }
            int i = 0;
            for (; PHT_EVALW_PAIR && i + 1 < m; i += 2) { // two terms per iteration (ILP)
                double a[RS], b[RS];
                load_rec_s<N, WIDE>(rec + (size_t)i * TS, a);
                load_rec_s<N, WIDE>(rec + (size_t)(i + 1) * TS, b);
                double pa, ta, pb, tb;
                phi_theta<N>(a, pl, tau, pa, ta);
                phi_theta<N>(b, pl, tau, pb, tb);
                acc.reduce(pa);
                acc.reduce(pb);
                const double2 wa = expcis(acc.reduced(pa), ta, sm.exptab, sm.cistab);
                const double2 wb = expcis(acc.reduced(pb), tb, sm.exptab, sm.cistab);
                acc.add(a, wa);
                acc.add(b, wb);
            }
            for (; i < m; ++i) {
                double a[RS];
                load_rec_s<N, WIDE>(rec + (size_t)i * TS, a);
                double pa, ta;
                phi_theta<N>(a, pl, tau, pa, ta);
                const double ya = acc.reduce(pa);
                acc.add(a, expcis(ya, ta, sm.exptab, sm.cistab));
            }
            double2 row[N + 2];
#pragma unroll
            for (int j = 0; j < N; ++j) row[j] = XM ? cmul(acc.g[j], W.inv[j][lane]) : acc.g[j];
            row[N] = XM ? make_double2(acc.gt.x * tinv, acc.gt.y * tinv) : acc.gt;
            row[N + 1] = acc.h;
            const int e = (int)acc.ed;
            const bool scaled = A.rexp != nullptr;
            if (!scaled) scale_row2<N + 2>(row, e);
            bool fin = true;
#pragma unroll
            for (int c = 0; c < N + 2; ++c) fin = fin && isfinite(row[c].x) && isfinite(row[c].y);
            if (!fin) st |= PT_NONFINITE;
            if (act && scaled) A.rexp[p * N + k] = e;
            if (PHT_EVALW_TMA && M.tma) {
                // the previous row's store must have finished reading the staging buffer
                if (pending && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    W.sj[lane][2 * j] = row[j].x;
                    W.sj[lane][2 * j + 1] = row[j].y;
                }
                W.st[lane][0] = row[N].x;
                W.st[lane][1] = row[N].y;
                W.sh[lane][0] = row[N + 1].x;
                W.sh[lane][1] = row[N + 1].y;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // visible to the TMA unit
                __syncwarp();
                if (lane == 0) {
                    const int q0 = (int)(grp * 32); // the map clips points >= P
                    if (A.J) tma_store3(&M.J, &W.sj[0][0], 0, k, q0);
                    if (A.Jt) tma_store3(&M.T, &W.st[0][0], 0, k, q0);
                    if (A.H) tma_store3(&M.H, &W.sh[0][0], 0, k, q0);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                pending = true;
            } else if (act) {
                const int64_t r = p * N + k;
                if (A.J) {
#pragma unroll
                    for (int j = 0; j < N; ++j) A.J[r * N + j] = row[j];
                }
                if (A.Jt) A.Jt[r] = row[N];
                if (A.H) A.H[r] = row[N + 1];
            }
        }
        if (act && A.status) A.status[p] = (uint8_t)st;
    }
    if (pending && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); // writes done
}

template <int N>
bool evalw_eligible(const DevSys &S)
{
    return N <= 12 && !S.proj && S.mt > 0;
}

// host: TMA maps for the outputs of one evaluate call (rank-3 views, FLOAT64 elements); 0 if the
// driver entry point is unavailable or a pointer is not 16-byte aligned (direct stores then)
int encode_eval_maps(EvalMaps &M, int n, int64_t P, void *J, void *Jt, void *H);

template <int N, int MODE, bool WIDE>
cudaError_t launch_evalw_r(const DevSys &S, const Args &A, const EvalMaps &M, size_t sb, cudaStream_t stream)
{
    const int64_t groups = (A.P + 31) / 32;
    static std::atomic<int64_t> conf_sb[64], last_sb[64], last_fg[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if ((int64_t)sb > conf_sb[dev & 63].load()) {
        cudaError_t e = cudaFuncSetAttribute(k_evalw<N, MODE, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
        if (e != cudaSuccess) return e;
        conf_sb[dev & 63].store((int64_t)sb);
    }
    int64_t fg = (last_sb[dev & 63].load() == (int64_t)sb) ? last_fg[dev & 63].load() : 0;
    if (fg == 0) {
        fg = persistent_grid(reinterpret_cast<const void *>(k_evalw<N, MODE, WIDE>), GeoEW<N>::NT, sb);
        last_fg[dev & 63].store(fg);
        last_sb[dev & 63].store((int64_t)sb);
    }
    const int64_t need = (groups + GeoEW<N>::WARPS - 1) / GeoEW<N>::WARPS;
    k_evalw<N, MODE, WIDE><<<dim3((unsigned)(need < fg ? need : fg)), dim3(GeoEW<N>::NT), sb, stream>>>(S, A, S.mt, M);
    return cudaGetLastError();
}

template <int N, int MODE>
cudaError_t launch_evalw(const DevSys &S, const Args &A, const EvalMaps &M, cudaStream_t stream)
{
    const int64_t groups = (A.P + 31) / 32;
    if (groups == 0) return cudaSuccess;
    const size_t base = (sizeof(SmemEW<N>) + 15) & ~(size_t)15;
    const size_t sw = base + (size_t)S.mt * N * RecW<N, true>::U * 16, sc = base + (size_t)S.mt * N * RecW<N>::U * 16;
    if (sw <= 200 * 1024) return launch_evalw_r<N, MODE, true>(S, A, M, sw, stream);
    if (sc <= 200 * 1024) return launch_evalw_r<N, MODE, false>(S, A, M, sc, stream);
    return cudaErrorNotSupported;
}
#endif // !__CUDACC_RTC__

} // namespace pht
