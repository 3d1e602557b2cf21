// pht_capi.cu — C ABI (include/pht.h): system loader / packer (the
// paper's Alg. 1 "Initialize") and the entry points that enqueue k_pht.
#include "../../include/pht.h"
#include "pht_dense.cuh"
#include "pht_evalw.cuh"
#include "pht_jit.h"
#include "pht_kernels.cuh"

#include <cudaTypedefs.h> // PFN_cuTensorMapEncodeTiled (driver entry point, no -lcuda)

#include <algorithm>
#include <cstdint>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

namespace pht {
#define PHT_DECL(N)                                                                             \
    extern template cudaError_t launch<N>(int, const DevSys &, const Args &, cudaStream_t, int); \
    extern template cudaError_t launch_track<N>(const DevSys &, const TrackArgs &, cudaStream_t, int, int); \
    extern template cudaError_t launch_dense<N>(int, const DevSys &, const DenseSys &, const Args &, cudaStream_t); \
    extern template cudaError_t launch_evalw<N, MODE_EVAL_X>(const DevSys &, const Args &, const EvalMaps &, cudaStream_t); \
    extern template cudaError_t launch_evalw<N, MODE_EVAL_Z>(const DevSys &, const Args &, const EvalMaps &, cudaStream_t);
PHT_DECL(1) PHT_DECL(2) PHT_DECL(3) PHT_DECL(4) PHT_DECL(5) PHT_DECL(6) PHT_DECL(7) PHT_DECL(8)
PHT_DECL(9) PHT_DECL(10) PHT_DECL(11) PHT_DECL(12) PHT_DECL(13) PHT_DECL(14) PHT_DECL(15)
PHT_DECL(16) PHT_DECL(17) PHT_DECL(18) PHT_DECL(19) PHT_DECL(20) PHT_DECL(21) PHT_DECL(22)
PHT_DECL(23) PHT_DECL(24)
#undef PHT_DECL

// TMA tensor maps of the evaluation outputs (k_evalw): Jx as [P][n][2n] doubles with box {2n, 1, 32},
// Jt and H as [P][n][2] with box {2, 1, 32}.  The encoder comes from the driver through the runtime's
// entry-point query (the library links no libcuda).
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder()
{
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

static bool encode3(CUtensorMap *m, void *base, int64_t d0, int64_t d1, int64_t d2, uint32_t b0)
{
    const cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
    const cuuint64_t strides[2] = {(cuuint64_t)(d0 * 8), (cuuint64_t)(d0 * d1 * 8)};
    const cuuint32_t box[3] = {b0, 1, 32}, estr[3] = {1, 1, 1};
    return tmap_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int encode_eval_maps(EvalMaps &M, int n, int64_t P, void *J, void *Jt, void *H)
{
    M.tma = 0;
    if (!tmap_encoder() || P <= 0 || P > ((int64_t)1 << 31)) return 0;
    for (void *ptr : {J, Jt, H})
        if (ptr && ((uintptr_t)ptr & 15u)) return 0;
    if (J && !encode3(&M.J, J, 2 * n, n, P, (uint32_t)(2 * n))) return 0;
    if (Jt && !encode3(&M.T, Jt, 2, n, P, 2)) return 0;
    if (H && !encode3(&M.H, H, 2, n, P, 2)) return 0;
    M.tma = 1;
    return 1;
}
} // namespace pht

static_assert(PHT_MAX_N == 24, "dispatch table below covers n = 1..24");

struct pht_system {
    int n = 0;
    int64_t M = 0;
    int max_terms = 0;
    int device = 0;
    int sms = 148;
    int dropped = 0; // terms with c = 0 removed by the packer
    int solver = 0;  // PHT_SOLVER_LU / PHT_SOLVER_QR (pht_system_set_solver)
    int proj = 0;    // projective system: n = n_eq + 1 homogeneous coordinates
    int kernels = 0; // PHT_KERNELS_* (pht_system_set_kernels)
    double2 *d_rec = nullptr;
    int *d_off = nullptr;
    double *d_exptab = nullptr;
    double2 *d_cistab = nullptr;
    double2 *d_logtab = nullptr; // log_split_t tables (pht_kernels.cuh)
    double *d_atantab = nullptr;
    // dense FP64 tensor-core path (pht_dense.cuh), built when the system is genuinely dense
    int dense = 0;
    double *d_b2phi = nullptr, *d_b2th = nullptr, *d_b4 = nullptr;
    int *d_tinfo = nullptr; // per n-tile equation / boundary info (build_dense)
    int max_ntk = 0; // most n-tiles one equation processes (k_dense staging size)
    int dense_ntiles = 0; // n-tiles of the packed term stream
    // packed tables on the host (input of the code generator, pht_system_specialize)
    std::vector<double> h_rec;
    std::vector<int> h_off;
    // system-specialised kernels (pht_jit.cu), or nullptr; replaced only under jit_mu, read by
    // the launchers under jit_mu (a snapshot); a replaced image stays loaded until destroy
    // (launches queued on streams may still use it)
    std::mutex jit_mu;
    pht::JitKernels *jit = nullptr;
    std::vector<pht::JitKernels *> jit_old;
    // workspace and copy/compute streams of the *_host entry points
    std::mutex ws_mu;
    // (copy-in, two compute, copy-out; per-chunk events: copy-in done, kernel done)
    cudaStream_t hs[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t hev_in[64] = {}, hev_k[64] = {}, hev_out[64] = {};
    cudaEvent_t hev0 = nullptr, hev_end = nullptr;
    // the previous host step (pht_pc_step_host_async chains): its point count and chunk count
    int64_t hprev_p = -1;
    int hprev_nch = 0;
    int64_t ws_cap = 0;
    void *ws = nullptr;
};

static thread_local std::string g_cuda_err;
static std::atomic<int64_t> g_launches{0};

static int cuda_fail(cudaError_t e)
{
    g_cuda_err = cudaGetErrorString(e);
    return PHT_ECUDA;
}

struct DevGuard {
    int prev = -1;
    bool ok = true;
    explicit DevGuard(int d)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != d) ok = cudaSetDevice(d) == cudaSuccess;
    }
    ~DevGuard()
    {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// a0: validate, drop zero coefficients, pack per-term records
//   [a_0 .. a_{n-1}, omega, log|c|, arg c, pad]   (DESIGN.md §2 "HBM/L1 layout")
static int pack_system(int32_t n_eq, int32_t n_var, const int64_t *off, const int32_t *exps, const double *coeffs,
                       const double *lifting, std::vector<double> &rec, std::vector<int> &doff, int &max_terms,
                       int64_t &M, int &n_dropped, bool homog = false)
{
    if (!off || !exps || !coeffs || !lifting) return PHT_EINVAL;
    if (n_eq != n_var || n_eq < 1 || n_eq > PHT_MAX_N) return PHT_ESHAPE;
    const int n = n_eq;
    if (off[0] != 0) return PHT_ESHAPE;
    for (int k = 0; k < n; ++k)
        if (off[k + 1] < off[k]) return PHT_ESHAPE;
    const int64_t M_in = off[n];
    if (M_in >= (int64_t)1 << 30) return PHT_ESHAPE;
    // projective: records over y in C^{n+1}, a^ = (a, deg(f_k) - 1^T a), homogenising
    // coordinate last, deg(f_k) = max 1^T a over the equation's terms
    const int NV = homog ? n + 1 : n;
    if (NV > PHT_MAX_N) return PHT_ESHAPE;
    const int RS = pht::rec_stride(NV);
    rec.clear();
    doff.assign(n + 1, 0);
    max_terms = 0;
    rec.reserve((size_t)M_in * RS);
    M = 0;
    n_dropped = 0;
    for (int k = 0; k < n; ++k) {
        int64_t deg = INT64_MIN;
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            int64_t d = 0;
            for (int j = 0; j < n; ++j) d += exps[i * n + j];
            deg = std::max(deg, d);
        }
        // a term is (a, omega): the same monomial may appear with different liftings (the
        // coefficient-parameter homotopy (1 - t) G + t F has x^a t^0 and x^a t^1 terms)
        std::set<std::pair<std::vector<int32_t>, double>> seen;
        int cnt = 0;
        for (int64_t i = off[k]; i < off[k + 1]; ++i) {
            std::vector<int32_t> a(exps + i * n, exps + (i + 1) * n);
            if (!seen.insert({a, lifting[i]}).second) return PHT_EDUPLICATE;
            for (int j = 0; j < n; ++j)
                if (a[j] > PHT_MAX_EXP || a[j] < -PHT_MAX_EXP) return PHT_ERANGE;
            const double cr = coeffs[2 * i], ci = coeffs[2 * i + 1], w = lifting[i];
            if (!std::isfinite(cr) || !std::isfinite(ci) || !std::isfinite(w)) return PHT_EINVAL;
            if (w < 0) return PHT_ERANGE;
            if (cr == 0.0 && ci == 0.0) { ++n_dropped; continue; }
            int64_t d = 0;
            for (int j = 0; j < n; ++j) {
                rec.push_back((double)a[j]);
                d += a[j];
            }
            if (homog) {
                if (deg - d > PHT_MAX_EXP) return PHT_ERANGE;
                rec.push_back((double)(deg - d));
            }
            rec.push_back(w);
            rec.push_back(std::log(std::hypot(cr, ci)));
            rec.push_back(std::atan2(ci, cr));
            for (int u = NV + 3; u < RS; ++u) rec.push_back(0.0);
            ++cnt;
            ++M;
        }
        if (cnt == 0) return PHT_EEMPTY;
        doff[k + 1] = (int)M;
        if (cnt > max_terms) max_terms = cnt;
    }
    return PHT_OK;
}

// FP64 tensor-core tables (pht_dense.cuh) from the packed records [a, omega, log|c|, arg c]:
// B operands pre-swizzled into mma.m8n8k4 fragment order.  Stage 2: B = [A; omega; log|c|] (phi)
// and [A; 0; arg c] (theta), K = n + 2 padded to 4; stage 4: B = [A_k | omega | 1] per 4-term
// half tile.  The terms of all equations form ONE stream cut into n-tiles of 8 slots: a tile may
// hold the end of one equation and the start of the next (at most one equation starts inside a
// tile; a second one is moved to the next tile, the skipped slots padded).  Per-equation tiles
// left the last tile of every 50-term equation 2/8 used (C4: 140 tiles for 1,000 terms; packed:
// 125).  Equation k processes the tiles that start with its terms and the boundary tile where it
// ends (tinfo, see pht_dense.cuh).
static int build_dense(pht_system *s)
{
    if (s->dense) return PHT_OK;
    const int n = s->n, RS = pht::rec_stride(n);
    const std::vector<double> &rec = s->h_rec;
    const std::vector<int> &off = s->h_off;
    const int KP = (n + 2 + 3) & ~3, KS = KP / 4, CT = (n + 2 + 7) / 8;
    // slot stream: global term index per slot, -1 = padding
    std::vector<int64_t> slot;
    std::vector<int> slot_eq;
    int max_ntk = 0;
    bool mid_start = false; // an equation already started inside the current tile
    for (int k = 0; k < n; ++k) {
        const int m = off[k + 1] - off[k];
        if (m == 0) return PHT_EINVAL;
        if (slot.size() % 8 != 0 && mid_start) // a second boundary in this tile: pad to the next tile
            while (slot.size() % 8 != 0) { slot.push_back(-1); slot_eq.push_back(k - 1); }
        mid_start = slot.size() % 8 != 0;
        for (int t = 0; t < m; ++t) {
            if (t > 0 && slot.size() % 8 == 0) mid_start = false; // crossed into a new tile
            slot.push_back(off[k] + t);
            slot_eq.push_back(k);
        }
    }
    while (slot.size() % 8 != 0) { slot.push_back(-1); slot_eq.push_back(n - 1); }
    const int NT = (int)(slot.size() / 8);
    // per equation k: the tiles [ts, te) it processes (those starting with its terms, plus the
    // boundary tile where it ends and k + 1 starts); sb = that tile's first slot of k + 1 (8: no
    // boundary tile); done: k lies entirely inside the previous boundary tile; endB: k + 1 ends
    // inside this equation's boundary tile
    std::vector<int> first(n, -1), last(n, -1);
    for (size_t u = 0; u < slot.size(); ++u) {
        if (slot[u] < 0) continue;
        const int k = slot_eq[u];
        if (first[k] < 0) first[k] = (int)u;
        last[k] = (int)u;
    }
    std::vector<int> tinfo(2 * n);
    max_ntk = 1;
    for (int k = 0; k < n; ++k) {
        const int ts = first[k] / 8 + (first[k] % 8 != 0 ? 1 : 0);
        const int tl = last[k] / 8;
        const bool done = ts > tl;
        int te = done ? ts : tl + 1, sb = 8;
        bool endB = false;
        if (!done && k + 1 < n && first[k + 1] / 8 == tl) { // k + 1 starts inside k's last tile
            sb = first[k + 1] % 8;
            endB = last[k + 1] / 8 == tl;
        }
        if (done) te = ts;
        max_ntk = std::max(max_ntk, te - ts);
        if (te > 0xffff) return PHT_EUNSUPPORTED;
        tinfo[2 * k] = ts | (te << 16);
        tinfo[2 * k + 1] = sb | ((int)done << 8) | ((int)endB << 9);
    }
    std::vector<double> b2p((size_t)NT * KS * 32), b2t((size_t)NT * KS * 32), b4((size_t)2 * NT * CT * 32);
    for (int ntg = 0; ntg < NT; ++ntg) {
        for (int lane = 0; lane < 32; ++lane) {
            const int g = lane >> 2, r = lane & 3;
            const int64_t i = slot[8 * ntg + g]; // stage 2: B[r][g] = slot 8t+g
            const bool real = i >= 0;
            const double *ri = rec.data() + (size_t)(real ? i : 0) * RS;
            for (int kk = 0; kk < KS; ++kk) {
                const int kr = 4 * kk + r;
                double vp = 0.0, vt = 0.0;
                if (real) {
                    if (kr < n) vp = vt = ri[kr];
                    else if (kr == n) vp = ri[n];
                    else if (kr == n + 1) { vp = ri[n + 1]; vt = ri[n + 2]; }
                } else if (kr == n + 1) {
                    vp = -1e300; // padding slot: exp -> 0
                }
                b2p[((size_t)ntg * KS + kk) * 32 + lane] = vp;
                b2t[((size_t)ntg * KS + kk) * 32 + lane] = vt;
            }
            for (int h = 0; h < 2; ++h) { // stage 4: B[r][g] = slot 8t+4h+r, column 8ct+g
                const int64_t i4 = slot[8 * ntg + 4 * h + r];
                for (int ct = 0; ct < CT; ++ct) {
                    const int c = 8 * ct + g;
                    double v = 0.0;
                    if (i4 >= 0) {
                        const double *r4 = rec.data() + (size_t)i4 * RS;
                        if (c < n) v = r4[c];
                        else if (c == n) v = r4[n];
                        else if (c == n + 1) v = 1.0;
                    }
                    b4[((size_t)(2 * ntg + h) * CT + ct) * 32 + lane] = v;
                }
            }
        }
    }
    DevGuard g(s->device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    cudaError_t e;
    if ((e = cudaMalloc(&s->d_b2phi, b2p.size() * 8)) != cudaSuccess ||
        (e = cudaMalloc(&s->d_b2th, b2t.size() * 8)) != cudaSuccess ||
        (e = cudaMalloc(&s->d_b4, b4.size() * 8)) != cudaSuccess ||
        (e = cudaMalloc(&s->d_tinfo, tinfo.size() * sizeof(int))) != cudaSuccess ||
        (e = cudaMemcpy(s->d_b2phi, b2p.data(), b2p.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_b2th, b2t.data(), b2t.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_b4, b4.data(), b4.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_tinfo, tinfo.data(), tinfo.size() * sizeof(int), cudaMemcpyHostToDevice)) != cudaSuccess)
        return e == cudaErrorMemoryAllocation ? PHT_ENOMEM : cuda_fail(e);
    s->max_ntk = max_ntk;
    s->dense_ntiles = NT;
    s->dense = 1;
    return PHT_OK;
}

static int create_impl(int32_t n_eq, int32_t n_var, const int64_t *off, const int32_t *exps, const double *coeffs,
                       const double *lifting, int32_t device, pht_system **out, bool proj)
{
    if (!out) return PHT_EINVAL;
    std::vector<double> rec;
    std::vector<int> doff;
    int max_terms = 0, n_dropped = 0;
    int64_t M = 0;
    const int prc = pack_system(n_eq, n_var, off, exps, coeffs, lifting, rec, doff, max_terms, M, n_dropped, proj);
    if (prc != PHT_OK) return prc;
    const int n = proj ? n_eq + 1 : n_eq; // kernel width: variables (rows = n_eq polynomials + y^*)

    // exp / cis tables, rounded from 80-bit long double
    std::vector<double> etab(256), ctab(512);
    const long double PI_L = 3.141592653589793238462643383279502884L;
    for (int j = 0; j < 256; ++j) {
        etab[j] = (double)exp2l((long double)j / 256.0L);
        ctab[2 * j] = (double)cosl(2.0L * PI_L * (long double)j / 256.0L);
        ctab[2 * j + 1] = (double)sinl(2.0L * PI_L * (long double)j / 256.0L);
    }
    // log / atan tables of log_split_t: (1/c_j rounded, -log of that rounded value) so that
    // r = m (1/c_j) - 1 carries the rounding of 1/c_j exactly, c_j = 1 + (j + 1/2)/128; atan(k/64)
    std::vector<double> ltab(256), atab(65);
    for (int j = 0; j < 128; ++j) {
        const double ic = (double)(1.0L / (1.0L + ((long double)j + 0.5L) / 128.0L));
        ltab[2 * j] = ic;
        ltab[2 * j + 1] = (double)(-logl((long double)ic));
    }
    for (int k = 0; k <= 64; ++k) atab[k] = (double)atanl((long double)k / 64.0L);

    DevGuard g(device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    pht_system *s = new (std::nothrow) pht_system();
    if (!s) return PHT_ENOMEM;
    s->n = n;
    s->M = M;
    s->max_terms = max_terms;
    s->device = device;
    s->dropped = n_dropped;
    s->proj = proj ? 1 : 0;
    s->h_rec = rec;
    s->h_off = doff;
    cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, device);
    {
        // the trackers' stream-ordered scratch (cudaMallocAsync) comes from the device's default
        // memory pool; by default the pool returns its memory to the OS at every synchronisation,
        // so the next allocation maps pages again inside the caller's stream (measured up to ~20 ms
        // stalls on a 6 ms tracking run).  Keep up to 64 MB of the pool resident instead.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = 0;
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            if (keep < (64ull << 20)) {
                keep = 64ull << 20;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
    }
    cudaError_t e;
    if ((e = cudaMalloc(&s->d_rec, rec.size() * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&s->d_off, doff.size() * sizeof(int))) != cudaSuccess ||
        (e = cudaMalloc(&s->d_exptab, 256 * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&s->d_cistab, 256 * sizeof(double2))) != cudaSuccess ||
        (e = cudaMemcpy(s->d_rec, rec.data(), rec.size() * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_off, doff.data(), doff.size() * sizeof(int), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_exptab, etab.data(), 256 * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_cistab, ctab.data(), 512 * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMalloc(&s->d_logtab, 128 * sizeof(double2))) != cudaSuccess ||
        (e = cudaMalloc(&s->d_atantab, 65 * sizeof(double))) != cudaSuccess ||
        (e = cudaMemcpy(s->d_logtab, ltab.data(), 256 * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(s->d_atantab, atab.data(), 65 * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess) {
        pht_system_destroy(s);
        return e == cudaErrorMemoryAllocation ? PHT_ENOMEM : cuda_fail(e);
    }
    // tensor-core evaluation tables: built for every affine system with n >= 10 (the AUTO policy
    // evaluates with DMMA from n = 11, profiles/r01_dense_tuning.txt), on demand otherwise
    // (pht_system_set_kernels(PHT_KERNELS_DENSE))
    if (n >= 10 && !proj) {
        const int rc = build_dense(s);
        if (rc != PHT_OK && rc != PHT_EUNSUPPORTED) { // (unsupported: > 65,535 n-tiles; no DMMA tables)
            pht_system_destroy(s);
            return rc;
        }
    }
    *out = s;
    return PHT_OK;
}

extern "C" int pht_system_create(int32_t n_eq, int32_t n_var, const int64_t *off, const int32_t *exps,
                                 const double *coeffs, const double *lifting, int32_t device,
                                 pht_system **out)
{
    return create_impl(n_eq, n_var, off, exps, coeffs, lifting, device, out, false);
}

extern "C" int pht_system_create_projective(int32_t n_eq, int32_t n_var, const int64_t *off, const int32_t *exps,
                                            const double *coeffs, const double *lifting, int32_t device,
                                            pht_system **out)
{
    return create_impl(n_eq, n_var, off, exps, coeffs, lifting, device, out, true);
}

extern "C" void pht_system_destroy(pht_system *s)
{
    if (!s) return;
    DevGuard g(s->device);
    // host steps still in flight (pht_pc_step_host_async without pht_host_wait) finish first:
    // their copies use the workspace, the events and the streams released below
    for (int u = 0; u < 4; ++u)
        if (s->hs[u]) cudaStreamSynchronize(s->hs[u]);
    cudaFree(s->d_rec);
    cudaFree(s->d_off);
    cudaFree(s->d_exptab);
    cudaFree(s->d_cistab);
    cudaFree(s->d_logtab);
    cudaFree(s->d_atantab);
    cudaFree(s->d_b2phi);
    cudaFree(s->d_b2th);
    cudaFree(s->d_b4);
    cudaFree(s->d_tinfo);
    cudaFree(s->ws);
    for (int u = 0; u < 4; ++u)
        if (s->hs[u]) cudaStreamDestroy(s->hs[u]);
    for (int c = 0; c < 64; ++c) {
        if (s->hev_in[c]) cudaEventDestroy(s->hev_in[c]);
        if (s->hev_k[c]) cudaEventDestroy(s->hev_k[c]);
        if (s->hev_out[c]) cudaEventDestroy(s->hev_out[c]);
    }
    if (s->hev0) cudaEventDestroy(s->hev0);
    if (s->hev_end) cudaEventDestroy(s->hev_end);
    pht::jit_free(s->jit);
    for (pht::JitKernels *J : s->jit_old) pht::jit_free(J);
    delete s;
}

extern "C" int pht_system_info(const pht_system *s, int32_t *n, int64_t *M, int32_t *max_terms,
                               int32_t *device)
{
    if (!s) return PHT_EINVAL;
    if (n) *n = s->n;
    if (M) *M = s->M;
    if (max_terms) *max_terms = s->max_terms;
    if (device) *device = s->device;
    return PHT_OK;
}

extern "C" int pht_system_flags(const pht_system *s)
{
    if (!s) return PHT_EINVAL;
    int f = s->dense ? PHT_SYS_DENSE : 0;
    if (s->jit) f |= PHT_SYS_SPECIALIZED;
    if (s->proj) f |= PHT_SYS_PROJECTIVE;
    return f;
}

extern "C" int pht_system_set_solver(pht_system *s, int32_t solver)
{
    if (!s || (solver != PHT_SOLVER_LU && solver != PHT_SOLVER_QR)) return PHT_EINVAL;
    s->solver = solver;
    return PHT_OK;
}

extern "C" int pht_system_set_kernels(pht_system *s, int32_t family)
{
    if (!s || family < PHT_KERNELS_AUTO || family > PHT_KERNELS_LANE) return PHT_EINVAL;
    if (family == PHT_KERNELS_DENSE) {
        if (s->proj) return PHT_EUNSUPPORTED;
        const int rc = build_dense(s);
        if (rc != PHT_OK) return rc;
    }
    if (family == PHT_KERNELS_SPECIALIZED) {
        std::lock_guard<std::mutex> lk(s->jit_mu);
        if (!s->jit) return PHT_EUNSUPPORTED;
    }
    s->kernels = family;
    return PHT_OK;
}

extern "C" int pht_system_kernels(const pht_system *s) { return s ? s->kernels : PHT_EINVAL; }

static pht::JitKernels *jit_snapshot(const pht_system *s)
{
    std::lock_guard<std::mutex> lk(const_cast<pht_system *>(s)->jit_mu);
    return s->jit;
}

// System-specialised kernels (pht_jit.cu): generate, compile (NVRTC, sm_100a), load.
static thread_local std::string g_jit_log;

// Size of the straight-line code a system would generate: sum over terms of (nonzero exponents
// + 8).  Above the limit the compile takes minutes and the code overflows the instruction caches
// (random dense n = 20 x 50 terms: ~24,000 units, 288 s of NVRTC for the step kernels).
static const int64_t kJitCodeLimit = 8000;
static int64_t jit_code_units(int n, const std::vector<double> &rec, const std::vector<int> &off)
{
    const int RS = pht::rec_stride(n);
    int64_t u = 0;
    for (int i = 0; i < off.back(); ++i) {
        u += 8;
        for (int j = 0; j < n; ++j) u += rec[(size_t)i * RS + j] != 0.0;
    }
    return u;
}

extern "C" int pht_system_specialize(pht_system *s, int32_t what)
{
    if (!s) return PHT_EINVAL;
    if (what == 0) what = PHT_SPEC_ALL;
    if (what & ~PHT_SPEC_ALL) return PHT_EINVAL;
    if (jit_code_units(s->n, s->h_rec, s->h_off) > kJitCodeLimit) return PHT_EUNSUPPORTED;
    std::lock_guard<std::mutex> lk(s->jit_mu);
    if (s->jit && (pht::jit_what(s->jit) & (unsigned)what) == (unsigned)what) return PHT_OK;
    const std::string src = pht::jit_source(s->n, s->h_rec, s->h_off);
    // process-wide cache of compiled images keyed by (generated source, kernel set): the same
    // system loaded again (another device, another handle) is not recompiled
    static std::mutex cache_mu;
    static std::map<std::string, std::pair<std::vector<char>, std::vector<std::string>>> cache;
    const std::string key = std::to_string(what) + "|" + src;
    std::vector<char> cubin;
    std::vector<std::string> names;
    {
        std::lock_guard<std::mutex> ck(cache_mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            cubin = it->second.first;
            names = it->second.second;
        }
    }
    if (cubin.empty()) {
        if (pht::jit_compile(s->n, src, (unsigned)what, cubin, names, g_jit_log) != 0) {
            g_cuda_err = "NVRTC: " + g_jit_log;
            return PHT_EJIT;
        }
        std::lock_guard<std::mutex> ck(cache_mu);
        cache[key] = {cubin, names};
    }
    DevGuard g(s->device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    cudaError_t e = cudaSuccess;
    pht::JitKernels *J = pht::jit_load(s->n, (unsigned)what, cubin, names, &e);
    if (!J) return cuda_fail(e);
    // the previous image may still be referenced by queued launches: unload it at destroy
    if (s->jit) s->jit_old.push_back(s->jit);
    s->jit = J;
    return PHT_OK;
}

extern "C" int pht_specialize_compile(int32_t n_eq, int32_t n_var, const int64_t *off, const int32_t *exps,
                                      const double *coeffs, const double *lifting, int32_t what,
                                      int64_t *cubin_bytes)
{
    std::vector<double> rec;
    std::vector<int> doff;
    int max_terms = 0, n_dropped = 0;
    int64_t M = 0;
    const int prc = pack_system(n_eq, n_var, off, exps, coeffs, lifting, rec, doff, max_terms, M, n_dropped);
    if (prc != PHT_OK) return prc;
    if (what == 0) what = PHT_SPEC_ALL;
    if (what & ~PHT_SPEC_ALL) return PHT_EINVAL;
    const std::string src = pht::jit_source(n_eq, rec, doff);
    std::vector<char> cubin;
    std::vector<std::string> names;
    if (pht::jit_compile(n_eq, src, (unsigned)what, cubin, names, g_jit_log) != 0) {
        g_cuda_err = "NVRTC: " + g_jit_log;
        return PHT_EJIT;
    }
    if (cubin_bytes) *cubin_bytes = (int64_t)cubin.size();
    return PHT_OK;
}

extern "C" int64_t pht_specialize_source(int32_t n_eq, int32_t n_var, const int64_t *off, const int32_t *exps,
                                         const double *coeffs, const double *lifting, char *buf, int64_t cap)
{
    std::vector<double> rec;
    std::vector<int> doff;
    int max_terms = 0, n_dropped = 0;
    int64_t M = 0;
    const int prc = pack_system(n_eq, n_var, off, exps, coeffs, lifting, rec, doff, max_terms, M, n_dropped);
    if (prc != PHT_OK) return prc;
    const std::string src = pht::jit_source(n_eq, rec, doff);
    if (buf && cap > 0) {
        const size_t c = std::min((size_t)cap - 1, src.size());
        memcpy(buf, src.data(), c);
        buf[c] = 0;
    }
    return (int64_t)src.size() + 1;
}

// Kernel choice per entry point (family = PHT_KERNELS_*, pht_system_set_kernels).  AUTO, the
// measured-best policy (DESIGN.md §3b/§3c, profiles/r01_dense_tuning.txt, r01_specialize.txt):
//   evaluation   specialised kernels if loaded; FP64 tensor cores (k_dense) for n >= 11 and for
//                pht_evaluate_log when the dense tables exist (n >= 10); else k_stepw<N, EVAL_X>
//                (n <= 12) or the tile kernel k_phte
//   directions / step   k_stepw for 10 <= n <= 12 (cyclic-10 604 vs 487 specialised, noon-10 578
//                vs 492, katsura-10 356 vs 344 M evals/s); the specialised tile kernel below n = 10
//                when loaded (cyclic-5 3080 vs 2760); else k_stepw (n <= 12) or k_pht
// A forced family applies wherever it implements the entry point, AUTO elsewhere.
// complex arrays are read and written as 16-byte vectors (double2), real arrays as doubles: a
// misaligned pointer would fault the context, so it is refused up front (PHT_EINVAL)
static bool al16(const void *p) { return ((uintptr_t)p & 15u) == 0; }
static bool al8(const void *p) { return ((uintptr_t)p & 7u) == 0; }

static int dispatch(const pht_system *s, int mode, const pht::Args &A0, void *stream)
{
    if (A0.P == 0) return PHT_OK;
    DevGuard g(s->device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    pht::DevSys S{s->d_rec, s->d_off, s->d_exptab, s->d_cistab, s->n, s->proj, s->max_terms, s->d_logtab, s->d_atantab};
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    pht::Args A = A0;
    A.solver = s->solver;
    const int fam = s->kernels;
    const bool evalm = mode == pht::MODE_EVAL_X || mode == pht::MODE_EVAL_Z;
    const unsigned need = evalm ? pht::JIT_EVAL : pht::JIT_STEP;
    const bool warp_step = s->n >= 10 && s->n <= 12 && !s->proj && s->solver == PHT_SOLVER_LU;
    pht::JitKernels *J = jit_snapshot(s);
    const bool jit_ok = J && (pht::jit_what(J) & need);
    bool use_jit = false;
    if (jit_ok) {
        if (fam == PHT_KERNELS_SPECIALIZED) use_jit = true;
        // AUTO: the generic point-per-lane evaluation (k_evalw, 6 <= n <= 12) beats the specialised
        // evaluation (cyclic-10 1.06 vs 0.81 G points/s); the specialised step below n = 10
        else if (fam == PHT_KERNELS_AUTO) use_jit = evalm ? (s->n < 6 || s->n > 12 || s->proj) : !warp_step;
    }
    if (use_jit) {
        e = pht::jit_launch(J, mode, S, A, st);
        if (e != cudaSuccess) return cuda_fail(e);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return PHT_OK;
    }
    bool dense = false;
    if (evalm && s->dense) {
        if (fam == PHT_KERNELS_DENSE) dense = true;
        else if (fam == PHT_KERNELS_AUTO || fam == PHT_KERNELS_SPECIALIZED) dense = s->n > 12;
    }
    const int lfam = fam == PHT_KERNELS_TILE ? pht::FAM_TILE : pht::FAM_AUTO;
    const pht::DenseSys D{s->d_b2phi, s->d_b2th, s->d_b4, s->d_tinfo, s->dense_ntiles, s->max_ntk};
    // point-per-lane evaluation (k_evalw): LANE for n <= 12, AUTO for 6 <= n <= 12 (measured, one B200,
    // G points/s: cyclic-10 1.06 vs 0.76 warp-per-group vs 0.62 tensor cores, noon-10 0.96 / 0.71 /
    // 0.61, katsura-10 (n = 11) 0.70 / 0.44 / 0.58; cyclic-5 2.85 vs 3.31 for the warp-per-group
    // kernel, which stays the AUTO choice for pht_evaluate below n = 6; pht_evaluate_log: cyclic-5 2.92
    // vs 2.77 tile); PHT_KERNELS_WARP keeps k_stepw<N, EVAL_X>
    const bool lane_eval = evalm && !s->proj && s->n <= 12 && s->max_terms > 0 && !dense &&
                           (fam == PHT_KERNELS_LANE ||
                            ((fam == PHT_KERNELS_AUTO || fam == PHT_KERNELS_SPECIALIZED) &&
                             (s->n >= 6 || mode == pht::MODE_EVAL_Z)));
    if (lane_eval) {
        pht::EvalMaps M{};
        pht::encode_eval_maps(M, s->n, A.P, A.J, A.Jt, A.H);
        e = cudaErrorNotSupported;
        switch (s->n) {
#define PHT_CASE(N) case N: e = mode == pht::MODE_EVAL_X ? pht::launch_evalw<N, pht::MODE_EVAL_X>(S, A, M, st) \
                                                        : pht::launch_evalw<N, pht::MODE_EVAL_Z>(S, A, M, st); break;
            PHT_CASE(1) PHT_CASE(2) PHT_CASE(3) PHT_CASE(4) PHT_CASE(5) PHT_CASE(6) PHT_CASE(7)
            PHT_CASE(8) PHT_CASE(9) PHT_CASE(10) PHT_CASE(11) PHT_CASE(12)
#undef PHT_CASE
        default: break;
        }
        if (e != cudaErrorNotSupported) {
            if (e != cudaSuccess) return cuda_fail(e);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            return PHT_OK;
        }
        cudaGetLastError(); // (too many terms for shared memory: the kernels below)
    }
    switch (s->n) {
#define PHT_CASE(N) case N: e = dense ? pht::launch_dense<N>(mode, S, D, A, st) : pht::launch<N>(mode, S, A, st, lfam); break;
        PHT_CASE(1) PHT_CASE(2) PHT_CASE(3) PHT_CASE(4) PHT_CASE(5) PHT_CASE(6) PHT_CASE(7)
        PHT_CASE(8) PHT_CASE(9) PHT_CASE(10) PHT_CASE(11) PHT_CASE(12) PHT_CASE(13) PHT_CASE(14)
        PHT_CASE(15) PHT_CASE(16) PHT_CASE(17) PHT_CASE(18) PHT_CASE(19) PHT_CASE(20) PHT_CASE(21)
        PHT_CASE(22) PHT_CASE(23) PHT_CASE(24)
#undef PHT_CASE
    default: return PHT_ESHAPE;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return PHT_OK;
}

extern "C" int pht_evaluate(const pht_system *s, int64_t p, const double *x, const double *t, double *H,
                            double *Jx, double *Jt, int32_t *row_exp2, uint8_t *status, void *stream)
{
    if (!s || p < 0 || (p > 0 && (!x || !t))) return PHT_EINVAL;
    if (!al16(x) || !al8(t) || !al16(H) || !al16(Jx) || !al16(Jt) || ((uintptr_t)row_exp2 & 3u)) return PHT_EINVAL;
    pht::Args A{};
    A.P = p;
    A.xin = (const double2 *)x;
    A.tin = t;
    A.H = (double2 *)H;
    A.J = (double2 *)Jx;
    A.Jt = (double2 *)Jt;
    A.rexp = row_exp2;
    A.status = status;
    return dispatch(s, pht::MODE_EVAL_X, A, stream);
}

extern "C" int pht_evaluate_log(const pht_system *s, int64_t p, const double *z, const double *tau, double *H,
                                double *Jz, double *Jtau, int32_t *row_exp2, uint8_t *status, void *stream)
{
    if (!s || p < 0 || (p > 0 && (!z || !tau))) return PHT_EINVAL;
    if (!al16(z) || !al8(tau) || !al16(H) || !al16(Jz) || !al16(Jtau) || ((uintptr_t)row_exp2 & 3u)) return PHT_EINVAL;
    pht::Args A{};
    A.P = p;
    A.xin = (const double2 *)z;
    A.tin = tau;
    A.H = (double2 *)H;
    A.J = (double2 *)Jz;
    A.Jt = (double2 *)Jtau;
    A.rexp = row_exp2;
    A.status = status;
    return dispatch(s, pht::MODE_EVAL_Z, A, stream);
}

extern "C" int pht_euler_newton(const pht_system *s, int64_t p, const double *x, const double *t, double *dE,
                                double *dN, uint8_t *status, void *stream)
{
    if (!s || p < 0 || (p > 0 && (!x || !t))) return PHT_EINVAL;
    if (!al16(x) || !al8(t) || !al16(dE) || !al16(dN)) return PHT_EINVAL;
    pht::Args A{};
    A.P = p;
    A.xin = (const double2 *)x;
    A.tin = t;
    A.dE = (double2 *)dE;
    A.dN = (double2 *)dN;
    A.status = status;
    return dispatch(s, pht::MODE_DIRS, A, stream);
}

extern "C" int pht_pc_step(const pht_system *s, int64_t p, double *x, double *tau, const double *dtau,
                           int32_t newton_iters, uint8_t *status, double *dn_norm, void *stream)
{
    if (!s || p < 0 || newton_iters < 0 || (p > 0 && (!x || !tau || !dtau))) return PHT_EINVAL;
    if (!al16(x) || !al8(tau) || !al8(dtau) || !al8(dn_norm)) return PHT_EINVAL;
    pht::Args A{};
    A.P = p;
    A.xio = (double2 *)x;
    A.tauio = tau;
    A.dtau = dtau;
    A.K = newton_iters;
    A.status = status;
    A.dnnorm = dn_norm;
    return dispatch(s, pht::MODE_STEP, A, stream);
}

// Host-buffer step, pipelined (the batch pipelining of P:807-824 as stream
// overlap): the points are cut into chunks and run through a three-stage stream pipeline --
// copy-in stream (H2D of every chunk back to back), compute (the step kernel of chunk c once its
// copy-in event fired; two streams taken alternately so the tail of one chunk's persistent kernel
// overlaps the start of the next), copy-out stream (D2H of chunk c once its kernel event fired).
// Each copy engine direction then streams without waiting on the other (pinned host memory needed
// for overlap).  Round 2 had chunk c's H2D, kernel and D2H in one of 3 round-robin streams, so a
// chunk's copy-in queued behind the copy-out of the chunk three places earlier.
#define PHT_HOST_CHUNKS 32
static int ensure_streams(pht_system *s)
{
    if (s->hs[0]) return PHT_OK;
    for (int u = 0; u < 4; ++u) {
        cudaError_t e = cudaStreamCreateWithFlags(&s->hs[u], cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    for (int c = 0; c < 64; ++c) {
        cudaError_t e = cudaEventCreateWithFlags(&s->hev_in[c], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->hev_k[c], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->hev_out[c], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    cudaError_t e = cudaEventCreateWithFlags(&s->hev0, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->hev_end, cudaEventDisableTiming);
    return e == cudaSuccess ? PHT_OK : cuda_fail(e);
}

static int host_step(const pht_system *cs, int64_t p, double *x, double *tau, const double *dtau, int32_t newton_iters,
                     uint8_t *status, double *dn_norm, void *stream, bool async)
{
    pht_system *s = const_cast<pht_system *>(cs);
    if (!s || p < 0 || newton_iters < 0 || (p > 0 && (!x || !tau || !dtau))) return PHT_EINVAL;
    if (!al8(x) || !al8(tau) || !al8(dtau) || !al8(dn_norm)) return PHT_EINVAL; // host buffers (copied)
    if (p == 0) return PHT_OK;
    std::lock_guard<std::mutex> lk(s->ws_mu);
    DevGuard g(s->device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    const int n = s->n;
    const size_t bx = (size_t)p * n * 16, bt = (size_t)p * 8, bs = (size_t)p;
    const size_t need = bx + 3 * bt + bs + 64;
    cudaError_t e;
    if ((int64_t)need > s->ws_cap) {
        if (s->hs[3] && (e = cudaStreamSynchronize(s->hs[3])) != cudaSuccess) return cuda_fail(e); // in-flight async steps
        cudaFree(s->ws);
        s->ws = nullptr;
        s->ws_cap = 0;
        if ((e = cudaMalloc(&s->ws, need)) != cudaSuccess) return e == cudaErrorMemoryAllocation ? PHT_ENOMEM : cuda_fail(e);
        s->ws_cap = (int64_t)need;
    }
    int rc = ensure_streams(s);
    if (rc != PHT_OK) return rc;
    char *w = (char *)s->ws;
    double *dx = (double *)w, *dtu = (double *)(w + bx), *ddt = (double *)(w + bx + bt),
           *ddn = (double *)(w + bx + 2 * bt);
    uint8_t *dst = (uint8_t *)(w + bx + 3 * bt);
    cudaStream_t st = (cudaStream_t)stream;
    cudaStream_t sin = s->hs[0], sout = s->hs[3];
    // the caller's stream orders us after its earlier work; we order it after our copies
    if ((e = cudaEventRecord(s->hev0, st)) != cudaSuccess) return cuda_fail(e);
    for (int u = 0; u < 4; ++u)
        if ((e = cudaStreamWaitEvent(s->hs[u], s->hev0, 0)) != cudaSuccess) return cuda_fail(e);
    // chunks: 1/32 of the batch, at least 32K points (launch and copy latency stay amortised); the
    // pipeline fill (first copy-in) and drain (last copy-out) are one chunk each
    int64_t chunk = (p + PHT_HOST_CHUNKS - 1) / PHT_HOST_CHUNKS;
    if (chunk < 32768) chunk = 32768;
    const int nch = (int)((p + chunk - 1) / chunk);
    // a previous host step may still be in flight (pht_pc_step_host_async): chunk c's copy-in
    // overwrites the workspace range (and the host x / tau) that step's chunk c copies out, so it
    // waits for that copy-out; a different point count (other chunking) waits for the whole step
    const bool chain = s->hprev_p == p && s->hprev_nch == nch;
    if (s->hprev_p >= 0 && !chain && (e = cudaStreamWaitEvent(sin, s->hev_end, 0)) != cudaSuccess) return cuda_fail(e);
    int c = 0;
    for (int64_t b = 0; b < p; b += chunk, ++c) {
        const int64_t m = (p - b < chunk) ? p - b : chunk;
        if (chain && (e = cudaStreamWaitEvent(sin, s->hev_out[c], 0)) != cudaSuccess) return cuda_fail(e);
        const size_t ox = (size_t)b * n * 2, mx = (size_t)m * n * 16, mt = (size_t)m * 8;
        cudaStream_t sk = s->hs[1 + (c & 1)];
        if ((e = cudaMemcpyAsync(dx + ox, x + ox, mx, cudaMemcpyHostToDevice, sin)) != cudaSuccess ||
            (e = cudaMemcpyAsync(dtu + b, tau + b, mt, cudaMemcpyHostToDevice, sin)) != cudaSuccess ||
            (e = cudaMemcpyAsync(ddt + b, dtau + b, mt, cudaMemcpyHostToDevice, sin)) != cudaSuccess ||
            (e = cudaEventRecord(s->hev_in[c], sin)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(sk, s->hev_in[c], 0)) != cudaSuccess)
            return cuda_fail(e);
        rc = pht_pc_step(s, m, dx + ox, dtu + b, ddt + b, newton_iters, dst + b, ddn + b, (void *)sk);
        if (rc != PHT_OK) return rc;
        if ((e = cudaEventRecord(s->hev_k[c], sk)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(sout, s->hev_k[c], 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(x + ox, dx + ox, mx, cudaMemcpyDeviceToHost, sout)) != cudaSuccess ||
            (e = cudaMemcpyAsync(tau + b, dtu + b, mt, cudaMemcpyDeviceToHost, sout)) != cudaSuccess ||
            (status && (e = cudaMemcpyAsync(status + b, dst + b, (size_t)m, cudaMemcpyDeviceToHost, sout)) != cudaSuccess) ||
            (dn_norm && (e = cudaMemcpyAsync(dn_norm + b, ddn + b, mt, cudaMemcpyDeviceToHost, sout)) != cudaSuccess) ||
            (e = cudaEventRecord(s->hev_out[c], sout)) != cudaSuccess)
            return cuda_fail(e);
    }
    s->hprev_p = p;
    s->hprev_nch = nch;
    // every chunk's copy-out is on sout, after its kernel; the caller's stream waits for the last
    // (the asynchronous variant leaves that to pht_host_wait)
    if ((e = cudaEventRecord(s->hev_end, sout)) != cudaSuccess) return cuda_fail(e);
    if (async) return PHT_OK;
    if ((e = cudaStreamWaitEvent(st, s->hev_end, 0)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e);
    return PHT_OK;
}

extern "C" int pht_pc_step_host(const pht_system *cs, int64_t p, double *x, double *tau, const double *dtau,
                                int32_t newton_iters, uint8_t *status, double *dn_norm, void *stream)
{
    return host_step(cs, p, x, tau, dtau, newton_iters, status, dn_norm, stream, false);
}

extern "C" int pht_pc_step_host_async(const pht_system *cs, int64_t p, double *x, double *tau, const double *dtau,
                                      int32_t newton_iters, uint8_t *status, double *dn_norm, void *stream)
{
    return host_step(cs, p, x, tau, dtau, newton_iters, status, dn_norm, stream, true);
}

extern "C" int pht_host_wait(const pht_system *cs, void *stream)
{
    pht_system *s = const_cast<pht_system *>(cs);
    if (!s) return PHT_EINVAL;
    std::lock_guard<std::mutex> lk(s->ws_mu);
    if (!s->hs[0] || s->hprev_p < 0) return PHT_OK; // no host step yet
    DevGuard g(s->device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if ((e = cudaStreamWaitEvent(st, s->hev_end, 0)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e);
    return PHT_OK;
}

// Affine points -> P^n (pht_homogenize): y = (x, 1) / ||(x, 1)||, x = e^z for log input.
// One thread per point; coordinates scaled by the largest magnitude before the norm.
__global__ void k_homogenize(int64_t p, int n, const double2 *x, int log_input, double2 *y)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= p) return;
    const double2 *xq = x + q * n;
    double lmax = 0.0; // log of the largest |coordinate| (the appended 1 included)
    for (int j = 0; j < n; ++j) {
        const double2 v = xq[j];
        lmax = fmax(lmax, log_input ? v.x : log(hypot(v.x, v.y)));
    }
    double s2 = 0.0;
    double2 *yq = y + q * (n + 1);
    for (int j = 0; j <= n; ++j) {
        double2 u;
        if (j == n) u = make_double2(exp(-lmax), 0.0);
        else if (log_input) {
            double sn, cs;
            sincos(xq[j].y, &sn, &cs);
            const double m = exp(xq[j].x - lmax);
            u = make_double2(m * cs, m * sn);
        } else {
            const double f = exp(-lmax);
            u = make_double2(xq[j].x * f, xq[j].y * f);
        }
        yq[j] = u;
        s2 = fma(u.x, u.x, fma(u.y, u.y, s2));
    }
    const double f = rsqrt(s2);
    for (int j = 0; j <= n; ++j) yq[j] = make_double2(yq[j].x * f, yq[j].y * f);
}

extern "C" int pht_homogenize(const pht_system *s, int64_t p, const double *x, int32_t log_input, double *y,
                              void *stream)
{
    if (!s || !s->proj || p < 0 || (p > 0 && (!x || !y))) return PHT_EINVAL;
    if (!al16(x) || !al16(y)) return PHT_EINVAL;
    if (p == 0) return PHT_OK;
    DevGuard g(s->device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    const int threads = 128;
    k_homogenize<<<(unsigned)((p + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
        p, s->n - 1, (const double2 *)x, log_input, (double2 *)y);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return PHT_OK;
}

extern "C" void pht_track_opts_default(pht_track_opts *o)
{
    if (!o) return;
    o->dtau_init = 0.05;
    o->dtau_min = 1e-12;
    o->dtau_max = 0.5;
    o->newton_tol = 1e-10;
    o->shrink = 0.5;
    o->grow = 2.0;
    o->final_tol = 1e-13;
    o->inf_norm = 1e8;
    o->newton_iters = 4;
    o->grow_after = 3;
    o->max_steps = 10000;
    o->final_iters = 5;
    o->log_state = 0;
    o->pred_log = -1;
    o->predictor = 0;
    o->pred_tol = 0.0; // classic grow_after rule (measured best, profiles/r01_tracker_control.txt)
    o->reuse_tangent = 0;
}

static int track_impl(const pht_system *s, int64_t p, double *x, double *tau, const double *cellw, int64_t ncells,
                      const int32_t *path_cell, const pht_track_opts *opts, int64_t *stats, uint8_t *status,
                      void *stream)
{
    if (!s || p < 0 || (p > 0 && (!x || !tau || !status))) return PHT_EINVAL;
    if (!al16(x) || !al8(tau) || !al8(stats) || !al8(cellw) || ((uintptr_t)path_cell & 3u)) return PHT_EINVAL;
    if (cellw && (!path_cell || ncells < 1 || ncells > INT32_MAX || s->dropped)) return PHT_EINVAL;
    if (p == 0) return PHT_OK;
    pht_track_opts o;
    if (opts) o = *opts;
    else pht_track_opts_default(&o);
    if (cellw) o.log_state = 1; // cell coordinates w are logarithmic
    if (s->proj && (cellw || o.log_state)) return PHT_EUNSUPPORTED; // projective: y state only
    if (s->proj) o.pred_log = 0;
    if (!(o.dtau_init > 0) || !(o.dtau_min > 0) || !(o.dtau_max > 0) || !(o.shrink > 0 && o.shrink < 1) ||
        !(o.grow >= 1) || o.newton_iters < 1 || o.grow_after < 1 || o.max_steps < 1 || o.final_iters < 1)
        return PHT_EINVAL;
    DevGuard g(s->device);
    if (!g.ok) return cuda_fail(cudaGetLastError());
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *ctr = nullptr;
    cudaError_t e;
    if ((e = cudaMallocAsync((void **)&ctr, sizeof(unsigned long long), st)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st)) != cudaSuccess) return cuda_fail(e);
    pht::DevSys S{s->d_rec, s->d_off, s->d_exptab, s->d_cistab, s->n, s->proj, s->max_terms, s->d_logtab, s->d_atantab};
    pht::TrackArgs A{};
    A.P = p;
    A.x = (double2 *)x;
    A.tau = tau;
    A.status = status;
    A.stats = (long long *)stats;
    A.queue = ctr;
    A.cellw = cellw;
    A.path_cell = path_cell;
    A.ncells = (int)ncells;
    A.M = (int)s->M;
    A.solver = s->solver;
    A.o = pht::TrackOpts{o.dtau_init, o.dtau_min, o.dtau_max, o.newton_tol, o.shrink, o.grow, o.final_tol,
                         o.inf_norm, o.newton_iters, o.grow_after, o.max_steps, o.final_iters, o.log_state,
                         o.pred_log < 0 ? o.log_state : o.pred_log, o.pred_tol, o.predictor, o.reuse_tangent};
    // AUTO: the warp-per-group tracker (k_trackw: n <= 12, LU, affine, Euler predictor) is faster
    // than the specialised tile tracker, which serves only where k_trackw does not apply and the
    // batch fills at least one wave of its (2-3x larger) tiles (measured: 70 paths 4x slower)
    const int fam = s->kernels;
    const bool warp_track = s->n <= 12 && !s->proj && s->solver == PHT_SOLVER_LU && o.predictor != 1;
    pht::JitKernels *J = jit_snapshot(s);
    const bool jit_ok = J && (pht::jit_what(J) & pht::JIT_TRACK);
    const bool use_jit = jit_ok && (fam == PHT_KERNELS_SPECIALIZED ||
                                    (fam == PHT_KERNELS_AUTO && !warp_track && p >= pht::jit_track_slots(J, s->sms)));
    const int lfam = fam == PHT_KERNELS_TILE ? pht::FAM_TILE : pht::FAM_AUTO;
    if (use_jit)
        e = pht::jit_launch_track(J, S, A, st, s->sms);
    else switch (s->n) {
#define PHT_CASE(N) case N: e = pht::launch_track<N>(S, A, st, s->sms, lfam); break;
        PHT_CASE(1) PHT_CASE(2) PHT_CASE(3) PHT_CASE(4) PHT_CASE(5) PHT_CASE(6) PHT_CASE(7)
        PHT_CASE(8) PHT_CASE(9) PHT_CASE(10) PHT_CASE(11) PHT_CASE(12) PHT_CASE(13) PHT_CASE(14)
        PHT_CASE(15) PHT_CASE(16) PHT_CASE(17) PHT_CASE(18) PHT_CASE(19) PHT_CASE(20) PHT_CASE(21)
        PHT_CASE(22) PHT_CASE(23) PHT_CASE(24)
#undef PHT_CASE
    default: e = cudaErrorInvalidValue;
    }
    cudaError_t e2 = cudaFreeAsync(ctr, st);
    if (e != cudaSuccess) return cuda_fail(e);
    if (e2 != cudaSuccess) return cuda_fail(e2);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return PHT_OK;
}

extern "C" int pht_track(const pht_system *s, int64_t p, double *x, double *tau, const pht_track_opts *opts,
                         int64_t *stats, uint8_t *status, void *stream)
{
    return track_impl(s, p, x, tau, nullptr, 0, nullptr, opts, stats, status, stream);
}

extern "C" int pht_track_cells(const pht_system *s, int64_t p, double *w, double *tau, const double *cell_lift,
                               int64_t ncells, const int32_t *path_cell, const pht_track_opts *opts,
                               int64_t *stats, uint8_t *status, void *stream)
{
    if (!cell_lift) return PHT_EINVAL;
    return track_impl(s, p, w, tau, cell_lift, ncells, path_cell, opts, stats, status, stream);
}

extern "C" int64_t pht_launch_count(void) { return g_launches.load(); }

extern "C" const char *pht_last_cuda_error(void) { return g_cuda_err.c_str(); }

extern "C" const char *pht_strerror(int code)
{
    switch (code) {
    case PHT_OK: return "ok";
    case PHT_EINVAL: return "invalid argument";
    case PHT_ESHAPE: return "shape error (square n in [1, PHT_MAX_N], monotone offsets)";
    case PHT_EDUPLICATE: return "duplicate (monomial, lifting) term in an equation";
    case PHT_EEMPTY: return "equation without a nonzero term";
    case PHT_ERANGE: return "exponent or lifting out of range";
    case PHT_ECUDA: return "CUDA error";
    case PHT_ENOMEM: return "out of memory";
    case PHT_EUNSUPPORTED: return "unsupported";
    case PHT_EJIT: return "run-time compilation of the specialised kernels failed (log: pht_last_cuda_error)";
    default: return "unknown error";
    }
}

extern "C" int pht_version(void) { return 4; }
