// microbench.cu — B200 FP64 microbenchmarks used to set the roofline denominators and to guide
// the kernel design.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -o microbench tools/microbench.cu ; run on the GPU box.  Prints one JSON object.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e_)); return 1; } } while (0)

// DFMA throughput: ILP independent chains per thread
template <int ILP>
__global__ void k_dfma(double *out, int iters, double a, double b)
{
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 123.456) out[0] = s;
}

// dependent-chain latency: one warp, clock64 around a chain
__global__ void k_dfma_lat(double *out, long long *cyc, int iters, double a, double b)
{
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    if (x == 123.456) out[0] = x;
}

__device__ __forceinline__ double2 libexpcis(double y, double th)
{
    double s, c;
    sincos(th, &s, &c);
    double m = exp(y);
    return make_double2(m * c, m * s);
}

__global__ void k_libexpcis(double *out, int iters)
{
    double y = -threadIdx.x * 1e-3, th = threadIdx.x * 1e-2 + 0.3;
    double2 acc = make_double2(0, 0);
    for (int it = 0; it < iters; ++it) {
        double2 w = libexpcis(y, th);
        acc.x += w.x; acc.y += w.y;
        y -= 1e-4; th += 0.37;
    }
    if (acc.x == 123.456) out[0] = acc.y;
}

__global__ void k_loglat(double *out, int iters)
{
    double x = 1.5 + threadIdx.x * 1e-3, y = 0.7, acc = 0;
    for (int it = 0; it < iters; ++it) {
        acc += 0.5 * log(fma(x, x, y * y)) + atan2(y, x);
        x += 1e-4; y -= 1e-4;
    }
    if (acc == 123.456) out[0] = acc;
}

// FP64 tensor core: mma.sync m8n8k4 f64 (lowers to DMMA on sm_100a), ILP independent accumulators
template <int ILP>
__global__ void k_dmma(double *out, int iters)
{
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
    double c[ILP][2];
#pragma unroll
    for (int i = 0; i < ILP; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
    if (s == 123.456) out[0] = s;
}

// conversion throughput: int32 -> double (I2F.F64), float -> double (F2F.F64.F32), and the
// magic-number int -> double (IADD + DADD), ILP 8 independent chains
template <int KIND>
__global__ void k_conv(double *out, int iters)
{
    int iv[8];
    float fv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { iv[i] = threadIdx.x + i; fv[i] = 0.5f * (threadIdx.x + i); }
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double d;
            if (KIND == 0) d = (double)iv[i];
            else if (KIND == 1) d = (double)fv[i];
            else d = __hiloint2double(0x43380000, iv[i] + 0x7fffffff) - 6755401602162687.0; // 2^52+2^51 bias
            acc[i] += d;
            iv[i] += 3;
            fv[i] += 1.0f;
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 123.456) out[0] = s;
}

// shared-memory LDS.128 with DISTINCT 16-byte addresses per warp (1, 3, 8, 32): cycles per warp load
template <int DISTINCT>
__global__ void k_lds(double *out, int iters)
{
    __shared__ double2 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_double2(i, -i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int idx = (lane % DISTINCT) * 7 % 1024;     // stride 7 (odd): distinct banks
    double2 acc = make_double2(0, 0);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 v = buf[(idx + u * 64) & 1023];
            acc.x += v.x;
            acc.y += v.y;
        }
        idx = (idx + 8) & 1023;
    }
    if (acc.x == 123.456) out[0] = acc.y;
}

int main()
{
    double *d;
    long long *c;
    CK(cudaMalloc(&d, 64));
    CK(cudaMalloc(&c, 64));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int mhz = 0;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    printf("{\"sms\": %d, \"clock_khz\": %d", sms, mhz);
    // throughput: 148*8 blocks x 256 threads, ILP 8
    {
        const int iters = 20000, blocks = sms * 8, threads = 256;
        k_dfma<8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_dfma<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)blocks * threads;
        printf(", \"dfma_tflops\": %.3f", flops / (ms * 1e-3) / 1e12);
    }
    // throughput vs warps per SM with ILP 1 (latency hiding curve)
    printf(", \"dfma_tflops_ilp1_by_warps_per_sm\": {");
    for (int wps = 2; wps <= 32; wps *= 2) {
        const int iters = 20000, blocks = sms, threads = 32 * wps;
        k_dfma<1><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dfma<1><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * iters * (double)blocks * threads;
        printf("%s\"%d\": %.3f", wps == 2 ? "" : ", ", wps, flops / (ms * 1e-3) / 1e12);
    }
    printf("}");
    printf(", \"dfma_tflops_ilp2_by_warps_per_sm\": {");
    for (int wps = 2; wps <= 32; wps *= 2) {
        const int iters = 20000, blocks = sms, threads = 32 * wps;
        k_dfma<2><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dfma<2><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 2 * iters * (double)blocks * threads;
        printf("%s\"%d\": %.3f", wps == 2 ? "" : ", ", wps, flops / (ms * 1e-3) / 1e12);
    }
    printf("}");
    {
        k_dfma_lat<<<1, 32>>>(d, c, 1000, 1.0000001, 1e-9);
        CK(cudaDeviceSynchronize());
        long long cy;
        cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf(", \"dfma_latency_cycles\": %.2f", cy / 4000.0);
    }
    {
        const int iters = 2000, blocks = sms * 4, threads = 256;
        k_libexpcis<<<blocks, threads>>>(d, 10);
        cudaEventRecord(e0);
        k_libexpcis<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"libdevice_exp_sincos_G_per_s\": %.3f", iters * (double)blocks * threads / (ms * 1e-3) / 1e9);
    }
    {
        const int iters = 2000, blocks = sms * 4, threads = 256;
        k_loglat<<<blocks, threads>>>(d, 10);
        cudaEventRecord(e0);
        k_loglat<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"libdevice_log_atan2_G_per_s\": %.3f", iters * (double)blocks * threads / (ms * 1e-3) / 1e9);
    }
    {
        const int iters = 20000, blocks = sms * 4, threads = 256;
        k_dmma<4><<<blocks, threads>>>(d, 10);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_dmma<4><<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        // each warp-level m8n8k4 = 8*8*4 = 256 FMAs = 512 flops
        double flops = 512.0 * 4 * iters * (double)blocks * (threads / 32);
        printf(", \"dmma_tflops\": %.3f", flops / (ms * 1e-3) / 1e12);
    }
    // co-issue: DMMA and DFMA kernels on two streams at the same time (only
    // worth splitting work across the tensor and FP64 pipes if the two overlap)
    {
        const int iters = 20000, blocks = sms * 4, threads = 256;
        cudaStream_t s1, s2;
        cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
        cudaEvent_t a0, a1;
        cudaEventCreate(&a0);
        cudaEventCreate(&a1);
        float ms_m, ms_f, ms_b;
        cudaEventRecord(a0, s1);
        k_dmma<4><<<blocks, threads, 0, s1>>>(d, iters);
        cudaEventRecord(a1, s1);
        CK(cudaEventSynchronize(a1));
        cudaEventElapsedTime(&ms_m, a0, a1);
        cudaEventRecord(a0, s1);
        k_dfma<8><<<blocks, threads, 0, s1>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(a1, s1);
        CK(cudaEventSynchronize(a1));
        cudaEventElapsedTime(&ms_f, a0, a1);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a0, 0);
        cudaEvent_t j0;
        cudaEventCreate(&j0);
        cudaEventRecord(j0, 0);
        cudaStreamWaitEvent(s1, j0, 0);
        cudaStreamWaitEvent(s2, j0, 0);
        k_dmma<4><<<blocks / 2, threads, 0, s1>>>(d, iters);
        k_dfma<8><<<blocks / 2, threads, 0, s2>>>(d, iters, 1.0000001, 1e-9);
        cudaEvent_t e1s, e2s;
        cudaEventCreate(&e1s);
        cudaEventCreate(&e2s);
        cudaEventRecord(e1s, s1);
        cudaEventRecord(e2s, s2);
        cudaStreamWaitEvent(0, e1s, 0);
        cudaStreamWaitEvent(0, e2s, 0);
        cudaEventRecord(a1, 0);
        CK(cudaEventSynchronize(a1));
        cudaEventElapsedTime(&ms_b, a0, a1);
        // half of each workload together vs the sum of the halves alone (ms_m/2 + ms_f/2)
        printf(", \"coissue\": {\"dmma_ms\": %.3f, \"dfma_ms\": %.3f, \"half_each_concurrent_ms\": %.3f, "
               "\"half_each_serial_ms\": %.3f}", ms_m, ms_f, ms_b, 0.5 * (ms_m + ms_f));
    }
    // conversions (G ops per second over the whole GPU)
    {
        const char *names[3] = {"i2f_f64", "f2f_f64_f32", "magic_int_to_f64"};
        printf(", \"conversions_G_per_s\": {");
        for (int kind = 0; kind < 3; ++kind) {
            const int iters = 20000, blocks = sms * 4, threads = 256;
            void (*k)(double *, int) = kind == 0 ? k_conv<0> : (kind == 1 ? k_conv<1> : k_conv<2>);
            k<<<blocks, threads>>>(d, 10);
            cudaEventRecord(e0);
            k<<<blocks, threads>>>(d, iters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s\"%s\": %.1f", kind ? ", " : "", names[kind], 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e9);
        }
        printf("}");
    }
    // LDS.128: warp loads per SM per cycle, by distinct addresses in the warp
    {
        printf(", \"lds128_warp_loads_per_sm_cycle\": {");
        const int ds[4] = {1, 3, 8, 32};
        for (int u = 0; u < 4; ++u) {
            const int iters = 20000, blocks = sms * 4, threads = 256;
            void (*k)(double *, int) = u == 0 ? k_lds<1> : (u == 1 ? k_lds<3> : (u == 2 ? k_lds<8> : k_lds<32>));
            k<<<blocks, threads>>>(d, 10);
            cudaEventRecord(e0);
            k<<<blocks, threads>>>(d, iters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double loads = 8.0 * iters * (double)blocks * (threads / 32);
            const double cyc = ms * 1e-3 * mhz * 1e3 * sms;
            printf("%s\"%d\": %.3f", u ? ", " : "", ds[u], loads / cyc);
        }
        printf("}");
    }
    printf("}\n");
    return 0;
}
