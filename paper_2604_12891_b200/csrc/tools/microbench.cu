// microbench.cu -- measured per-chip issue peaks used as roofline denominators by bench.py for
// the stages that are bound by the SFU (MUFU.EX2) or the FMA pipe rather than by HBM or the
// tensor cores ("Add ex2-throughput and FFMA-throughput microbenchmarks to the bench
// so these derived peaks are measured, not assumed").  Built as libtcl_microbench.so; not part of
// the scoring path.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256) k_ex2(float* out, int iters, float seed) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j) * 1e-6f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float seed) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j);
    const float b = 0.999f, c = 1e-3f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_ffma2(float* out, int iters, float seed) {
    float2 a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = make_float2(seed * (threadIdx.x + j), seed * j);
    const float2 b = make_float2(0.999f, 0.998f), c = make_float2(1e-3f, 2e-3f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __ffma2_rn(a[j], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y;
    if (s == 12345.f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_tanh(float* out, int iters, float seed) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j) * 1e-6f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a[j]));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.f) out[0] = s;
}

extern "C" {
// Returns ops/s over the whole chip (0: MUFU.EX2, 1: FFMA, 2: FFMA2 (2 per lane), 3: MUFU.TANH);
// < 0 on error.
double tclmb_run(int which, int iters) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out;
    if (cudaMalloc(&out, 4) != cudaSuccess) return -1;
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms up
        cudaEventRecord(a);
        if (which == 0) k_ex2<<<blocks, threads>>>(out, iters, 0.5f);
        else if (which == 1) k_ffma<<<blocks, threads>>>(out, iters, 0.5f);
        else if (which == 2) k_ffma2<<<blocks, threads>>>(out, iters, 0.5f);
        else k_tanh<<<blocks, threads>>>(out, iters, 0.5f);
        cudaEventRecord(b);
    }
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess || ms <= 0) return -1;
    // lanes of work per second (FFMA2 counts 2 per lane)
    return (double)blocks * threads * iters * 8 * (which == 2 ? 2 : 1) / (ms * 1e-3);
}
}
