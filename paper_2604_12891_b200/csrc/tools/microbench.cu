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

// The selective scan's per-state instruction mix (mixer_fused.cu, ZOH): per pair of states one
// FMUL2 for the exponent argument, two MUFU.EX2, FMUL2 x2 for v = B u / A, FADD2 + FFMA2 for the
// update, FFMA2 for y += C s.  Its throughput is the achievable ceiling of the scan loop on this
// chip (MUFU and the FMA pipe are both busy; neither reaches its solo peak).  Counts exps.
__global__ void __launch_bounds__(256) k_scanmix(float* out, int iters, float seed) {
    float2 s[8], A2[8], iA[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
        s[n] = make_float2(0.f, 0.f);
        A2[n] = make_float2(-seed * (2 * n + 1) * 1.01f, -seed * (2 * n + 2) * 0.99f);
        iA[n] = make_float2(1.f / (2 * n + 1.5f), 1.f / (2 * n + 2.5f));
    }
    float dl = seed * threadIdx.x * 1e-3f, u = 0.1f * seed;
    float2 y = make_float2(0.f, 0.f);
    for (int i = 0; i < iters; ++i) {
        const float2 dl2 = make_float2(dl, dl), u2 = make_float2(u, u);
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            const float2 x2 = __fmul2_rn(dl2, A2[n]);
            float e0, e1;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(x2.x));
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(x2.y));
            const float2 v = __fmul2_rn(__fmul2_rn(A2[n], u2), iA[n]);
            const float2 t = __fadd2_rn(s[n], v);
            s[n] = __ffma2_rn(make_float2(e0, e1), t, make_float2(-v.x, -v.y));
            y = __ffma2_rn(iA[n], s[n], y);
        }
        dl += 1e-7f;
        u += 1e-7f;
    }
    float acc = y.x + y.y;
#pragma unroll
    for (int n = 0; n < 8; ++n) acc += s[n].x + s[n].y;
    if (acc == 12345.f) out[0] = acc;
}

extern "C" {
// Returns ops/s over the whole chip (0: MUFU.EX2, 1: FFMA, 2: FFMA2 (2 per lane), 3: MUFU.TANH,
// 4: exps of the scan instruction mix (16 per lane per iteration));
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
        else if (which == 3) k_tanh<<<blocks, threads>>>(out, iters, 0.5f);
        else k_scanmix<<<sms * 2, threads>>>(out, iters, 0.5f);   // 16 warps/SM, as the mixer
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
    if (which == 4) return (double)sms * 2 * threads * iters * 16 / (ms * 1e-3);
    return (double)blocks * threads * iters * 8 * (which == 2 ? 2 : 1) / (ms * 1e-3);
}
}
