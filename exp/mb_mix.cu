// Microbenchmark: throughput of the scan's instruction mix (MUFU.EX2 + packed FMA) per SM sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float seed) {
    float2 s[8], A2[8], iA[8];
    for (int n = 0; n < 8; ++n) { s[n] = make_float2(0.f, 0.f); A2[n] = make_float2(-seed * (2 * n + 1) * 1.01f, -seed * (2 * n + 2) * 0.99f); iA[n] = make_float2(1.f / (2 * n + 1.5f), 1.f / (2 * n + 2.5f)); }
    float dl = seed * threadIdx.x, u = 0.1f * seed;
    float2 y = make_float2(0.f, 0.f);
    for (int i = 0; i < iters; ++i) {
        const float2 dl2 = make_float2(dl, dl), u2 = make_float2(u, u);
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            if (MODE == 0) {  // scan pair: 2 MUFU + 6 FMA2
                const float2 x2 = __fmul2_rn(dl2, A2[n]);
                const float2 ab = make_float2(ex2(x2.x), ex2(x2.y));
                const float2 v = __fmul2_rn(__fmul2_rn(A2[n], u2), iA[n]);
                const float2 t = __fadd2_rn(s[n], v);
                s[n] = __ffma2_rn(ab, t, make_float2(-v.x, -v.y));
                y = __ffma2_rn(iA[n], s[n], y);
            } else if (MODE == 1) {  // FMA part only
                const float2 x2 = __fmul2_rn(dl2, A2[n]);
                const float2 ab = x2;
                const float2 v = __fmul2_rn(__fmul2_rn(A2[n], u2), iA[n]);
                const float2 t = __fadd2_rn(s[n], v);
                s[n] = __ffma2_rn(ab, t, make_float2(-v.x, -v.y));
                y = __ffma2_rn(iA[n], s[n], y);
            } else if (MODE == 2) {  // MUFU part only (+ the FMUL2 feeding it)
                const float2 x2 = __fmul2_rn(dl2, A2[n]);
                s[n] = __fadd2_rn(s[n], make_float2(ex2(x2.x), ex2(x2.y)));
            } else if (MODE == 3) {  // scan pair in scalar FFMA
                float ab0 = ex2(dl * A2[n].x), ab1 = ex2(dl * A2[n].y);
                float v0 = A2[n].x * u * iA[n].x, v1 = A2[n].y * u * iA[n].y;
                s[n].x = fmaf(ab0, s[n].x + v0, -v0); s[n].y = fmaf(ab1, s[n].y + v1, -v1);
                y.x = fmaf(iA[n].x, s[n].x, y.x); y.y = fmaf(iA[n].y, s[n].y, y.y);
            } else if (MODE == 5) {  // x2 and v packed, update + y scalar
                const float2 x2 = __fmul2_rn(dl2, A2[n]);
                const float2 ab = make_float2(ex2(x2.x), ex2(x2.y));
                const float2 v = __fmul2_rn(__fmul2_rn(A2[n], u2), iA[n]);
                s[n].x = fmaf(ab.x, s[n].x + v.x, -v.x); s[n].y = fmaf(ab.y, s[n].y + v.y, -v.y);
                y.x = fmaf(iA[n].x, s[n].x, y.x); y.y = fmaf(iA[n].y, s[n].y, y.y);
            } else if (MODE == 6) {  // packed except y
                const float2 x2 = __fmul2_rn(dl2, A2[n]);
                const float2 ab = make_float2(ex2(x2.x), ex2(x2.y));
                const float2 v = __fmul2_rn(__fmul2_rn(A2[n], u2), iA[n]);
                const float2 t = __fadd2_rn(s[n], v);
                s[n] = __ffma2_rn(ab, t, make_float2(-v.x, -v.y));
                y.x = fmaf(iA[n].x, s[n].x, y.x); y.y = fmaf(iA[n].y, s[n].y, y.y);
            } else if (MODE == 4) {  // pure MUFU
                s[n].x = ex2(s[n].x); s[n].y = ex2(s[n].y);
            }
        }
        dl += 1e-7f; u += 1e-7f;
    }
    float acc = y.x + y.y;
    for (int n = 0; n < 8; ++n) acc += s[n].x + s[n].y;
    if (acc == 12345.f) out[0] = acc;
}

template <int MODE>
void run(const char* name, int blocks_per_sm) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, 4);
    const int iters = 4096;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<MODE><<<sms * blocks_per_sm, 256>>>(out, 16, 1e-3f);
    cudaEventRecord(a);
    k<MODE><<<sms * blocks_per_sm, 256>>>(out, iters, 1e-3f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double pairs = (double)sms * blocks_per_sm * 256 / 32 * iters * 8;   // warp-pairs
    double cyc = ms * 1e-3 * 1.965e9;  // at max clock
    printf("%-28s bps=%d  %.3f ms  SMSP cycles per warp-pair: %.2f\n", name, blocks_per_sm, ms, cyc * sms * 4 / pairs);
}

int main() {
    for (int bps : {2, 4}) {
        run<0>("scan pair (2 MUFU + 6 FMA2)", bps);
        run<1>("FMA2 part only", bps);
        run<3>("scan pair scalar FFMA", bps);
        run<5>("x2,v packed; s,y scalar", bps);
        run<6>("packed except y", bps);
        run<4>("pure MUFU.EX2 x2", bps);
    }
    return 0;
}
