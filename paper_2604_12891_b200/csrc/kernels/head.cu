// head.cu -- SURVEY §8(a) a9: final LayerNorm ("normalized again"), masked mean
// over the T real tokens (reading R9), decoder of three linears 64,32,1 with SiLU
// after the first two (reading R1), plus the MC-dropout sites dec h1/h2 and the
// per-candidate Welford accumulation over passes (reading R17).
// The pool kernels reduce each candidate's rows in order t = 0..T-1 (one warp per candidate); the
// decoder runs as three small GEMMs over the candidates (gemm_simt.cu); every reduction has a
// fixed order -> batch-invariant scores.
#include <cuda_bf16.h>
#include <math.h>

#include "../kernels.h"

namespace tcl {

// LN_f of every real row and the masked mean over the candidate's T rows; one warp per candidate
// (8 candidates per CTA), rows summed in order t = 0..T-1 -> batch-invariant.
template <int PER>
__global__ void __launch_bounds__(256) k_pool(const float* __restrict__ H, int ldh,
                                              const float* __restrict__ g, const float* __restrict__ b,
                                              float eps, const int32_t* __restrict__ cu,
                                              const int32_t* __restrict__ lens, int max_len, int64_t n,
                                              float* __restrict__ pooled) {
    constexpr int dm = 32 * PER;
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int T = lens[i];
    float acc[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j] = 0.0f;
    if (T >= 1 && T <= max_len) {
        const float* h = H + (int64_t)cu[i] * ldh;
        float gv[PER], bv[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) { gv[j] = __ldg(g + lane + 32 * j); bv[j] = __ldg(b + lane + 32 * j); }
        for (int t = 0; t < T; ++t) {
            float v[PER];
            float sm = 0.f;
#pragma unroll
            for (int j = 0; j < PER; ++j) { v[j] = h[(int64_t)t * ldh + lane + 32 * j]; sm += v[j]; }
            const float mean = warp_sum(sm) * (1.0f / dm);
            float q = 0.f;
#pragma unroll
            for (int j = 0; j < PER; ++j) { const float e = v[j] - mean; q = fmaf(e, e, q); }
            const float rstd = rsqrtf(warp_sum(q) * (1.0f / dm) + eps);
#pragma unroll
            for (int j = 0; j < PER; ++j) acc[j] += (v[j] - mean) * rstd * gv[j] + bv[j];
        }
        const float invT = 1.0f / (float)T;
#pragma unroll
        for (int j = 0; j < PER; ++j) acc[j] *= invT;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) pooled[i * dm + lane + 32 * j] = acc[j];
}

void launch_pool(const float* H, int ldh, int dm, const float* lnf_w, const float* lnf_b, float eps,
                 const int32_t* cu, const int32_t* lens, int max_len, int64_t n, float* pooled,
                 cudaStream_t s) {
    if (n == 0) return;
    dim3 grid((unsigned)((n + 7) / 8));
    switch (dm / 32) {
#define TCL_POOL(P) case P: k_pool<P><<<grid, 256, 0, s>>>(H, ldh, lnf_w, lnf_b, eps, cu, lens, max_len, n, pooled); break;
        TCL_POOL(1) TCL_POOL(2) TCL_POOL(3) TCL_POOL(4) TCL_POOL(5) TCL_POOL(6) TCL_POOL(7) TCL_POOL(8)
#undef TCL_POOL
        default: break;
    }
}

// Masked mean of bf16 rows that are already LN_f(H): one warp per candidate, rows summed in order.
template <int PER>
__global__ void __launch_bounds__(256) k_pool_bf16(const __nv_bfloat16* __restrict__ F, int ldf,
                                                   const int32_t* __restrict__ cu,
                                                   const int32_t* __restrict__ lens, int max_len, int64_t n,
                                                   float* __restrict__ pooled) {
    constexpr int dm = 64 * PER;  // lane handles 2 * PER columns (bf16x2 loads)
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int T = lens[i];
    float acc[2 * PER];
#pragma unroll
    for (int j = 0; j < 2 * PER; ++j) acc[j] = 0.0f;
    if (T >= 1 && T <= max_len) {
        const __nv_bfloat16* f = F + (int64_t)cu[i] * ldf;
#pragma unroll 4
        for (int t = 0; t < T; ++t) {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(f + (int64_t)t * ldf + 2 * (lane + 32 * j));
                const float2 fv = __bfloat1622float2(v);
                acc[2 * j] += fv.x;
                acc[2 * j + 1] += fv.y;
            }
        }
        const float invT = 1.0f / (float)T;
#pragma unroll
        for (int j = 0; j < 2 * PER; ++j) acc[j] *= invT;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j)
        *reinterpret_cast<float2*>(pooled + i * dm + 2 * (lane + 32 * j)) = make_float2(acc[2 * j], acc[2 * j + 1]);
}

void launch_pool_bf16(const void* F, int ldf, int dm, const int32_t* cu, const int32_t* lens, int max_len,
                      int64_t n, float* pooled, cudaStream_t s) {
    if (n == 0) return;
    dim3 grid((unsigned)((n + 7) / 8));
    const auto* f = reinterpret_cast<const __nv_bfloat16*>(F);
    switch (dm / 64) {
        case 1: k_pool_bf16<1><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        case 2: k_pool_bf16<2><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        case 3: k_pool_bf16<3><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        case 4: k_pool_bf16<4><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        default: break;
    }
}

__global__ void k_welford(const float* __restrict__ score, const int32_t* __restrict__ lens, int max_len,
                          int64_t n, int pass, float* __restrict__ mean, float* __restrict__ m2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int T = lens[i];
    if (T < 1 || T > max_len) { mean[i] = NAN; m2[i] = NAN; return; }
    const float v = score[i];
    const float m_old = pass == 0 ? 0.0f : mean[i];
    const float q_old = pass == 0 ? 0.0f : m2[i];
    const float delta = v - m_old;
    const float m_new = m_old + delta / (float)(pass + 1);
    mean[i] = m_new;
    m2[i] = q_old + delta * (v - m_new);
}

void launch_welford(const float* score, const int32_t* lens, int max_len, int64_t n, int pass, float* mean,
                    float* m2, cudaStream_t s) {
    if (n == 0) return;
    k_welford<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(score, lens, max_len, n, pass, mean, m2);
}

__global__ void k_mask_invalid(const int32_t* __restrict__ lens, int max_len, int64_t n, float* __restrict__ sc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int T = lens[i];
    if (T < 1 || T > max_len) sc[i] = NAN;
}

void launch_mask_invalid(const int32_t* lens, int max_len, int64_t n, float* scores, cudaStream_t s) {
    if (n == 0) return;
    k_mask_invalid<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lens, max_len, n, scores);
}

__global__ void k_mc_finalize(const float* __restrict__ m2, int64_t n, int passes,
                              float* __restrict__ var) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) var[i] = m2[i] / (float)passes;
}

void launch_mc_finalize(const float* m2, int64_t n, int passes, float* var, cudaStream_t s) {
    if (n == 0) return;
    k_mc_finalize<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(m2, n, passes, var);
}

}  // namespace tcl
