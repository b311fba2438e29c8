// norm.cu -- LayerNorm of the residual stream ("After normalization ... normalized
// again"; reading R2: affine LayerNorm, biased variance, eps inside the square root).
// One warp per row; the row lives in registers (two-pass mean / variance, no cancellation).
#include <cuda_bf16.h>

#include "../kernels.h"

namespace tcl {

template <int PER>  // dm = 32 * PER
__global__ void __launch_bounds__(256) k_layernorm(const float* __restrict__ H, int ldh,
                                                   const float* __restrict__ g,
                                                   const float* __restrict__ b, float eps,
                                                   float* __restrict__ Y, __nv_bfloat16* __restrict__ Yb,
                                                   int ldy, const int32_t* __restrict__ p_rows) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= *p_rows) return;
    constexpr int dm = 32 * PER;
    float v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = H[(int64_t)row * ldh + lane + 32 * j];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) s += v[j];
    const float mean = warp_sum(s) * (1.0f / dm);
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) { float t = v[j] - mean; q = fmaf(t, t, q); }
    const float rstd = rsqrtf(warp_sum(q) * (1.0f / dm) + eps);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        float o = (v[j] - mean) * rstd * __ldg(g + c) + __ldg(b + c);
        if (Y) Y[(int64_t)row * ldy + c] = o;
        if (Yb) Yb[(int64_t)row * ldy + c] = __float2bfloat16_rn(o);
    }
}

void launch_layernorm(const float* H, int ldh, int dm, const float* g, const float* b, float eps,
                      float* Y, void* Yb, int ldy, int max_rows, const int32_t* p_rows,
                      cudaStream_t s) {
    if (max_rows <= 0) return;
    dim3 grid((max_rows + 7) / 8);
    auto* yb = (__nv_bfloat16*)Yb;
    switch (dm / 32) {
        case 1: k_layernorm<1><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        case 2: k_layernorm<2><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        case 4: k_layernorm<4><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        case 8: k_layernorm<8><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        case 3: k_layernorm<3><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        case 5: k_layernorm<5><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        case 6: k_layernorm<6><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        case 7: k_layernorm<7><<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows); break;
        default: break;  // validated on the host (dm % 32 == 0, dm <= 256)
    }
}

}  // namespace tcl
