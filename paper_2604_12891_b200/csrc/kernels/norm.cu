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

// d_model 128: the same arithmetic in the same order as the LayerNorm fused into the fp32 GEMM
// epilogue (gemm_simt.cu, EPI_RESID_LN / EPI_LN): virtual thread t < 16 sums columns
// {4t..4t+3, 64+4t..64+4t+3} in that order, then a 16-lane xor tree (1, 2, 4, 8); lanes 16..31
// mirror lanes 0..15.  The fused and unfused forwards therefore give bit-identical rows (the KB + AC
// model, which keeps this kernel, equals the plain model bit for bit when its gates are closed).
__global__ void __launch_bounds__(256) k_layernorm128(const float* __restrict__ H, int ldh,
                                                      const float* __restrict__ g,
                                                      const float* __restrict__ b, float eps,
                                                      float* __restrict__ Y, __nv_bfloat16* __restrict__ Yb,
                                                      int ldy, const int32_t* __restrict__ p_rows) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= *p_rows) return;
    const int t = lane & 15;
    const float* hr = H + (int64_t)row * ldh;
    const float4 h0 = *reinterpret_cast<const float4*>(hr + 4 * t);
    const float4 h1 = *reinterpret_cast<const float4*>(hr + 64 + 4 * t);
    const float v[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
    float sm = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) sm += v[q];
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
    const float mean = sm * (1.0f / 128);
    float sq = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) { const float d = v[q] - mean; sq = fmaf(d, d, sq); }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const float rstd = rsqrtf(sq * (1.0f / 128) + eps);
    if (lane < 16) {
#pragma unroll
        for (int jh = 0; jh < 2; ++jh) {
            const int c = 4 * t + 64 * jh;
            float r[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) r[q] = (v[4 * jh + q] - mean) * rstd * __ldg(g + c + q) + __ldg(b + c + q);
            if (Y) *reinterpret_cast<float4*>(Y + (int64_t)row * ldy + c) = make_float4(r[0], r[1], r[2], r[3]);
            if (Yb) {
#pragma unroll
                for (int q = 0; q < 4; ++q) Yb[(int64_t)row * ldy + c + q] = __float2bfloat16_rn(r[q]);
            }
        }
    }
}

void launch_layernorm(const float* H, int ldh, int dm, const float* g, const float* b, float eps,
                      float* Y, void* Yb, int ldy, int max_rows, const int32_t* p_rows,
                      cudaStream_t s, bool gemm_epilogue_order) {
    if (max_rows <= 0) return;
    dim3 grid((max_rows + 7) / 8);
    auto* yb = (__nv_bfloat16*)Yb;
    if (gemm_epilogue_order && dm == 128 && (ldh % 4) == 0 && (ldy % 4) == 0) {
        k_layernorm128<<<grid, 256, 0, s>>>(H, ldh, g, b, eps, Y, yb, ldy, p_rows);
        return;
    }
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
