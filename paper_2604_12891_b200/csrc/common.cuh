// common.cuh -- shared device helpers of libtcl (product path; independent of oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace tcl {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// Per-launch "fast" transcendental helpers.  MUFU.EX2 via ex2.approx.ftz (max rel. err ~2^-22).
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// SiLU(v) = v * sigmoid(v) (reading R1).  One MUFU.EX2 + one MUFU.RCP.
__device__ __forceinline__ float silu(float v) { return v * rcp(1.0f + ex2(-v * kLog2e)); }
// bf16-path SiLU: h (1 + tanh h), h = v / 2 -- one MUFU.TANH (tanh.approx, relative error ~2^-11,
// below the bf16 rounding of the output it feeds).
__device__ __forceinline__ float silu_tanh(float v) {
    const float h = 0.5f * v;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    return fmaf(h, t, h);
}
// softplus(v) = log(1 + e^v) (reading R13): v > 20 -> v (error < 2.1e-9); log1pf for accuracy.
__device__ __forceinline__ float softplus(float v) {
    return v > 20.0f ? v : log1pf(__expf(v));
}

// Philox4x32-10 (Salmon et al. SC'11, the Random123 constants).  Reading R17.
struct u32x4 { uint32_t x, y, z, w; };
__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        u32x4 n = {hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        c = n;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Dropout keep decision of (unit, token, site, pass, global index) -- integer only.
struct DropoutCtx {
    uint64_t seed;
    uint32_t thr;        // floor(p * 2^32)
    float scale;         // 1 / (1 - p)
    int32_t pass;
    int64_t index_base;
    int enabled;
    // MC passes batched into one forward (tcl_score_mc): virtual candidate v of the launch is
    // candidate v mod pass_n of pass (pass + v / pass_n); 0 = one pass per launch (v = candidate)
    uint32_t pass_n;
};
// Philox counter of (unit group, token, site, pass, global candidate index)
__device__ __forceinline__ u32x4 dropout_counter(const DropoutCtx& d, int unit4, int token, int site,
                                                 int64_t cand) {
    uint32_t pass = (uint32_t)d.pass, local = (uint32_t)cand;
    if (d.pass_n) {
        const uint32_t q = local / d.pass_n;
        pass += q;
        local -= q * d.pass_n;
    }
    return {(uint32_t)unit4 >> 2, ((uint32_t)token << 2) | (uint32_t)site, pass,
            (uint32_t)(d.index_base + local)};
}
__device__ __forceinline__ bool dropout_keep(const DropoutCtx& d, int unit, int token, int site,
                                             int64_t cand) {
    u32x4 c = dropout_counter(d, unit, token, site, cand);
    u32x4 w = philox4x32_10(c, (uint32_t)d.seed, (uint32_t)(d.seed >> 32));
    uint32_t word = (unit & 3) == 0 ? w.x : (unit & 3) == 1 ? w.y : (unit & 3) == 2 ? w.z : w.w;
    return word >= d.thr;
}

// The keep words of units [4 g, 4 g + 3] from one Philox call (dropout_keep(d, u, ...) reads word
// u & 3 of the call for unit4 = u & ~3): epilogues that own 4 consecutive units draw once.
__device__ __forceinline__ u32x4 dropout_words(const DropoutCtx& d, int unit4, int token, int site,
                                               int64_t cand) {
    return philox4x32_10(dropout_counter(d, unit4, token, site, cand), (uint32_t)d.seed, (uint32_t)(d.seed >> 32));
}
__device__ __forceinline__ float dropout_apply_word(const DropoutCtx& d, float v, uint32_t word) {
    return word >= d.thr ? v * d.scale : 0.0f;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace tcl
