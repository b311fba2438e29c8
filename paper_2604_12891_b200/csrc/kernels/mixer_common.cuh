// mixer_common.cuh -- device helpers of the bf16-path mixer kernels (mixer_split.cu): warp-level
// MMA fragments, the one-MUFU softplus and the bulk-copy wrappers.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "../common.cuh"
#include "../tc_ptx.cuh"

namespace tcl {

__device__ __forceinline__ uint32_t pk_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// softplus(v) = max(v, 0) + log(1 + y), y = e^{-|v|} in (0, 1]: one MUFU.EX2 for y, log1p(y) as
// y * P4(y) on the FMA pipe (Chebyshev fit of log1p(y)/y on [0, 1], relative error 1.2e-4 in fp32
// Horner form: an exponent error of 1.2e-4 |Delta A| in exp(Delta A), far below the bf16
// rounding of the path).  The dt_proj phase issues 32 softplus per thread at once and was
// MUFU-throttled with the former ex2 + lg2 pair.
__device__ __forceinline__ float softplus_fast(float v) {
    const float y = ex2(-fabsf(v) * kLog2e);
    float p = fmaf(0.041064512f, y, -0.15602843f);
    p = fmaf(p, y, 0.30467236f);
    p = fmaf(p, y, -0.49636829f);
    p = fmaf(p, y, 0.99988794f);
    return fmaf(y, p, fmaxf(v, 0.0f));
}

// softplus_fast on a pair, the polynomial in packed fp32x2 (bit-identical to two softplus_fast)
__device__ __forceinline__ float2 softplus_fast2(float2 v) {
    const float2 y = make_float2(ex2(-fabsf(v.x) * kLog2e), ex2(-fabsf(v.y) * kLog2e));
    float2 p = __ffma2_rn(make_float2(0.041064512f, 0.041064512f), y, make_float2(-0.15602843f, -0.15602843f));
    p = __ffma2_rn(p, y, make_float2(0.30467236f, 0.30467236f));
    p = __ffma2_rn(p, y, make_float2(-0.49636829f, -0.49636829f));
    p = __ffma2_rn(p, y, make_float2(0.99988794f, 0.99988794f));
    return __ffma2_rn(y, p, make_float2(fmaxf(v.x, 0.0f), fmaxf(v.y, 0.0f)));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            tc::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
        : "memory");
}

// bulk copy shared -> global (one bulk group per issuing thread)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(tc::smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// A candidate range [c0, c1) and its packed rows [r0, r_end) (a k_scan work group).
struct RowRange {
    int64_t c0, c1, r0, r_end;
};

// Static partition: CTA b of G owns the candidates whose first row lies in [P b / G, P (b + 1) / G).
__device__ __forceinline__ RowRange cta_rows(const int32_t* cu, int64_t n) {
    const int64_t P = cu[n];
    auto cand_at = [&](int64_t target) -> int64_t {   // first candidate i with cu[i] >= target
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cu[mid] < target) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    RowRange r;
    r.c0 = cand_at(P * blockIdx.x / gridDim.x);
    r.c1 = cand_at(P * (blockIdx.x + 1) / gridDim.x);
    r.r0 = cu[r.c0];
    r.r_end = cu[r.c1];
    return r;
}

}  // namespace tcl
