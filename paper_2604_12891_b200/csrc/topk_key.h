// topk_key.h -- the (score desc, index asc) total order of the top-k ("selects the best
// K"; reading R15) as one uint64 key, shared by the device kernels and the host-side C ABI
// (tcl_topk_key) so that every rank of a multi-GPU job and the host agree bit for bit:
//   key = orderable_u32(score) << 32 | (0xFFFFFFFF - global_index)
// NaN counts as -inf, -0 as +0; the k largest keys are exactly the top-k.  Key 0 never encodes a
// real candidate (the smallest real high word is orderable(-inf) = 0x007FFFFF): padding sentinel.
#pragma once
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define TCL_HD __host__ __device__ __forceinline__
#else
#define TCL_HD inline
#endif

namespace tcl {

TCL_HD uint32_t float_bits(float f) {
#ifdef __CUDA_ARCH__
    return __float_as_uint(f);
#else
    uint32_t b;
    memcpy(&b, &f, 4);
    return b;
#endif
}

TCL_HD unsigned long long topk_key(float f, uint32_t gidx) {
    if (f != f) f = -__builtin_huge_valf();   // NaN -> -inf
    if (f == 0.0f) f = 0.0f;                  // -0 == +0 in the score order
    const uint32_t b = float_bits(f);
    const uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((unsigned long long)ord << 32) | (unsigned long long)(0xFFFFFFFFu - gidx);
}

}  // namespace tcl
