// pack.cu -- SURVEY §8(a) a1: length validation, exclusive prefix sum, varlen row gather.
//
// The feature tensor arrives padded [n][L][d_in] ("26x22 on CPU"; SPEC.md:154
// padding trails).  Work downstream must be proportional to sum(T_i), not n*L, so the real rows
// are packed contiguously: candidate i owns rows [cu[i], cu[i+1]).  Padded slots are never read.
#include <cuda_bf16.h>

#include "../kernels.h"

namespace tcl {

// One block of 1024 threads; each thread scans a contiguous strip of lengths.
__global__ void __launch_bounds__(1024) k_lens_prefix(const int32_t* __restrict__ lens, int64_t n,
                                                      int32_t max_len, int32_t* __restrict__ cu,
                                                      int* __restrict__ err) {
    __shared__ int32_t warp_tot[32];
    const int tid = threadIdx.x;
    const int64_t per = (n + 1023) / 1024;
    const int64_t lo = tid * per, hi = min(n, lo + per);
    int32_t local = 0;
    bool bad = false;
    for (int64_t i = lo; i < hi; ++i) {
        int32_t T = lens[i];
        bool ok = (T >= 1 && T <= max_len);
        bad |= !ok;
        local += ok ? T : 0;
    }
    if (bad) atomicOr(err, ERR_LEN);
    // block exclusive scan of `local`
    const int lane = tid & 31, wid = tid >> 5;
    int32_t v = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) warp_tot[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int32_t w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    int32_t run = v - local + (wid > 0 ? warp_tot[wid - 1] : 0);
    for (int64_t i = lo; i < hi; ++i) {
        cu[i] = run;
        int32_t T = lens[i];
        run += (T >= 1 && T <= max_len) ? T : 0;
    }
    if (tid == 1023) cu[n] = warp_tot[31];
}

void launch_lens_prefix(const int32_t* lens, int64_t n, int32_t max_len, int32_t* cu, int* err,
                        cudaStream_t s) {
    k_lens_prefix<<<1, 1024, 0, s>>>(lens, n, max_len, cu, err);
}

// One warp per padded slot (i, t): lanes copy the d_in columns when t < T_i.
__global__ void __launch_bounds__(256) k_pack(const float* __restrict__ feats,
                                              const int32_t* __restrict__ lens,
                                              const int32_t* __restrict__ cu, int64_t n, int L,
                                              int d_in, int ldx, float* __restrict__ X,
                                              __nv_bfloat16* __restrict__ Xb,
                                              int32_t* __restrict__ row_cand) {
    const int64_t slot = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (slot >= n * L) return;
    const int64_t i = slot / L;
    const int t = (int)(slot - i * L);
    const int32_t T = lens[i];
    if (T < 1 || T > L || t >= T) return;
    const int64_t row = cu[i] + t;
    const float* src = feats + slot * d_in;
    for (int c = lane; c < ldx; c += 32) {
        float v = c < d_in ? __ldg(src + c) : 0.0f;
        if (X) X[row * ldx + c] = v;
        if (Xb) Xb[row * ldx + c] = __float2bfloat16_rn(v);
    }
    if (lane == 0) row_cand[row] = (int32_t)i;
}

void launch_pack(const float* feats, const int32_t* lens, const int32_t* cu, int64_t n, int L,
                 int d_in, int ldx, float* X, void* x_bf16, int32_t* row_cand, cudaStream_t s) {
    int64_t slots = n * L;
    if (slots == 0) return;
    k_pack<<<(unsigned)((slots + 7) / 8), 256, 0, s>>>(feats, lens, cu, n, L, d_in, ldx, X,
                                                       (__nv_bfloat16*)x_bf16, row_cand);
}

}  // namespace tcl
