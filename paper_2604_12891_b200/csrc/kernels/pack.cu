// pack.cu -- SURVEY §8(a) a1: length validation, exclusive prefix sum, varlen row gather.
//
// The feature tensor arrives padded [n][L][d_in] ("26x22 on CPU"; SPEC.md:154
// padding trails).  Work downstream must be proportional to sum(T_i), not n*L, so the real rows
// are packed contiguously: candidate i owns rows [cu[i], cu[i+1]).  Padded slots are never read.
#include <cuda_bf16.h>

#include "../kernels.h"

namespace tcl {

// One block of 1024 threads walks the lengths in coalesced tiles of 4096 (int4 per thread):
// block-wide exclusive scan per tile + running carry.  Invalid lengths count as 0 rows.
__global__ void __launch_bounds__(1024) k_lens_prefix(const int32_t* __restrict__ lens, int64_t n,
                                                      int32_t max_len, int32_t* __restrict__ cu,
                                                      int* __restrict__ err) {
    __shared__ int32_t warp_tot[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int32_t carry = 0;
    bool bad = false;
    for (int64_t base = 0; base < n; base += 4096) {
        int32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = base + tid * 4 + j;
            int32_t T = i < n ? lens[i] : 1;
            const bool ok = T >= 1 && T <= max_len;
            bad |= (i < n) && !ok;
            v[j] = (i < n && ok) ? T : 0;
        }
        const int32_t local = v[0] + v[1] + v[2] + v[3];
        int32_t x = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int32_t w = warp_tot[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t t = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += t;
            }
            warp_tot[lane] = w;  // inclusive
        }
        __syncthreads();
        int32_t run = carry + (x - local) + (wid > 0 ? warp_tot[wid - 1] : 0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = base + tid * 4 + j;
            if (i < n) cu[i] = run;
            run += v[j];
        }
        carry += warp_tot[31];
        __syncthreads();
    }
    if (bad) atomicOr(err, ERR_LEN);
    if (tid == 0) cu[n] = carry;
}

void launch_lens_prefix(const int32_t* lens, int64_t n, int32_t max_len, int32_t* cu, int* err,
                        cudaStream_t s) {
    k_lens_prefix<<<1, 1024, 0, s>>>(lens, n, max_len, cu, err);
}

// One warp per candidate.  The candidate's real rows are one contiguous run of T * d_in floats in
// the padded input, so the warp streams it as float2 pairs (consecutive lanes, consecutive 8-byte
// loads; d_in is even, so a pair never straddles two rows) and scatters each pair to its packed
// row (bf16x2 or float2), then zero-fills the pad columns [d_in, ldx) of its rows.  Padded slots
// t >= T are never read.
__global__ void __launch_bounds__(256) k_pack(const float* __restrict__ feats,
                                              const int32_t* __restrict__ lens,
                                              const int32_t* __restrict__ cu, int64_t n, int L,
                                              int d_in, int ldx, float* __restrict__ X,
                                              __nv_bfloat16* __restrict__ Xb,
                                              int32_t* __restrict__ row_cand, int64_t n_src) {
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int32_t T = lens[i];
    if (T < 1 || T > L) return;
    const int64_t row0 = cu[i];
    const int64_t isrc = i % n_src;                 // batched MC passes re-read the same features
    if (d_in & 1) {   // odd feature width: column per lane
        const float* srcs = feats + isrc * (int64_t)L * d_in;
        for (int t = 0; t < T; ++t) {
            const int64_t row = row0 + t;
            for (int c = lane; c < ldx; c += 32) {
                const float v = c < d_in ? __ldg(srcs + t * d_in + c) : 0.0f;
                if (X) X[row * ldx + c] = v;
                if (Xb) Xb[row * ldx + c] = __float2bfloat16_rn(v);
            }
            if (lane == 0) row_cand[row] = (int32_t)i;
        }
        return;
    }
    const int hp = d_in >> 1;                       // pairs per row
    const float2* src = reinterpret_cast<const float2*>(feats + isrc * (int64_t)L * d_in);
    const int npairs = T * hp;
    for (int p = lane; p < npairs; p += 32) {
        const int t = p / hp, c = 2 * (p - t * hp);
        const float2 v = __ldg(src + p);
        const int64_t o = (row0 + t) * ldx + c;
        if (X) *reinterpret_cast<float2*>(X + o) = v;
        if (Xb) *reinterpret_cast<__nv_bfloat162*>(Xb + o) = __floats2bfloat162_rn(v.x, v.y);
    }
    const int pad = (ldx - d_in) >> 1;             // zero pairs per row
    for (int p = lane; p < T * pad; p += 32) {
        const int t = p / pad, c = d_in + 2 * (p - t * pad);
        const int64_t o = (row0 + t) * ldx + c;
        if (X) *reinterpret_cast<float2*>(X + o) = make_float2(0.f, 0.f);
        if (Xb) *reinterpret_cast<__nv_bfloat162*>(Xb + o) = __floats2bfloat162_rn(0.f, 0.f);
    }
    for (int t = lane; t < T; t += 32) row_cand[row0 + t] = (int32_t)i;
}

void launch_pack(const float* feats, const int32_t* lens, const int32_t* cu, int64_t n, int L,
                 int d_in, int ldx, float* X, void* x_bf16, int32_t* row_cand, cudaStream_t s,
                 int64_t n_src) {
    if (n == 0) return;
    k_pack<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(feats, lens, cu, n, L, d_in, ldx, X,
                                                   (__nv_bfloat16*)x_bf16, row_cand, n_src > 0 ? n_src : n);
}

}  // namespace tcl
