// topk.cu -- SURVEY §8(a) a11: "selects the best K".
//
// Total order (score desc, index asc) with NaN -> -inf (reading R15) is encoded in one uint64 key:
//   key = orderable_u32(score) << 32 | (0xFFFFFFFF - global_index)
// so the k largest keys are exactly the top-k.  Key 0 never encodes a real candidate (the
// smallest real high word is orderable(-inf) = 0x007FFFFF) and is used as the padding sentinel.
// Selection, k <= 1024: each CTA takes up to 8,192 keys, finds its k-th largest key by an
// MSB-first radix select (8-bit digits, shared-memory histograms, early exit once the boundary
// digit holds exactly the keys still needed), gathers the keys above it and bitonic-sorts only
// those k; rounds repeat over the survivors until one CTA's worth remains (k_topk_radix).
// k > 1024: a tournament in which each CTA bitonic-sorts a chunk of keys in shared memory and
// keeps its best k, rounds repeating until one chunk remains (k_topk_chunk).  Integer-only ->
// bit-exact in both paths.
#include <math.h>

#include "../kernels.h"
#include "../topk_key.h"

namespace tcl {

typedef unsigned long long u64;

__device__ __forceinline__ u64 make_key(float f, uint32_t gidx) { return topk_key(f, gidx); }

template <bool FROM_SCORES, int C>
__global__ void __launch_bounds__(1024) k_topk_chunk(const float* __restrict__ scores,
                                                     const u64* __restrict__ keys_in, int64_t count,
                                                     int64_t index_base, int k, u64* __restrict__ out) {
    extern __shared__ u64 sk[];
    const int64_t lo = (int64_t)blockIdx.x * C;
    const int64_t m = min((int64_t)C, count - lo);
    for (int j = threadIdx.x; j < C; j += blockDim.x) {
        u64 v = 0;
        if (j < m) v = FROM_SCORES ? make_key(scores[lo + j], (uint32_t)(index_base + lo + j)) : keys_in[lo + j];
        sk[j] = v;
    }
    __syncthreads();
    for (int size = 2; size <= C; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int j = threadIdx.x; j < C / 2; j += blockDim.x) {
                const int a = 2 * stride * (j / stride) + (j % stride);
                const int b = a + stride;
                const bool desc = (a & size) == 0;
                const u64 x = sk[a], y = sk[b];
                if ((x < y) == desc) { sk[a] = y; sk[b] = x; }
            }
            __syncthreads();
        }
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) out[(int64_t)blockIdx.x * k + j] = sk[j];
}

// k <= 1024: each CTA takes a chunk of up to 8,192 keys and selects its k-th largest key by an
// MSB-first radix select (8-bit digits; shared-memory histograms; stops once the boundary digit
// holds exactly the keys still needed), gathers the keys above it and sorts only those k keys -- far
// fewer barrier rounds than a full bitonic sort of the chunk.  One CTA finishes a tuning round
// (~4,096 candidates); 65,536 take two rounds (8 CTAs, then 1).  Keys are unique except the 0
// padding, so the selection is exact and integer-only (bit-exact).
template <bool FROM_SCORES>
__global__ void __launch_bounds__(1024) k_topk_radix(const float* __restrict__ scores,
                                                     const u64* __restrict__ keys_in, int64_t count,
                                                     int64_t index_base, int k, u64* __restrict__ out) {
    constexpr int PER = 8;
    __shared__ uint32_t hist[256];
    __shared__ u64 sel[1024];
    __shared__ u64 s_prefix;
    __shared__ int s_kk, s_done, s_ngt;
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t lo = (int64_t)blockIdx.x * (PER * 1024);
    out += (int64_t)blockIdx.x * k;
    u64 v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int64_t i = lo + tid + (int64_t)j * 1024;
        v[j] = i < count ? (FROM_SCORES ? make_key(scores[i], (uint32_t)(index_base + i)) : keys_in[i]) : 0ull;
    }
    u64 prefix = 0;
    int kk = k, done = 0;
    for (int byte = 7; byte >= 0 && !done; --byte) {
        const u64 hmask = byte == 7 ? 0ull : (~0ull << (8 * (byte + 1)));
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if ((v[j] & hmask) == prefix) atomicAdd(&hist[(uint32_t)(v[j] >> (8 * byte)) & 0xFFu], 1u);
        __syncthreads();
        if (tid < 32) {
            uint32_t c[8], sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) { c[q] = hist[8 * lane + q]; sum += c[q]; }
            uint32_t incl = sum;   // keys in digits >= 8 lane
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += t;
            }
            const uint32_t excl = incl - sum;   // keys in digits above this lane's
            if (excl < (uint32_t)kk && (uint32_t)kk <= incl) {
                uint32_t run = excl;
#pragma unroll
                for (int q = 7; q >= 0; --q) {
                    if (run + c[q] >= (uint32_t)kk) {
                        s_prefix = prefix | ((u64)(8 * lane + q) << (8 * byte));
                        s_kk = kk - (int)run;
                        s_done = (c[q] == (uint32_t)(kk - (int)run)) ? 1 : 0;   // the whole bin is taken
                        break;
                    }
                    run += c[q];
                }
            }
        }
        __syncthreads();
        prefix = s_prefix;
        kk = s_kk;
        done = s_done;
    }
    // threshold: keys whose top bytes match `prefix` on the resolved digits (done) or equal it
    if (tid == 0) s_ngt = 0;
    __syncthreads();
    if (done) {   // every key >= prefix is selected (exactly k of them)
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (v[j] >= prefix) sel[atomicAdd(&s_ngt, 1)] = v[j];
        __syncthreads();
    } else {      // prefix is the k-th key itself; kk copies of it are needed (only 0 repeats)
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (v[j] > prefix) sel[atomicAdd(&s_ngt, 1)] = v[j];
        __syncthreads();
        if (tid < kk) sel[k - kk + tid] = prefix;
        __syncthreads();
    }
    // sort the k selected keys descending (bitonic over the next power of two, 0-padded)
    int K2 = 1;
    while (K2 < k) K2 <<= 1;
    if (tid >= k && tid < K2) sel[tid] = 0ull;
    __syncthreads();
    for (int size = 2; size <= K2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (tid < K2 / 2) {
                const int a = 2 * stride * (tid / stride) + (tid % stride);
                const int b = a + stride;
                const bool desc = (a & size) == 0;
                const u64 x = sel[a], y = sel[b];
                if ((x < y) == desc) { sel[a] = y; sel[b] = x; }
            }
            __syncthreads();
        }
    }
    if (tid < k) out[tid] = sel[tid];
}

__global__ void k_topk_decode(const u64* __restrict__ keys, int k, int64_t* __restrict__ idx,
                              float* __restrict__ score) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    const u64 key = keys[j];
    if (key == 0) { idx[j] = -1; score[j] = -INFINITY; return; }
    const uint32_t ord = (uint32_t)(key >> 32);
    const uint32_t b = (ord & 0x80000000u) ? (ord & 0x7FFFFFFFu) : ~ord;
    idx[j] = (int64_t)(0xFFFFFFFFu - (uint32_t)key);
    score[j] = __uint_as_float(b);
}

size_t topk_tmp_keys(int64_t n, int k) {
    const int64_t blocks = (n + 2047) / 2048;  // smallest chunk size -> most first-round blocks
    return (size_t)(2 * blocks * k + 2 * kTopkChunk);
}

template <int C>
static void launch_chunk(bool from_scores, unsigned blocks, const float* scores, const u64* src, int64_t cur,
                         int64_t index_base, int k, u64* dst, cudaStream_t s) {
    const int smem = C * (int)sizeof(u64);
    prepare_kernel(k_topk_chunk<true, C>, smem);
    prepare_kernel(k_topk_chunk<false, C>, smem);
    if (from_scores)
        k_topk_chunk<true, C><<<blocks, 1024, smem, s>>>(scores, nullptr, cur, index_base, k, dst);
    else
        k_topk_chunk<false, C><<<blocks, 1024, smem, s>>>(nullptr, src, cur, 0, k, dst);
}

// Chunk size: >= 4k (each round shrinks the candidate set >= 4x) and small enough that the first
// round spreads over many CTAs.
static int chunk_for(int k) { return k <= 512 ? 2048 : (k <= 1024 ? 4096 : kTopkChunk); }

// Rounds of the tournament; writes exactly k keys (descending, 0-padded) to `out`.
static int tournament(const float* scores, const u64* keys, int64_t count, int k,
                      int64_t index_base, u64* out, u64* tmp, cudaStream_t s) {
    int launched = 0;
    if (k <= 1024) {   // radix-select rounds over 8,192-key chunks until one chunk remains
        const int64_t blocks0 = (count + kTopkChunk - 1) / kTopkChunk;
        u64* rb[2] = {tmp, tmp + blocks0 * k};
        int w = 0;
        const u64* src = keys;
        bool from_scores = scores != nullptr;
        int64_t cur = count;
        for (;;) {
            int64_t blocks = (cur + kTopkChunk - 1) / kTopkChunk;
            if (blocks < 1) blocks = 1;
            u64* dst = blocks == 1 ? out : rb[w];
            if (from_scores) k_topk_radix<true><<<(unsigned)blocks, 1024, 0, s>>>(scores, nullptr, cur, index_base, k, dst);
            else k_topk_radix<false><<<(unsigned)blocks, 1024, 0, s>>>(nullptr, src, cur, 0, k, dst);
            ++launched;
            if (blocks == 1) break;
            cur = blocks * k;
            src = dst;
            w ^= 1;
            from_scores = false;
        }
        return launched;
    }
    // a set that fits one CTA's chunk is selected in a single round (no cross-CTA tournament)
    const int64_t need = count > k ? count : k;   // the chunk must also hold the k outputs
    const int C = need <= 2048 ? 2048 : need <= 4096 ? 4096 : need <= kTopkChunk ? kTopkChunk : chunk_for(k);
    const int64_t blocks0 = (count + C - 1) / C;
    u64* buf[2] = {tmp, tmp + blocks0 * k + kTopkChunk};
    int which = 0;
    const u64* src = keys;
    bool from_scores = scores != nullptr;
    int64_t cur = count;
    for (;;) {
        int64_t blocks = (cur + C - 1) / C;
        if (blocks < 1) blocks = 1;
        u64* dst = blocks == 1 ? out : buf[which];
        if (C == 2048) launch_chunk<2048>(from_scores, (unsigned)blocks, scores, src, cur, index_base, k, dst, s);
        else if (C == 4096) launch_chunk<4096>(from_scores, (unsigned)blocks, scores, src, cur, index_base, k, dst, s);
        else launch_chunk<kTopkChunk>(from_scores, (unsigned)blocks, scores, src, cur, index_base, k, dst, s);
        ++launched;
        if (blocks == 1) break;
        cur = blocks * k;
        src = dst;
        which ^= 1;
        from_scores = false;
    }
    return launched;
}

int launch_topk_keys(const float* scores, int64_t n, int k, int64_t index_base, u64* out_keys,
                     u64* tmp, cudaStream_t s) {
    return tournament(scores, nullptr, n, k, index_base, out_keys, tmp, s);
}

int launch_topk_decode(const u64* keys, int k, int64_t* idx, float* score, cudaStream_t s) {
    k_topk_decode<<<(k + 255) / 256, 256, 0, s>>>(keys, k, idx, score);
    return 1;
}

int launch_topk_merge(const u64* keys, int64_t count, int k, int64_t* idx, float* score, u64* tmp,
                      cudaStream_t s) {
    u64* fin = tmp;  // k keys, then the tournament scratch
    int launched = tournament(nullptr, keys, count, k, 0, fin, tmp + k, s);
    k_topk_decode<<<(k + 255) / 256, 256, 0, s>>>(fin, k, idx, score);
    return launched + 1;
}

}  // namespace tcl
