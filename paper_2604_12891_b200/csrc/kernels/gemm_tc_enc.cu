// gemm_tc_enc.cu -- the first two encoder linears of the bf16 path chained in ONE tcgen05 kernel
// (reading R1: SiLU after linears 1 and 2; MC-dropout sites 0
// and 1, reading R17):
//
//   E1 = SiLU(X W1^T + b1)      X [P][32] bf16 (22 features + zero pad), W1 [e1][32]
//   E2 = SiLU(E1 W2^T + b2)     W2 [e2][e1]  ->  E2 [P][e2] bf16 (the operand of enc3 + LN_0)
//
// E1 never leaves the SM: the epilogue of the first MMA writes it (bias, SiLU, dropout, bf16) into
// shared memory in the 128B-swizzled K-major layout the second MMA reads, so the HBM traffic per
// row is the 64-byte feature row in and the e2-wide bf16 row out (the unfused pair also wrote and
// re-read E1).  Persistent CTA per SM, warp-specialised like gemm_tc.cu: warp 0 = TMA producer
// (W1, W2 once; X row tiles through a 2-stage ring), warp 1 = TMEM allocator + single-thread MMA
// issuer, warps 2..9 = epilogue (warp w drains TMEM lanes 32 (w % 4) .., column half (w - 2) / 4).
// TMEM: acc1 double-buffered (2 x e1 columns), acc2 (e2 columns); E1 double-buffered in shared
// memory.  MMA1 of tile j+1 is issued before MMA2 of tile j, and the epilogue warps form E1 of tile
// j+1 while MMA2 of tile j runs, then drain E2 of tile j.  SiLU in both epilogues is the one-MUFU
// tanh form (h (1 + tanh h), h = v/2): the two SiLUs per E1/E2 element are the epilogue's cost.
#include <cuda_bf16.h>

#include "../kernels.h"
#include "../kernels_tc.h"
#include "../tc_ptx.cuh"

namespace tcl {
namespace enc {

constexpr int kBM = 128;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kXStages = 2;

template <int E1N, int E2N>
struct Smem {
    static constexpr int kKB1 = E1N / 64;                       // K-blocks of MMA2
    static constexpr int kOffW1 = 0;                            // [E1N rows][128 B]
    static constexpr int kOffW2 = kOffW1 + E1N * 128;           // kKB1 x [E2N rows][128 B]
    static constexpr int kOffX = kOffW2 + kKB1 * E2N * 128;     // kXStages x [128 rows][128 B]
    static constexpr int kOffE1 = kOffX + kXStages * kBM * 128; // [2] x kKB1 x [128 rows][128 B]
    static constexpr int kE1Bytes = kKB1 * kBM * 128;
    static constexpr int kOffStg = kOffE1 + 2 * kE1Bytes;       // kEpiWarps x [32 rows][128 B]
    static constexpr int kOffPar = kOffStg + kEpiWarps * 32 * 128;
    static constexpr int kOffBar = kOffPar + (E1N + E2N) * 4;
    static constexpr int kBytes = kOffBar + 256 + 1024;
    static_assert(kBytes <= 232448, "gemm_tc_enc shared memory");
    static_assert(2 * E1N + E2N <= 512, "TMEM columns");
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
// one Philox draw per 4 consecutive units (inlined: the out-of-line call kept a stack frame)
__device__ __forceinline__ u32x4 drop_words_enc(const DropoutCtx& d, int unit4, int token, int site, int64_t cand) {
    return dropout_words(d, unit4, token, site, cand);
}

template <int E1N, int E2N, bool DROP>
__global__ void __launch_bounds__(kThreads, 1) k_enc12(const __grid_constant__ CUtensorMap tmX,
                                                       const __grid_constant__ CUtensorMap tmW1,
                                                       const __grid_constant__ CUtensorMap tmW2,
                                                       const __grid_constant__ CUtensorMap tmE2,
                                                       const EncParams p) {
    using S = Smem<E1N, E2N>;
    constexpr int KB1 = S::kKB1;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment (128B-swizzled TMA tiles) as an offset from the shared array, so that every
    // access below stays in the shared state space (LDS / STS, not generic LD / ST)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sW1 = smem + S::kOffW1;
    uint8_t* sW2 = smem + S::kOffW2;
    uint8_t* sX = smem + S::kOffX;
    uint8_t* sE1 = smem + S::kOffE1;
    float* s_b1 = reinterpret_cast<float*>(smem + S::kOffPar);
    float* s_b2 = s_b1 + E1N;
    uint64_t* bfull = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
    uint64_t* xfull = bfull + 1;            // [kXStages]
    uint64_t* xempty = xfull + kXStages;    // [kXStages]
    uint64_t* a1full = xempty + kXStages;   // [2]
    uint64_t* a1empty = a1full + 2;         // [2]
    uint64_t* e1full = a1empty + 2;         // [2] (E1 smem double buffer)
    uint64_t* a2full = e1full + 2;
    uint64_t* a2empty = a2full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a2empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = *p.p_rows;
    const int num_m = (rows + kBM - 1) / kBM;
    const int n_my = blockIdx.x < num_m ? (num_m - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

    if (threadIdx.x == 0) {
        tc::mbar_init(bfull, 1);
        for (int st = 0; st < kXStages; ++st) { tc::mbar_init(&xfull[st], 1); tc::mbar_init(&xempty[st], 1); }
        for (int a = 0; a < 2; ++a) { tc::mbar_init(&a1full[a], 1); tc::mbar_init(&a1empty[a], kEpiWarps); }
        tc::mbar_init(&e1full[0], kEpiWarps);
        tc::mbar_init(&e1full[1], kEpiWarps);
        tc::mbar_init(a2full, 1);
        tc::mbar_init(a2empty, kEpiWarps);
        tc::fence_mbar_init();
    }
    for (int j = threadIdx.x; j < E1N; j += kThreads) s_b1[j] = __ldg(p.b1 + j);
    for (int j = threadIdx.x; j < E2N; j += kThreads) s_b2[j] = __ldg(p.b2 + j);
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t t_acc2 = tmem_base + 2 * E1N;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            tc::tma_prefetch(&tmX);
            tc::mbar_arrive_expect_tx(bfull, E1N * 128 + KB1 * E2N * 128);
            tc::tma_load_2d(sW1, &tmW1, 0, 0, bfull);
            for (int kb = 0; kb < KB1; ++kb) tc::tma_load_2d(sW2 + kb * E2N * 128, &tmW2, kb * 64, 0, bfull);
            const uint64_t pol = tc::policy_evict_first();
            for (int j = 0; j < n_my; ++j) {
                const int st = j % kXStages;
                const uint32_t ph = (j / kXStages) & 1;
                tc::mbar_wait(&xempty[st], ph ^ 1);
                tc::mbar_arrive_expect_tx(&xfull[st], kBM * 128);
                tc::tma_load_2d_hint(sX + st * kBM * 128, &tmX, 0, (blockIdx.x + j * gridDim.x) * kBM, &xfull[st], pol);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint32_t id1 = tc::idesc_bf16_f32(kBM, E1N);
            constexpr uint32_t id2 = tc::idesc_bf16_f32(kBM, E2N);
            tc::mbar_wait(bfull, 0);
            tc::tc_fence_after();
            const uint32_t aW1 = tc::smem_u32(sW1), aW2 = tc::smem_u32(sW2), aX = tc::smem_u32(sX),
                           aE1 = tc::smem_u32(sE1);
            auto mma1 = [&](int j) {
                const int st = j % kXStages;
                tc::mbar_wait(&xfull[st], (j / kXStages) & 1);
                tc::mbar_wait(&a1empty[j & 1], ((j >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                // K = 32 real feature columns: two K=16 steps (columns 32..63 of the box are zero)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    tc::mma_bf16(tmem_base + (j & 1) * E1N, tc::sw128_kmajor_desc(aX + st * kBM * 128 + k * 32),
                                 tc::sw128_kmajor_desc(aW1 + k * 32), id1, k != 0);
                tc::mma_commit(&xempty[st]);
                tc::mma_commit(&a1full[j & 1]);
            };
            if (n_my > 0) mma1(0);
            for (int j = 0; j < n_my; ++j) {
                if (j + 1 < n_my) mma1(j + 1);
                tc::mbar_wait(&e1full[j & 1], (j >> 1) & 1);   // E1 of tile j in shared memory
                tc::mbar_wait(a2empty, (j & 1) ^ 1);  // acc2 drained (tile j-1)
                tc::tc_fence_after();
#pragma unroll
                for (int kb = 0; kb < KB1; ++kb)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc::mma_bf16(t_acc2, tc::sw128_kmajor_desc(aE1 + (j & 1) * S::kE1Bytes + kb * kBM * 128 + k * 32),
                                     tc::sw128_kmajor_desc(aW2 + kb * E2N * 128 + k * 32), id2, (kb | k) != 0);
                tc::mma_commit(a2full);                // also: E1 buffer j & 1 free again
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue warps
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = quarter * 32 + lane;          // tile row = TMEM lane
        uint8_t* stg = smem + S::kOffStg + (warp - 2) * (32 * 128);
        uint32_t stores = 0;
        auto rowinfo = [&](int j, int& m, int& row, int& cand, int& token) {
            m = blockIdx.x + j * gridDim.x;
            row = m * kBM + r;
            cand = 0; token = 0;
            if (DROP && row < rows) { cand = p.row_cand[row]; token = row - p.cu[cand]; }
        };
        auto epi1 = [&](int j) {
            int m, row, cand, token;
            rowinfo(j, m, row, cand, token);
            // ---- E1 = SiLU(acc1 + b1) (+ dropout site 0) -> bf16 -> swizzled smem (MMA2's A)
            tc::mbar_wait(&a1full[j & 1], (j >> 1) & 1);
            tc::tc_fence_after();
            const uint32_t tb1 = tmem_base + ((uint32_t)(quarter * 32) << 16) + (j & 1) * E1N;
#pragma unroll 1
            for (int c = half * (E1N / 64); c < (half + 1) * (E1N / 64); ++c) {   // 32-column chunks
                uint32_t v[32];
                tc::tmem_ld32(tb1 + c * 32, v);
                tc::tmem_ld_wait();
                uint32_t pk[16];
#pragma unroll
                for (int q = 0; q < 32; q += 4) {
                    float x[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) x[e] = silu_tanh(__uint_as_float(v[q + e]) + s_b1[c * 32 + q + e]);
                    if (DROP) {
                        const u32x4 wd = drop_words_enc(p.drop, c * 32 + q, token, 0, cand);
                        x[0] = dropout_apply_word(p.drop, x[0], wd.x);
                        x[1] = dropout_apply_word(p.drop, x[1], wd.y);
                        x[2] = dropout_apply_word(p.drop, x[2], wd.z);
                        x[3] = dropout_apply_word(p.drop, x[3], wd.w);
                    }
                    pk[q / 2] = pack_bf16x2(x[0], x[1]);
                    pk[q / 2 + 1] = pack_bf16x2(x[2], x[3]);
                }
                const int kb = (c * 32) / 64;               // K-block of MMA2
                const int piece0 = ((c * 32) % 64) / 8;      // first 16-byte piece of the 128-byte row
                uint8_t* dst = sE1 + (j & 1) * S::kE1Bytes + kb * kBM * 128 + r * 128;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<uint4*>(dst + (((piece0 + q) ^ (r & 7)) << 4)) =
                        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            }
            tc::fence_proxy_async();     // generic-proxy smem writes -> visible to tcgen05.mma
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) { tc::mbar_arrive(&e1full[j & 1]); tc::mbar_arrive(&a1empty[j & 1]); }
        };
        auto epi2 = [&](int j) {
            int m, row, cand, token;
            rowinfo(j, m, row, cand, token);
            // ---- E2 = SiLU(acc2 + b2) (+ dropout site 1) -> bf16 -> TMA store
            tc::mbar_wait(a2full, j & 1);
            tc::tc_fence_after();
            const uint32_t tb2 = t_acc2 + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
            for (int c = half * (E2N / 64); c < (half + 1) * (E2N / 64); ++c) {
                uint32_t v[32];
                tc::tmem_ld32(tb2 + c * 32, v);
                tc::tmem_ld_wait();
                uint32_t pk[16];
#pragma unroll
                for (int q = 0; q < 32; q += 4) {
                    float x[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) x[e] = silu_tanh(__uint_as_float(v[q + e]) + s_b2[c * 32 + q + e]);
                    if (DROP) {
                        const u32x4 wd = drop_words_enc(p.drop, c * 32 + q, token, 1, cand);
                        x[0] = dropout_apply_word(p.drop, x[0], wd.x);
                        x[1] = dropout_apply_word(p.drop, x[1], wd.y);
                        x[2] = dropout_apply_word(p.drop, x[2], wd.z);
                        x[3] = dropout_apply_word(p.drop, x[3], wd.w);
                    }
                    pk[q / 2] = pack_bf16x2(x[0], x[1]);
                    pk[q / 2 + 1] = pack_bf16x2(x[2], x[3]);
                }
                const int k = c - half * (E2N / 64);        // chunk within this warp's columns
                if ((k & 1) == 0 && stores > 0) {            // staging reuse: previous store read it
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int piece = (k & 1) * 4 + q;
                    *reinterpret_cast<uint4*>(stg + lane * 128 + ((piece ^ (lane & 7)) << 4)) =
                        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                }
                if (k & 1) {
                    tc::fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                reinterpret_cast<uint64_t>(&tmE2)),
                            "r"((c - 1) * 32), "r"(m * kBM + quarter * 32), "r"(tc::smem_u32(stg))
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    ++stores;
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(a2empty);
        };
        // E1 of tile j+1 is formed while MMA2 of tile j runs (its E1 buffer was freed by MMA2 of j-1)
        if (n_my > 0) epi1(0);
        for (int j = 0; j < n_my; ++j) {
            if (j + 1 < n_my) epi1(j + 1);
            epi2(j);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

template <int E1N, int E2N, bool DROP>
static cudaError_t launch_k(const CUtensorMap& x, const CUtensorMap& w1, const CUtensorMap& w2,
                            const CUtensorMap& e2, const EncParams& p, int num_sms, cudaStream_t s) {
    constexpr int smem = Smem<E1N, E2N>::kBytes;
    auto kern = k_enc12<E1N, E2N, DROP>;
    cudaError_t e = prepare_kernel(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<num_sms, kThreads, smem, s>>>(x, w1, w2, e2, p);
    return cudaGetLastError();
}

}  // namespace enc

bool enc12_supported(int e1, int e2, int d_in) { return d_in <= 32 && ((e1 == 128 && e2 == 256) || (e1 == 64 && e2 == 128)); }

cudaError_t launch_enc12(const CUtensorMap& x, const CUtensorMap& w1, const CUtensorMap& w2, const CUtensorMap& e2,
                         const EncParams& p, int e1n, int e2n, int num_sms, cudaStream_t s) {
    const bool drop = p.drop.enabled != 0;
    if (e1n == 128 && e2n == 256)
        return drop ? enc::launch_k<128, 256, true>(x, w1, w2, e2, p, num_sms, s)
                    : enc::launch_k<128, 256, false>(x, w1, w2, e2, p, num_sms, s);
    if (e1n == 64 && e2n == 128)
        return drop ? enc::launch_k<64, 128, true>(x, w1, w2, e2, p, num_sms, s)
                    : enc::launch_k<64, 128, false>(x, w1, w2, e2, p, num_sms, s);
    return cudaErrorInvalidValue;
}

}  // namespace tcl
