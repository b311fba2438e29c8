// gemm_tc.cu -- the projections of the bf16 path on the 5th-generation tensor cores (tcgen05).
//
//   out_proj  H <- H + g W_out^T, then LN_{l+1}(H)   (a8 + a3 of the next layer, fused epilogue;
//             the d_model < 128 configurations -- gemm_tc_ln.cu takes d_model 128 / 256)
//   encoder   SiLU(X W1^T + b1), SiLU(. W2^T + b2), . W3^T + b3 (+ LN_0)   (a2)
//             (the linears that k_enc12 / gemm_tc_ln do not take)
// (in_proj runs in k_inconv, inconv.cu, fused with the conv.)
//
// Design (B200-first): persistent, warp-specialised, weight-stationary.  Each CTA keeps its
// [BN x K] slice of the weight matrix resident in shared memory for the whole launch (loaded once
// by TMA), and streams 128-row activation tiles through a 4-stage TMA ring (128B-swizzled,
// K-major).  One elected thread issues tcgen05.mma (M=128, N=BN, K=16 per instruction) into a
// double-buffered fp32 accumulator in TMEM (2 x BN columns), so the epilogue of tile i overlaps
// the MMAs of tile i+1.  Four epilogue warps drain TMEM with tcgen05.ld (one row per thread) and
// apply the fused epilogue (bias, SiLU, MC-dropout, bf16 pack; or residual add + LayerNorm of the
// next layer computed in-thread from the full row).
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2..5 = epilogue (warp w drains TMEM lanes 32*(w%4) .. 32*(w%4)+31).
#include <cuda_bf16.h>

#include "../kernels.h"
#include "../kernels_tc.h"
#include "../tc_ptx.cuh"

namespace tcl {

constexpr int kBM = 128;
constexpr int kABytes = kBM * 128;  // one 128 x 64 bf16 K-block of A
constexpr int kEpiWarps = 8;        // two warps per TMEM lane quarter (column halves)
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN, int KB, int EPI>
struct TcSmem {
    static constexpr bool kTmaStore = EPI < 3 && BN >= 128;          // bf16 out through TMA stores
    // staging per epilogue warp: [32 rows][128 B] x kStgBufs (one TMA store per 64 columns; BN = 128
    // issues a single store per tile and warp, so one buffer suffices and the smem goes to the A ring;
    // a 128 KB weight slice also leaves room for only one)
    static constexpr int kBBytes = KB * BN * 128;
    static constexpr int kStgBufs = (BN <= 128 || kBBytes > 96 * 1024) ? 1 : 2;
    static constexpr int kStgBytes = kTmaStore ? kEpiWarps * kStgBufs * 32 * 128 : 0;
    static constexpr int kStagesRaw = (216 * 1024 - kBBytes - kStgBytes) / kABytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : (kStagesRaw < 2 ? 2 : kStagesRaw);
    static constexpr int kOffB = 0;
    static constexpr int kOffA = kOffB + kBBytes;
    static constexpr int kOffStg = kOffA + kStages * kABytes;         // 1024-aligned (swizzled staging)
    static constexpr int kOffPar = kOffStg + kStgBytes;               // bias, ln_g, ln_b  [3][BN] fp32
    static constexpr int kOffRed = kOffPar + 3 * BN * 4;              // LN partials [2][128] float2
    static constexpr int kOffBar = kOffRed + 2 * 128 * 8;
    static constexpr int kBytes = kOffBar + 256 + 1024;               // + barriers, + alignment slack
    static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per block");
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// MC-dropout keep words, inlined (an out-of-line call kept a stack frame and extra registers in every
// dropout epilogue: measured slower)
__device__ __forceinline__ u32x4 drop_words(const DropoutCtx& d, int unit4, int token, int site, int64_t cand) {
    return dropout_words(d, unit4, token, site, cand);
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// EPI: 0 = bf16 out; 1 = bf16 out of SiLU(acc + bias); 2 = same + MC dropout;
//      3 = residual/bias into fp32 H, then LayerNorm(H) -> bf16 out (BN == full row)
template <int BN, int KB, int EPI>
__global__ void __launch_bounds__(kThreads, 1) k_gemm_tc(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         const __grid_constant__ CUtensorMap tmC,
                                                         const TcGemmParams p) {
    using S = TcSmem<BN, KB, EPI>;
    constexpr int kStages = S::kStages;
    constexpr int NCH = BN / 32;  // 32-column chunks of the accumulator
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment (128B-swizzled TMA tiles) as an offset from the shared array, so that every
    // access below stays in the shared state space (LDS / STS, not generic LD / ST)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem + S::kOffB;
    uint8_t* sA = smem + S::kOffA;
    float* s_bias = reinterpret_cast<float*>(smem + S::kOffPar);
    float* s_g = s_bias + BN;
    float* s_b = s_g + BN;
    float2* s_red = reinterpret_cast<float2*>(smem + S::kOffRed);  // [2 halves][128 rows]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
    uint64_t* empty = full + kStages;
    uint64_t* bfull = empty + kStages;
    uint64_t* tfull = bfull + 1;      // [2]
    uint64_t* tempty = tfull + 2;     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = *p.p_rows;
    const int num_m = (rows + kBM - 1) / kBM;
    const int n_tile = blockIdx.x % p.n_tiles;
    const int m_first = blockIdx.x / p.n_tiles;
    const int m_step = gridDim.x / p.n_tiles;

    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st) { tc::mbar_init(&full[st], 1); tc::mbar_init(&empty[st], 1); }
        tc::mbar_init(bfull, 1);
        for (int a = 0; a < 2; ++a) { tc::mbar_init(&tfull[a], 1); tc::mbar_init(&tempty[a], kEpiWarps); }
        tc::fence_mbar_init();
    }
    for (int j = threadIdx.x; j < BN; j += kThreads) {
        const int n = n_tile * BN + j;
        s_bias[j] = p.bias ? __ldg(p.bias + n) : 0.0f;
        if (EPI == 3) { s_g[j] = __ldg(p.ln_g + j); s_b[j] = __ldg(p.ln_b + j); }
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            tc::tma_prefetch(&tmA);
            tc::tma_prefetch(&tmB);
            tc::mbar_arrive_expect_tx(bfull, S::kBBytes);
            for (int kb = 0; kb < KB; ++kb)
                tc::tma_load_2d(sB + kb * BN * 128, &tmB, kb * 64, n_tile * BN, bfull);
            const uint64_t pol = tc::policy_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            for (int m = m_first; m < num_m; m += m_step) {
                for (int kb = 0; kb < KB; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], kABytes);
                    tc::tma_load_2d_hint(sA + stage * kABytes, &tmA, kb * 64, m * kBM, &full[stage], pol);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread)
            constexpr uint32_t idesc = tc::idesc_bf16_f32(kBM, BN);
            tc::mbar_wait(bfull, 0);
            tc::tc_fence_after();
            const uint32_t sA_addr = tc::smem_u32(sA), sB_addr = tc::smem_u32(sB);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int m = m_first; m < num_m; m += m_step) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kb = 0; kb < KB; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t ad = tc::sw128_kmajor_desc(sA_addr + stage * kABytes + k * 32);
                        const uint64_t bd = tc::sw128_kmajor_desc(sB_addr + kb * BN * 128 + k * 32);
                        tc::mma_bf16(d, ad, bd, idesc, (kb | k) != 0);
                    }
                    tc::mma_commit(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue warps: warp w drains TMEM lanes 32*(w%4).., column half h
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        const int rloc = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t groups = 0;  // TMA-store groups issued by this warp (staging double buffer)
        for (int m = m_first; m < num_m; m += m_step) {
            const int row = m * kBM + rloc;
            const bool valid = row < rows;
            // residual stream: prefetch this row's first H chunk before waiting for the MMAs
            float4 hn[8];
            if constexpr (EPI == 3) {
                if (p.residual && valid) {
                    const float4* h4 = reinterpret_cast<const float4*>(p.H + (int64_t)row * p.ldh + half * 32);
#pragma unroll
                    for (int q = 0; q < 8; ++q) hn[q] = h4[q];
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) hn[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
            if constexpr (EPI != 3) {
                int cand = 0, token = 0;
                if (EPI == 2 && valid) { cand = p.row_cand[row]; token = row - p.cu[cand]; }
                __nv_bfloat16* orow = p.out + (int64_t)row * p.ldo + n_tile * BN;
                // S::kTmaStore: this warp owns the contiguous columns [half*BN/2, (half+1)*BN/2),
                // staged 64 columns at a time in a 128B-swizzled [32 rows][128 B] buffer, stored by TMA.
                constexpr int C0 = S::kTmaStore ? 1 : 2;   // chunk stride
#pragma unroll 1
                for (int k = 0; k < (S::kTmaStore ? NCH / 2 : (NCH + 1 - half) / 2); ++k) {
                    const int c = S::kTmaStore ? half * (NCH / 2) + k : half + k * C0;
                    uint32_t r[32];
                    tc::tmem_ld32(tbase + c * 32, r);
                    tc::tmem_ld_wait();
                    uint32_t pk[16];
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        float x[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            x[e] = __uint_as_float(r[j + e]);
                            if (EPI >= 1) x[e] = silu_tanh(x[e] + s_bias[c * 32 + j + e]);
                        }
                        if (EPI == 2) {   // one Philox draw for the 4 consecutive units
                            const u32x4 wd = drop_words(p.drop, n_tile * BN + c * 32 + j, token, p.site, cand);
                            x[0] = dropout_apply_word(p.drop, x[0], wd.x);
                            x[1] = dropout_apply_word(p.drop, x[1], wd.y);
                            x[2] = dropout_apply_word(p.drop, x[2], wd.z);
                            x[3] = dropout_apply_word(p.drop, x[3], wd.w);
                        }
                        pk[j / 2] = pack_bf16x2(x[0], x[1]);
                        pk[j / 2 + 1] = pack_bf16x2(x[2], x[3]);
                    }
                    if constexpr (S::kTmaStore) {
                        // chunk parity picks the 64-byte half of the 128-byte staged row
                        const int buf = S::kStgBufs == 2 ? (groups & 1) : 0;
                        uint8_t* stg = smem + S::kOffStg + ((warp - 2) * S::kStgBufs + buf) * (32 * 128);
                        if ((k & 1) == 0 && groups >= (uint32_t)S::kStgBufs) {  // buffer reuse: its store must have read smem
                            if (lane == 0) {
                                if (S::kStgBufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                                else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                            }
                            __syncwarp();
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int piece = (k & 1) * 4 + q;              // 16-byte piece of the 128-byte row
                            const int sw = piece ^ (lane & 7);
                            *reinterpret_cast<uint4*>(stg + lane * 128 + sw * 16) =
                                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                        }
                        if (k & 1) {
                            tc::fence_proxy_async();
                            __syncwarp();
                            if (lane == 0) {
                                const int col = n_tile * BN + (c - 1) * 32;
                                asm volatile(
                                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                                    ::"l"(reinterpret_cast<uint64_t>(&tmC)), "r"(col),
                                    "r"(m * kBM + quarter * 32), "r"(tc::smem_u32(stg))
                                    : "memory");
                                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                            }
                            ++groups;
                        }
                    } else if (valid) {
                        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
                        for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                    }
                }
            } else {
                // pass 1: v = acc + bias (+ H_old); store H; keep v in TMEM; partial row sum
                float* hrow = p.H + (int64_t)row * p.ldh;
                float sum = 0.f;
#pragma unroll 1
                for (int c = half; c < NCH; c += 2) {
                    uint32_t r[32];
                    tc::tmem_ld32(tbase + c * 32, r);
                    float hv[32];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        hv[4 * q] = hn[q].x; hv[4 * q + 1] = hn[q].y; hv[4 * q + 2] = hn[q].z; hv[4 * q + 3] = hn[q].w;
                    }
                    if (p.residual && valid && c + 2 < NCH) {  // prefetch the next chunk
                        const float4* h4 = reinterpret_cast<const float4*>(hrow + (c + 2) * 32);
#pragma unroll
                        for (int q = 0; q < 8; ++q) hn[q] = h4[q];
                    }
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float v = __uint_as_float(r[j]) + s_bias[c * 32 + j] + hv[j];
                        hv[j] = v;
                        sum += v;
                        r[j] = __float_as_uint(v);
                    }
                    if (valid) {
                        float4* o4 = reinterpret_cast<float4*>(hrow + c * 32);
#pragma unroll
                        for (int q = 0; q < 8; ++q) o4[q] = make_float4(hv[4 * q], hv[4 * q + 1], hv[4 * q + 2], hv[4 * q + 3]);
                    }
                    tc::tmem_st32(tbase + c * 32, r);
                }
                tc::tmem_st_wait();
                // exchange the halves' partial sums (named barrier of the 2 warps of this quarter)
                s_red[half * 128 + rloc].x = sum;
                named_bar(1 + quarter, 64);
                const float mean = (s_red[rloc].x + s_red[128 + rloc].x) * (1.0f / BN);
                // pass 2: sum of squared deviations (two-pass variance, no cancellation)
                float sq = 0.f;
#pragma unroll 1
                for (int c = half; c < NCH; c += 2) {
                    uint32_t r[32];
                    tc::tmem_ld32(tbase + c * 32, r);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float e = __uint_as_float(r[j]) - mean;
                        sq = fmaf(e, e, sq);
                    }
                }
                s_red[half * 128 + rloc].y = sq;
                named_bar(1 + quarter, 64);
                const float var = (s_red[rloc].y + s_red[128 + rloc].y) * (1.0f / BN);
                const float rstd = rsqrtf(var + p.eps);
                // pass 3: normalise -> bf16
                if (p.out) {
                    __nv_bfloat16* arow = p.out + (int64_t)row * p.ldo;
#pragma unroll 1
                    for (int c = half; c < NCH; c += 2) {
                        uint32_t r[32];
                        tc::tmem_ld32(tbase + c * 32, r);
                        tc::tmem_ld_wait();
                        uint32_t pk[16];
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            const int n = c * 32 + j;
                            const float a0 = (__uint_as_float(r[j]) - mean) * rstd * s_g[n] + s_b[n];
                            const float a1 = (__uint_as_float(r[j + 1]) - mean) * rstd * s_g[n + 1] + s_b[n + 1];
                            pk[j / 2] = pack_bf16x2(a0, a1);
                        }
                        if (valid) {
                            uint4* dst = reinterpret_cast<uint4*>(arow + c * 32);
#pragma unroll
                            for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                        }
                    }
                }
                named_bar(1 + quarter, 64);  // s_red reuse guard for the next tile
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    if constexpr (S::kTmaStore) {
        if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 2 * BN);
    }
}

// ------------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

static bool make_tmap(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tmap_f32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                   uint32_t box_inner, uint32_t box_outer) {
    return make_tmap(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, inner, outer, row_bytes, box_inner, box_outer);
}

bool make_tmap_f32_sw64(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                        uint32_t box_outer) {
    return make_tmap(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, inner, outer, row_bytes, 16, box_outer,
                     CU_TENSOR_MAP_SWIZZLE_64B);
}

bool make_tmap_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                    uint32_t box_inner, uint32_t box_outer) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BN, int KB, int EPI>
static cudaError_t launch_impl(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                               const TcGemmParams& p, int grid, cudaStream_t s) {
    const int smem = TcSmem<BN, KB, EPI>::kBytes;
    auto kern = k_gemm_tc<BN, KB, EPI>;
    cudaError_t e = prepare_kernel(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(a, b, c, p);
    return cudaGetLastError();
}

template <int BN, int KB>
static cudaError_t launch_epi(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                              const TcGemmParams& p, int grid, cudaStream_t s) {
    if (p.epi == TC_EPI_RESID_LN) return launch_impl<BN, KB, 3>(a, b, c, p, grid, s);
    if (p.drop.enabled) return launch_impl<BN, KB, 2>(a, b, c, p, grid, s);
    if (p.act_silu) return launch_impl<BN, KB, 1>(a, b, c, p, grid, s);
    return launch_impl<BN, KB, 0>(a, b, c, p, grid, s);
}

cudaError_t launch_gemm_tc(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                           const TcGemmParams& p, int bn, int kb, int num_sms, cudaStream_t s) {
    // grid: one persistent CTA per SM, a multiple of the number of N tiles
    const int grid = (num_sms / p.n_tiles) * p.n_tiles;
    if (p.epi == TC_EPI_BF16 && p.act_silu == 0 && p.bias) return cudaErrorInvalidValue;  // unsupported combo
#define TCL_TC_CASE(BN_, KB_) if (bn == BN_ && kb == KB_) return launch_epi<BN_, KB_>(a, b, c, p, grid, s);
    TCL_TC_CASE(256, 1) TCL_TC_CASE(256, 2) TCL_TC_CASE(256, 3) TCL_TC_CASE(256, 4)
    TCL_TC_CASE(128, 1) TCL_TC_CASE(128, 2) TCL_TC_CASE(128, 3) TCL_TC_CASE(128, 4)
    TCL_TC_CASE(64, 1) TCL_TC_CASE(64, 2) TCL_TC_CASE(64, 3) TCL_TC_CASE(64, 4)
    TCL_TC_CASE(32, 1) TCL_TC_CASE(32, 2) TCL_TC_CASE(32, 3) TCL_TC_CASE(32, 4)
#undef TCL_TC_CASE
    return cudaErrorInvalidValue;
}

}  // namespace tcl
