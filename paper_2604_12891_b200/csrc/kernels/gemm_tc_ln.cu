// gemm_tc_ln.cu -- tcgen05 GEMM with the residual + LayerNorm epilogue (bf16 path):
//
//   H <- (residual ? H : 0) + acc (+ bias);   out = bf16(LN(H) * g + b)
//
// used for out_proj (+ the next layer's pre-norm; SURVEY §8(a) a8 + a3) and for
// the encoder's last linear (+ LN_0).  The row of H is d_model wide (BN = d_model <= 256), so one
// CTA owns full rows and computes the LayerNorm statistics itself.
//
// Differences from gemm_tc.cu (which keeps its weight slice resident): the weight tile is
// streamed with each K-block (it is L2-resident, < 4 MB for the whole model), which frees the
// shared memory for TMA staging of the fp32 residual stream: every epilogue warp moves its
// 32-row x 32-column fp32 chunks of H in and out with cp.async.bulk.tensor (128B-swizzled, so the
// row-per-thread TMEM layout reads and writes shared memory without bank conflicts), and the
// bf16 LayerNorm output leaves through TMA stores as well.  All global traffic of the epilogue is
// therefore full-line bulk copies instead of per-thread strided accesses (the L1 wavefront limit
// of the previous version).
#include <cuda_bf16.h>

#include "../kernels.h"
#include "../kernels_tc.h"
#include "../tc_ptx.cuh"

namespace tcl {

namespace ln {

constexpr int kBM = 128;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN, int KB>
struct Smem {
    static constexpr int kStageBytes = kBM * 128 + BN * 128;          // A k-block + B k-block
    static constexpr int kStages = BN >= 256 ? 2 : 3;
    static constexpr int kStgPerWarp = 3 * 32 * 128;                  // H buf[2] + out buf
    static constexpr int kOffStage = 0;
    static constexpr int kOffStg = kOffStage + kStages * kStageBytes;
    static constexpr int kOffPar = kOffStg + kEpiWarps * kStgPerWarp;
    static constexpr int kOffRed = kOffPar + 3 * BN * 4;
    static constexpr int kOffBar = kOffRed + 2 * 128 * 8;
    static constexpr int kBytes = kOffBar + 512 + 1024;
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(tc::smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void store_read_wait_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// 16-byte piece p (0..7) of row r in a 128B-swizzled [rows][128 B] tile
__device__ __forceinline__ uint32_t sw_off(int r, int p) { return r * 128 + ((p ^ (r & 7)) << 4); }

template <int BN, int KB>
__global__ void __launch_bounds__(kThreads, 1) k_gemm_ln(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         const __grid_constant__ CUtensorMap tmH,
                                                         const __grid_constant__ CUtensorMap tmO,
                                                         const TcGemmParams p) {
    using S = Smem<BN, KB>;
    constexpr int kStages = S::kStages;
    constexpr int NC = BN / 64;  // 32-column chunks per epilogue warp (its column half)
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment (128B-swizzled TMA tiles) as an offset from the shared array, so that every
    // access below stays in the shared state space (LDS / STS, not generic LD / ST)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    float* s_bias = reinterpret_cast<float*>(smem + S::kOffPar);
    float* s_g = s_bias + BN;
    float* s_b = s_g + BN;
    float2* s_red = reinterpret_cast<float2*>(smem + S::kOffRed);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;   // [2]
    uint64_t* tempty = tfull + 2;        // [2]
    uint64_t* hbar = tempty + 2;         // [kEpiWarps][2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hbar + 2 * kEpiWarps);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = *p.p_rows;
    const int num_m = (rows + kBM - 1) / kBM;

    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st) { tc::mbar_init(&full[st], 1); tc::mbar_init(&empty[st], 1); }
        for (int a = 0; a < 2; ++a) { tc::mbar_init(&tfull[a], 1); tc::mbar_init(&tempty[a], kEpiWarps); }
        for (int k = 0; k < 2 * kEpiWarps; ++k) tc::mbar_init(&hbar[k], 1);
        tc::fence_mbar_init();
    }
    for (int j = threadIdx.x; j < BN; j += kThreads) {
        s_bias[j] = p.bias ? __ldg(p.bias + j) : 0.0f;
        s_g[j] = p.out ? __ldg(p.ln_g + j) : 0.0f;
        s_b[j] = p.out ? __ldg(p.ln_b + j) : 0.0f;
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer: A and B k-blocks per stage
            tc::tma_prefetch(&tmA);
            tc::tma_prefetch(&tmB);
            const uint64_t pol = tc::policy_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            for (int m = blockIdx.x; m < num_m; m += gridDim.x) {
                for (int kb = 0; kb < KB; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smem + S::kOffStage + stage * S::kStageBytes;
                    tc::mbar_arrive_expect_tx(&full[stage], S::kStageBytes);
                    tc::tma_load_2d_hint(st, &tmA, kb * 64, m * kBM, &full[stage], pol);
                    tc::tma_load_2d(st + kBM * 128, &tmB, kb * 64, 0, &full[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint32_t idesc = tc::idesc_bf16_f32(kBM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int m = blockIdx.x; m < num_m; m += gridDim.x) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kb = 0; kb < KB; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t sa = tc::smem_u32(smem + S::kOffStage + stage * S::kStageBytes);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t ad = tc::sw128_kmajor_desc(sa + k * 32);
                        const uint64_t bd = tc::sw128_kmajor_desc(sa + kBM * 128 + k * 32);
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
        // ---------------- epilogue warps: rows 32*quarter + lane, columns [half*BN/2, (half+1)*BN/2)
        const int ew = warp - 2;
        const int quarter = warp & 3;
        const int half = ew >> 2;
        const int rloc = quarter * 32 + lane;
        const int col0 = half * (BN / 2);
        uint8_t* hb = smem + S::kOffStg + ew * S::kStgPerWarp;   // H buffers [2][32][128 B]
        uint8_t* ob = hb + 2 * 32 * 128;                          // out staging [32][128 B]
        uint64_t* hbw = hbar + 2 * ew;
        uint32_t hph = 0;   // phase bits of hbw[0], hbw[1]
        int acc = 0;
        uint32_t acc_phase = 0;
        const bool res = p.residual != 0;
        auto load_h = [&](int m, int c, int b) {  // lane 0 only
            tc::mbar_arrive_expect_tx(&hbw[b], 32 * 128);
            tc::tma_load_2d(hb + b * 32 * 128, &tmH, col0 + c * 32, m * kBM + quarter * 32, &hbw[b]);
        };
        int m = blockIdx.x;
        if (res && m < num_m && lane == 0) {
            for (int c = 0; c < NC && c < 2; ++c) load_h(m, c, c);
        }
        for (; m < num_m; m += gridDim.x) {
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + col0;
            // ---- pass 1: v = acc + bias (+ H); H out via TMA; v kept in TMEM; partial row sum
            float sum = 0.f;
#pragma unroll 1
            for (int c = 0; c < NC; ++c) {
                const int b = c & 1;
                uint32_t r[32];
                tc::tmem_ld32(tbase + c * 32, r);
                uint8_t* buf = hb + b * 32 * 128;
                if (res) {
                    tc::mbar_wait(&hbw[b], (hph >> b) & 1u);
                    hph ^= 1u << b;
                } else {
                    if (lane == 0) store_read_wait_all();   // buffer b's previous store has read it
                    __syncwarp();
                }
                float4 hv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    hv[q] = res ? *reinterpret_cast<const float4*>(buf + sw_off(lane, q)) : make_float4(0.f, 0.f, 0.f, 0.f);
                tc::tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int n = col0 + c * 32 + 4 * q;
                    float4 v;
                    v.x = __uint_as_float(r[4 * q]) + s_bias[n] + hv[q].x;
                    v.y = __uint_as_float(r[4 * q + 1]) + s_bias[n + 1] + hv[q].y;
                    v.z = __uint_as_float(r[4 * q + 2]) + s_bias[n + 2] + hv[q].z;
                    v.w = __uint_as_float(r[4 * q + 3]) + s_bias[n + 3] + hv[q].w;
                    sum += (v.x + v.y) + (v.z + v.w);
                    r[4 * q] = __float_as_uint(v.x); r[4 * q + 1] = __float_as_uint(v.y);
                    r[4 * q + 2] = __float_as_uint(v.z); r[4 * q + 3] = __float_as_uint(v.w);
                    *reinterpret_cast<float4*>(buf + sw_off(lane, q)) = v;
                }
                tc::tmem_st32(tbase + c * 32, r);
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    if (!p.skip_h_store) tma_store_2d(&tmH, col0 + c * 32, m * kBM + quarter * 32, buf);
                    if (res && c + 2 < NC) {           // refill this buffer with chunk c + 2
                        store_read_wait_all();
                        load_h(m, c + 2, b);
                    }
                }
                __syncwarp();
            }
            tc::tmem_st_wait();
            // prefetch the next tile's first H chunks (overlaps the LN passes and the next MMAs)
            const int mn = m + gridDim.x;
            if (res && mn < num_m && lane == 0) {
                store_read_wait_all();
                for (int c = 0; c < NC && c < 2; ++c) load_h(mn, c, c);
            }
            __syncwarp();
            // ---- LayerNorm statistics of the full row (two-pass, halves exchanged via smem)
            s_red[half * 128 + rloc].x = sum;
            named_bar(1 + quarter, 64);
            const float mean = (s_red[rloc].x + s_red[128 + rloc].x) * (1.0f / BN);
            float sq = 0.f;
#pragma unroll 1
            for (int c = 0; c < NC; ++c) {
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
            const float rstd = rsqrtf((s_red[rloc].y + s_red[128 + rloc].y) * (1.0f / BN) + p.eps);
            named_bar(1 + quarter, 64);  // s_red reads done before the next tile writes it
            // ---- pass 3: normalise -> bf16, 64-column boxes through the out staging buffer
            if (p.out) {
#pragma unroll 1
                for (int c = 0; c < NC; ++c) {
                    uint32_t r[32];
                    tc::tmem_ld32(tbase + c * 32, r);
                    tc::tmem_ld_wait();
                    if ((c & 1) == 0) {
                        if (lane == 0) store_read_wait_all();
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t pk[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int j = 8 * q + 2 * e;
                            const int n = col0 + c * 32 + j;
                            const float a0 = (__uint_as_float(r[j]) - mean) * rstd * s_g[n] + s_b[n];
                            const float a1 = (__uint_as_float(r[j + 1]) - mean) * rstd * s_g[n + 1] + s_b[n + 1];
                            pk[e] = pack_bf16x2(a0, a1);
                        }
                        *reinterpret_cast<uint4*>(ob + sw_off(lane, (c & 1) * 4 + q)) =
                            make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                    if (c & 1) {
                        tc::fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) tma_store_2d(&tmO, col0 + (c - 1) * 32, m * kBM + quarter * 32, ob);
                        __syncwarp();
                    }
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 2 * BN);
    }
}

template <int BN, int KB>
static cudaError_t launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& h, const CUtensorMap& o,
                          const TcGemmParams& p, int num_sms, cudaStream_t s) {
    constexpr int smem = Smem<BN, KB>::kBytes;
    cudaError_t e = prepare_kernel(k_gemm_ln<BN, KB>, smem);
    if (e != cudaSuccess) return e;
    k_gemm_ln<BN, KB><<<num_sms, kThreads, smem, s>>>(a, b, h, o, p);
    return cudaGetLastError();
}

}  // namespace ln

cudaError_t launch_gemm_tc_ln(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& h,
                              const CUtensorMap& o, const TcGemmParams& p, int bn, int kb, int num_sms,
                              cudaStream_t s) {
#define TCL_LN_CASE(BN_, KB_) if (bn == BN_ && kb == KB_) return ln::launch<BN_, KB_>(a, b, h, o, p, num_sms, s);
    TCL_LN_CASE(256, 1) TCL_LN_CASE(256, 2) TCL_LN_CASE(256, 3) TCL_LN_CASE(256, 4)
    TCL_LN_CASE(128, 1) TCL_LN_CASE(128, 2) TCL_LN_CASE(128, 3) TCL_LN_CASE(128, 4)
#undef TCL_LN_CASE
    return cudaErrorInvalidValue;
}

}  // namespace tcl
