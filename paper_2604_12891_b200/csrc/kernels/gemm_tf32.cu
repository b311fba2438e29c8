// gemm_tf32.cu -- the row GEMMs of the fp32 path on the 5th-generation tensor cores, fp32-accurate
// by the 3xTF32 split (the fp32 configurations' encoder linears, in_proj and
// out_proj: PAPER.md:446, :449-451, trained and evaluated in fp32):
//
//   a = a_hi + a_lo,  a_hi = a with the low 13 mantissa bits cleared (exactly a tf32 number),
//                     a_lo = tf32_rna(a - a_hi)                       (the same split for W)
//   a . w  ~=  a_hi w_hi + a_hi w_lo + a_lo w_hi      (a_lo w_lo ~ 2^-21 |a w| is dropped)
//
// Three tcgen05.mma.kind::tf32 (M = 128, N = BN, K = 8 each) per 8-deep k step accumulate into
// ONE fp32 TMEM accumulator, so each product keeps ~21 bits and the fp32 path's 1e-4 score bound
// holds with two orders of margin (measured: DESIGN.md).  The operands are exact tf32 numbers, so
// the tensor core's own fp32 -> tf32 handling (truncation or rounding) never matters.
//
// Design (as gemm_tc.cu): persistent CTA per SM, weight-stationary (the CTA's [BN x K] slice of
// W_hi and W_lo stays in shared memory, loaded once by TMA), 128-row activation tiles streamed by
// TMA through a ring of K-blocks (16 fp32 = 64 B per row, 64B-swizzled, K-major: half-size stages,
// so that 4+ A loads are in flight next to the resident weights).  Roles (448 threads):
//   warp 0       TMA producer
//   warp 1       TMEM allocator + single-thread MMA issuer (6 MMAs per K-block)
//   warps 2..5   split: A_hi in place (mask) and A_lo (another smem buffer) per landed K-block; the
//                element-wise split keeps the swizzled layout, so no address math is needed
//   warps 6..13  epilogue: warp w drains TMEM lanes 32 (w % 4).., column half (w - 6) / 4
// fp32 accumulators double-buffered in TMEM (2 x BN columns): the epilogue of tile i overlaps the
// MMAs of tile i+1.  Epilogues (fp32 outputs; thread = row for the arithmetic, global rows read and
// written coalesced through a per-warp staging tile, EpiStage):
//   0  Y = acc                                   (in_proj)
//   1  Y = SiLU(acc + b) [inverted dropout]      (encoder linears 1, 2; MC sites 0, 1, R17)
//   3  H = [H +] acc + b, then A = LN(H) if out   (out_proj + residual (+ next LN); encoder linear 3)
// Every output element's value depends on its own row only: batch-invariant.
#include "../kernels.h"
#include "../kernels_tc.h"
#include "../tc_ptx.cuh"

namespace tcl {
namespace tf {

constexpr int kBM = 128;
constexpr int kKBBytes = kBM * 64;    // one 128-row x 16-fp32 K-block (64-byte rows, 64B swizzle)
constexpr int kSplitWarps = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * (kSplitWarps + kEpiWarps);
constexpr int kEpi0 = 2 + kSplitWarps;   // first epilogue warp

// KB counts 32-wide K units (the dispatcher's kb = ceil(K / 32)); the ring moves 16-wide K-blocks
// (K2 = 2 KB of them): half-size stages, twice as many in the same shared memory, so more A loads
// are in flight (measured with 32-wide blocks: 2 stages, the split warps waiting on TMA)
template <int BN, int KB>
struct Smem {
    static constexpr int K2 = 2 * KB;                                // 16-wide K-blocks
    static constexpr int kBBytes = K2 * BN * 64;                     // one weight matrix (hi or lo)
    static constexpr int kStageBytes = 2 * kKBBytes;                 // A_hi + A_lo of one K-block
    static constexpr int kStgBytes = kEpiWarps * 32 * 16 * 4;         // epilogue staging [warp][32 rows][16 fp32]
    static constexpr int kStagesRaw = (220 * 1024 - kStgBytes - 2 * kBBytes) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static constexpr int kOffB = 0;                                  // W_hi, then W_lo
    static constexpr int kOffA = 2 * kBBytes;                        // stage s: A_hi at s*2K, A_lo at s*2K + K
    static constexpr int kOffStg = kOffA + kStages * kStageBytes;
    static constexpr int kOffPar = kOffStg + kStgBytes;              // bias, ln_g, ln_b  [3][BN] fp32
    static constexpr int kOffRed = kOffPar + 3 * BN * 4;             // LN partials [2][128] float2
    static constexpr int kOffBar = kOffRed + 2 * 128 * 8;
    static constexpr int kBytes = kOffBar + 512 + 1024;
    static_assert(kStagesRaw >= 2, "weight slice too large for the 3xTF32 GEMM");
    static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per block");
};

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32 (fp32 accumulate), issued by one thread.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Instruction descriptor, kind::tf32: fp32 accumulator (c_format 1 at [4,6)), A = B = TF32 (2 at
// [7,10) and [10,13)), both K-major, N >> 3 at [17,23), M >> 4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ u32x4 drop_words_tf(const DropoutCtx& d, int unit4, int token, int site, int64_t cand) {
    return dropout_words(d, unit4, token, site, cand);
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Epilogue staging of one warp: 32 rows x 16 fp32 (2 KB), 16-byte group g of row r stored at group
// g ^ ((r >> 1) & 3).  The TMEM layout gives thread = row; global rows are written and read
// coalesced through this tile instead (lane -> row 8 i + lane / 4, group lane % 4: one 128-bit
// access covers 8 rows x 64 contiguous bytes, against 32 rows x 16 bytes per thread-row access).
// Both access patterns are bank-conflict-free (each 8-lane phase covers all 32 banks).
struct EpiStage {
    float* t;
    int lane;
    __device__ __forceinline__ float4* at(int r, int g) const { return reinterpret_cast<float4*>(t + r * 16 + 4 * (g ^ ((r >> 1) & 3))); }
    // thread = row: write / read its 16 values
    __device__ __forceinline__ void put_row(const float* x) const {
#pragma unroll
        for (int g = 0; g < 4; ++g) *at(lane, g) = make_float4(x[4 * g], x[4 * g + 1], x[4 * g + 2], x[4 * g + 3]);
    }
    __device__ __forceinline__ void get_row(float* x) const {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const float4 v = *at(lane, g);
            x[4 * g] = v.x; x[4 * g + 1] = v.y; x[4 * g + 2] = v.z; x[4 * g + 3] = v.w;
        }
    }
    // coalesced: rows [0, 32) of the warp at base (row stride ld floats), rows >= nvalid skipped
    __device__ __forceinline__ void load_global(float4 (&v)[4], const float* base, int64_t ld, int nvalid) const {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = 8 * i + (lane >> 2);
            v[i] = r < nvalid ? *reinterpret_cast<const float4*>(base + r * ld + 4 * (lane & 3)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __device__ __forceinline__ void put_global(const float4 (&v)[4]) const {
#pragma unroll
        for (int i = 0; i < 4; ++i) *at(8 * i + (lane >> 2), lane & 3) = v[i];
    }
    __device__ __forceinline__ void store_global(float* base, int64_t ld, int nvalid) const {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = 8 * i + (lane >> 2);
            if (r < nvalid) *reinterpret_cast<float4*>(base + r * ld + 4 * (lane & 3)) = *at(r, lane & 3);
        }
    }
};

template <int BN, int KB, int EPI>
__global__ void __launch_bounds__(kThreads, 1) k_gemm_tf32(const __grid_constant__ CUtensorMap tmA,
                                                           const __grid_constant__ CUtensorMap tmB,
                                                           const __grid_constant__ CUtensorMap tmBlo,
                                                           const Tf32GemmParams p) {
    using S = Smem<BN, KB>;
    constexpr int kStages = S::kStages;
    constexpr int NCH = BN / 32;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment (128B-swizzled TMA tiles) as an offset from the shared array, so that every
    // access below stays in the shared state space (LDS / STS, not generic LD / ST)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sB = smem + S::kOffB;
    uint8_t* sA = smem + S::kOffA;
    float* s_bias = reinterpret_cast<float*>(smem + S::kOffPar);
    float* s_g = s_bias + BN;
    float* s_b = s_g + BN;
    float2* s_red = reinterpret_cast<float2*>(smem + S::kOffRed);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);   // TMA landed
    uint64_t* split = full + kStages;                                   // hi / lo ready
    uint64_t* empty = split + kStages;                                  // MMAs done with the stage
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
        for (int st = 0; st < kStages; ++st) {
            tc::mbar_init(&full[st], 1);
            tc::mbar_init(&split[st], kSplitWarps);
            tc::mbar_init(&empty[st], 1);
        }
        tc::mbar_init(bfull, 1);
        for (int a = 0; a < 2; ++a) { tc::mbar_init(&tfull[a], 1); tc::mbar_init(&tempty[a], kEpiWarps); }
        tc::fence_mbar_init();
    }
    for (int j = threadIdx.x; j < BN; j += kThreads) {
        const int n = n_tile * BN + j;
        s_bias[j] = p.bias ? __ldg(p.bias + n) : 0.0f;
        if (EPI == 3 && p.out) { s_g[j] = __ldg(p.ln_g + j); s_b[j] = __ldg(p.ln_b + j); }
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer: W_hi, W_lo once; A K-blocks through the ring
            tc::tma_prefetch(&tmA);
            tc::mbar_arrive_expect_tx(bfull, 2 * S::kBBytes);
            for (int kb = 0; kb < S::K2; ++kb) {
                tc::tma_load_2d(sB + kb * BN * 64, &tmB, kb * 16, n_tile * BN, bfull);
                tc::tma_load_2d(sB + S::kBBytes + kb * BN * 64, &tmBlo, kb * 16, n_tile * BN, bfull);
            }
            const uint64_t pol = tc::policy_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            for (int m = m_first; m < num_m; m += m_step) {
                for (int kb = 0; kb < S::K2; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], kKBBytes);
                    tc::tma_load_2d_hint(sA + stage * S::kStageBytes, &tmA, kb * 16, m * kBM, &full[stage], pol);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer: per 8-deep k step  hi.hi + hi.lo + lo.hi
            constexpr uint32_t idesc = idesc_tf32(kBM, BN);
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
                for (int kb = 0; kb < S::K2; ++kb) {
                    tc::mbar_wait(&split[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_hi = sA_addr + stage * S::kStageBytes, a_lo = a_hi + kKBBytes;
                    const uint32_t b_hi = sB_addr + kb * BN * 64, b_lo = b_hi + S::kBBytes;
#pragma unroll
                    for (int k = 0; k < 2; ++k) {   // two 8-deep k steps per 64-byte row
                        const uint64_t ah = tc::sw64_kmajor_desc(a_hi + k * 32), al = tc::sw64_kmajor_desc(a_lo + k * 32);
                        const uint64_t bh = tc::sw64_kmajor_desc(b_hi + k * 32), bl = tc::sw64_kmajor_desc(b_lo + k * 32);
                        mma_tf32(d, ah, bh, idesc, (kb | k) != 0);
                        mma_tf32(d, ah, bl, idesc, 1);
                        mma_tf32(d, al, bh, idesc, 1);
                    }
                    tc::mma_commit(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp < kEpi0) {
        // ---------------- split warps: A_hi = mask(A) in place, A_lo = tf32(A - A_hi)
        const int t = threadIdx.x - 64;   // 0 .. 127
        int stage = 0;
        uint32_t phase = 0;
        for (int m = m_first; m < num_m; m += m_step) {
            for (int kb = 0; kb < S::K2; ++kb) {
                tc::mbar_wait(&full[stage], phase);
                uint4* hi = reinterpret_cast<uint4*>(sA + stage * S::kStageBytes);
                uint4* lo = reinterpret_cast<uint4*>(sA + stage * S::kStageBytes + kKBBytes);
#pragma unroll
                for (int i = 0; i < kKBBytes / 16 / 128; ++i) {
                    const int idx = t + 128 * i;
                    const uint4 v = hi[idx];
                    uint4 h, l;
                    h.x = v.x & 0xFFFFE000u; l.x = tf32_rna(__uint_as_float(v.x) - __uint_as_float(h.x));
                    h.y = v.y & 0xFFFFE000u; l.y = tf32_rna(__uint_as_float(v.y) - __uint_as_float(h.y));
                    h.z = v.z & 0xFFFFE000u; l.z = tf32_rna(__uint_as_float(v.z) - __uint_as_float(h.z));
                    h.w = v.w & 0xFFFFE000u; l.w = tf32_rna(__uint_as_float(v.w) - __uint_as_float(h.w));
                    hi[idx] = h;
                    lo[idx] = l;
                }
                tc::fence_proxy_async();     // generic-proxy smem writes -> visible to tcgen05.mma
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&split[stage]);
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ---------------- epilogue warps
        const int quarter = warp & 3;
        const int half = (warp - kEpi0) >> 2;
        const int rloc = quarter * 32 + lane;
        const EpiStage st{reinterpret_cast<float*>(smem + S::kOffStg) + (warp - kEpi0) * 32 * 16, lane};
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int m = m_first; m < num_m; m += m_step) {
            const int row = m * kBM + rloc;
            const int row0 = m * kBM + quarter * 32;          // the warp's first row
            const int nvalid = rows - row0;                    // rows of the warp inside [0, rows)
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
            if constexpr (EPI != 3) {
                int cand = 0, token = 0;
                if (EPI == 1 && p.drop.enabled && row < rows) { cand = p.row_cand[row]; token = row - p.cu[cand]; }
                float* obase = p.Y + (int64_t)row0 * p.ldy + n_tile * BN;
#pragma unroll 1
                for (int c = half; c < NCH; c += 2) {
                    uint32_t r[32];
                    tc::tmem_ld32(tbase + c * 32, r);
                    tc::tmem_ld_wait();
                    float x[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        x[j] = __uint_as_float(r[j]);
                        if (EPI == 1) x[j] = silu(x[j] + s_bias[c * 32 + j]);
                    }
                    if (EPI == 1 && p.drop.enabled) {   // one Philox draw per 4 consecutive units
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const u32x4 wd = drop_words_tf(p.drop, n_tile * BN + c * 32 + j, token, p.site, cand);
                            x[j] = dropout_apply_word(p.drop, x[j], wd.x);
                            x[j + 1] = dropout_apply_word(p.drop, x[j + 1], wd.y);
                            x[j + 2] = dropout_apply_word(p.drop, x[j + 2], wd.z);
                            x[j + 3] = dropout_apply_word(p.drop, x[j + 3], wd.w);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        st.put_row(x + 16 * h);
                        __syncwarp();
                        st.store_global(obase + c * 32 + 16 * h, p.ldy, nvalid);
                        __syncwarp();
                    }
                }
            } else {
                // pass 1: v = [H +] acc + b; store H; keep v in TMEM; partial row sum.  The residual
                // rows arrive coalesced (issued before the TMEM load) and are transposed through
                // the staging tile.
                float* hbase = p.H + (int64_t)row0 * p.ldh + n_tile * BN;   // this CTA's columns
                float sum = 0.f;
#pragma unroll 1
                for (int c = half; c < NCH; c += 2) {
                    float4 hg[4];
                    if (p.residual) st.load_global(hg, hbase + c * 32, p.ldh, nvalid);
                    uint32_t r[32];
                    tc::tmem_ld32(tbase + c * 32, r);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float hv[16];
                        if (p.residual) {
                            st.put_global(hg);
                            __syncwarp();
                            if (h == 0) st.load_global(hg, hbase + c * 32 + 16, p.ldh, nvalid);   // next half in flight
                            st.get_row(hv);
                        } else {
#pragma unroll
                            for (int q = 0; q < 16; ++q) hv[q] = 0.0f;
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int jj = 16 * h + j;
                            const float v = hv[j] + (__uint_as_float(r[jj]) + s_bias[c * 32 + jj]);
                            hv[j] = v;
                            sum += v;
                            r[jj] = __float_as_uint(v);
                        }
                        st.put_row(hv);   // own row only: no hazard with this thread's get_row above
                        __syncwarp();
                        st.store_global(hbase + c * 32 + 16 * h, p.ldh, nvalid);
                        __syncwarp();
                    }
                    if (p.out) tc::tmem_st32(tbase + c * 32, r);
                }
                if (p.out) {
                    tc::tmem_st_wait();
                    s_red[half * 128 + rloc].x = sum;
                    named_bar(1 + quarter, 64);
                    const float mean = (s_red[rloc].x + s_red[128 + rloc].x) * (1.0f / BN);
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
                    const float rstd = rsqrtf((s_red[rloc].y + s_red[128 + rloc].y) * (1.0f / BN) + p.eps);
                    float* abase = p.out + (int64_t)row0 * p.ldo;
#pragma unroll 1
                    for (int c = half; c < NCH; c += 2) {
                        uint32_t r[32];
                        tc::tmem_ld32(tbase + c * 32, r);
                        tc::tmem_ld_wait();
                        float a[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            a[j] = (__uint_as_float(r[j]) - mean) * rstd * s_g[c * 32 + j] + s_b[c * 32 + j];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            st.put_row(a + 16 * h);
                            __syncwarp();
                            st.store_global(abase + c * 32 + 16 * h, p.ldo, nvalid);
                            __syncwarp();
                        }
                    }
                    named_bar(1 + quarter, 64);  // s_red reuse guard for the next tile
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 2 * BN);
    }
}

template <int BN, int KB, int EPI>
static cudaError_t launch_impl(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& blo,
                               const Tf32GemmParams& p, int grid, cudaStream_t s) {
    constexpr int smem = Smem<BN, KB>::kBytes;
    auto kern = k_gemm_tf32<BN, KB, EPI>;
    cudaError_t e = prepare_kernel(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(a, b, blo, p);
    return cudaGetLastError();
}

template <int BN, int KB>
static cudaError_t launch_epi(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& blo,
                              const Tf32GemmParams& p, int grid, cudaStream_t s) {
    if (p.epi == 3) return launch_impl<BN, KB, 3>(a, b, blo, p, grid, s);
    if (p.epi == 1) return launch_impl<BN, KB, 1>(a, b, blo, p, grid, s);
    return launch_impl<BN, KB, 0>(a, b, blo, p, grid, s);
}

__global__ void k_tf32_split(const float* __restrict__ w, int64_t n, float* __restrict__ hi, float* __restrict__ lo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float v = w[i];
    const uint32_t h = __float_as_uint(v) & 0xFFFFE000u;
    hi[i] = __uint_as_float(h);
    lo[i] = __uint_as_float(tf32_rna(v - __uint_as_float(h)));
}

}  // namespace tf

void launch_tf32_split(const float* w, int64_t n, float* hi, float* lo, cudaStream_t s) {
    if (n > 0) tf::k_tf32_split<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w, n, hi, lo);
}

// Exactly the (bn, kb) pairs instantiated in launch_gemm_tf32 below.
bool tf32_gemm_supported(int bn, int k) {
    const int kb = (k + 31) / 32;
    return (bn == 32 || bn == 64 || bn == 128 || bn == 256) && (kb == 1 || kb == 2 || kb == 4 || kb == 8) &&
           kb * bn <= 512;   // both weight halves resident + a 2-stage ring of A K-blocks
}

cudaError_t launch_gemm_tf32(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& blo,
                             const Tf32GemmParams& p, int bn, int k, int num_sms, cudaStream_t s) {
    const int kb = (k + 31) / 32;
    if (p.epi == 3 && p.out && p.n_tiles != 1) return cudaErrorInvalidValue;   // LN needs whole rows
    const int grid = (num_sms / p.n_tiles) * p.n_tiles;
#define TCL_TF_CASE(BN_, KB_) \
    if (bn == BN_ && kb == KB_) return tf::launch_epi<BN_, KB_>(a, b, blo, p, grid, s);
    TCL_TF_CASE(32, 1) TCL_TF_CASE(32, 2) TCL_TF_CASE(32, 4) TCL_TF_CASE(32, 8)
    TCL_TF_CASE(64, 1) TCL_TF_CASE(64, 2) TCL_TF_CASE(64, 4) TCL_TF_CASE(64, 8)
    TCL_TF_CASE(128, 1) TCL_TF_CASE(128, 2) TCL_TF_CASE(128, 4)
    TCL_TF_CASE(256, 1) TCL_TF_CASE(256, 2)
#undef TCL_TF_CASE
    return cudaErrorInvalidValue;
}

}  // namespace tcl
