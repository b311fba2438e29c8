// inconv.cu -- in_proj + SiLU(z) + causal depthwise conv + SiLU of the bf16 path in ONE tcgen05
// kernel (PAPER.md:446 in_proj, P:570 conv; readings R4, R25):
//
//   [x | z] = LN_l(H) W_in^T                      (tcgen05: M = 128 rows, N = 2 HC channels)
//   GZ = SiLU(z)                                  -> [P][DI] bf16, the scan's gate
//   u  = SiLU(b_conv + causal conv_4(x))          -> the mixer packet's u columns (fp16)
//
// x never leaves the SM: as an in_proj GEMM followed by a conv kernel, x made a round trip through
// HBM (1 KB per token and layer at `large`).  k_xdt (mixer_split.cu) then turns u into dt_r, B, C
// and Delta.
//
// Layout: the epilogue drains SiLU(z) and x from TMEM (thread = row, 16-byte shared stores) into
// 128B-swizzled staging tiles [rows][channels]; the conv then walks the x tile with lane = HC/32
// consecutive channels and warp = one row at a time (8-byte shared loads / stores, conflict-free),
// writes u in place, and TMA stores move SiLU(z) and u to HBM.  Every memory instruction is 8-16
// bytes wide per lane (2-byte per-lane stores, global or shared, were the bound of the transposed
// variants -- in_proj as W . A^T with TMEM lane = channel -- at ~2.7-6.6 cycles per warp instruction).
//
// Tiles overlap: tile m covers the packed rows [125 m - 3, 125 m + 125); its first d_conv - 1 = 3
// rows are the conv halo of row 125 m (recomputed by the MMA, never stored), so a tile needs
// nothing from its neighbours.  The conv window is cleared at candidate starts (the taps before a
// start are dropped exactly; the rows after it shift valid x in): every row's result is
// independent of the tiling (batch-invariant).
//
// DI = 256: the 512 x 256 bf16 in_proj weight does not fit one SM, so CTA h of a 2-CTA cluster owns
// channels [128 h, 128 h + 128) of x and of z (a 256-row, 128 KB weight slice, resident); both
// CTAs take the same row tiles and share each A tile by TMA multicast (each fetches 64 rows).
// DI <= 128: one CTA owns all channels (DI = 64 runs with N = 128).
//
// Roles (576 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + single-thread MMA issuer,
// warps 2..9 = group Z (the TMEM side: SiLU(z) -> staging -> TMA store, then x -> the x tile),
// warps 10..17 = group X (conv -> u in place -> TMA store).  The groups hand the x tile back and
// forth through two mbarriers (x staged / u store has read it), so SiLU(z) and the x staging of
// tile j + 1 overlap the conv of tile j.  TMEM: two accumulator buffers of [x | z] (2 HC columns)
// freed once group Z has drained them: the MMAs of tile j + 1 run while the epilogue works on j.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "../kernels.h"
#include "../kernels_mixer.h"
#include "../kernels_tc.h"
#include "../tc_ptx.cuh"
#include "mixer_common.cuh"

namespace tcl {
namespace inconv {

// Phase timeline of the first two CTAs (experiment builds only: -DTCL_INCONV_TRACE, read by
// exp/inconv_trace.py through tcl_diag_inconv_trace; the product build compiles TR() to nothing).
#ifdef TCL_INCONV_TRACE
__device__ unsigned long long g_trace[2][256][8];
#define TR(ev) do { if (blockIdx.x < 2 && j < 256) g_trace[blockIdx.x][j][ev] = clock64(); } while (0)
#else
#define TR(ev) do { } while (0)
#endif

constexpr int kBM = 128;                 // rows per tile (the MMA's M)
constexpr int kHalo = 3;                 // d_conv - 1
constexpr int kOut = kBM - kHalo;        // rows stored per tile
constexpr int kZWarps = 8;              // group Z: warps 2 .. 9
constexpr int kXWarps = 8;              // group X: warps 10 .. 17
constexpr int kEpiWarps = kZWarps + kXWarps;
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int KB, int HC>
struct Smem {
    static constexpr int NIN = 2 * HC;                     // MMA N: [x | z] channels of this CTA
    static constexpr int kWBytes = KB * NIN * 128;         // KB x [NIN rows][128 B]
    // staging tiles: SiLU(z) one 64-channel box at a time (shared memory goes to the A ring), for its
    // TMA store; x of all HC channels, then u in place, for its TMA store.  [rows][128 B] blocks,
    // 128B-swizzled.
    static constexpr int kZBytes = kBM * 128;
    static constexpr int kXBytes = (HC / 64) * kBM * 128;
    static constexpr int kFixed = kWBytes + kXBytes + kZBytes + 256 + 1024;
    static constexpr int kStagesRaw = (232448 - kFixed) / (kBM * 128);
    static constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
    static constexpr int kOffW = 0;
    static constexpr int kOffZ = kOffW + kWBytes;          // SiLU(z) staging
    static constexpr int kOffX = kOffZ + kZBytes;          // x, then u in place
    static constexpr int kOffA = kOffX + kXBytes;
    static constexpr int kOffBar = kOffA + kStages * kBM * 128;
    static constexpr int kBytes = kOffBar + 256 + 1024;
    static_assert(kStages >= 3, "A ring: three stages keep the A loads off the critical path");
    static_assert(kBytes <= 232448, "exceeds the 227 KB of shared memory per block");
    static_assert(2 * NIN <= 512, "TMEM columns");
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(tc::smem_u32(src))
                 : "memory");
}
// 16-byte chunk `ck` (0..7) of row `r` in a 128B-swizzled [rows][128 B] block
__device__ __forceinline__ uint32_t sw_off(int r, int ck) { return (uint32_t)(r * 128 + ((ck ^ (r & 7)) << 4)); }

template <int KB, int HC, int SPLIT>
__global__ void __launch_bounds__(kThreads, 1) k_inconv(const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmW,
                                                        const __grid_constant__ CUtensorMap tmGZ,
                                                        const __grid_constant__ CUtensorMap tmU,
                                                        const InConvParams p) {
    using S = Smem<KB, HC>;
    constexpr int NIN = S::NIN;
    constexpr int kStages = S::kStages;
    constexpr int HB = HC / 64;          // 64-channel blocks (K-blocks of the tiles, TMA store boxes)
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned base by an offset from smem_raw (keeps the shared state space: LDS / STS, not generic)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sW = smem + S::kOffW;
    uint8_t* sZ = smem + S::kOffZ;
    uint8_t* sX = smem + S::kOffX;
    uint8_t* sA = smem + S::kOffA;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
    uint64_t* empty = full + kStages;
    uint64_t* bfull = empty + kStages;
    uint64_t* afull = bfull + 1;     // [2] in_proj accumulators
    uint64_t* aempty = afull + 2;    // [2]
    uint64_t* xfull = aempty + 2;    // the x tile holds x of the next tile (group Z -> group X)
    uint64_t* xfree = xfull + 1;     // the u store has read the x tile (group X -> group Z)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfree + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = SPLIT == 2 ? tc::cluster_ctarank() : 0u;
    const int ch0 = (int)rank * HC;                  // first channel of this CTA
    const int rows = *p.p_rows;
    const int num_m = (rows + kOut - 1) / kOut;
    const int unit = SPLIT == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int n_units = SPLIT == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int n_my = unit < num_m ? (num_m - 1 - unit) / n_units + 1 : 0;

    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st) { tc::mbar_init(&full[st], 1); tc::mbar_init(&empty[st], SPLIT); }
        tc::mbar_init(bfull, 1);
        for (int a = 0; a < 2; ++a) { tc::mbar_init(&afull[a], 1); tc::mbar_init(&aempty[a], kZWarps); }
        tc::mbar_init(xfull, 32 * kZWarps);
        tc::mbar_init(xfree, 1);
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * NIN);
    tc::tc_fence_before();
    __syncthreads();
    if (SPLIT == 2) tc::cluster_sync();   // the peer's barriers exist before any multicast lands
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            tc::tma_prefetch(&tmA);
            tc::mbar_arrive_expect_tx(bfull, S::kWBytes);
            for (int kb = 0; kb < KB; ++kb) {
                tc::tma_load_2d(sW + kb * NIN * 128, &tmW, kb * 64, ch0, bfull);                 // x rows
                tc::tma_load_2d(sW + kb * NIN * 128 + HC * 128, &tmW, kb * 64, p.DI + ch0, bfull); // z rows
            }
            const uint64_t pol = tc::policy_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            for (int j = 0; j < n_my; ++j) {
                const int g0 = (unit + j * n_units) * kOut - kHalo;   // may be negative: zero fill
                for (int kb = 0; kb < KB; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], kBM * 128);
                    if (SPLIT == 1)
                        tc::tma_load_2d_hint(sA + stage * kBM * 128, &tmA, kb * 64, g0, &full[stage], pol);
                    else
                        tc::tma_load_2d_mcast(sA + stage * kBM * 128 + rank * 64 * 128, &tmA, kb * 64, g0 + (int)rank * 64,
                                              &full[stage], (uint16_t)3);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer: [x | z] of tile j into buffer j & 1
            constexpr uint32_t id_in = tc::idesc_bf16_f32(kBM, NIN);
            tc::mbar_wait(bfull, 0);
            tc::tc_fence_after();
            const uint32_t aA = tc::smem_u32(sA), aW = tc::smem_u32(sW);
            int stage = 0;
            uint32_t phase = 0;
            for (int j = 0; j < n_my; ++j) {
                const int b = j & 1;
                tc::mbar_wait(&aempty[b], ((j >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                TR(7);
                for (int kb = 0; kb < KB; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc::mma_bf16(tmem_base + b * NIN, tc::sw128_kmajor_desc(aA + stage * kBM * 128 + k * 32),
                                     tc::sw128_kmajor_desc(aW + kb * NIN * 128 + k * 32), id_in, (kb | k) != 0);
                    if (SPLIT == 1) tc::mma_commit(&empty[stage]);
                    else tc::mma_commit_mcast(&empty[stage], (uint16_t)3);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit(&afull[b]);
            }
        }
        __syncwarp();
    } else if (warp < 10) {
        // ---------------- group Z (warps 2..9): the TMEM side.  SiLU(z) -> staging -> TMA store, then x ->
        // the x tile for group X.  Lane quarter warp % 4, 32-channel half (warp - 2) / 4 of each
        // 64-channel block; thread = row.
        const int zt = threadIdx.x - 64;              // 0 .. 255
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        const int r = quarter * 32 + lane;
        for (int j = 0; j < n_my; ++j) {
            const int m = unit + j * n_units;
            const int b = j & 1;
            tc::mbar_wait(&afull[b], (j >> 1) & 1);
            tc::tc_fence_after();
            const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + b * NIN + HC;   // z columns
            // one 64-channel box at a time (the staging tile holds one box: shared memory goes to the A ring);
            // the two column halves of the group take 32 channels of the box each
#pragma unroll
            for (int bx = 0; bx < HB; ++bx) {
                if (zt == 0) bulk_wait_read0();       // the previous SiLU(z) box store has read the staging tile
                named_bar(1, 256);
                {
                    const int col = bx * 64 + half * 32;    // 32 columns: one TMEM load, one wait
                    uint32_t v[32];
                    tc::tmem_ld32(tb + col, v);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t zs[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            zs[q] = pk_bf16(silu_tanh(__uint_as_float(v[16 * c + 2 * q])),
                                            silu_tanh(__uint_as_float(v[16 * c + 2 * q + 1])));
                        const int ck = (col % 64) / 8 + 2 * c;
                        *reinterpret_cast<uint4*>(sZ + sw_off(r, ck)) = make_uint4(zs[0], zs[1], zs[2], zs[3]);
                        *reinterpret_cast<uint4*>(sZ + sw_off(r, ck + 1)) = make_uint4(zs[4], zs[5], zs[6], zs[7]);
                    }
                }
                tc::fence_proxy_async();
                named_bar(1, 256);
                if (zt == 0) {   // SiLU(z) rows 3 .. 127 -> GZ (the box starts at tile row 3: 128-byte aligned,
                                 // the 128B swizzle follows the shared address bits)
                    tma_store_2d(&tmGZ, ch0 + bx * 64, m * kOut, sZ + kHalo * 128);
                    bulk_commit();
                }
            }
            // ---- x -> registers (bf16: the conv's input precision of the unfused path), the TMEM buffer
            // freed, then -> the x tile once group X's u store of the previous tile has read it
            uint32_t xs[HC / 32][8];
#pragma unroll
            for (int bx = 0; bx < HB; ++bx) {
                uint32_t v[32];
                tc::tmem_ld32(tb - HC + bx * 64 + half * 32, v);   // 32 columns: one TMEM load, one wait
                tc::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        xs[2 * bx + c][q] = pk_bf16(__uint_as_float(v[16 * c + 2 * q]), __uint_as_float(v[16 * c + 2 * q + 1]));
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&aempty[b]);   // x and z of tile j are read
            if (j > 0) tc::mbar_wait(xfree, (j - 1) & 1);
#pragma unroll
            for (int k = 0; k < HC / 32; ++k) {
                const int col = (k / 2) * 64 + half * 32 + 16 * (k % 2);
                uint8_t* xb = sX + (col / 64) * (kBM * 128);
                *reinterpret_cast<uint4*>(xb + sw_off(r, (col % 64) / 8)) = make_uint4(xs[k][0], xs[k][1], xs[k][2], xs[k][3]);
                *reinterpret_cast<uint4*>(xb + sw_off(r, (col % 64) / 8 + 1)) = make_uint4(xs[k][4], xs[k][5], xs[k][6], xs[k][7]);
            }
            tc::mbar_arrive(xfull);                        // (release: this thread's x row is in the tile)
        }
        if (zt == 0) bulk_wait0();
    } else {
        // ---------------- group X (warps 10..17): conv + SiLU over the x tile group Z staged -> u in place ->
        // TMA store.  Warp = rows [16 xw, 16 xw + 16) (+ the 3 halo rows before them), lane = CPL
        // consecutive channels.
        constexpr int CPL = HC / 32;                  // conv channels per lane
        constexpr int CP = CPL / 2;                   // channel pairs per lane
        constexpr int RW = kBM / kXWarps;             // conv rows per warp
        const int xt = threadIdx.x - 64 - 32 * kZWarps;   // 0 .. 255
        const int xw = warp - 2 - kZWarps;            // 0 .. 7
        const int64_t P = rows;
        float2 wc[CP][4], bc[CP];                     // taps / bias pre-halved: SiLU(v) = h (1 + tanh h), h = v / 2
#pragma unroll
        for (int q = 0; q < CP; ++q) {
            const int ch = ch0 + CPL * lane + 2 * q;
            bc[q] = make_float2(0.5f * __ldg(p.b_conv + ch), 0.5f * __ldg(p.b_conv + ch + 1));
#pragma unroll
            for (int k = 0; k < 4; ++k)
                wc[q][k] = make_float2(0.5f * __ldg(p.w_conv + ch * 4 + k), 0.5f * __ldg(p.w_conv + (ch + 1) * 4 + k));
        }
        const int lc = CPL * lane;                    // this lane's first channel (local)
        uint8_t* xl = sX + (lc / 64) * (kBM * 128) + (lc % 8) * 2;   // + sw_off(row, xck)
        const int xck = (lc % 64) / 8;
        using V = typename std::conditional<CPL == 4, uint2, uint32_t>::type;
        auto cand_of = [&](int64_t g) -> int { return (g >= 0 && g < P) ? __ldg(p.row_cand + g) : -1 - (int)(g & 3); };
        auto ld = [&](int row, float2 (&x)[CP]) {
            const V v = *reinterpret_cast<const V*>(xl + sw_off(row, xck));
            const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int q = 0; q < CP; ++q) x[q] = __bfloat1622float2(e[q]);
        };
        const int rw = RW * xw;                       // first conv row of this warp
        const bool in = lane < RW + kHalo;
        // candidate ids of rows rw - 3 + lane of the tile, loaded one tile ahead (the row_cand reads miss
        // L2 under the streaming traffic: ~1 us, off the critical path this way)
        auto cand_tile = [&](int jj) -> int {
            return (jj < n_my && in) ? cand_of((int64_t)(unit + jj * n_units) * kOut - kHalo + rw - kHalo + lane) : -7;
        };
        int cc_next = cand_tile(0);
        for (int j = 0; j < n_my; ++j) {
            const int m = unit + j * n_units;
            const int cc = cc_next;
            cc_next = cand_tile(j + 1);
            if (xt == 0) TR(0);
            tc::mbar_wait(xfull, j & 1);              // group Z has staged x of tile j
            if (xt == 0) TR(2);
            // candidate starts of rows rw - 3 .. rw + RW - 1 (bit l = row rw - 3 + l)
            const int cp = __shfl_up_sync(0xffffffffu, cc, 1);
            const uint32_t starts = __ballot_sync(0xffffffffu, lane >= 1 && in && cc != cp);
            named_bar(2, 32 * kXWarps);
            if (xt == 0) TR(3);
            // ---- conv + SiLU -> u (fp16) in place (rows in batches of 8), then TMA-stored
            {
                float2 win[kHalo][CP];   // x of rows t-1, t-2, t-3
#pragma unroll
                for (int i = 0; i < kHalo; ++i)
#pragma unroll
                    for (int q = 0; q < CP; ++q) win[i][q] = make_float2(0.f, 0.f);
                float2 xh[kHalo][CP];
#pragma unroll
                for (int i = 0; i < kHalo; ++i) {
                    const int row = rw - kHalo + i;
                    if (row >= 0) ld(row, xh[i]);
                    else
#pragma unroll
                        for (int q = 0; q < CP; ++q) xh[i][q] = make_float2(0.f, 0.f);
                }
                named_bar(2, 32 * kXWarps);   // every halo is read before any row is overwritten with u
                // the halo rows: a start among them clears the window before they shift in
#pragma unroll
                for (int i = 0; i < kHalo; ++i) {
                    if ((starts >> i) & 1u)
#pragma unroll
                        for (int k = 0; k < kHalo; ++k)
#pragma unroll
                            for (int q = 0; q < CP; ++q) win[k][q] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int q = 0; q < CP; ++q) { win[2][q] = win[1][q]; win[1][q] = win[0][q]; win[0][q] = xh[i][q]; }
                }
#pragma unroll
                for (int t0 = 0; t0 < RW; t0 += 8) {
                    float2 xv[8][CP];
#pragma unroll
                    for (int t = 0; t < 8; ++t) ld(rw + t0 + t, xv[t]);
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        if ((starts >> (kHalo + t0 + t)) & 1u)   // warp-uniform
#pragma unroll
                            for (int k = 0; k < kHalo; ++k)
#pragma unroll
                                for (int q = 0; q < CP; ++q) win[k][q] = make_float2(0.f, 0.f);
                        uint32_t uo[CP];
#pragma unroll
                        for (int q = 0; q < CP; ++q) {
                            float2 h = __ffma2_rn(wc[q][3], xv[t][q], bc[q]);
                            h = __ffma2_rn(wc[q][2], win[0][q], h);
                            h = __ffma2_rn(wc[q][1], win[1][q], h);
                            h = __ffma2_rn(wc[q][0], win[2][q], h);
                            win[2][q] = win[1][q]; win[1][q] = win[0][q]; win[0][q] = xv[t][q];
                            float2 th;
                            asm("tanh.approx.f32 %0, %1;" : "=f"(th.x) : "f"(h.x));
                            asm("tanh.approx.f32 %0, %1;" : "=f"(th.y) : "f"(h.y));
                            const __half2 u2 = __float22half2_rn(__ffma2_rn(h, th, h));
                            uo[q] = *reinterpret_cast<const uint32_t*>(&u2);
                        }
                        V o;
                        if constexpr (CPL == 4) o = make_uint2(uo[0], uo[1]); else o = uo[0];
                        *reinterpret_cast<V*>(xl + sw_off(rw + t0 + t, xck)) = o;
                    }
                }
            }
            if (xt == 0) TR(4);
            tc::fence_proxy_async();
            named_bar(2, 32 * kXWarps);
            if (xt == 0) {   // u rows 3 .. 127 -> the packet's u columns (the box starts at tile row 3)
#pragma unroll
                for (int bx = 0; bx < HB; ++bx) tma_store_2d(&tmU, ch0 + bx * 64, m * kOut, sX + bx * (kBM * 128) + kHalo * 128);
                bulk_commit();
                bulk_wait_read0();                    // the store has read the tile: group Z may refill it
                tc::mbar_arrive(xfree);
            }
            if (xt == 0) TR(5);
        }
        if (xt == 0) bulk_wait0();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (SPLIT == 2) tc::cluster_sync();   // no CTA leaves while its peer may still multicast / commit into it
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 2 * NIN);
    }
}

template <int KB, int HC, int SPLIT>
static cudaError_t launch_k(const CUtensorMap& a, const CUtensorMap& w, const CUtensorMap& gz, const CUtensorMap& um,
                            const InConvParams& p, int num_sms, cudaStream_t s) {
    constexpr int smem = Smem<KB, HC>::kBytes;
    auto kern = k_inconv<KB, HC, SPLIT>;
    cudaError_t e = prepare_kernel(kern, smem);
    if (e != cudaSuccess) return e;
    const int grid = SPLIT == 2 ? (num_sms / 2) * 2 : num_sms;
    if (SPLIT == 1) {
        kern<<<grid, kThreads, smem, s>>>(a, w, gz, um, p);
    } else {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, a, w, gz, um, p);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

template <int HC, int SPLIT>
static cudaError_t launch_kb(int kb, const CUtensorMap& a, const CUtensorMap& w, const CUtensorMap& gz,
                             const CUtensorMap& um, const InConvParams& p, int num_sms, cudaStream_t s) {
    if (kb == 1) return launch_k<1, HC, SPLIT>(a, w, gz, um, p, num_sms, s);
    if (kb == 2) return launch_k<2, HC, SPLIT>(a, w, gz, um, p, num_sms, s);
    if (kb == 4) return launch_k<4, HC, SPLIT>(a, w, gz, um, p, num_sms, s);
    return cudaErrorInvalidValue;
}

}  // namespace inconv

#ifdef TCL_INCONV_TRACE
extern "C" int tcl_diag_inconv_trace(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, inconv::g_trace, sizeof(inconv::g_trace));
}
#endif

int inconv_split(int di) { return di == 256 ? 2 : 1; }
int inconv_channels(int di) { return di / inconv_split(di); }

cudaError_t launch_inconv(const CUtensorMap& a, const CUtensorMap& w, const CUtensorMap& gz, const CUtensorMap& um,
                          const InConvParams& p, int dm, int num_sms, cudaStream_t s) {
    if ((dm != 64 && dm != 128 && dm != 256) || p.d_conv != 4) return cudaErrorInvalidValue;
    const int kb = dm / 64;
    if (p.DI == 256) return inconv::launch_kb<128, 2>(kb, a, w, gz, um, p, num_sms, s);
    if (p.DI == 128) return inconv::launch_kb<128, 1>(kb, a, w, gz, um, p, num_sms, s);
    if (p.DI == 64) return inconv::launch_kb<64, 1>(kb, a, w, gz, um, p, num_sms, s);
    return cudaErrorInvalidValue;
}

}  // namespace tcl
