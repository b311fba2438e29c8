// mixer_fused.cu -- the Mamba mixer of the bf16 path in ONE persistent kernel
// (SURVEY §8(a) a5-a7):
//
//   u   = SiLU(b_conv + causal depthwise conv_{d_conv}(x))            (R4)
//   [dt_r | B | C] = u W_x^T                                           (input-dependent selection; R7)
//   Delta = softplus(dt_r W_dt^T + b_dt)
//   s_t = exp(Delta A) s_{t-1} + (exp(Delta A) - 1)/A * B_t u_t        (Eqs. 4-5 with ZOH; R5)
//   y_t = C_t . s_t + D u_t ;  g_t = y_t * SiLU(z_t)                   (R6; gate: SiLU(z) is formed
//                                                                       by the in_proj epilogue)
//
// Work decomposition: a persistent CTA of DI threads owns the packed rows of a contiguous range of
// candidates (balanced by rows); thread d owns channel d and keeps its N SSM states in registers,
// resetting them (and the conv window) at every candidate start.  The rows are processed in chunks
// of 16 consecutive rows that may span candidates, so chunks are full (no per-candidate ragged
// tail paying the x_proj / dt_proj / barrier cost of a whole chunk):
//   0. the chunk's 16 rows of the in_proj output [x | z] (bf16, contiguous in the packed layout)
//      arrive by one TMA bulk copy (cp.async.bulk) into a double buffer; the copy of the NEXT
//      chunk is issued before this chunk is computed, so HBM latency is hidden;
//   1. causal conv + SiLU from a register window of the previous d_conv-1 inputs -> u (smem);
//   2. x_proj on the tensor cores: mma.sync m16n8k16 (bf16 in, fp32 accumulate) of the 16 x DI
//      chunk by W_x^T (weights staged once per CTA in padded shared memory);
//   3. dt_proj on the tensor cores (B fragments held in registers for the whole launch) with the
//      softplus epilogue -> Delta (smem);
//   4. the selective scan: exp(Delta A) = 2^(Delta * A log2 e) on MUFU.EX2 (A pre-scaled at model
//      creation); all other arithmetic in packed fp32x2 (FFMA2/FMUL2/FADD2) so that the SFU, not
//      instruction issue, bounds the loop; D skip; gate by the SiLU(z) the in_proj epilogue
//      stored (one MUFU op per (t, d) moved out of the SFU-bound scan); g stored as bf16.
// The 16 x 48 x 256 and 16 x 256 x 16 contractions per chunk are far too small for a TMEM
// accumulator round trip, so the warp-level MMA is the right unit here.
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstdio>

#include "../kernels.h"
#include "../kernels_mixer.h"
#include "../tc_ptx.cuh"
#include "mixer_common.cuh"

namespace tcl {

constexpr int kTC = 16;  // tokens per chunk (= MMA M)

template <int DI, int NXP>
struct MixerSmem {
    static constexpr int kWxld = DI + 8;   // bf16 row stride of W_x (+16 B: conflict-free B fragments)
    static constexpr int kDbcld = NXP + 4;
    static constexpr int kUld = DI + 4;
    static constexpr int kXZ = 0;                                  // bf16 [2][16][2 DI] (TMA bulk dst)
    static constexpr int kU = kXZ + 2 * kTC * 2 * DI * 2;          // float [16][DI + 4]
    static constexpr int kDl = kU + kTC * kUld * 4;                // float [16][DI]
    static constexpr int kDbc = kDl + kTC * DI * 4;                // float [16][NXP + 4]
    static constexpr int kUb = kDbc + kTC * kDbcld * 4;            // bf16  [16][DI + 8] (MMA A operand)
    static constexpr int kWx = kUb + kTC * kWxld * 2;              // bf16  [NXP][DI + 8]
    static constexpr int kBar = kWx + NXP * kWxld * 2;             // 2 mbarriers
    // candidate-start bits of the CTA's rows, 16 per chunk (more chunks than this fall back to
    // walking cu[] per chunk)
    static constexpr int kStartWords = 1024;
    static constexpr int kStarts = kBar + 16;                      // u32 [kStartWords]
    static constexpr int kBytes = kStarts + 4 * kStartWords;
};

template <int DI, int N, int RP, int NXP, int DC, int DISC, int SU>
__global__ void __launch_bounds__(DI, 2) k_mixer_fused(MixerArgs a) {
    constexpr int NW = DI / 32;
    using L = MixerSmem<DI, NXP>;
    extern __shared__ __align__(128) uint8_t msm[];
    __nv_bfloat16* xz_s = reinterpret_cast<__nv_bfloat16*>(msm + L::kXZ);   // [2][16][2 DI]
    float* u_s = reinterpret_cast<float*>(msm + L::kU);                       // [16][DI + 4]
    float* dl_s = reinterpret_cast<float*>(msm + L::kDl);                     // [16][DI]
    float* dbc_s = reinterpret_cast<float*>(msm + L::kDbc);                   // [16][NXP + 4]
    __nv_bfloat16* wx_s = reinterpret_cast<__nv_bfloat16*>(msm + L::kWx);    // [NXP][DI + 8]
    __nv_bfloat16* u_b = reinterpret_cast<__nv_bfloat16*>(msm + L::kUb);     // [16][DI + 8]
    uint64_t* bar = reinterpret_cast<uint64_t*>(msm + L::kBar);

    const int d = threadIdx.x;
    const int warp = d >> 5, lane = d & 31;
    const int g = lane >> 2, tq = lane & 3;

    // ---- once per CTA: W_x into padded smem, W_dt fragments into registers, per-channel constants
    for (int idx = d; idx < NXP * DI / 8; idx += DI) {
        const int r = idx / (DI / 8), c8 = idx - r * (DI / 8);
        *reinterpret_cast<uint4*>(wx_s + r * L::kWxld + c8 * 8) =
            __ldg(reinterpret_cast<const uint4*>(a.Wx_b + (int64_t)r * DI + c8 * 8));
    }
    constexpr int NT_DT = DI / 8 / NW;  // dt_proj n-tiles per warp
    // W_dt fragments / b_dt held in registers for the whole launch
    uint32_t wdt[NT_DT][RP / 16][2];
#pragma unroll
    for (int j = 0; j < NT_DT; ++j) {
        const __nv_bfloat16* wrow = a.Wdt_b + (int64_t)((warp + j * NW) * 8 + g) * RP;
#pragma unroll
        for (int ks = 0; ks < RP / 16; ++ks) {
            wdt[j][ks][0] = __ldg(reinterpret_cast<const unsigned int*>(wrow + ks * 16 + 2 * tq));
            wdt[j][ks][1] = __ldg(reinterpret_cast<const unsigned int*>(wrow + ks * 16 + 8 + 2 * tq));
        }
    }
    float2 bdt[NT_DT];  // dt_proj bias of this thread's output columns
#pragma unroll
    for (int j = 0; j < NT_DT; ++j) bdt[j] = __ldg(reinterpret_cast<const float2*>(a.b_dt + (warp + j * NW) * 8 + 2 * tq));
    float2 A2[N / 2], iA[N / 2];
#pragma unroll
    for (int n = 0; n < N / 2; ++n) {
        A2[n] = __ldg(reinterpret_cast<const float2*>(a.A2 + d * N) + n);
        iA[n] = __ldg(reinterpret_cast<const float2*>(a.invA + d * N) + n);
    }
    const float Dv = __ldg(a.Dv + d);
    const float bconv = 0.5f * __ldg(a.b_conv + d);   // pre-halved for the SiLU below
    float wc[DC];
#pragma unroll
    for (int k = 0; k < DC; ++k) wc[k] = 0.5f * __ldg(a.w_conv + d * DC + k);
    if (d == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        tc::fence_mbar_init();
    }
    __syncthreads();

    // ---- row-chunk iterator: this CTA owns the packed rows of a contiguous candidate range
    // [c0, c1), balanced by rows (binary search in cu); chunks are 16 consecutive rows that may
    // span candidates (states and conv window reset at candidate starts), so no chunk is ragged
    // except the CTA's last one.
    const int64_t P = a.cu[a.n];
    auto cand_at = [&](int64_t target) -> int64_t {   // first candidate i with cu[i] >= target
        int64_t lo = 0, hi = a.n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (a.cu[mid] < target) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    const int64_t c0 = cand_at(P * blockIdx.x / gridDim.x);
    const int64_t c1 = cand_at(P * (blockIdx.x + 1) / gridDim.x);
    const int64_t r_end = a.cu[c1];
    int64_t r0 = a.cu[c0];
    int64_t k_next = c0;   // next candidate whose start row is >= r0
    auto issue = [&](int64_t r, int b) {
        if (d == 0 && r < r_end) {
            const uint32_t bytes = (uint32_t)(r_end - r < kTC ? r_end - r : kTC) * 2 * DI * 2;
            tc::mbar_arrive_expect_tx(&bar[b], bytes);
            bulk_g2s(xz_s + b * kTC * 2 * DI, a.XZ + r * (int64_t)a.ldxz, bytes, &bar[b]);
        }
    };
    // candidate starts of the CTA's rows as a bit array in shared memory, built once: the chunk
    // loop then reads 16 bits per chunk instead of walking cu[] (dependent global loads on the
    // critical path of every chunk)
    uint32_t* st_w = reinterpret_cast<uint32_t*>(msm + L::kStarts);
    const int64_t n_chunks = (r_end - r0 + kTC - 1) / kTC;
    const bool bits = L::kStartWords > 0 && (n_chunks + 2) / 2 <= L::kStartWords;
    if (bits) {
        const int nw = (int)(n_chunks + 2) / 2;
        for (int w = d; w < nw; w += DI) st_w[w] = 0u;
        __syncthreads();
        for (int64_t i = c0 + d; i < c1; i += DI) {
            const int64_t off = a.cu[i] - r0;
            atomicOr(&st_w[off >> 5], 1u << (off & 31));
        }
        __syncthreads();
    }
    issue(r0, 0);
    uint32_t parity = 0;  // bit b = phase parity of buffer b
    int buf = 0;
    int chunk = 0;

    float2 s[N / 2];
    float win[DC];
#pragma unroll
    for (int n = 0; n < N / 2; ++n) s[n] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < DC; ++k) win[k] = 0.0f;
    while (r0 < r_end) {
        const int tc = (int)(r_end - r0 < kTC ? r_end - r0 : kTC);
        // rows of this chunk that start a candidate (zero-length candidates share a start row)
        uint32_t starts = 0;
        if (bits) {
            starts = (st_w[chunk >> 1] >> ((chunk & 1) * 16)) & 0xFFFFu;
        } else {
            while (k_next < c1 && a.cu[k_next] < r0 + tc) {
                starts |= 1u << (int)(a.cu[k_next] - r0);
                ++k_next;
            }
        }
        issue(r0 + kTC, buf ^ 1);   // prefetch the next chunk into the other buffer

        tc::mbar_wait(&bar[buf], (parity >> buf) & 1u);
        parity ^= 1u << buf;
        const __nv_bfloat16* xz = xz_s + buf * kTC * 2 * DI;

        // ---- 1. causal conv + SiLU
        // (rows tt >= tc of the chunk are left stale: MMA rows are independent and never read back)
        // fully unrolled over the 16 rows (the window shift is register renaming): 16 independent
        // conv + SiLU chains in flight instead of 4 (measured 4.40 -> 4.24 ms at `large`)
        // SiLU(v) = h (1 + tanh h) with h = v / 2: the conv weights and bias are pre-halved (exact).
        auto conv_tok = [&](int tt) {
            if ((starts >> tt) & 1u) {
#pragma unroll
                for (int k = 0; k < DC; ++k) win[k] = 0.0f;
            }
            const float x = __bfloat162float(xz[tt * 2 * DI + d]);
            float h = fmaf(wc[DC - 1], x, bconv);
#pragma unroll
            for (int k = 0; k < DC - 1; ++k) h = fmaf(wc[DC - 2 - k], win[k], h);
#pragma unroll
            for (int k = DC - 1; k > 0; --k) win[k] = win[k - 1];
            win[0] = x;
            float th;
            asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(h));
            const float u = fmaf(h, th, h);
            u_s[tt * L::kUld + d] = u;
            u_b[tt * L::kWxld + d] = __float2bfloat16_rn(u);
        };
        {
            if (tc == kTC) {
#pragma unroll
                for (int tt = 0; tt < kTC; ++tt) conv_tok(tt);
            } else {
#pragma unroll
                for (int tt = 0; tt < kTC; ++tt) {
                    if (tt >= tc) break;
                    conv_tok(tt);
                }
            }
        }
        __syncthreads();
        // ---- 2. x_proj on the tensor cores: dbc[16][NXP] = u[16][DI] . W_x^T
        for (int nt = warp; nt < NXP / 8; nt += NW) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            // fragments by ldmatrix: A (16 x 16 of u) one x4 per k-step, B (8 rows of W_x) one x4
            // per two k-steps
            const uint32_t a_addr = tc::smem_u32(u_b + (lane & 15) * L::kWxld + 8 * (lane >> 4));
            const uint32_t b_addr = tc::smem_u32(wx_s + (nt * 8 + (lane & 7)) * L::kWxld + 8 * (lane >> 3));
#pragma unroll 4
            for (int k0 = 0; k0 < DI; k0 += 32) {
                uint32_t af[4], af2[4], bf[4];
                ldsm_x4(af, a_addr + k0 * 2);
                ldsm_x4(af2, a_addr + (k0 + 16) * 2);
                ldsm_x4(bf, b_addr + k0 * 2);
                mma_16816(acc, af, bf[0], bf[1]);
                mma_16816(acc, af2, bf[2], bf[3]);
            }
            const int c = nt * 8 + 2 * tq;
            *reinterpret_cast<float2*>(dbc_s + g * L::kDbcld + c) = make_float2(acc[0], acc[1]);
            *reinterpret_cast<float2*>(dbc_s + (g + 8) * L::kDbcld + c) = make_float2(acc[2], acc[3]);
        }
        __syncthreads();
        // ---- 3. dt_proj + softplus: dl[16][DI] = softplus(dt_r[16][RP] . W_dt^T + b_dt)
        {
            uint32_t af[RP / 16][4];
#pragma unroll
            for (int ks = 0; ks < RP / 16; ++ks) {
                const int k0 = ks * 16;
                auto ld2 = [&](int r, int k) -> uint32_t {
                    const float v0 = (k < a.R) ? dbc_s[r * L::kDbcld + k] : 0.0f;
                    const float v1 = (k + 1 < a.R) ? dbc_s[r * L::kDbcld + k + 1] : 0.0f;
                    return pk_bf16(v0, v1);
                };
                af[ks][0] = ld2(g, k0 + 2 * tq);
                af[ks][1] = ld2(g + 8, k0 + 2 * tq);
                af[ks][2] = ld2(g, k0 + 8 + 2 * tq);
                af[ks][3] = ld2(g + 8, k0 + 8 + 2 * tq);
            }
#pragma unroll
            for (int j = 0; j < NT_DT; ++j) {
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int ks = 0; ks < RP / 16; ++ks) mma_16816(acc, af[ks], wdt[j][ks][0], wdt[j][ks][1]);
                const int c = (warp + j * NW) * 8 + 2 * tq;
                const float2 bj = bdt[j];
                const float b0v = bj.x, b1v = bj.y;
                *reinterpret_cast<float2*>(dl_s + g * DI + c) =
                    make_float2(softplus_fast(acc[0] + b0v), softplus_fast(acc[1] + b1v));
                *reinterpret_cast<float2*>(dl_s + (g + 8) * DI + c) =
                    make_float2(softplus_fast(acc[2] + b0v), softplus_fast(acc[3] + b1v));
            }
        }
        __syncthreads();
        // ---- 4. selective scan + D skip + gate (packed fp32x2 arithmetic, MUFU.EX2 for exp)
        __nv_bfloat16* gout = a.G + r0 * DI + d;   // ldg == DI (checked at launch)
        const float* up = u_s + d;
        const float* dlp = dl_s + d;
        const __nv_bfloat16* gzp = xz + DI + d;
        const float* bcp = dbc_s + a.R;
        // one token of the scan; the row pointers advance by compile-time strides (G rows are DI
        // wide on this path), so in the unrolled full-chunk loop every access is base + immediate
        auto scan_tok = [&](int tt) {
            if ((starts >> tt) & 1u) {
#pragma unroll
                for (int n = 0; n < N / 2; ++n) s[n] = make_float2(0.f, 0.f);
            }
            const float u = up[0];
            const float dl = dlp[0];
            const float gz = __bfloat162float(gzp[0]);   // SiLU(z), formed by the in_proj epilogue
            const float4* B4 = reinterpret_cast<const float4*>(bcp);
            const float4* C4 = reinterpret_cast<const float4*>(bcp + N);
            const float2 dl2 = make_float2(dl, dl);
            const float2 u2 = make_float2(u, u);
            float2 y2 = make_float2(0.f, 0.f), y2b = make_float2(0.f, 0.f);
            if (DISC == 1) {
                const float2 du2 = __fmul2_rn(dl2, u2);
#pragma unroll
                for (int q = 0; q < N / 4; ++q) {
                    const float4 b4 = B4[q], c4 = C4[q];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int n = 2 * q + h;
                        const float2 x2 = __fmul2_rn(dl2, A2[n]);
                        const float2 ab = make_float2(ex2(x2.x), ex2(x2.y));
                        const float2 bb = h ? make_float2(b4.z, b4.w) : make_float2(b4.x, b4.y);
                        const float2 cc = h ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
                        s[n] = __ffma2_rn(ab, s[n], __fmul2_rn(bb, du2));
                        if (h) y2b = __ffma2_rn(cc, s[n], y2b); else y2 = __ffma2_rn(cc, s[n], y2);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < N / 4; ++q) {
                    const float4 b4 = B4[q], c4 = C4[q];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int n = 2 * q + h;
                        const float2 x2 = __fmul2_rn(dl2, A2[n]);
                        const float2 ab = make_float2(ex2(x2.x), ex2(x2.y));
                        const float2 bb = h ? make_float2(b4.z, b4.w) : make_float2(b4.x, b4.y);
                        const float2 cc = h ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
                        // Bbar u = (Ab - 1) v with v = B u / A;  s <- Ab (s + v) - v
                        const float2 v = __fmul2_rn(__fmul2_rn(bb, u2), iA[n]);
                        const float2 t = __fadd2_rn(s[n], v);
                        s[n] = __ffma2_rn(ab, t, make_float2(-v.x, -v.y));
                        if (h) y2b = __ffma2_rn(cc, s[n], y2b); else y2 = __ffma2_rn(cc, s[n], y2);
                    }
                }
            }
            const float y = fmaf(Dv, u, (y2.x + y2b.x) + (y2.y + y2b.y));
            gout[0] = __float2bfloat16_rn(y * gz);
            up += L::kUld;
            dlp += DI;
            gzp += 2 * DI;
            bcp += L::kDbcld;
            gout += DI;
        };
        {
            if (tc == kTC && SU > 1) {
#pragma unroll 1
                for (int t0 = 0; t0 < kTC; t0 += SU) {
#pragma unroll
                    for (int j = 0; j < SU; ++j) scan_tok(t0 + j);
                }
            } else {
#pragma unroll 1
                for (int tt = 0; tt < tc; ++tt) scan_tok(tt);
            }
        }
        __syncthreads();
        buf ^= 1;
        r0 += kTC;
        ++chunk;
    }
}

template <int DI, int N, int RP, int NXP, int DC, int DISC, int SU>
static cudaError_t mixer_launch_k(const MixerArgs& a, int num_sms, cudaStream_t s) {
    constexpr int smem = MixerSmem<DI, NXP>::kBytes;
    auto kern = k_mixer_fused<DI, N, RP, NXP, DC, DISC, SU>;
    if (a.ldg != DI) return cudaErrorInvalidValue;
    int blocks_per_sm = 0;
    cudaError_t e = prepare_kernel(kern, smem, DI, &blocks_per_sm);
    if (e != cudaSuccess) return e;
    int64_t grid = (int64_t)num_sms * blocks_per_sm;
    if (grid > a.n) grid = a.n;
    kern<<<(unsigned)grid, DI, smem, s>>>(a);
    return cudaGetLastError();
}

// scan tokens per unrolled step of a full chunk: 2 (measured at `large`: 1 -> 4.14 ms, 2 -> 4.03,
// 4 -> 4.08-4.12, 16 -> 4.24 with spills)
template <int DI, int N, int RP, int NXP>
static cudaError_t mixer_launch(const MixerArgs& a, int num_sms, cudaStream_t s) {
    if (a.d_conv != 4) return cudaErrorInvalidValue;  // validated on the host
    return a.disc == 1 ? mixer_launch_k<DI, N, RP, NXP, 4, 1, 2>(a, num_sms, s)
                       : mixer_launch_k<DI, N, RP, NXP, 4, 0, 2>(a, num_sms, s);
}

template <int DI, int N>
static cudaError_t mixer_rp(const MixerArgs& a, int num_sms, cudaStream_t s) {
    const int nxp = ((a.R + 2 * N) + 7) / 8 * 8;
    if (a.RP == 16) {
        if (nxp <= 24) return mixer_launch<DI, N, 16, 24>(a, num_sms, s);
        if (nxp <= 48) return mixer_launch<DI, N, 16, 48>(a, num_sms, s);
    } else if (a.RP == 32) {
        if (nxp <= 64) return mixer_launch<DI, N, 32, 64>(a, num_sms, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_mixer_fused(const MixerArgs& a, int num_sms, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    if (a.DI == 256) return a.N == 16 ? mixer_rp<256, 16>(a, num_sms, s) : mixer_rp<256, 8>(a, num_sms, s);
    if (a.DI == 128) return a.N == 16 ? mixer_rp<128, 16>(a, num_sms, s) : mixer_rp<128, 8>(a, num_sms, s);
    if (a.DI == 64) return a.N == 16 ? mixer_rp<64, 16>(a, num_sms, s) : mixer_rp<64, 8>(a, num_sms, s);
    return cudaErrorInvalidValue;
}

}  // namespace tcl
