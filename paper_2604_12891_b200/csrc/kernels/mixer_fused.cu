// mixer_fused.cu -- the Mamba mixer of the bf16 path in ONE kernel:
//
//   u   = SiLU(b_conv + causal depthwise conv_{d_conv}(x))            (R4)
//   [dt_r | B | C] = u W_x^T                                           (input-dependent selection; R7)
//   Delta = softplus(dt_r W_dt^T + b_dt)
//   s_t = exp(Delta A) s_{t-1} + (exp(Delta A) - 1)/A * B_t u_t        (Eqs. 4-5 with ZOH; R5)
//   y_t = C_t . s_t + D u_t ;  g_t = y_t * SiLU(z_t)                   (R6; gate)
//
// One CTA per candidate, one thread per channel d (the N states of channel d live in registers
// for the whole sequence, never in memory).  The candidate is walked in chunks of 16 tokens:
//   1. conv + SiLU from a register window of the last d_conv-1 inputs (coalesced bf16 loads of x
//      and z from the in_proj output), u kept fp32 in shared memory + a bf16 copy for the MMA;
//   2. x_proj on the tensor cores: mma.sync m16n8k16 (bf16 in, fp32 out) of the 16 x DI chunk
//      by W_x^T (these contractions are 16 x 48 x 256 and 16 x 256 x 16 per chunk: far too small
//      for a TMEM accumulator round trip, so the warp-level MMA is the right unit here);
//   3. dt_proj on the tensor cores, softplus epilogue -> Delta in shared memory;
//   4. the selective scan (ex2.approx on MUFU, exp(Delta A) = 2^(Delta * A log2 e) with A
//      pre-scaled at model creation) + D skip + SiLU(z) gate, g written as bf16 for out_proj.
// Nothing but x, z (in) and g (out) touches HBM.
#include <cuda_bf16.h>

#include "../kernels.h"
#include "../kernels_mixer.h"

namespace tcl {

constexpr int kTC = 16;  // tokens per chunk (= MMA M)

template <int DI, int NXP>
struct MixerSmem {
    static constexpr int kUbld = DI + 8;   // bf16 row stride (+16 B: conflict-free fragment loads)
    static constexpr int kDbcld = NXP + 4;
    static constexpr int kU = 0;                                   // float [16][DI]
    static constexpr int kDl = kU + kTC * DI * 4;                  // float [16][DI]
    static constexpr int kZ = kDl + kTC * DI * 4;                  // bf16  [16][DI]
    static constexpr int kUb = kZ + kTC * DI * 2;                  // bf16  [16][DI + 8]
    static constexpr int kDbc = kUb + kTC * kUbld * 2;             // float [16][NXP + 4]
    static constexpr int kBytes = kDbc + kTC * kDbcld * 4;
};

__device__ __forceinline__ uint32_t pk_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int DI, int N, int RP, int NXP, int DC>
__global__ void __launch_bounds__(DI) k_mixer_fused(MixerArgs a) {
    constexpr int NW = DI / 32;
    using L = MixerSmem<DI, NXP>;
    extern __shared__ __align__(16) uint8_t msm[];
    float (*u_s)[DI] = reinterpret_cast<float (*)[DI]>(msm + L::kU);
    float (*dl_s)[DI] = reinterpret_cast<float (*)[DI]>(msm + L::kDl);
    __nv_bfloat16 (*z_s)[DI] = reinterpret_cast<__nv_bfloat16 (*)[DI]>(msm + L::kZ);
    __nv_bfloat16 (*u_b)[L::kUbld] = reinterpret_cast<__nv_bfloat16 (*)[L::kUbld]>(msm + L::kUb);
    float (*dbc_s)[L::kDbcld] = reinterpret_cast<float (*)[L::kDbcld]>(msm + L::kDbc);

    const int64_t i = blockIdx.x;
    const int d = threadIdx.x;
    const int warp = d >> 5, lane = d & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int T = a.lens[i];
    if (T < 1 || T > a.max_len) return;
    const int64_t base = a.cu[i];

    // per-channel constants
    float A2[N], iA[N], s[N];
#pragma unroll
    for (int n = 0; n < N; ++n) {
        A2[n] = __ldg(a.A2 + d * N + n);
        iA[n] = __ldg(a.invA + d * N + n);
        s[n] = 0.0f;
    }
    const float Dv = __ldg(a.Dv + d);
    const float bconv = __ldg(a.b_conv + d);
    float wc[DC];
#pragma unroll
    for (int k = 0; k < DC; ++k) wc[k] = __ldg(a.w_conv + d * DC + k);
    float win[DC];  // x[t-1], x[t-2], ... (window of previous inputs, zero before the candidate)
#pragma unroll
    for (int k = 0; k < DC; ++k) win[k] = 0.0f;

    for (int t0 = 0; t0 < T; t0 += kTC) {
        const int tc = min(kTC, T - t0);
        // ---- 1. conv + SiLU, z staging
        for (int tt = 0; tt < kTC; ++tt) {
            float u = 0.0f, z = 0.0f;
            if (tt < tc) {
                const __nv_bfloat16* xr = a.XZ + (base + t0 + tt) * a.ldxz;
                const float x = __bfloat162float(xr[d]);
                z = __bfloat162float(xr[DI + d]);
                // c = b + sum_k w[k] * x[t - (dc-1) + k]; tap dc-1 is the current token
                float acc = fmaf(wc[DC - 1], x, bconv);
#pragma unroll
                for (int k = 0; k < DC - 1; ++k) acc = fmaf(wc[DC - 2 - k], win[k], acc);
#pragma unroll
                for (int k = DC - 1; k > 0; --k) win[k] = win[k - 1];
                win[0] = x;
                u = silu(acc);
            }
            u_s[tt][d] = u;
            z_s[tt][d] = __float2bfloat16_rn(z);
            u_b[tt][d] = __float2bfloat16_rn(u);
        }
        __syncthreads();
        // ---- 2. x_proj: dbc[16][NXP] = u_b[16][DI] . W_x^T   (warp w -> n-tiles w, w+NW, ...)
        for (int nt = warp; nt < NXP / 8; nt += NW) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const __nv_bfloat16* wrow = a.Wx_b + (int64_t)(nt * 8 + g) * DI;
#pragma unroll 4
            for (int k0 = 0; k0 < DI; k0 += 16) {
                uint32_t af[4];
                af[0] = *reinterpret_cast<const uint32_t*>(&u_b[g][k0 + 2 * tq]);
                af[1] = *reinterpret_cast<const uint32_t*>(&u_b[g + 8][k0 + 2 * tq]);
                af[2] = *reinterpret_cast<const uint32_t*>(&u_b[g][k0 + 8 + 2 * tq]);
                af[3] = *reinterpret_cast<const uint32_t*>(&u_b[g + 8][k0 + 8 + 2 * tq]);
                const uint32_t b0 = __ldg(reinterpret_cast<const unsigned int*>(wrow + k0 + 2 * tq));
                const uint32_t b1 = __ldg(reinterpret_cast<const unsigned int*>(wrow + k0 + 8 + 2 * tq));
                mma_16816(acc, af, b0, b1);
            }
            const int c = nt * 8 + 2 * tq;
            dbc_s[g][c] = acc[0];
            dbc_s[g][c + 1] = acc[1];
            dbc_s[g + 8][c] = acc[2];
            dbc_s[g + 8][c + 1] = acc[3];
        }
        __syncthreads();
        // ---- 3. dt_proj + softplus: dl[16][DI] = softplus(dt_r[16][RP] . W_dt^T + b_dt)
        {
            uint32_t af[RP / 16][4];
#pragma unroll
            for (int ks = 0; ks < RP / 16; ++ks) {
                const int k0 = ks * 16;
                auto ld2 = [&](int r, int k) -> uint32_t {
                    const float v0 = (k < a.R) ? dbc_s[r][k] : 0.0f;
                    const float v1 = (k + 1 < a.R) ? dbc_s[r][k + 1] : 0.0f;
                    return pk_bf16(v0, v1);
                };
                af[ks][0] = ld2(g, k0 + 2 * tq);
                af[ks][1] = ld2(g + 8, k0 + 2 * tq);
                af[ks][2] = ld2(g, k0 + 8 + 2 * tq);
                af[ks][3] = ld2(g + 8, k0 + 8 + 2 * tq);
            }
            for (int nt = warp; nt < DI / 8; nt += NW) {
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                const __nv_bfloat16* wrow = a.Wdt_b + (int64_t)(nt * 8 + g) * RP;
#pragma unroll
                for (int ks = 0; ks < RP / 16; ++ks) {
                    const uint32_t b0 = __ldg(reinterpret_cast<const unsigned int*>(wrow + ks * 16 + 2 * tq));
                    const uint32_t b1 = __ldg(reinterpret_cast<const unsigned int*>(wrow + ks * 16 + 8 + 2 * tq));
                    mma_16816(acc, af[ks], b0, b1);
                }
                const int c = nt * 8 + 2 * tq;
                const float b0v = __ldg(a.b_dt + c), b1v = __ldg(a.b_dt + c + 1);
                dl_s[g][c] = softplus(acc[0] + b0v);
                dl_s[g][c + 1] = softplus(acc[1] + b1v);
                dl_s[g + 8][c] = softplus(acc[2] + b0v);
                dl_s[g + 8][c + 1] = softplus(acc[3] + b1v);
            }
        }
        __syncthreads();
        // ---- 4. selective scan + D skip + gate
        for (int tt = 0; tt < tc; ++tt) {
            const float u = u_s[tt][d];
            const float dl = dl_s[tt][d];
            const float z = __bfloat162float(z_s[tt][d]);
            const float* Bt = &dbc_s[tt][a.R];
            const float* Ct = Bt + N;
            float y = 0.0f;
            if (a.disc == 1) {
                const float du = dl * u;
#pragma unroll
                for (int n = 0; n < N; ++n) {
                    const float Ab = ex2(dl * A2[n]);
                    s[n] = fmaf(Ab, s[n], du * Bt[n]);
                    y = fmaf(Ct[n], s[n], y);
                }
            } else {
#pragma unroll
                for (int n = 0; n < N; ++n) {
                    const float Ab = ex2(dl * A2[n]);
                    const float v = (Bt[n] * u) * iA[n];
                    s[n] = fmaf(Ab, s[n] + v, -v);
                    y = fmaf(Ct[n], s[n], y);
                }
            }
            y = fmaf(Dv, u, y);
            a.G[(base + t0 + tt) * a.ldg + d] = __float2bfloat16_rn(y * silu(z));
        }
        __syncthreads();
    }
}

template <int DI, int N, int RP, int NXP, int DC>
static cudaError_t mixer_launch_dc(const MixerArgs& a, cudaStream_t s) {
    constexpr int smem = MixerSmem<DI, NXP>::kBytes;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_mixer_fused<DI, N, RP, NXP, DC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_mixer_fused<DI, N, RP, NXP, DC><<<(unsigned)a.n, DI, smem, s>>>(a);
    return cudaGetLastError();
}

template <int DI, int N, int RP, int NXP>
static cudaError_t mixer_launch(const MixerArgs& a, cudaStream_t s) {
    switch (a.d_conv) {
        case 4: return mixer_launch_dc<DI, N, RP, NXP, 4>(a, s);
        case 3: return mixer_launch_dc<DI, N, RP, NXP, 3>(a, s);
        case 2: return mixer_launch_dc<DI, N, RP, NXP, 2>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int DI, int N>
static cudaError_t mixer_rp(const MixerArgs& a, cudaStream_t s) {
    const int nxp = ((a.R + 2 * N) + 7) / 8 * 8;
    if (a.RP == 16) {
        if (nxp <= 24) return mixer_launch<DI, N, 16, 24>(a, s);
        if (nxp <= 48) return mixer_launch<DI, N, 16, 48>(a, s);
    } else if (a.RP == 32) {
        if (nxp <= 48) return mixer_launch<DI, N, 32, 48>(a, s);
        if (nxp <= 64) return mixer_launch<DI, N, 32, 64>(a, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_mixer_fused(const MixerArgs& a, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    if (a.DI == 256) return a.N == 16 ? mixer_rp<256, 16>(a, s) : mixer_rp<256, 8>(a, s);
    if (a.DI == 128) return a.N == 16 ? mixer_rp<128, 16>(a, s) : mixer_rp<128, 8>(a, s);
    if (a.DI == 64) return a.N == 16 ? mixer_rp<64, 16>(a, s) : mixer_rp<64, 8>(a, s);
    return cudaErrorInvalidValue;
}

}  // namespace tcl
