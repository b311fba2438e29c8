// mixer_ws.cu -- warp-specialised fused Mamba mixer for the bf16 path.
//
// Same arithmetic as mixer_fused.cu (conv + SiLU, x_proj, dt_proj + softplus, ZOH selective scan,
// D skip, SiLU(z) gate; readings R4-R7), reorganised so that the SFU-bound
// scan never waits for the rest:
//
//   producer warps (4):  TMA bulk copy of the next chunk's [x | z] rows (3-deep ring),
//                        causal conv + SiLU, x_proj and dt_proj on mma.sync, softplus
//                        -> u, Delta, B, C of chunk c+1 in a double-buffered slot
//   scan warps (DI/32):  thread d = channel d, N states in registers, walks chunk c
//
// Producer and scan hand chunks over through mbarriers (full[slot] / empty[slot]); the scan warps
// execute no __syncthreads.  In the scan, exp(Delta A) = 2^(Delta A log2 e) runs on MUFU.EX2 for
// most state pairs and, for OFF of the N/2 pairs, as a degree-3 polynomial on the FMA pipe
// (Cody-Waite split 2^x = 2^j 2^f, |f| <= 1/2, relative error 1.0e-4; exponent inserted with
// integer ops), which balances MUFU against instruction issue.  All other scan arithmetic is
// packed fp32x2 (FFMA2 / FMUL2 / FADD2).
#include <cuda_bf16.h>

#include "../kernels.h"
#include "../kernels_mixer.h"
#include "../tc_ptx.cuh"

namespace tcl {

namespace ws {

constexpr int kTC = 16;       // tokens per chunk (= MMA M)
constexpr int kProdWarps = 4;

template <int DI, int NXP>
struct Smem {
    static constexpr int kXZld = 2 * DI;           // bf16, row = [x | z]
    static constexpr int kUld = DI + 4;            // fp32
    static constexpr int kUbld = DI + 8;           // bf16 (+16 B: conflict-free MMA fragments)
    static constexpr int kDbcld = NXP + 4;         // fp32
    static constexpr int kXZslot = kTC * kXZld * 2;
    static constexpr int kXZ = 0;                                       // [3][16][2 DI] bf16
    static constexpr int kU = kXZ + 3 * kXZslot;                        // [2][16][DI + 4] fp32
    static constexpr int kDl = kU + 2 * kTC * kUld * 4;                 // [2][16][DI] fp32
    static constexpr int kDbc = kDl + 2 * kTC * DI * 4;                 // [2][16][NXP + 4] fp32
    static constexpr int kUb = kDbc + 2 * kTC * kDbcld * 4;             // [16][DI + 8] bf16
    static constexpr int kWx = kUb + kTC * kUbld * 2;                   // [NXP][DI + 8] bf16
    static constexpr int kBar = kWx + NXP * kUbld * 2;                  // tma[3], full[2], empty[2]
    static constexpr int kBytes = kBar + 8 * 8;
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
__device__ __forceinline__ float silu_fast(float v) {  // v * (0.5 + 0.5 tanh(v / 2)), one MUFU
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * v));
    return v * fmaf(0.5f, t, 0.5f);
}
__device__ __forceinline__ float softplus_fast(float v) {  // max(v,0) + log(1 + e^-|v|), branch-free
    return fmaxf(v, 0.0f) + __logf(1.0f + __expf(-fabsf(v)));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            tc::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// 2^x for a pair, x <= 0, on the FMA + ALU pipes: x = j + f (j integer, |f| <= 1/2),
// 2^f ~ 1 + f (c1 + f (c2 + f c3)) (near-minimax, max relative error 1.0e-4), 2^j inserted into
// the exponent field with an integer shift/add.  Inputs are clamped to -125 (result >= 2^-125).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
    x.x = fmaxf(x.x, -125.0f);
    x.y = fmaxf(x.y, -125.0f);
    const float2 magic = make_float2(12582912.0f, 12582912.0f);  // 1.5 * 2^23
    const float2 t = __fadd2_rn(x, magic);                       // round(x) in the low mantissa bits
    const float2 j = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
    const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
    float2 p = __ffma2_rn(f, make_float2(0.05500858f, 0.05500858f), make_float2(0.24221037f, 0.24221037f));
    p = __ffma2_rn(p, f, make_float2(0.6932829f, 0.6932829f));
    p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
    const uint32_t rx = __float_as_uint(p.x) + (__float_as_uint(t.x) << 23);
    const uint32_t ry = __float_as_uint(p.y) + (__float_as_uint(t.y) << 23);
    return make_float2(__uint_as_float(rx), __uint_as_float(ry));
}

// Deterministic per-CTA chunk sequence (both roles walk it independently).
struct ChunkIter {
    const int32_t* lens; int64_t n; int max_len; int stride;
    int64_t i; int t0;
    __device__ int64_t first_valid(int64_t j) const {
        for (; j < n; j += stride) {
            const int T = lens[j];
            if (T >= 1 && T <= max_len) return j;
        }
        return j;
    }
    __device__ void start(int64_t j0) { i = first_valid(j0); t0 = 0; }
    __device__ bool valid() const { return i < n; }
    __device__ void next() {
        const int T = lens[i];
        t0 += kTC;
        if (t0 >= T) { i = first_valid(i + stride); t0 = 0; }
    }
};

// SPLIT threads per channel: each scan thread owns N/SPLIT of the channel's states; the partial
// outputs C.s of a channel are combined with one shuffle (SPLIT = 2 doubles the scan warps per SM
// at the same register budget -> better latency hiding for the MUFU-bound recurrence).
template <int DI, int N, int RP, int NXP, int DC, int DISC, int SPLIT>
__global__ void __launch_bounds__(SPLIT * DI + 32 * kProdWarps, 1) k_mixer_ws(MixerArgs a) {
    using L = Smem<DI, NXP>;
    constexpr int OFF = 0;                // polynomial exp pairs (FMA pipe already ~45% busy)
    constexpr int NSW = SPLIT * DI / 32;  // scan warps
    constexpr int NPT = 32 * kProdWarps;  // producer threads
    constexpr int CPT = DI / NPT;         // channels per producer thread
    extern __shared__ __align__(128) uint8_t msm[];
    __nv_bfloat16* xz_s = reinterpret_cast<__nv_bfloat16*>(msm + L::kXZ);
    float* u_s = reinterpret_cast<float*>(msm + L::kU);
    float* dl_s = reinterpret_cast<float*>(msm + L::kDl);
    float* dbc_s = reinterpret_cast<float*>(msm + L::kDbc);
    __nv_bfloat16* u_b = reinterpret_cast<__nv_bfloat16*>(msm + L::kUb);
    __nv_bfloat16* wx_s = reinterpret_cast<__nv_bfloat16*>(msm + L::kWx);
    uint64_t* tmab = reinterpret_cast<uint64_t*>(msm + L::kBar);   // [3]
    uint64_t* full = tmab + 3;                                      // [2] producer -> scan
    uint64_t* empty = full + 2;                                     // [2] scan -> producer

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    for (int idx = tid; idx < NXP * DI / 8; idx += blockDim.x) {
        const int r = idx / (DI / 8), c8 = idx - r * (DI / 8);
        *reinterpret_cast<uint4*>(wx_s + r * L::kUbld + c8 * 8) =
            __ldg(reinterpret_cast<const uint4*>(a.Wx_b + (int64_t)r * DI + c8 * 8));
    }
    if (tid == 0) {
        for (int k = 0; k < 3; ++k) tc::mbar_init(&tmab[k], 1);
        for (int k = 0; k < 2; ++k) { tc::mbar_init(&full[k], NPT); tc::mbar_init(&empty[k], NSW); }
        tc::fence_mbar_init();
    }
    __syncthreads();

    ChunkIter it{a.lens, a.n, a.max_len, (int)gridDim.x, 0, 0};
    it.start(blockIdx.x);

    if (warp >= NSW) {
        // =============================== producer warps ===============================
        const int p = tid - SPLIT * DI;     // 0 .. NPT-1
        const int pw = warp - NSW;          // producer warp 0..3
        const int g = lane >> 2, tq = lane & 3;
        constexpr int NT_DT = DI / 8 / kProdWarps;
        uint32_t wdt[NT_DT][RP / 16][2];
#pragma unroll
        for (int j = 0; j < NT_DT; ++j) {
            const __nv_bfloat16* wrow = a.Wdt_b + (int64_t)((pw + j * kProdWarps) * 8 + g) * RP;
#pragma unroll
            for (int ks = 0; ks < RP / 16; ++ks) {
                wdt[j][ks][0] = __ldg(reinterpret_cast<const unsigned int*>(wrow + ks * 16 + 2 * tq));
                wdt[j][ks][1] = __ldg(reinterpret_cast<const unsigned int*>(wrow + ks * 16 + 8 + 2 * tq));
            }
        }
        float wc[CPT][DC], bc[CPT], win[CPT][DC];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const int d = p + q * NPT;
            bc[q] = __ldg(a.b_conv + d);
#pragma unroll
            for (int k = 0; k < DC; ++k) { wc[q][k] = __ldg(a.w_conv + d * DC + k); win[q][k] = 0.0f; }
        }
        // TMA issue helper: chunk (i, t0) into ring slot r
        auto issue = [&](int64_t i, int t0, int r) {
            const int T = a.lens[i];
            const int tc = min(kTC, T - t0);
            const uint32_t bytes = (uint32_t)tc * L::kXZld * 2;
            tc::mbar_arrive_expect_tx(&tmab[r], bytes);
            bulk_g2s(xz_s + r * kTC * L::kXZld, a.XZ + (a.cu[i] + t0) * (int64_t)a.ldxz, bytes, &tmab[r]);
        };
        ChunkIter pre = it;  // TMA runs one chunk ahead of the producer's compute
        if (p == 0 && pre.valid()) issue(pre.i, pre.t0, 0);
        if (pre.valid()) pre.next();
        uint32_t c = 0;  // chunk counter
        while (it.valid()) {
            const int slot = c & 1, r = c % 3;
            const int T = a.lens[it.i];
            const int tc = min(kTC, T - it.t0);
            if (it.t0 == 0) {
#pragma unroll
                for (int q = 0; q < CPT; ++q)
#pragma unroll
                    for (int k = 0; k < DC; ++k) win[q][k] = 0.0f;
            }
            // slot reuse: the scan must have finished chunk c-2 (which also frees ring slot (c+1)%3)
            if (c >= 2) tc::mbar_wait(&empty[slot], ((c >> 1) - 1) & 1);
            if (p == 0 && pre.valid()) issue(pre.i, pre.t0, (c + 1) % 3);
            if (pre.valid()) pre.next();
            tc::mbar_wait(&tmab[r], (c / 3) & 1);
            const __nv_bfloat16* xz = xz_s + r * kTC * L::kXZld;
            float* us = u_s + slot * kTC * L::kUld;
            float* dls = dl_s + slot * kTC * DI;
            float* dbcs = dbc_s + slot * kTC * L::kDbcld;
            // ---- conv + SiLU
#pragma unroll 4
            for (int tt = 0; tt < kTC; ++tt) {
#pragma unroll
                for (int q = 0; q < CPT; ++q) {
                    const int d = p + q * NPT;
                    float u = 0.0f;
                    if (tt < tc) {
                        const float x = __bfloat162float(xz[tt * L::kXZld + d]);
                        float acc = fmaf(wc[q][DC - 1], x, bc[q]);
#pragma unroll
                        for (int k = 0; k < DC - 1; ++k) acc = fmaf(wc[q][DC - 2 - k], win[q][k], acc);
#pragma unroll
                        for (int k = DC - 1; k > 0; --k) win[q][k] = win[q][k - 1];
                        win[q][0] = x;
                        u = silu_fast(acc);
                    }
                    us[tt * L::kUld + d] = u;
                    u_b[tt * L::kUbld + d] = __float2bfloat16_rn(u);
                }
            }
            named_bar(1, NPT);
            // ---- x_proj: dbc[16][NXP] = u[16][DI] . W_x^T
            for (int nt = pw; nt < NXP / 8; nt += kProdWarps) {
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                const __nv_bfloat16* wrow = wx_s + (nt * 8 + g) * L::kUbld;
#pragma unroll 4
                for (int k0 = 0; k0 < DI; k0 += 16) {
                    uint32_t af[4];
                    af[0] = *reinterpret_cast<const uint32_t*>(u_b + g * L::kUbld + k0 + 2 * tq);
                    af[1] = *reinterpret_cast<const uint32_t*>(u_b + (g + 8) * L::kUbld + k0 + 2 * tq);
                    af[2] = *reinterpret_cast<const uint32_t*>(u_b + g * L::kUbld + k0 + 8 + 2 * tq);
                    af[3] = *reinterpret_cast<const uint32_t*>(u_b + (g + 8) * L::kUbld + k0 + 8 + 2 * tq);
                    const uint32_t b0 = *reinterpret_cast<const uint32_t*>(wrow + k0 + 2 * tq);
                    const uint32_t b1 = *reinterpret_cast<const uint32_t*>(wrow + k0 + 8 + 2 * tq);
                    mma_16816(acc, af, b0, b1);
                }
                const int cc = nt * 8 + 2 * tq;
                *reinterpret_cast<float2*>(dbcs + g * L::kDbcld + cc) = make_float2(acc[0], acc[1]);
                *reinterpret_cast<float2*>(dbcs + (g + 8) * L::kDbcld + cc) = make_float2(acc[2], acc[3]);
            }
            named_bar(1, NPT);
            // ---- dt_proj + softplus
            {
                uint32_t af[RP / 16][4];
#pragma unroll
                for (int ks = 0; ks < RP / 16; ++ks) {
                    const int k0 = ks * 16;
                    auto ld2 = [&](int row, int k) -> uint32_t {
                        const float v0 = (k < a.R) ? dbcs[row * L::kDbcld + k] : 0.0f;
                        const float v1 = (k + 1 < a.R) ? dbcs[row * L::kDbcld + k + 1] : 0.0f;
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
                    const int cc = (pw + j * kProdWarps) * 8 + 2 * tq;
                    const float b0v = __ldg(a.b_dt + cc), b1v = __ldg(a.b_dt + cc + 1);
                    *reinterpret_cast<float2*>(dls + g * DI + cc) =
                        make_float2(softplus_fast(acc[0] + b0v), softplus_fast(acc[1] + b1v));
                    *reinterpret_cast<float2*>(dls + (g + 8) * DI + cc) =
                        make_float2(softplus_fast(acc[2] + b0v), softplus_fast(acc[3] + b1v));
                }
            }
            tc::mbar_arrive(&full[slot]);  // all NPT producer threads arrive (release their writes)
            named_bar(1, NPT);             // u_b reuse guard for the next chunk
            it.next();
            ++c;
        }
    } else {
        // =============================== scan warps ===============================
        constexpr int NP = N / 2 / SPLIT;         // state pairs per thread
        const int d = SPLIT == 1 ? tid : warp * 16 + (lane >> 1);
        const int hh = SPLIT == 1 ? 0 : (lane & 1);
        float2 A2[NP], iA[NP];
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            A2[n] = __ldg(reinterpret_cast<const float2*>(a.A2 + d * N) + hh * NP + n);
            iA[n] = __ldg(reinterpret_cast<const float2*>(a.invA + d * N) + hh * NP + n);
        }
        const float Dv = __ldg(a.Dv + d);
        float2 s[NP];
        uint32_t c = 0;
        while (it.valid()) {
            const int slot = c & 1, r = c % 3;
            const int T = a.lens[it.i];
            const int tc = min(kTC, T - it.t0);
            if (it.t0 == 0) {
#pragma unroll
                for (int n = 0; n < NP; ++n) s[n] = make_float2(0.f, 0.f);
            }
            tc::mbar_wait(&full[slot], (c >> 1) & 1);
            tc::mbar_wait(&tmab[r], (c / 3) & 1);  // z rows (async-proxy writes) visible here too
            const __nv_bfloat16* zp = xz_s + r * kTC * L::kXZld + DI + d;
            const float* up = u_s + slot * kTC * L::kUld + d;
            const float* dlp = dl_s + slot * kTC * DI + d;
            const float* bp = dbc_s + slot * kTC * L::kDbcld + a.R + hh * 2 * NP;
            __nv_bfloat16* gout = a.G + (a.cu[it.i] + it.t0) * (int64_t)a.ldg + d;
            for (int tt = 0; tt < tc; ++tt) {
                const float u = *up;
                const float dl = *dlp;
                const float z = __bfloat162float(*zp);
                const float2 dl2 = make_float2(dl, dl);
                const float2 u2 = make_float2(u, u);
                const float2 du2 = __fmul2_rn(dl2, u2);
                float2 y2 = make_float2(0.f, 0.f), y2b = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < NP / 2; ++q) {
                    const float4 b4 = reinterpret_cast<const float4*>(bp)[q];
                    const float4 c4 = reinterpret_cast<const float4*>(bp + N)[q];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int n = 2 * q + h;
                        const float2 x2 = __fmul2_rn(dl2, A2[n]);
                        const float2 ab = (n >= NP - OFF) ? exp2_poly2(x2)
                                                          : make_float2(ex2(x2.x), ex2(x2.y));
                        const float2 bb = h ? make_float2(b4.z, b4.w) : make_float2(b4.x, b4.y);
                        const float2 cc = h ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
                        if (DISC == 1) {
                            s[n] = __ffma2_rn(ab, s[n], __fmul2_rn(bb, du2));
                        } else {
                            // Bbar u = (Ab - 1) v, v = B u / A:  s <- Ab (s + v) - v
                            const float2 v = __fmul2_rn(__fmul2_rn(bb, u2), iA[n]);
                            s[n] = __ffma2_rn(ab, __fadd2_rn(s[n], v), make_float2(-v.x, -v.y));
                        }
                        if (h) y2b = __ffma2_rn(cc, s[n], y2b); else y2 = __ffma2_rn(cc, s[n], y2);
                    }
                }
                float yp = (y2.x + y2b.x) + (y2.y + y2b.y);
                if (SPLIT == 2) yp += __shfl_xor_sync(0xffffffffu, yp, 1);
                const float y = fmaf(Dv, u, yp);
                const __nv_bfloat16 gv = __float2bfloat16_rn(y * silu_fast(z));
                if (hh == 0) gout[(int64_t)tt * a.ldg] = gv;
                up += L::kUld;
                dlp += DI;
                zp += L::kXZld;
                bp += L::kDbcld;
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[slot]);
            it.next();
            ++c;
        }
    }
}

template <int DI, int N, int RP, int NXP, int SPLIT>
static cudaError_t launch_k(const MixerArgs& a, int num_sms, cudaStream_t s) {
    constexpr int smem = Smem<DI, NXP>::kBytes;
    constexpr int threads = SPLIT * DI + 32 * kProdWarps;
    auto kern = a.disc == 1 ? k_mixer_ws<DI, N, RP, NXP, 4, 1, SPLIT> : k_mixer_ws<DI, N, RP, NXP, 4, 0, SPLIT>;
    static bool attr[2] = {false, false};
    if (!attr[a.disc]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr[a.disc] = true;
    }
    int64_t grid = num_sms;
    if (grid > a.n) grid = a.n;
    kern<<<(unsigned)grid, threads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int DI, int N>
static cudaError_t launch_rp(const MixerArgs& a, int num_sms, cudaStream_t s) {
    const int nxp = ((a.R + 2 * N) + 7) / 8 * 8;
    constexpr int SPLIT = N == 16 ? 2 : 1;  // two threads per channel when the state is large
    if (a.RP == 16) {
        if (nxp <= 24) return launch_k<DI, N, 16, 24, SPLIT>(a, num_sms, s);
        if (nxp <= 48) return launch_k<DI, N, 16, 48, SPLIT>(a, num_sms, s);
    } else if (a.RP == 32) {
        if (nxp <= 64) return launch_k<DI, N, 32, 64, SPLIT>(a, num_sms, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace ws

cudaError_t launch_mixer_ws(const MixerArgs& a, int num_sms, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    if (a.d_conv != 4) return cudaErrorInvalidValue;
    if (a.DI == 256) return a.N == 16 ? ws::launch_rp<256, 16>(a, num_sms, s) : ws::launch_rp<256, 8>(a, num_sms, s);
    if (a.DI == 128) return a.N == 16 ? ws::launch_rp<128, 16>(a, num_sms, s) : ws::launch_rp<128, 8>(a, num_sms, s);
    return cudaErrorInvalidValue;
}

}  // namespace tcl
