// head.cu -- SURVEY §8(a) a9: final LayerNorm ("normalized again"), masked mean
// over the T real tokens (reading R9), decoder of three linears 64,32,1 with SiLU
// after the first two (reading R1), plus the MC-dropout sites dec h1/h2 and the
// per-candidate Welford accumulation over passes (reading R17).
// The pool kernels reduce each candidate's rows in order t = 0..T-1 (one warp per candidate); the
// decoder runs as three small GEMMs over the candidates (gemm_simt.cu); every reduction has a
// fixed order -> batch-invariant scores.
#include <cuda_bf16.h>
#include <math.h>

#include "../kernels.h"

namespace tcl {

// LN_f of every real row and the masked mean over the candidate's T rows; one warp per candidate
// (8 candidates per CTA), rows summed in order t = 0..T-1 -> batch-invariant.
template <int PER>
__global__ void __launch_bounds__(256) k_pool(const float* __restrict__ H, int ldh,
                                              const float* __restrict__ g, const float* __restrict__ b,
                                              float eps, const int32_t* __restrict__ cu,
                                              const int32_t* __restrict__ lens, int max_len, int64_t n,
                                              float* __restrict__ pooled) {
    constexpr int dm = 32 * PER;
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int T = lens[i];
    float acc[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j] = 0.0f;
    if (T >= 1 && T <= max_len) {
        const float* h = H + (int64_t)cu[i] * ldh;
        float gv[PER], bv[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) { gv[j] = __ldg(g + lane + 32 * j); bv[j] = __ldg(b + lane + 32 * j); }
        for (int t = 0; t < T; ++t) {
            float v[PER];
            float sm = 0.f;
#pragma unroll
            for (int j = 0; j < PER; ++j) { v[j] = h[(int64_t)t * ldh + lane + 32 * j]; sm += v[j]; }
            const float mean = warp_sum(sm) * (1.0f / dm);
            float q = 0.f;
#pragma unroll
            for (int j = 0; j < PER; ++j) { const float e = v[j] - mean; q = fmaf(e, e, q); }
            const float rstd = rsqrtf(warp_sum(q) * (1.0f / dm) + eps);
#pragma unroll
            for (int j = 0; j < PER; ++j) acc[j] += (v[j] - mean) * rstd * gv[j] + bv[j];
        }
        const float invT = 1.0f / (float)T;
#pragma unroll
        for (int j = 0; j < PER; ++j) acc[j] *= invT;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) pooled[i * dm + lane + 32 * j] = acc[j];
}

void launch_pool(const float* H, int ldh, int dm, const float* lnf_w, const float* lnf_b, float eps,
                 const int32_t* cu, const int32_t* lens, int max_len, int64_t n, float* pooled,
                 cudaStream_t s) {
    if (n == 0) return;
    dim3 grid((unsigned)((n + 7) / 8));
    switch (dm / 32) {
#define TCL_POOL(P) case P: k_pool<P><<<grid, 256, 0, s>>>(H, ldh, lnf_w, lnf_b, eps, cu, lens, max_len, n, pooled); break;
        TCL_POOL(1) TCL_POOL(2) TCL_POOL(3) TCL_POOL(4) TCL_POOL(5) TCL_POOL(6) TCL_POOL(7) TCL_POOL(8)
#undef TCL_POOL
        default: break;
    }
}

// Masked mean of bf16 rows that are already LN_f(H): one warp per candidate, rows summed in order.
template <int PER>
__global__ void __launch_bounds__(256) k_pool_bf16(const __nv_bfloat16* __restrict__ F, int ldf,
                                                   const int32_t* __restrict__ cu,
                                                   const int32_t* __restrict__ lens, int max_len, int64_t n,
                                                   float* __restrict__ pooled) {
    constexpr int dm = 64 * PER;  // lane handles 2 * PER columns (bf16x2 loads)
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int T = lens[i];
    float acc[2 * PER];
#pragma unroll
    for (int j = 0; j < 2 * PER; ++j) acc[j] = 0.0f;
    if (T >= 1 && T <= max_len) {
        const __nv_bfloat16* f = F + (int64_t)cu[i] * ldf;
#pragma unroll 4
        for (int t = 0; t < T; ++t) {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(f + (int64_t)t * ldf + 2 * (lane + 32 * j));
                const float2 fv = __bfloat1622float2(v);
                acc[2 * j] += fv.x;
                acc[2 * j + 1] += fv.y;
            }
        }
        const float invT = 1.0f / (float)T;
#pragma unroll
        for (int j = 0; j < 2 * PER; ++j) acc[j] *= invT;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j)
        *reinterpret_cast<float2*>(pooled + i * dm + 2 * (lane + 32 * j)) = make_float2(acc[2 * j], acc[2 * j + 1]);
}

void launch_pool_bf16(const void* F, int ldf, int dm, const int32_t* cu, const int32_t* lens, int max_len,
                      int64_t n, float* pooled, cudaStream_t s) {
    if (n == 0) return;
    dim3 grid((unsigned)((n + 7) / 8));
    const auto* f = reinterpret_cast<const __nv_bfloat16*>(F);
    switch (dm / 64) {
        case 1: k_pool_bf16<1><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        case 2: k_pool_bf16<2><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        case 3: k_pool_bf16<3><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        case 4: k_pool_bf16<4><<<grid, 256, 0, s>>>(f, ldf, cu, lens, max_len, n, pooled); break;
        default: break;
    }
}

// ---------------------------------------------------------------------------- fused head
// The whole head in ONE kernel (one launch instead of five): a CTA of 256 threads takes 32
// candidates; (1) each warp pools 4 of them exactly as k_pool / k_pool_bf16 (rows in order
// t = 0..T-1) into shared memory; (2)-(4) the three decoder linears, each output one sequential
// FFMA chain over k in order (the weights staged 32 k at a time, transposed, in shared memory),
// v = acc + b, SiLU (+ inverted dropout, sites 2 / 3, token 0) -- the arithmetic of the SIMT
// GEMMs it replaces, so the scores are bit-identical to the five-launch head; (5) the score is
// stored (NaN for an invalid length) or folded into the MC Welford statistics.
template <int CT, int K, int NO, int NOP, bool ACT, int TA = 4>
__device__ __forceinline__ void head_linear(const float* __restrict__ inT, const float* __restrict__ W,
                                            const float* __restrict__ bias, float* __restrict__ outT,
                                            float* ws, const DropoutCtx& drop, int site, int64_t cand0,
                                            int64_t n) {
    // inT [K][CT + 4], outT [NO][CT + 4] (transposed: 4 consecutive candidates are one float4).
    // Thread -> a TA x 4 register tile: columns 4 jq .. 4 jq + 3, candidates TA cq .. TA cq + TA - 1;
    // each output is one sequential FFMA chain over k (TA / 4 + 1 LDS.128 per 4 TA FFMA).
    static_assert(TA % 4 == 0, "TA: whole float4 candidate groups");
    constexpr int LD = CT + 4;
    constexpr int JQ = NOP / 4, CQ = CT / TA;
    static_assert(JQ * CQ <= 256, "head_linear: more register tiles than threads");
    const int jq = threadIdx.x % JQ, cq = threadIdx.x / JQ;
    const bool act_thr = cq < CQ && 4 * jq < NO;
    float acc[TA][4];
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
    // W is staged 32 k at a time into ws[2][32][NOP] (double-buffered: the next slice's global
    // loads are in flight while this slice is consumed).  Layout: row kk, float4 group g of
    // columns 4 g .. 4 g + 3 stored at group g ^ (kk & 7): a warp loads 4 rows x 8 consecutive k
    // (32-byte segments) and its 32 stores hit 32 distinct banks; the float4 reads of a row stay
    // conflict-free (a permutation of the row's groups).
    static_assert(NOP >= 32, "ws swizzle needs >= 8 float4 groups per row");
    constexpr int kPer = (NO * 32 + 255) / 256;
    constexpr int kSlices = (K + 31) / 32;
    float pre[kPer];
    auto gload = [&](int k0) {
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int idx = threadIdx.x + 256 * e, lane = idx & 31, c = idx >> 5;
            const int kk = 8 * (c & 3) + (lane & 7), jj = 4 * (c >> 2) + (lane >> 3);
            pre[e] = (idx < NO * 32 && jj < NO && k0 + kk < K) ? __ldg(W + (int64_t)jj * K + k0 + kk) : 0.0f;
        }
    };
    auto sstore = [&](float* buf) {
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int idx = threadIdx.x + 256 * e, lane = idx & 31, c = idx >> 5;
            const int kk = 8 * (c & 3) + (lane & 7), g = c >> 2;
            if (idx < NO * 32) buf[kk * NOP + 4 * (g ^ (kk & 7)) + (lane >> 3)] = pre[e];
        }
    };
    gload(0);
    __syncthreads();   // ws reuse (and the producer of inT is done)
    sstore(ws);
    __syncthreads();
    for (int sl = 0; sl < kSlices; ++sl) {
        const int k0 = 32 * sl;
        const float* cur = ws + (sl & 1) * 32 * NOP;
        if (sl + 1 < kSlices) gload(k0 + 32);
        if (act_thr) {
#pragma unroll 4
            for (int kk = 0; kk < 32; ++kk) {
                if (k0 + kk >= K) break;
                const float4 wv = *reinterpret_cast<const float4*>(cur + kk * NOP + 4 * (jq ^ (kk & 7)));
                const float wsv[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                for (int g = 0; g < TA / 4; ++g) {
                    const float4 xv = *reinterpret_cast<const float4*>(inT + (k0 + kk) * LD + TA * cq + 4 * g);
                    const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) acc[4 * g + a][b] = fmaf(xs[a], wsv[b], acc[4 * g + a][b]);
                }
            }
        }
        if (sl + 1 < kSlices) sstore(ws + ((sl + 1) & 1) * 32 * NOP);
        __syncthreads();
    }
    if (act_thr) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = 4 * jq + b;
            if (j >= NO) continue;
            const float bj = __ldg(bias + j);
#pragma unroll
            for (int g = 0; g < TA / 4; ++g) {
                float v4[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int c = TA * cq + 4 * g + a;
                    float v = acc[4 * g + a][b] + bj;
                    if (ACT) {
                        v = silu(v);
                        if (drop.enabled && cand0 + c < n) v = dropout_keep(drop, j, 0, site, cand0 + c) ? v * drop.scale : 0.0f;
                    }
                    v4[a] = v;
                }
                *reinterpret_cast<float4*>(outT + j * LD + TA * cq + 4 * g) = make_float4(v4[0], v4[1], v4[2], v4[3]);
            }
        }
    }
}

// CT candidates per CTA.  A candidate's arithmetic does not depend on CT.
template <int PER, bool BF16, int H1, int H2, int CT>
__global__ void __launch_bounds__(256) k_head(HeadArgs a) {
    constexpr int kHeadCT = CT;
    constexpr int dm = 32 * PER;
    constexpr int H1P = H1 <= 32 ? 32 : (H1 <= 64 ? 64 : (H1 <= 128 ? 128 : 256));
    constexpr int H2P = H2 <= 32 ? 32 : (H2 <= 64 ? 64 : (H2 <= 128 ? 128 : 256));
    constexpr int LD = CT + 4;   // transposed activations: [feature][candidate], float4 rows
    extern __shared__ __align__(16) float hsm[];
    float* pooledT = hsm;                         // [dm][LD]
    float* h1T = pooledT + dm * LD;               // [H1][LD]
    float* h2T = h1T + H1 * LD;                   // [H2][LD]
    float* ws = h2T + H2 * LD;                    // [2][32][max(H1P, H2P)]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.x * kHeadCT;
    // ---- (1) masked mean (of LN_f(H) rows: computed here on the fp32 path, stored bf16 on the bf16 path)
    for (int cc = warp; cc < kHeadCT; cc += 8) {
        const int64_t i = c0 + cc;
        const int T = i < a.n ? a.lens[i] : 0;
        const bool ok = T >= 1 && T <= a.max_len;
        if (!BF16) {
            float acc[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) acc[j] = 0.0f;
            if (ok) {
                const float* h = a.H + (int64_t)a.cu[i] * a.ldh;
                float gv[PER], bv[PER];
#pragma unroll
                for (int j = 0; j < PER; ++j) { gv[j] = __ldg(a.lnf_w + lane + 32 * j); bv[j] = __ldg(a.lnf_b + lane + 32 * j); }
                for (int t = 0; t < T; ++t) {
                    float v[PER];
                    float sm = 0.f;
#pragma unroll
                    for (int j = 0; j < PER; ++j) { v[j] = h[(int64_t)t * a.ldh + lane + 32 * j]; sm += v[j]; }
                    const float mean = warp_sum(sm) * (1.0f / dm);
                    float q = 0.f;
#pragma unroll
                    for (int j = 0; j < PER; ++j) { const float e = v[j] - mean; q = fmaf(e, e, q); }
                    const float rstd = rsqrtf(warp_sum(q) * (1.0f / dm) + a.eps);
#pragma unroll
                    for (int j = 0; j < PER; ++j) acc[j] += (v[j] - mean) * rstd * gv[j] + bv[j];
                }
                const float invT = 1.0f / (float)T;
#pragma unroll
                for (int j = 0; j < PER; ++j) acc[j] *= invT;
            }
#pragma unroll
            for (int j = 0; j < PER; ++j) pooledT[(lane + 32 * j) * LD + cc] = acc[j];
        } else {
            constexpr int PB = PER / 2;   // bf16x2 pairs per lane
            float acc[2 * PB];
#pragma unroll
            for (int j = 0; j < 2 * PB; ++j) acc[j] = 0.0f;
            if (ok) {
                const __nv_bfloat16* f = a.F + (int64_t)a.cu[i] * a.ldf;
#pragma unroll 4
                for (int t = 0; t < T; ++t) {
#pragma unroll
                    for (int j = 0; j < PB; ++j) {
                        const float2 fv = __bfloat1622float2(
                            *reinterpret_cast<const __nv_bfloat162*>(f + (int64_t)t * a.ldf + 2 * (lane + 32 * j)));
                        acc[2 * j] += fv.x;
                        acc[2 * j + 1] += fv.y;
                    }
                }
                const float invT = 1.0f / (float)T;
#pragma unroll
                for (int j = 0; j < 2 * PB; ++j) acc[j] *= invT;
            }
#pragma unroll
            for (int j = 0; j < PB; ++j) {
                pooledT[(2 * (lane + 32 * j)) * LD + cc] = acc[2 * j];
                pooledT[(2 * (lane + 32 * j) + 1) * LD + cc] = acc[2 * j + 1];
            }
        }
    }
    // ---- (2)-(4) decoder
    // candidates per thread: 4, or as many as put every thread to work on a CT-candidate batch
    constexpr int TA1 = CT * (H1P / 4) > 1024 ? CT * (H1P / 4) / 256 : 4;
    constexpr int TA2 = CT * (H2P / 4) > 1024 ? CT * (H2P / 4) / 256 : 4;
    head_linear<CT, dm, H1, H1P, true, TA1>(pooledT, a.W1, a.b1, h1T, ws, a.drop, 2, c0, a.n);
    head_linear<CT, H1, H2, H2P, true, TA2>(h1T, a.W2, a.b2, h2T, ws, a.drop, 3, c0, a.n);
    __syncthreads();
    // ---- (3) score, then store / Welford
    if (threadIdx.x < kHeadCT) {
        const int cc = threadIdx.x;
        const int64_t i = c0 + cc;
        if (i < a.n) {
            float acc = 0.0f;
#pragma unroll 8
            for (int k = 0; k < H2; ++k) acc = fmaf(h2T[k * LD + cc], __ldg(a.W3 + k), acc);
            const float v = acc + __ldg(a.b3);
            const int T = a.lens[i];
            const bool ok = T >= 1 && T <= a.max_len;
            if (!a.mc_mean) {
                a.scores[i] = ok ? v : NAN;
            } else if (!ok) {
                a.mc_mean[i] = NAN;
                a.m2[i] = NAN;
            } else {   // Welford over passes (as k_welford)
                const int pass = a.drop.pass;
                const float m_old = pass == 0 ? 0.0f : a.mc_mean[i];
                const float q_old = pass == 0 ? 0.0f : a.m2[i];
                const float delta = v - m_old;
                const float m_new = m_old + delta / (float)(pass + 1);
                a.mc_mean[i] = m_new;
                a.m2[i] = q_old + delta * (v - m_new);
            }
        }
    }
}

template <int PER, bool BF16, int CT>
static bool head_dims(const HeadArgs& a, cudaStream_t s) {
    const dim3 grid((unsigned)((a.n + CT - 1) / CT));
#define TCL_HEAD(H1_, H2_)                                                                                 \
    if (a.h1 == H1_ && a.h2 == H2_) {                                                                 \
        constexpr int H1P = H1_ <= 32 ? 32 : (H1_ <= 64 ? 64 : (H1_ <= 128 ? 128 : 256));           \
        const int smem = 4 * ((CT + 4) * (32 * PER + H1_ + H2_) + 2 * 32 * H1P);                     \
        auto kern = k_head<PER, BF16, H1_, H2_, CT>;                                            \
        if (prepare_kernel(kern, smem) != cudaSuccess) return false;                                  \
        kern<<<grid, 256, smem, s>>>(a);                                                              \
        return true;                                                                                  \
    }
    TCL_HEAD(32 * PER / 2, 32 * PER / 4)   // reading R10: decoder [d_model / 2, d_model / 4, 1]
#undef TCL_HEAD
    return false;
}

template <int PER, bool BF16>
static bool head_pick(const HeadArgs& a, cudaStream_t s) {
    // small batches (launch-bound): everything in one launch, 8 candidates per CTA.  Large batches
    // return false: the caller's pool kernel + SIMT decoder GEMMs keep more rows in flight and
    // reuse each weight tile across 64-128 candidates (measured: the one-launch head at 65,536
    // candidates took 0.53 ms for the decoder alone, re-staging W1 per 32 candidates, vs 0.41 ms
    // for the whole five-launch head).  Both compute every candidate with the same operations in
    // the same order: bit-identical, so the switch does not break batch invariance (tested).
    // (measured again with a 64-candidate decoder launch after the pool kernel, weights staged
    // double-buffered: 0.48 ms for pool + decoder at 65,536 candidates vs 0.42 ms for pool + SIMT
    // GEMMs -- 8 warps per SM do not hide the FFMA / shared-memory latencies that the SIMT GEMMs'
    // 24+ warps do)
    if (a.n < 8192) return head_dims<PER, BF16, 8>(a, s);
    return false;
}

bool launch_head_fused(const HeadArgs& a, cudaStream_t s) {
    if (a.n == 0) return true;
    if (a.h1 != a.dm / 2 || a.h2 != a.dm / 4) return false;
    const bool bf = a.F != nullptr;
    switch (a.dm) {
        case 64: return bf ? head_pick<2, true>(a, s) : head_pick<2, false>(a, s);
        case 128: return bf ? head_pick<4, true>(a, s) : head_pick<4, false>(a, s);
        case 256: return bf ? head_pick<8, true>(a, s) : head_pick<8, false>(a, s);
        default: return false;
    }
}

__global__ void k_welford(const float* __restrict__ score, const int32_t* __restrict__ lens, int max_len,
                          int64_t n, int pass, float* __restrict__ mean, float* __restrict__ m2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int T = lens[i];
    if (T < 1 || T > max_len) { mean[i] = NAN; m2[i] = NAN; return; }
    const float v = score[i];
    const float m_old = pass == 0 ? 0.0f : mean[i];
    const float q_old = pass == 0 ? 0.0f : m2[i];
    const float delta = v - m_old;
    const float m_new = m_old + delta / (float)(pass + 1);
    mean[i] = m_new;
    m2[i] = q_old + delta * (v - m_new);
}

void launch_welford(const float* score, const int32_t* lens, int max_len, int64_t n, int pass, float* mean,
                    float* m2, cudaStream_t s) {
    if (n == 0) return;
    k_welford<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(score, lens, max_len, n, pass, mean, m2);
}

__global__ void k_mask_invalid(const int32_t* __restrict__ lens, int max_len, int64_t n, float* __restrict__ sc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int T = lens[i];
    if (T < 1 || T > max_len) sc[i] = NAN;
}

void launch_mask_invalid(const int32_t* lens, int max_len, int64_t n, float* scores, cudaStream_t s) {
    if (n == 0) return;
    k_mask_invalid<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lens, max_len, n, scores);
}

// Batched MC passes: the per-pass scores of candidate i are score[ps * n + i]; Welford in pass order
// with k_welford's arithmetic (bit-identical to the pass-by-pass fold), then var = M2 / passes.
__global__ void k_mc_reduce(const float* __restrict__ score, const int32_t* __restrict__ lens, int max_len,
                            int64_t n, int passes, float* __restrict__ mean, float* __restrict__ var) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int T = lens[i];
    if (T < 1 || T > max_len) { mean[i] = NAN; var[i] = NAN; return; }
    float m = 0.0f, q = 0.0f;
    for (int pass = 0; pass < passes; ++pass) {
        const float v = score[(int64_t)pass * n + i];
        const float delta = v - m;
        const float m_new = m + delta / (float)(pass + 1);
        q = q + delta * (v - m_new);
        m = m_new;
    }
    mean[i] = m;
    var[i] = q / (float)passes;
}

void launch_mc_reduce(const float* score, const int32_t* lens, int max_len, int64_t n, int passes, float* mean,
                      float* var, cudaStream_t s) {
    if (n == 0) return;
    k_mc_reduce<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(score, lens, max_len, n, passes, mean, var);
}

__global__ void k_mc_finalize(const float* __restrict__ m2, int64_t n, int passes,
                              float* __restrict__ var) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) var[i] = m2[i] / (float)passes;
}

void launch_mc_finalize(const float* m2, int64_t n, int passes, float* var, cudaStream_t s) {
    if (n == 0) return;
    k_mc_finalize<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(m2, n, passes, var);
}

}  // namespace tcl
