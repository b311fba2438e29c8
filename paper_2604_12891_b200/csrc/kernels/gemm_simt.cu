// gemm_simt.cu -- fp32 CUDA-core GEMM Y = epi(X W^T + b) for the FP32 precision mode.
//
// Used for every linear of the fp32 path (encoder P:451, in_proj / x_proj / dt_proj / out_proj
// of the Mamba block P:446) and for the small projections of the bf16 path.  Exact fp32
// FFMA accumulation in a fixed k order: a row's result never depends on the other rows of the
// tile, so scores are batch-invariant (reading R19).
// Tile 64x64x16, 256 threads, 4x4 outputs per thread, operands staged k-major in shared memory.
#include <cstdlib>

#include "../kernels.h"

namespace tcl {

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256) k_gemm_simt(GemmArgs a) {
    __shared__ __align__(16) float As[BK][BM + 4];
    __shared__ __align__(16) float Ws[BK][BN + 4];
    const int rows = a.p_rows ? *a.p_rows : a.rows_const;
    const int m0 = blockIdx.x * BM;
    if (m0 >= rows) return;
    const int n0 = blockIdx.y * BN;
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    // loader mapping: 64 rows x 16 k = 1024 floats = 256 threads x float4
    const int lr = tid >> 2, lk = (tid & 3) * 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

    const int k_end = a.K + a.K2;
    for (int k0 = 0; k0 < k_end; k0 += BK) {
        {
            // k in [0, K): X / W; k in [K, K + K2): the lateral pair X2 / W2 (K2 > 0 only)
            const bool second = k0 >= a.K;
            const float* X = second ? a.X2 : a.X;
            const float* W = second ? a.W2 : a.W;
            const int ldx = second ? a.ldx2 : a.ldx, ldw = second ? a.ldw2 : a.ldw;
            const int kk_end = second ? a.K2 : a.K;
            const int gm = m0 + lr, gk = (second ? k0 - a.K : k0) + lk;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (gm < rows && gk < kk_end) v = *reinterpret_cast<const float4*>(X + (int64_t)gm * ldx + gk);
            As[lk + 0][lr] = v.x; As[lk + 1][lr] = v.y; As[lk + 2][lr] = v.z; As[lk + 3][lr] = v.w;
            const int gn = n0 + lr;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (a.wT && !second) {   // W stored [K][N]: four strided scalars
                if (gn < a.N) {
                    if (gk + 0 < kk_end) w.x = __ldg(W + (int64_t)(gk + 0) * ldw + gn);
                    if (gk + 1 < kk_end) w.y = __ldg(W + (int64_t)(gk + 1) * ldw + gn);
                    if (gk + 2 < kk_end) w.z = __ldg(W + (int64_t)(gk + 2) * ldw + gn);
                    if (gk + 3 < kk_end) w.w = __ldg(W + (int64_t)(gk + 3) * ldw + gn);
                }
            } else if (gn < a.N && gk < kk_end) {
                w = __ldg(reinterpret_cast<const float4*>(W + (int64_t)gn * ldw + gk));
            }
            Ws[lk + 0][lr] = w.x; Ws[lk + 1][lr] = w.y; Ws[lk + 2][lr] = w.z; Ws[lk + 3][lr] = w.w;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
            float4 wv = *reinterpret_cast<const float4*>(&Ws[kk][tx * 4]);
            float ar[4] = {av.x, av.y, av.z, av.w}, wr[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], wr[j], acc[i][j]);
        }
        __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= rows) continue;
        int cand = 0, token = 0;
        u32x4 wd = {0u, 0u, 0u, 0u};
        if (a.epi == EPI_SILU && a.drop.enabled) {
            cand = a.rows_are_cands ? gm : a.row_cand[gm];
            token = a.rows_are_cands ? 0 : gm - a.cu[cand];
            wd = dropout_words(a.drop, n0 + tx * 4, token, a.site, cand);   // this thread's 4 units
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= a.N) continue;
            float v = acc[i][j] + (a.bias ? __ldg(a.bias + gn) : 0.0f);
            float* dst = a.Y + (int64_t)gm * a.ldy + gn;
            if (a.Ypre) a.Ypre[(int64_t)gm * a.ldy + gn] = v;
            switch (a.epi) {
                case EPI_SILU:
                    v = silu(v);
                    if (a.drop.enabled)
                        v = dropout_apply_word(a.drop, v, j == 0 ? wd.x : j == 1 ? wd.y : j == 2 ? wd.z : wd.w);
                    break;
                case EPI_SOFTPLUS: v = softplus(v); break;
                case EPI_RESID: v = *dst + v; break;
                default: break;
            }
            *dst = v;
        }
    }
}

// Wide variant for N >= 128 (in_proj, out_proj, the encoder's 2nd/3rd linears of the fp32 path):
// tile 128x128x8, 256 threads, 8x8 outputs per thread (rows ty*4 + {0..3, 64..67}, columns
// tx*4 + {0..3, 64..67}: four 128-bit smem loads feed 64 FFMA per k step), smem double-buffered
// with register prefetch of the next k-block (one barrier per k-block).  The k order of every
// output is the same sequential 0..K-1 FFMA chain as k_gemm_simt, so results are bit-identical.
constexpr int BM2 = 128, BN2 = 128;

__device__ __forceinline__ void epi_store(const GemmArgs& a, int gm, int gn, float acc, int cand, int token) {
    float v = acc + (a.bias ? __ldg(a.bias + gn) : 0.0f);
    float* dst = a.Y + (int64_t)gm * a.ldy + gn;
    if (a.Ypre) a.Ypre[(int64_t)gm * a.ldy + gn] = v;
    switch (a.epi) {
        case EPI_SILU:
            v = silu(v);
            if (a.drop.enabled) v = dropout_keep(a.drop, gn, token, a.site, cand) ? v * a.drop.scale : 0.0f;
            break;
        case EPI_SOFTPLUS: v = softplus(v); break;
        case EPI_RESID: v = *dst + v; break;
        default: break;
    }
    *dst = v;
}

// BK: k depth per shared-memory stage (8 or 16); SEG2: the KB + AC lateral K segment is present.
template <int BK, bool SEG2>
__global__ void __launch_bounds__(256) k_gemm_simt128(GemmArgs a) {
    constexpr int NV = BK / 8;   // float4 loads per thread and operand per stage
    __shared__ __align__(16) float As[2][BK][BM2 + 4];
    __shared__ __align__(16) float Ws[2][BK][BN2 + 4];
    const int rows = a.p_rows ? *a.p_rows : a.rows_const;
    const int m0 = blockIdx.x * BM2;
    if (m0 >= rows) return;
    const int n0 = blockIdx.y * BN2;
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    // loader: 128 rows x BK k = 256 threads x NV float4 (row tid/2, k offset (tid&1) * BK/2)
    const int lr = tid >> 1, lk = (tid & 1) * (BK / 2);
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

    const int k_end = a.K + (SEG2 ? a.K2 : 0);
    float4 xv[NV], wv[NV];
    auto load = [&](int k0) {
        const bool second = SEG2 && k0 >= a.K;
        const float* X = second ? a.X2 : a.X;
        const float* W = second ? a.W2 : a.W;
        const int ldx = second ? a.ldx2 : a.ldx, ldw = second ? a.ldw2 : a.ldw;
        const int kk_end = second ? a.K2 : a.K;
        const int gm = m0 + lr, gn = n0 + lr;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int gk = (second ? k0 - a.K : k0) + lk + 4 * v;
            xv[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            wv[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (gm < rows && gk < kk_end) xv[v] = *reinterpret_cast<const float4*>(X + (int64_t)gm * ldx + gk);
            if (gn < a.N && gk < kk_end) wv[v] = __ldg(reinterpret_cast<const float4*>(W + (int64_t)gn * ldw + gk));
        }
    };
    auto stash = [&](int b) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int k = lk + 4 * v;
            As[b][k + 0][lr] = xv[v].x; As[b][k + 1][lr] = xv[v].y; As[b][k + 2][lr] = xv[v].z; As[b][k + 3][lr] = xv[v].w;
            Ws[b][k + 0][lr] = wv[v].x; Ws[b][k + 1][lr] = wv[v].y; Ws[b][k + 2][lr] = wv[v].z; Ws[b][k + 3][lr] = wv[v].w;
        }
    };
    load(0);
    stash(0);
    __syncthreads();
    int b = 0;
    for (int k0 = 0; k0 < k_end; k0 += BK) {
        const bool more = k0 + BK < k_end;
        if (more) load(k0 + BK);    // global loads in flight during this k-block's math
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[b][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[b][kk][ty * 4 + 64]);
            const float4 w0 = *reinterpret_cast<const float4*>(&Ws[b][kk][tx * 4]);
            const float4 w1 = *reinterpret_cast<const float4*>(&Ws[b][kk][tx * 4 + 64]);
            const float ar[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float wr[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(ar[i], wr[j], acc[i][j]);
        }
        if (more) {
            stash(b ^ 1);   // the other buffer: last read before the previous barrier
            __syncthreads();
            b ^= 1;
        }
    }

    if (a.epi == EPI_RESID_LN || a.epi == EPI_LN) {
        // whole 128-wide rows in this CTA: the 16 threads of a half-warp (same ty) hold one row's
        // 128 columns (8 each) -> two-pass mean / variance by 16-lane shuffles, as norm.cu
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int gm = m0 + ty * 4 + (i & 3) + (i >> 2) * 64;
            const bool valid = gm < rows;
            float v[8];
#pragma unroll
            for (int jh = 0; jh < 2; ++jh) {
                const int gn0 = tx * 4 + jh * 64;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                float* dst = a.Y + (int64_t)gm * a.ldy + gn0;
                if (valid && a.epi == EPI_RESID_LN) o = *reinterpret_cast<const float4*>(dst);
                const float b0 = a.bias ? __ldg(a.bias + gn0) : 0.f, b1 = a.bias ? __ldg(a.bias + gn0 + 1) : 0.f,
                            b2 = a.bias ? __ldg(a.bias + gn0 + 2) : 0.f, b3 = a.bias ? __ldg(a.bias + gn0 + 3) : 0.f;
                v[jh * 4 + 0] = o.x + (acc[i][jh * 4 + 0] + b0);
                v[jh * 4 + 1] = o.y + (acc[i][jh * 4 + 1] + b1);
                v[jh * 4 + 2] = o.z + (acc[i][jh * 4 + 2] + b2);
                v[jh * 4 + 3] = o.w + (acc[i][jh * 4 + 3] + b3);
                if (valid) *reinterpret_cast<float4*>(dst) = make_float4(v[jh * 4], v[jh * 4 + 1], v[jh * 4 + 2], v[jh * 4 + 3]);
            }
            float sm = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) sm += v[q];
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
            const float mean = sm * (1.0f / 128);
            float sq = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) { const float t = v[q] - mean; sq = fmaf(t, t, sq); }
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            const float rstd = rsqrtf(sq * (1.0f / 128) + a.ln_eps);
            if (valid) {
#pragma unroll
                for (int jh = 0; jh < 2; ++jh) {
                    const int c = tx * 4 + jh * 64;
                    float r[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) r[q] = (v[jh * 4 + q] - mean) * rstd * __ldg(a.ln_g + c + q) + __ldg(a.ln_b + c + q);
                    *reinterpret_cast<float4*>(a.Y2 + (int64_t)gm * a.ldy2 + c) = make_float4(r[0], r[1], r[2], r[3]);
                }
            }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int gm = m0 + ty * 4 + (i & 3) + (i >> 2) * 64;
        if (gm >= rows) continue;
        int cand = 0, token = 0;
        if (a.epi == EPI_SILU && a.drop.enabled) {
            cand = a.rows_are_cands ? gm : a.row_cand[gm];
            token = a.rows_are_cands ? 0 : gm - a.cu[cand];
        }
#pragma unroll
        for (int jh = 0; jh < 2; ++jh) {
            const int gn0 = n0 + tx * 4 + jh * 64;
            if (gn0 + 3 < a.N && !a.Ypre && (a.ldy & 3) == 0 && (reinterpret_cast<uintptr_t>(a.Y) & 15) == 0) {
                // 4 consecutive columns: one 128-bit load / store
                float v[4];
                const float4 bv = a.bias ? make_float4(__ldg(a.bias + gn0), __ldg(a.bias + gn0 + 1), __ldg(a.bias + gn0 + 2),
                                                       __ldg(a.bias + gn0 + 3))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                v[0] = acc[i][jh * 4 + 0] + bv.x; v[1] = acc[i][jh * 4 + 1] + bv.y;
                v[2] = acc[i][jh * 4 + 2] + bv.z; v[3] = acc[i][jh * 4 + 3] + bv.w;
                float4* dst = reinterpret_cast<float4*>(a.Y + (int64_t)gm * a.ldy + gn0);
                if (a.epi == EPI_RESID) {
                    const float4 o = *dst;
                    v[0] = o.x + v[0]; v[1] = o.y + v[1]; v[2] = o.z + v[2]; v[3] = o.w + v[3];
                } else if (a.epi == EPI_SILU) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[q] = silu(v[q]);
                    if (a.drop.enabled) {   // gn0 % 4 == 0: one Philox draw for the 4 units
                        const u32x4 wd = dropout_words(a.drop, gn0, token, a.site, cand);
                        v[0] = dropout_apply_word(a.drop, v[0], wd.x);
                        v[1] = dropout_apply_word(a.drop, v[1], wd.y);
                        v[2] = dropout_apply_word(a.drop, v[2], wd.z);
                        v[3] = dropout_apply_word(a.drop, v[3], wd.w);
                    }
                } else if (a.epi == EPI_SOFTPLUS) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[q] = softplus(v[q]);
                }
                *dst = make_float4(v[0], v[1], v[2], v[3]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int gn = gn0 + q;
                    if (gn < a.N) epi_store(a, gm, gn, acc[i][jh * 4 + q], cand, token);
                }
            }
        }
    }
}

void launch_gemm_simt(const GemmArgs& a, cudaStream_t s) {
    if (a.max_rows <= 0) return;
    const bool ln = a.epi == EPI_RESID_LN || a.epi == EPI_LN;
    if (ln && (a.N != 128 || a.wT || (a.K % 16) != 0 || (a.K2 % 16) != 0)) return;   // callers guarantee
    if (a.N >= 128 && !a.wT && (a.K % 16) == 0 && (a.K2 % 16) == 0) {
        dim3 grid2((a.max_rows + BM2 - 1) / BM2, (a.N + BN2 - 1) / BN2);
        if (a.K2 > 0) k_gemm_simt128<16, true><<<grid2, 256, 0, s>>>(a);
        else k_gemm_simt128<16, false><<<grid2, 256, 0, s>>>(a);
        return;
    }
    dim3 grid((a.max_rows + BM - 1) / BM, (a.N + BN - 1) / BN);
    k_gemm_simt<<<grid, 256, 0, s>>>(a);
}

}  // namespace tcl
