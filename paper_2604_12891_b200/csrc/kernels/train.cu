// train.cu -- training-side kernels of the fp32 path (reading R24):
// the LambdaRank loss and its score gradient (Eq. 6), the backward pass of every layer
// of the cost model (encoder, pre-norm, in_proj, causal conv + SiLU, x_proj / dt_proj + softplus,
// the selective scan with ZOH, gate, out_proj, final norm + masked mean, decoder) and Adam.
//
// Design: the forward that precedes these saves every activation the backward needs (per layer:
// the block input, LN output, [x|z], u, [dt_r|B|C], Delta, the scan states after every step, the
// gated output); the backward is a chain of row-parallel kernels plus weight-gradient reductions
// dW = dY^T X computed as split-row partial tiles reduced in a fixed order (deterministic).
#include <algorithm>
#include <cmath>

#include "../kernels.h"

namespace tcl {

namespace trn {

__device__ __forceinline__ float sigm(float v) { return 1.0f / (1.0f + expf(-v)); }
// d SiLU(v) / dv = s (1 + v (1 - s)), s = sigmoid(v)
__device__ __forceinline__ float dsilu(float v) {
    const float s = sigm(v);
    return s * (1.0f + v * (1.0f - s));
}

// ---------------------------------------------------------------- weight gradients
// part[split][j][k] = sum over this split's rows m of dY[m][j] * X[m][k]
constexpr int WB = 64, WK = 16;
__global__ void __launch_bounds__(256) k_wgrad(const float* __restrict__ dY, int lddy, const float* __restrict__ X,
                                               int ldx, int Nout, int K, const int32_t* __restrict__ p_rows,
                                               int rows_const, int rows_per_split, float* __restrict__ part) {
    __shared__ float Ys[WK][WB + 4];
    __shared__ float Xs[WK][WB + 4];
    const int rows = p_rows ? *p_rows : rows_const;
    const int j0 = blockIdx.x * WB, k0 = blockIdx.y * WB;
    const int m_begin = blockIdx.z * rows_per_split;
    const int m_end = min(rows, m_begin + rows_per_split);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    float acc[4][4] = {};
    for (int m0 = m_begin; m0 < m_end; m0 += WK) {
        for (int e = tid; e < WK * WB; e += 256) {
            const int mm = e / WB, c = e - mm * WB;
            const int m = m0 + mm;
            Ys[mm][c] = (m < m_end && j0 + c < Nout) ? dY[(int64_t)m * lddy + j0 + c] : 0.0f;
            Xs[mm][c] = (m < m_end && k0 + c < K) ? X[(int64_t)m * ldx + k0 + c] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int mm = 0; mm < WK; ++mm) {
            float yv[4], xv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { yv[i] = Ys[mm][ty * 4 + i]; xv[i] = Xs[mm][tx * 4 + i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(yv[i], xv[q], acc[i][q]);
        }
        __syncthreads();
    }
    float* out = part + (size_t)blockIdx.z * Nout * K;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int j = j0 + ty * 4 + i;
        if (j >= Nout) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = k0 + tx * 4 + q;
            if (k < K) out[(size_t)j * K + k] = acc[i][q];
        }
    }
}

// out[j * ldo + k] = sum_split part[split][j][k]   (fixed order)
__global__ void k_reduce_parts(const float* __restrict__ part, int splits, int Nout, int K, float* __restrict__ out,
                               int ldo) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)Nout * K) return;
    const int j = (int)(e / K), k = (int)(e - (int64_t)j * K);
    // loads are independent of the (in-order) additions: unrolled so the L2 latencies overlap
    float s = 0.0f;
    int p = 0;
    for (; p + 8 <= splits; p += 8) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = part[(size_t)(p + q) * Nout * K + e];
#pragma unroll
        for (int q = 0; q < 8; ++q) s += v[q];
    }
    for (; p < splits; ++p) s += part[(size_t)p * Nout * K + e];
    out[(size_t)j * ldo + k] = s;
}

// part[split][j] = sum over the split's rows of dY[m][j]
__global__ void k_colsum(const float* __restrict__ dY, int lddy, int Ncol, const int32_t* __restrict__ p_rows,
                         int rows_const, int rows_per_split, float* __restrict__ part) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= Ncol) return;
    const int rows = p_rows ? *p_rows : rows_const;
    const int m_begin = blockIdx.y * rows_per_split;
    const int m_end = min(rows, m_begin + rows_per_split);
    float s = 0.0f;
    int m = m_begin;
    for (; m + 8 <= m_end; m += 8) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = dY[(int64_t)(m + q) * lddy + j];
#pragma unroll
        for (int q = 0; q < 8; ++q) s += v[q];
    }
    for (; m < m_end; ++m) s += dY[(int64_t)m * lddy + j];
    part[(size_t)blockIdx.y * Ncol + j] = s;
}

// ---------------------------------------------------------------- elementwise
// dPre[m][j] = dPost[m][j] * SiLU'(pre[m][j])   (in place allowed: dPre == dPost)
__global__ void k_silu_bwd(const float* dPost, int ldp, const float* __restrict__ pre, int ldpre, float* dPre,
                           int ldo, int Ncol, const int32_t* __restrict__ p_rows, int rows_const) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int rows = p_rows ? *p_rows : rows_const;
    const int64_t m = e / Ncol;
    const int j = (int)(e - m * Ncol);
    if (m >= rows) return;
    dPre[m * ldo + j] = dPost[m * ldp + j] * dsilu(pre[m * ldpre + j]);
}

// decoder output layer (N = 1): dPre2[c][j] = ds[c] * W3[j] * SiLU'(pre2[c][j])
__global__ void k_dec_out_bwd(const float* __restrict__ ds, const float* __restrict__ W3, const float* __restrict__ pre2,
                              int h2, int64_t n, float* __restrict__ dpre2) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * h2) return;
    const int64_t c = e / h2;
    const int j = (int)(e - c * h2);
    dpre2[e] = ds[c] * __ldg(W3 + j) * dsilu(pre2[e]);
}

// ---------------------------------------------------------------- LayerNorm backward
// Row m: x = H[m], y = LN(x) g + b, dY given (or, pool mode, dY[m][c] = dpooled[cand][c] / T).
// dx = rstd (dxh - mean(dxh) - xh mean(dxh xh)), dxh = dY g.  dH[m] = (accumulate ? dH[m] : 0) + dx;
// also writes xhdy[m][c] = dY xh (for the gamma gradient) and, in pool mode, dYout[m][c] = dY.
template <int PER>
__global__ void __launch_bounds__(256) k_ln_bwd(const float* __restrict__ H, int dm, const float* __restrict__ g,
                                                float eps, const float* __restrict__ dY,
                                                const float* __restrict__ dpooled, const int32_t* __restrict__ row_cand,
                                                const int32_t* __restrict__ lens, float* __restrict__ dYout,
                                                float* __restrict__ dH, int accumulate, float* __restrict__ xhdy,
                                                const int32_t* __restrict__ p_rows) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= *p_rows) return;
    float v[PER], dy[PER];
    float invT = 0.f;
    int cand = 0;
    if (dpooled) {
        cand = row_cand[row];
        invT = 1.0f / (float)lens[cand];
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        v[j] = H[(int64_t)row * dm + c];
        dy[j] = dpooled ? dpooled[(int64_t)cand * dm + c] * invT : dY[(int64_t)row * dm + c];
        if (dYout) dYout[(int64_t)row * dm + c] = dy[j];
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) s += v[j];
    const float mean = warp_sum(s) / dm;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) { const float t = v[j] - mean; q = fmaf(t, t, q); }
    const float rstd = 1.0f / sqrtf(warp_sum(q) / dm + eps);
    float xh[PER], dxh[PER], s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        xh[j] = (v[j] - mean) * rstd;
        dxh[j] = dy[j] * __ldg(g + c);
        s1 += dxh[j];
        s2 = fmaf(dxh[j], xh[j], s2);
        xhdy[(int64_t)row * dm + c] = dy[j] * xh[j];
    }
    const float m1 = warp_sum(s1) / dm, m2 = warp_sum(s2) / dm;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        const float dx = rstd * (dxh[j] - m1 - xh[j] * m2);
        float* dst = dH + (int64_t)row * dm + c;
        *dst = accumulate ? *dst + dx : dx;
    }
}

// ---------------------------------------------------------------- conv backward
// dpre[row][d] = dU[row][d] * SiLU'(pre), pre = b + sum_k w[d][k] x[t-(dc-1)+k]
__global__ void k_conv_pre_bwd(const float* __restrict__ X, int ldx, const float* __restrict__ w,
                               const float* __restrict__ b, int di, int dc, const float* __restrict__ dU,
                               float* __restrict__ dpre, const int32_t* __restrict__ row_cand,
                               const int32_t* __restrict__ cu, const int32_t* __restrict__ p_rows) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = idx / di;
    const int d = (int)(idx - row * di);
    if (row >= *p_rows) return;
    const int t = (int)(row - cu[row_cand[row]]);
    float acc = __ldg(b + d);
    for (int k = 0; k < dc; ++k) {
        const int back = dc - 1 - k;
        if (t >= back) acc = fmaf(__ldg(w + d * dc + k), X[(row - back) * ldx + d], acc);
    }
    dpre[row * di + d] = dU[row * di + d] * dsilu(acc);
}

// dX[row][d] = sum_k w[d][k] dpre[row + (dc-1-k)][d] over rows of the same candidate
__global__ void k_conv_dx(const float* __restrict__ dpre, const float* __restrict__ w, int di, int dc,
                          float* __restrict__ dX, int lddx, const int32_t* __restrict__ row_cand,
                          const int32_t* __restrict__ cu, const int32_t* __restrict__ lens,
                          const int32_t* __restrict__ p_rows) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = idx / di;
    const int d = (int)(idx - row * di);
    if (row >= *p_rows) return;
    const int cand = row_cand[row];
    const int t = (int)(row - cu[cand]);
    const int T = lens[cand];
    float acc = 0.0f;
    for (int k = 0; k < dc; ++k) {
        const int fwd = dc - 1 - k;
        if (t + fwd < T) acc = fmaf(__ldg(w + d * dc + k), dpre[(row + fwd) * di + d], acc);
    }
    dX[row * lddx + d] = acc;
}

// part[split][d][k] = sum_rows dpre[row][d] x[row-(dc-1-k)][d] (t >= dc-1-k); part[split][d][dc] = sum dpre
__global__ void k_conv_wgrad(const float* __restrict__ dpre, const float* __restrict__ X, int ldx, int di, int dc,
                             const int32_t* __restrict__ row_cand, const int32_t* __restrict__ cu,
                             const int32_t* __restrict__ p_rows, int rows_per_split, float* __restrict__ part) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= di) return;
    const int rows = *p_rows;
    const int m_begin = blockIdx.y * rows_per_split, m_end = min(rows, m_begin + rows_per_split);
    float acc[9] = {};
#pragma unroll 4
    for (int row = m_begin; row < m_end; ++row) {
        const float g = dpre[(int64_t)row * di + d];
        const int t = row - cu[row_cand[row]];
        for (int k = 0; k < dc; ++k) {
            const int back = dc - 1 - k;
            if (t >= back) acc[k] = fmaf(g, X[(int64_t)(row - back) * ldx + d], acc[k]);
        }
        acc[dc] += g;
    }
    float* out = part + ((size_t)blockIdx.y * di + d) * (dc + 1);
    for (int k = 0; k <= dc; ++k) out[k] = acc[k];
}

// part [splits][di][dc+1] -> dw [di][dc], db [di]
__global__ void k_conv_reduce(const float* __restrict__ part, int splits, int di, int dc, float* __restrict__ dw,
                              float* __restrict__ db) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= di * (dc + 1)) return;
    const int d = e / (dc + 1), k = e - d * (dc + 1);
    float s = 0.0f;
    for (int p = 0; p < splits; ++p) s += part[(size_t)p * di * (dc + 1) + e];
    if (k < dc) dw[d * dc + k] = s;
    else db[d] = s;
}

// ---------------------------------------------------------------- selective scan backward
// One block per candidate, one thread per channel d (blockDim = di).  Reverse time with the state
// adjoint ds in registers; s_t read back from the forward's saved states.  Writes dz (gate), du
// (scan input; x_proj's contribution is added later), dDelta_pre (softplus folded in), dB and dC
// (block reductions over channels), and per-candidate partials of dA_log and dD.
template <int N, int DISC>
__global__ void k_scan_bwd(ScanBwdArgs a) {
    extern __shared__ float sm[];  // sBC [T][2N] | red [di/32][2N]
    const int64_t i = blockIdx.x;
    const int d = threadIdx.x;
    const int T = a.lens[i];
    if (T < 1 || T > a.max_len) return;
    const int64_t base = a.cu[i];
    float* sBC = sm;
    float* red = sm + a.max_len * 2 * N;
    for (int idx = threadIdx.x; idx < T * 2 * N; idx += blockDim.x) {
        const int t = idx / (2 * N), j = idx - t * 2 * N;
        sBC[idx] = a.BC[(base + t) * a.ldbc + (j < N ? a.b_off + j : a.c_off + j - N)];
    }
    __syncthreads();
    const int di = a.di, lane = d & 31, warp = d >> 5, nwarps = blockDim.x >> 5;
    float A[N], ds[N], dA[N];
#pragma unroll
    for (int n = 0; n < N; ++n) {
        A[n] = -expf(__ldg(a.A_log + d * N + n));
        ds[n] = 0.0f;
        dA[n] = 0.0f;
    }
    const float Dv = __ldg(a.Dv + d);
    float dD = 0.0f;
    for (int t = T - 1; t >= 0; --t) {
        const int64_t row = base + t;
        const float u = a.U[row * di + d];
        const float dl = a.Delta[row * di + d];
        const float z = a.Z[row * a.ldz + d];
        const float dg = a.dG[row * di + d];
        const float* Bt = sBC + t * 2 * N;
        const float* Ct = Bt + N;
        const float* st = a.S + (row * di + d) * N;
        const float* sp = t > 0 ? a.S + ((row - 1) * di + d) * N : nullptr;
        float y = Dv * u;
#pragma unroll
        for (int n = 0; n < N; ++n) y = fmaf(Ct[n], st[n], y);
        // gate g = y SiLU(z)
        const float sz = z * sigm(z);
        const float dy = dg * sz;
        a.dZ[row * a.lddz + d] = dg * y * dsilu(z);
        dD = fmaf(dy, u, dD);
        float du = dy * Dv, ddl = 0.0f;
        float pB[N], pC[N];
#pragma unroll
        for (int n = 0; n < N; ++n) {
            ds[n] = fmaf(dy, Ct[n], ds[n]);
            pC[n] = dy * st[n];
            const float x = dl * A[n];
            const float Ab = expf(x);
            const float sprev = sp ? sp[n] : 0.0f;
            const float dAb = ds[n] * sprev;
            const float dBb = ds[n] * u;
            float coef, dcoef_dA, dBb_ddl;
            if (DISC == 0) {   // ZOH: Bbar = (e^x - 1) / A * B
                const float em1 = expm1f(x);
                coef = em1 / A[n];
                // d coef / dA = (x e^x - expm1(x)) / A^2; series for small |x| (cancellation)
                float h;
                if (fabsf(x) < 0.1f)
                    h = x * x *
                        fmaf(x, fmaf(x, fmaf(x, fmaf(x, fmaf(x, 1.0f / 840, 1.0f / 144), 1.0f / 30), 1.0f / 8), 1.0f / 3),
                             0.5f);
                else
                    h = x * Ab - em1;
                dcoef_dA = h / (A[n] * A[n]);
                dBb_ddl = Ab * Bt[n];
            } else {           // Euler-B: Bbar = Delta B
                coef = dl;
                dcoef_dA = 0.0f;
                dBb_ddl = Bt[n];
            }
            du = fmaf(ds[n], coef * Bt[n], du);
            pB[n] = dBb * coef;
            ddl = fmaf(dAb, A[n] * Ab, ddl);
            ddl = fmaf(dBb, dBb_ddl, ddl);
            dA[n] = fmaf(dAb, dl * Ab, dA[n]);
            dA[n] = fmaf(dBb * Bt[n], dcoef_dA, dA[n]);
            ds[n] *= Ab;   // adjoint carried to t - 1
        }
        a.dU[row * di + d] = du;
        a.dDpre[row * di + d] = ddl * (-expm1f(-dl));   // softplus'(v) = sigmoid(v) = 1 - e^{-Delta}
        // dB[t][n], dC[t][n] = sums over the di channels
#pragma unroll
        for (int n = 0; n < N; ++n) {
            const float b = warp_sum(pB[n]);
            const float c = warp_sum(pC[n]);
            if (lane == 0) {
                red[warp * 2 * N + n] = b;
                red[warp * 2 * N + N + n] = c;
            }
        }
        __syncthreads();
        if (d < 2 * N) {
            float s = 0.0f;
            for (int w = 0; w < nwarps; ++w) s += red[w * 2 * N + d];
            a.dBC[row * a.ldbc + (d < N ? a.b_off + d : a.c_off + d - N)] = s;
        }
        __syncthreads();
    }
    // per-candidate partials: dA_log = dA * A (A = -exp(A_log)), dD
#pragma unroll
    for (int n = 0; n < N; ++n) a.dAlog_part[(i * di + d) * N + n] = dA[n] * A[n];
    a.dD_part[i * di + d] = dD;
}

// ---------------------------------------------------------------- LambdaRank (Eq. 6)
// One block per group (<= 4096 members, shared memory).  Ranks by (score desc, index asc) via
// bitonic sort of u64 keys; ideal DCG from the relevance sorted descending; dL/ds_i and the
// group's loss from all ordered pairs with y_i > y_j.  Group results are divided by n_groups.
__device__ __forceinline__ unsigned long long score_key(float s, uint32_t j) {
    uint32_t b = __float_as_uint(s != s ? -INFINITY : s);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((unsigned long long)b << 32) | (0xFFFFFFFFu - j);
}

__device__ void bitonic_desc(unsigned long long* keys, int P) {
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
                const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const unsigned long long x = keys[lo], y = keys[hi];
                if (desc ? (x < y) : (x > y)) { keys[lo] = y; keys[hi] = x; }
            }
            __syncthreads();
        }
}

__device__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float s = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];   // fixed order
    return s;
}

__global__ void __launch_bounds__(1024) k_lambdarank(const float* __restrict__ scores, const float* __restrict__ lat,
                                                     const int64_t* __restrict__ off, int64_t n_groups, int max_group,
                                                     int64_t n_total, float sigma, float* __restrict__ dscores,
                                                     float* __restrict__ gloss, int* __restrict__ err) {
    extern __shared__ unsigned long long keys[];   // [P]
    __shared__ float red[32];
    const int64_t g = blockIdx.x;
    const int64_t o = off[g];
    const int64_t n64 = off[g + 1] - o;
    // shared memory is sized for max_group on the host: a group outside [1, max_group] or outside
    // [0, n_total) is skipped (loss term 0, its candidates keep the zero gradient set by the
    // launcher) and raises ERR_TASK (tcl_sync_error -> TCL_ESHAPE)
    if (n64 < 1 || n64 > max_group || o < 0 || o + n64 > n_total) {
        if (threadIdx.x == 0) {
            gloss[g] = 0.0f;
            atomicOr(err, ERR_TASK);
        }
        return;
    }
    const int n = (int)n64;
    int P = 1;
    while (P < n) P <<= 1;
    float* ys = reinterpret_cast<float*>(keys + P);    // [n] relevance
    float* G = ys + P;                                  // [n] gain / maxDCG
    float* invD = G + P;                                // [n] 1 / log2(1 + rank)
    float* sc = invD + P;                               // [n] scores
    // relevance y_i = min latency / latency_i
    float mn = INFINITY;
    for (int j = threadIdx.x; j < n; j += blockDim.x) mn = fminf(mn, lat[o + j]);
    for (int s_ = 16; s_ > 0; s_ >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, s_));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
    __syncthreads();
    mn = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mn = fminf(mn, red[w]);
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        ys[j] = mn / lat[o + j];
        sc[j] = scores[o + j];
    }
    // ideal ordering: keys on relevance (desc); gains 2^y - 1 are monotone in y
    for (int j = threadIdx.x; j < P; j += blockDim.x) keys[j] = j < n ? score_key(ys[j], (uint32_t)j) : 0ull;
    __syncthreads();
    bitonic_desc(keys, P);
    float part = 0.0f;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const int j = (int)(0xFFFFFFFFu - (uint32_t)(keys[r] & 0xFFFFFFFFull));
        part += (exp2f(ys[j]) - 1.0f) / log2f((float)r + 2.0f);
    }
    const float max_dcg = block_sum(part, red);
    __syncthreads();
    // predicted ranking
    for (int j = threadIdx.x; j < P; j += blockDim.x) keys[j] = j < n ? score_key(sc[j], (uint32_t)j) : 0ull;
    __syncthreads();
    bitonic_desc(keys, P);
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const int j = (int)(0xFFFFFFFFu - (uint32_t)(keys[r] & 0xFFFFFFFFull));
        invD[j] = 1.0f / log2f((float)r + 2.0f);
        G[j] = (exp2f(ys[j]) - 1.0f) / max_dcg;
    }
    __syncthreads();
    const float inv_groups = 1.0f / (float)n_groups;
    const float kInvLn2 = 1.4426950408889634f;
    float lsum = 0.0f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        float gi = 0.0f;
        for (int j = 0; j < n; ++j) {
            if (ys[i] == ys[j]) continue;
            const bool hi = ys[i] > ys[j];
            const float dndcg = fabsf(G[i] - G[j]) * fabsf(invD[i] - invD[j]);
            const float x = hi ? sigma * (sc[i] - sc[j]) : sigma * (sc[j] - sc[i]);   // s_high - s_low
            // pair term dndcg * log2(1 + e^{-x}); d/ds_high = -dndcg sigma sigmoid(-x) / ln 2
            const float lam = dndcg * sigma * kInvLn2 * sigm(-x);
            gi += hi ? -lam : lam;
            if (hi) lsum += dndcg * kInvLn2 * (fmaxf(-x, 0.0f) + log1pf(expf(-fabsf(x))));
        }
        dscores[o + i] = gi * inv_groups;
    }
    const float L = block_sum(lsum, red);
    if (threadIdx.x == 0) gloss[g] = L;
}

__global__ void k_loss_mean(const float* __restrict__ gloss, int64_t n_groups, float* __restrict__ loss) {
    __shared__ float red[32];
    float s = 0.0f;
    for (int64_t g = threadIdx.x; g < n_groups; g += blockDim.x) s += gloss[g];
    s = block_sum(s, red);
    if (threadIdx.x == 0) *loss = s / (float)n_groups;
}

// ---------------------------------------------------------------- Adam + derived weights
// step counter and bias corrections live on the device, so a captured step graph replays correctly
__global__ void k_adam_count(int* __restrict__ step, float b1, float b2, float* __restrict__ corr) {
    const int t = ++*step;
    corr[0] = 1.0f - powf(b1, (float)t);
    corr[1] = 1.0f - powf(b2, (float)t);
}

__global__ void k_adam(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                       int64_t n, float lr, float b1, float b2, float eps, const float* __restrict__ corr) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const float c1 = corr[0], c2 = corr[1];
    const float gg = g[e];
    const float mm = b1 * m[e] + (1.0f - b1) * gg;
    const float vv = b2 * v[e] + (1.0f - b2) * gg * gg;
    m[e] = mm;
    v[e] = vv;
    w[e] -= lr * (mm / c1) / (sqrtf(vv / c2) + eps);
}

// W1p [e1][ldp] <- W1 [e1][d_in] (zero-padded)
__global__ void k_refresh_w1(const float* __restrict__ W1, int e1, int d_in, int ldp, float* __restrict__ W1p) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e1 * ldp) return;
    const int o = e / ldp, i = e - o * ldp;
    W1p[e] = i < d_in ? W1[o * d_in + i] : 0.0f;
}
// A2 = -exp(A_log) log2(e); invA = 1 / A  (as at model creation, in double)
__global__ void k_refresh_a(const float* __restrict__ alog, int diN, float* __restrict__ A2, float* __restrict__ invA) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= diN) return;
    const double A = -exp((double)alog[e]);
    A2[e] = (float)(A * 1.4426950408889634);
    invA[e] = (float)(1.0 / A);
}

}  // namespace trn

// ---------------------------------------------------------------- launchers
static int splits_for(int tiles, int rows) {
    int s = (2 * 148 + tiles - 1) / tiles;
    s = std::max(1, std::min(s, (rows + 63) / 64));
    return s;
}

void launch_wgrad(const float* dY, int lddy, const float* X, int ldx, int Nout, int K, const int32_t* p_rows,
                  int max_rows, float* part, size_t part_cap, float* out, int ldo, cudaStream_t s) {
    const int tj = (Nout + trn::WB - 1) / trn::WB, tk = (K + trn::WB - 1) / trn::WB;
    int splits = splits_for(tj * tk, max_rows);
    while (splits > 1 && (size_t)splits * Nout * K > part_cap) --splits;
    const int rps = ((max_rows + splits - 1) / splits + trn::WK - 1) / trn::WK * trn::WK;
    splits = std::max(1, (max_rows + rps - 1) / rps);
    trn::k_wgrad<<<dim3(tj, tk, splits), 256, 0, s>>>(dY, lddy, X, ldx, Nout, K, p_rows, max_rows, rps, part);
    const int64_t tot = (int64_t)Nout * K;
    trn::k_reduce_parts<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(part, splits, Nout, K, out, ldo);
}

void launch_colsum(const float* dY, int lddy, int Ncol, const int32_t* p_rows, int max_rows, float* part,
                   size_t part_cap, float* out, cudaStream_t s) {
    const int tj = (Ncol + 127) / 128;
    int splits = std::max(1, std::min((2 * 148 + tj - 1) / tj, (max_rows + 31) / 32));
    while (splits > 1 && (size_t)splits * Ncol > part_cap) --splits;
    const int rps = (max_rows + splits - 1) / splits;
    splits = std::max(1, (max_rows + rps - 1) / std::max(1, rps));
    trn::k_colsum<<<dim3(tj, splits), 128, 0, s>>>(dY, lddy, Ncol, p_rows, max_rows, std::max(1, rps), part);
    trn::k_reduce_parts<<<(Ncol + 255) / 256, 256, 0, s>>>(part, splits, 1, Ncol, out, Ncol);
}

void launch_silu_bwd(const float* dPost, int ldp, const float* pre, int ldpre, float* dPre, int ldo, int Ncol,
                     const int32_t* p_rows, int max_rows, cudaStream_t s) {
    const int64_t tot = (int64_t)max_rows * Ncol;
    if (tot == 0) return;
    trn::k_silu_bwd<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(dPost, ldp, pre, ldpre, dPre, ldo, Ncol, p_rows,
                                                                   max_rows);
}

void launch_dec_out_bwd(const float* ds, const float* W3, const float* pre2, int h2, int64_t n, float* dpre2,
                        cudaStream_t s) {
    const int64_t tot = n * h2;
    trn::k_dec_out_bwd<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(ds, W3, pre2, h2, n, dpre2);
}

void launch_ln_bwd(const float* H, int dm, const float* g, float eps, const float* dY, const float* dpooled,
                   const int32_t* row_cand, const int32_t* lens, float* dYout, float* dH, int accumulate,
                   float* xhdy, int max_rows, const int32_t* p_rows, cudaStream_t s) {
    dim3 grid((max_rows + 7) / 8);
#define LNB(P) trn::k_ln_bwd<P><<<grid, 256, 0, s>>>(H, dm, g, eps, dY, dpooled, row_cand, lens, dYout, dH, accumulate, xhdy, p_rows)
    switch (dm / 32) {
        case 1: LNB(1); break; case 2: LNB(2); break; case 3: LNB(3); break; case 4: LNB(4); break;
        case 5: LNB(5); break; case 6: LNB(6); break; case 7: LNB(7); break; case 8: LNB(8); break;
        default: break;
    }
#undef LNB
}

void launch_conv_bwd(const float* X, int ldx, const float* w, const float* b, int di, int dc, const float* dU,
                     float* dpre, float* dX, int lddx, const int32_t* row_cand, const int32_t* cu,
                     const int32_t* lens, const int32_t* p_rows, int max_rows, float* part, size_t part_cap,
                     float* dw, float* db, cudaStream_t s) {
    const int64_t tot = (int64_t)max_rows * di;
    if (tot == 0) return;
    trn::k_conv_pre_bwd<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(X, ldx, w, b, di, dc, dU, dpre, row_cand, cu,
                                                                        p_rows);
    trn::k_conv_dx<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(dpre, w, di, dc, dX, lddx, row_cand, cu, lens, p_rows);
    const int tb = (di + 127) / 128;
    int splits = std::max(1, std::min((2 * 148 + tb - 1) / tb, (max_rows + 63) / 64));
    while (splits > 1 && (size_t)splits * di * (dc + 1) > part_cap) --splits;
    const int rps = (max_rows + splits - 1) / splits;
    trn::k_conv_wgrad<<<dim3(tb, splits), 128, 0, s>>>(dpre, X, ldx, di, dc, row_cand, cu, p_rows, rps, part);
    trn::k_conv_reduce<<<(di * (dc + 1) + 255) / 256, 256, 0, s>>>(part, splits, di, dc, dw, db);
}

void launch_scan_bwd(const ScanBwdArgs& a, cudaStream_t s) {
    if (a.n == 0) return;
    const size_t smem = ((size_t)a.max_len * 2 * a.N + (size_t)(a.di / 32) * 2 * a.N) * sizeof(float);
    dim3 grid((unsigned)a.n);
    if (a.N == 8) {
        if (a.disc == 1) trn::k_scan_bwd<8, 1><<<grid, a.di, smem, s>>>(a);
        else trn::k_scan_bwd<8, 0><<<grid, a.di, smem, s>>>(a);
    } else {
        if (a.disc == 1) trn::k_scan_bwd<16, 1><<<grid, a.di, smem, s>>>(a);
        else trn::k_scan_bwd<16, 0><<<grid, a.di, smem, s>>>(a);
    }
}

cudaError_t launch_lambdarank(const float* scores, const float* lat, const int64_t* off, int64_t n_groups,
                              int max_group, int64_t n_total, float sigma, float* dscores, float* gloss, float* loss,
                              int* err, cudaStream_t s) {
    int P = 1;
    while (P < max_group) P <<= 1;
    const size_t smem = (size_t)P * 8 + (size_t)P * 4 * 4;
    // opted in once per device for the largest group (4096): the first (direct) step does it, so a
    // graph capture never needs to
    cudaError_t e = prepare_kernel(trn::k_lambdarank, 4096 * (8 + 16));
    if (e != cudaSuccess) return e;
    // candidates outside every group get dL/ds = 0 (not stale values)
    if ((e = cudaMemsetAsync(dscores, 0, sizeof(float) * (size_t)n_total, s)) != cudaSuccess) return e;
    trn::k_lambdarank<<<(unsigned)n_groups, 1024, smem, s>>>(scores, lat, off, n_groups, max_group, n_total, sigma,
                                                             dscores, gloss, err);
    trn::k_loss_mean<<<1, 1024, 0, s>>>(gloss, n_groups, loss);
    return cudaGetLastError();
}

void launch_adam(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
                 int* step_dev, float* corr_dev, cudaStream_t s) {
    trn::k_adam_count<<<1, 1, 0, s>>>(step_dev, b1, b2, corr_dev);
    trn::k_adam<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w, g, m, v, n, lr, b1, b2, eps, corr_dev);
}

void launch_refresh_w1(const float* W1, int e1, int d_in, int ldp, float* W1p, cudaStream_t s) {
    trn::k_refresh_w1<<<(e1 * ldp + 255) / 256, 256, 0, s>>>(W1, e1, d_in, ldp, W1p);
}

void launch_refresh_a(const float* alog, int diN, float* A2, float* invA, cudaStream_t s) {
    trn::k_refresh_a<<<(diN + 255) / 256, 256, 0, s>>>(alog, diN, A2, invA);
}

}  // namespace tcl
