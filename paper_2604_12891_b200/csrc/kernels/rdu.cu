// rdu.cu -- RDU acquisition on the GPU: one selection round of
// PAPER.md Algorithm 1 (lines 16-31) with the diversity / uncertainty / total scores of Eqs. 1-3.
//
// Given the cost model's predictions for the unlabeled pool D_u and the labeled set D_l:
//   f^      = min-max normalised predictions over D_u u D_l ("normalized before being used")
//   d_s(i)  = min_{j in D_l} |f^_i - f^_j|                                   (Eq. 1; 1 if D_l empty)
//   mu      = (f^_i + S) / (M + 1),  S = sum_j f^_j                          (Eq. 2)
//   u_s(i)  = ((f^_i - mu)^2 + (Q - 2 mu S + M mu^2)) / (M + 1),  Q = sum_j f^_j^2   (Eq. 3)
//   t_s(i)  = f^_i d_s(i) + u_s(i)                                           (Alg. 1 line 24)
// then repeatedly take the argmax of t_s (ties: higher f^, then lower index), skipping
// operator types whose budget B_t * prob(op) is exhausted (lines 25-31), add the pick to D_l and
// update d_s, S, Q, M.  Reading R21: every score is evaluated in fp32 with the fixed
// operation order above (no contraction), so the CPU oracle takes the same integer decisions.
//
// One cooperative persistent kernel: the pool is spread over the CTAs' registers; each pick is a
// CTA-level argmax, one grid-wide barrier, and a redundant (identical) reduction of the per-CTA
// winners in every CTA -- no host round trip between picks.
#include <cooperative_groups.h>

#include <cmath>

#include "../kernels.h"

namespace cg = cooperative_groups;

namespace tcl {

namespace rdu {

constexpr int kThreads = 256;
constexpr int kMaxPer = 16;   // candidates per thread held in registers
constexpr int kMaxOps = 256;

struct Best { float ts, f; int64_t idx; };

__device__ __forceinline__ bool better(const Best& a, const Best& b) {  // a before b
    if (a.idx < 0) return false;
    if (b.idx < 0) return true;
    if (a.ts != b.ts) return a.ts > b.ts;
    if (a.f != b.f) return a.f > b.f;
    return a.idx < b.idx;
}

__device__ __forceinline__ Best warp_best(Best v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Best w;
        w.ts = __shfl_xor_sync(0xffffffffu, v.ts, o);
        w.f = __shfl_xor_sync(0xffffffffu, v.f, o);
        w.idx = __shfl_xor_sync(0xffffffffu, v.idx, o);
        if (better(w, v)) v = w;
    }
    return v;
}

// Eq. 2-3 + line 24 in fp32, fixed order, no contraction (must match oracle/tcl_oracle.c).
__device__ __forceinline__ float total_score(float fi, float ds, float S, float Q, float Mf) {
    const float m1 = __fadd_rn(Mf, 1.0f);
    const float mu = __fdiv_rn(__fadd_rn(fi, S), m1);
    const float a = __fsub_rn(fi, mu);
    const float a2 = __fmul_rn(a, a);
    const float t1 = __fmul_rn(mu, S);
    const float t2 = __fadd_rn(t1, t1);
    const float t3 = __fmul_rn(mu, mu);
    const float t4 = __fmul_rn(Mf, t3);
    const float b = __fadd_rn(__fsub_rn(Q, t2), t4);
    const float us = __fdiv_rn(__fadd_rn(a2, b), m1);
    return __fadd_rn(__fmul_rn(fi, ds), us);
}

__global__ void k_minmax_hist(const float* __restrict__ pool, int64_t n_pool, const float* __restrict__ lab,
                              int64_t n_lab, const int32_t* __restrict__ ops, int n_ops,
                              unsigned int* __restrict__ mm, unsigned long long* __restrict__ hist) {
    float lo = INFINITY, hi = -INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pool + n_lab;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float v = i < n_pool ? pool[i] : lab[i - n_pool];
        if (isfinite(v)) {  // only finite predictions take part (reading R21)
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
        }
        if (i < n_pool) {
            const int op = ops[i];
            if (op >= 0 && op < n_ops) atomicAdd(&hist[op], 1ull);
        }
    }
    // orderable-uint encoding for atomic min / max of floats
    auto ord = [](float f) { uint32_t b = __float_as_uint(f); return (b & 0x80000000u) ? ~b : (b | 0x80000000u); };
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], ord(lo));
        atomicMax(&mm[1], ord(hi));
    }
}

__device__ __forceinline__ float unord(uint32_t o) {
    const uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
    return __uint_as_float(b);
}

struct SelArgs {
    const float* pool; const int32_t* ops; int64_t n_pool;
    const float* lab; int64_t n_lab;
    int n_ops; int budget_total; int per;
    const unsigned int* mm; const unsigned long long* hist;
    float* keys;                 // [2][gridDim][3] per-CTA winners (ts, f, idx as float bits x2)
    int64_t* out; int32_t* n_out;
};

__global__ void __launch_bounds__(kThreads) k_rdu_select(SelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ float s_budget[kMaxOps];
    __shared__ int s_sel[kMaxOps];
    __shared__ Best s_warp[kThreads / 32];
    __shared__ float s_lab_stats[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float lo = unord(a.mm[0]), hi = unord(a.mm[1]);
    const bool flat = !(hi > lo);
    const float range = __fsub_rn(hi, lo);
    auto norm = [&](float v) { return flat ? 0.5f : __fdiv_rn(__fsub_rn(v, lo), range); };
    // per-op budgets B_t * count / n_pool (Alg. 1 lines 17-19), compared as selected < budget
    for (int op = tid; op < a.n_ops; op += kThreads) {
        s_budget[op] = (float)((double)a.budget_total * (double)a.hist[op] / (double)a.n_pool);
        s_sel[op] = 0;
    }
    // S, Q, M of the initial labeled set: sequential sums in index order (one thread, every CTA)
    if (tid == 0) {
        float S = 0.f, Q = 0.f, M = 0.f;
        for (int64_t j = 0; j < a.n_lab; ++j) {
            if (!isfinite(a.lab[j])) continue;
            const float f = norm(a.lab[j]);
            S = __fadd_rn(S, f);
            Q = __fadd_rn(Q, __fmul_rn(f, f));
            M = __fadd_rn(M, 1.0f);
        }
        s_lab_stats[0] = S;
        s_lab_stats[1] = Q;
        s_lab_stats[2] = M;
    }
    // this thread's candidates: i = (blockIdx * kThreads + tid) * per + k
    float fv[kMaxPer], dv[kMaxPer];
    int opv[kMaxPer];
    bool alive[kMaxPer];
    const int64_t base = ((int64_t)blockIdx.x * kThreads + tid) * a.per;
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
        const int64_t i = base + k;
        alive[k] = k < a.per && i < a.n_pool;
        if (alive[k] && !isfinite(a.pool[i])) alive[k] = false;
        fv[k] = alive[k] ? norm(a.pool[i]) : 0.f;
        opv[k] = alive[k] ? a.ops[i] : -1;
        float ds = INFINITY;
        if (alive[k])
            for (int64_t j = 0; j < a.n_lab; ++j)
                if (isfinite(a.lab[j])) ds = fminf(ds, fabsf(__fsub_rn(fv[k], norm(a.lab[j]))));
        dv[k] = ds == INFINITY ? 1.0f : ds;  // Eq. 1 with an empty labeled set: maximal novelty 1
        if (alive[k] && (opv[k] < 0 || opv[k] >= a.n_ops || !isfinite(fv[k]))) alive[k] = false;
    }
    __syncthreads();
    float S = s_lab_stats[0], Q = s_lab_stats[1];
    float Mf = s_lab_stats[2];
    int picks = 0;
    for (int p = 0; p < a.budget_total; ++p) {
        Best b{0.f, 0.f, -1};
#pragma unroll
        for (int k = 0; k < kMaxPer; ++k) {
            if (!alive[k] || !((float)s_sel[opv[k]] < s_budget[opv[k]])) continue;
            const Best c{total_score(fv[k], dv[k], S, Q, Mf), fv[k], base + k};
            if (better(c, b)) b = c;
        }
        b = warp_best(b);
        if (lane == 0) s_warp[warp] = b;
        __syncthreads();
        if (warp == 0) {
            Best w = lane < kThreads / 32 ? s_warp[lane] : Best{0.f, 0.f, -1};
            w = warp_best(w);
            if (lane == 0) {
                float* kp = a.keys + ((size_t)(p & 1) * gridDim.x + blockIdx.x) * 4;
                kp[0] = w.ts;
                kp[1] = w.f;
                reinterpret_cast<int64_t*>(kp)[1] = w.idx;
            }
        }
        grid.sync();
        // every CTA reduces the per-CTA winners in the same order -> the same global pick
        Best g{0.f, 0.f, -1};
        for (int c = lane; c < (int)gridDim.x; c += 32) {
            const float* kp = a.keys + ((size_t)(p & 1) * gridDim.x + c) * 4;
            const Best w{kp[0], kp[1], reinterpret_cast<const int64_t*>(kp)[1]};
            if (better(w, g)) g = w;
        }
        g = warp_best(g);  // all warps compute it (identical)
        if (g.idx < 0) break;
        const float fs = g.f;
        const int ops = a.ops[g.idx];
        if (tid == 0) s_sel[ops] += 1;
        S = __fadd_rn(S, fs);
        Q = __fadd_rn(Q, __fmul_rn(fs, fs));
        Mf = __fadd_rn(Mf, 1.0f);
#pragma unroll
        for (int k = 0; k < kMaxPer; ++k) {
            if (base + k == g.idx) alive[k] = false;
            dv[k] = fminf(dv[k], fabsf(__fsub_rn(fv[k], fs)));
        }
        if (blockIdx.x == 0 && tid == 0) a.out[p] = g.idx;
        ++picks;
        __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) *a.n_out = picks;
}

}  // namespace rdu

size_t rdu_scratch_bytes(int grid_max, int n_ops) {
    return 16 + (size_t)n_ops * 8 + (size_t)2 * grid_max * 16;
}

cudaError_t launch_rdu_select(const float* pool, const int32_t* ops, int64_t n_pool, const float* lab,
                              int64_t n_lab, int n_ops, int budget_total, int64_t* out, int32_t* n_out,
                              void* scratch, int num_sms, cudaStream_t s) {
    using namespace rdu;
    if (n_ops < 1 || n_ops > kMaxOps) return cudaErrorInvalidValue;
    const int64_t per_block_max = (int64_t)kThreads * kMaxPer;
    int grid = (int)std::min<int64_t>(num_sms, (n_pool + kThreads - 1) / kThreads);
    if (grid < 1) grid = 1;
    const int64_t per = (n_pool + (int64_t)grid * kThreads - 1) / ((int64_t)grid * kThreads);
    if (per > kMaxPer || n_pool > per_block_max * num_sms) return cudaErrorInvalidValue;
    uint8_t* sp = reinterpret_cast<uint8_t*>(scratch);
    unsigned int* mm = reinterpret_cast<unsigned int*>(sp);
    unsigned long long* hist = reinterpret_cast<unsigned long long*>(sp + 16);
    float* keys = reinterpret_cast<float*>(sp + 16 + (size_t)n_ops * 8);
    cudaError_t e = cudaMemsetAsync(mm, 0xFF, 4, s);   // running min (orderable encoding)
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(mm + 1, 0, 4, s)) != cudaSuccess) return e;   // running max
    if ((e = cudaMemsetAsync(hist, 0, (size_t)n_ops * 8, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(n_out, 0, sizeof(int32_t), s)) != cudaSuccess) return e;
    k_minmax_hist<<<std::max(1, std::min(1024, (int)((n_pool + n_lab + 255) / 256))), 256, 0, s>>>(
        pool, n_pool, lab, n_lab, ops, n_ops, mm, hist);
    SelArgs a{pool, ops, n_pool, lab, n_lab, n_ops, budget_total, (int)per, mm, hist, keys, out, n_out};
    void* args[] = {&a};
    e = cudaLaunchCooperativeKernel((void*)k_rdu_select, dim3(grid), dim3(kThreads), args, 0, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace tcl
