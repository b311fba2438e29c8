// rdu.cu -- RDU acquisition on the GPU: one selection round of
// PAPER.md Algorithm 1 (lines 16-31) with the diversity / uncertainty / total scores of Eqs. 1-3.
//
// Given the cost model's predictions for the unlabeled pool D_u and the labeled set D_l:
//   f^      = min-max normalised predictions over D_u u D_l ("normalized before being used")
//   d_s(i)  = min_{j in D_l} |f^_i - f^_j|                                   (Eq. 1; 1 if D_l empty)
//   mu      = (f^_i + S) r,  S = sum_j f^_j,  r = 1 / (M + 1)                (Eq. 2)
//   u_s(i)  = ((f^_i - mu)^2 + (Q - 2 mu S + M mu^2)) r,  Q = sum_j f^_j^2   (Eq. 3)
//   t_s(i)  = f^_i d_s(i) + u_s(i)                                           (Alg. 1 line 24)
// then repeatedly take the argmax of t_s (ties: higher f^, then lower index), skipping
// operator types whose budget B_t * prob(op) is exhausted (lines 25-31), add the pick to D_l and
// update d_s, S, Q, M.  Reading R21: every score is evaluated in fp32 with the fixed
// operation order above (no contraction; r is one IEEE division per pick), so the CPU oracle
// takes the same integer decisions.
//
// Two kernels, no host round trip between picks:
//  * k_rdu_cluster (n_pool <= 32768): a thread-block cluster of C <= 8 CTAs x 1024 threads,
//    each CTA holding its slice (f^, d_s, op) in shared memory.  A pick = CTA argmax (warp
//    shuffles + shared memory), one cluster barrier, and every CTA reducing the C per-CTA winners
//    read over DSMEM (double-buffered slots: one cluster barrier per pick).
//  * k_rdu_select (larger pools, up to 16 x 256 x SMs): the same protocol over a cooperative grid,
//    candidates in registers, one grid-wide barrier per pick.
#include <cooperative_groups.h>

#include <cmath>

#include "../kernels.h"

namespace cg = cooperative_groups;

namespace tcl {

namespace rdu {

constexpr int kThreads = 256;     // cooperative kernel
constexpr int kMaxPer = 16;       // candidates per thread (registers / shared memory)
constexpr int kMaxOps = 256;
constexpr int kCThreads = 1024;   // cluster kernel
constexpr int kPerCta = kCThreads * kMaxPer;   // 16384 candidates per CTA
constexpr int kMaxCluster = 8;

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
__device__ __forceinline__ float total_score(float fi, float ds, float S, float Q, float Mf, float r) {
    const float mu = __fmul_rn(__fadd_rn(fi, S), r);
    const float a = __fsub_rn(fi, mu);
    const float a2 = __fmul_rn(a, a);
    const float t1 = __fmul_rn(mu, S);
    const float t2 = __fadd_rn(t1, t1);
    const float t3 = __fmul_rn(mu, mu);
    const float t4 = __fmul_rn(Mf, t3);
    const float b = __fadd_rn(__fsub_rn(Q, t2), t4);
    const float us = __fmul_rn(__fadd_rn(a2, b), r);
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
    float* keys;                 // cooperative kernel: [2][gridDim][4] per-CTA winners
    int64_t* out; int32_t* n_out;
};

// f^ = (v - lo) / (hi - lo), or 0.5 for a flat pool
struct Norm {
    float lo, range;
    bool flat;
    __device__ float operator()(float v) const { return flat ? 0.5f : __fdiv_rn(__fsub_rn(v, lo), range); }
};

__device__ __forceinline__ Norm make_norm(const unsigned int* mm) {
    Norm n;
    n.lo = unord(mm[0]);
    const float hi = unord(mm[1]);
    n.flat = !(hi > n.lo);
    n.range = __fsub_rn(hi, n.lo);
    return n;
}

// S, Q, M of the labeled set: sequential sums in index order (one thread)
__device__ __forceinline__ void lab_sums(const SelArgs& a, const Norm& norm, float* out3) {
    float S = 0.f, Q = 0.f, M = 0.f;
    for (int64_t j = 0; j < a.n_lab; ++j) {
        if (!isfinite(a.lab[j])) continue;
        const float f = norm(a.lab[j]);
        S = __fadd_rn(S, f);
        Q = __fadd_rn(Q, __fmul_rn(f, f));
        M = __fadd_rn(M, 1.0f);
    }
    out3[0] = S;
    out3[1] = Q;
    out3[2] = M;
}

__device__ __forceinline__ float init_ds(const SelArgs& a, const Norm& norm, float f) {
    float ds = INFINITY;
    for (int64_t j = 0; j < a.n_lab; ++j)
        if (isfinite(a.lab[j])) ds = fminf(ds, fabsf(__fsub_rn(f, norm(a.lab[j]))));
    return ds == INFINITY ? 1.0f : ds;   // Eq. 1 with an empty labeled set: maximal novelty 1
}

// ---------------------------------------------------------------- cluster kernel
__global__ void __launch_bounds__(kCThreads, 1) k_rdu_cluster(SelArgs a) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) uint8_t rsm[];
    const int kk = (a.per + kCThreads - 1) / kCThreads;              // candidates per thread (<= 16)
    const int cap = kk * kCThreads;
    float* f_s = reinterpret_cast<float*>(rsm);                       // [cap]
    float* d_s = f_s + cap;                                            // [cap]
    int16_t* op_s = reinterpret_cast<int16_t*>(d_s + cap);             // [cap], -1 = not eligible
    __shared__ float s_budget[kMaxOps];
    __shared__ int s_sel[kMaxOps];
    __shared__ Best s_warp[kCThreads / 32];
    __shared__ Best s_slot[2];      // this CTA's winner of pick p in slot p & 1 (read over DSMEM)
    __shared__ Best s_pick;
    __shared__ float s_lab[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
    const Norm norm = make_norm(a.mm);
    for (int op = tid; op < a.n_ops; op += kCThreads) {
        s_budget[op] = (float)((double)a.budget_total * (double)a.hist[op] / (double)a.n_pool);
        s_sel[op] = 0;
    }
    if (tid == 0) lab_sums(a, norm, s_lab);
    const int64_t base = (int64_t)rank * a.per;   // this CTA's slice [base, base + per)
    for (int j = tid; j < cap; j += kCThreads) {
        const int64_t i = base + j;
        bool ok = j < a.per && i < a.n_pool;
        float f = 0.f;
        int op = -1;
        if (ok) {
            const float v = a.pool[i];
            op = a.ops[i];
            ok = isfinite(v) && op >= 0 && op < a.n_ops;
            f = norm(v);
            ok = ok && isfinite(f);
        }
        f_s[j] = f;
        d_s[j] = ok ? init_ds(a, norm, f) : 0.f;
        op_s[j] = ok ? (int16_t)op : (int16_t)-1;
    }
    __syncthreads();
    float S = s_lab[0], Q = s_lab[1], Mf = s_lab[2];
    int picks = 0;
    for (int p = 0; p < a.budget_total; ++p) {
        const float r = __fdiv_rn(1.0f, __fadd_rn(Mf, 1.0f));
        Best b{0.f, 0.f, -1};
        for (int k = 0; k < kk; ++k) {
            const int j = tid + k * kCThreads;
            const int op = op_s[j];
            if (op < 0 || !((float)s_sel[op] < s_budget[op])) continue;
            const float f = f_s[j];
            const Best c{total_score(f, d_s[j], S, Q, Mf, r), f, base + j};
            if (better(c, b)) b = c;
        }
        b = warp_best(b);
        if (lane == 0) s_warp[warp] = b;
        __syncthreads();
        if (warp == 0) {
            Best w = s_warp[lane];
            w = warp_best(w);
            if (lane == 0) s_slot[p & 1] = w;
        }
        cluster.sync();   // every CTA's slot p & 1 is written (release / acquire)
        if (warp == 0) {
            Best g{0.f, 0.f, -1};
            if (lane < (int)csize) g = *cluster.map_shared_rank(&s_slot[p & 1], (unsigned)lane);
            g = warp_best(g);   // same order in every CTA -> the same global pick
            if (lane == 0) s_pick = g;
        }
        __syncthreads();
        const Best g = s_pick;
        if (g.idx < 0) break;
        const float fs = g.f;
        if (tid == 0) s_sel[a.ops[g.idx]] += 1;
        S = __fadd_rn(S, fs);
        Q = __fadd_rn(Q, __fmul_rn(fs, fs));
        Mf = __fadd_rn(Mf, 1.0f);
        const int64_t loc = g.idx - base;
        for (int k = 0; k < kk; ++k) {
            const int j = tid + k * kCThreads;
            if (j == loc) op_s[j] = -1;
            d_s[j] = fminf(d_s[j], fabsf(__fsub_rn(f_s[j], fs)));
        }
        if (rank == 0 && tid == 0) a.out[p] = g.idx;
        ++picks;
        __syncthreads();
    }
    if (rank == 0 && tid == 0) *a.n_out = picks;
    cluster.sync();   // no CTA exits while another may still read its slots
}

// ---------------------------------------------------------------- cooperative grid kernel
__global__ void __launch_bounds__(kThreads) k_rdu_select(SelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ float s_budget[kMaxOps];
    __shared__ int s_sel[kMaxOps];
    __shared__ Best s_warp[kThreads / 32];
    __shared__ float s_lab[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Norm norm = make_norm(a.mm);
    for (int op = tid; op < a.n_ops; op += kThreads) {
        s_budget[op] = (float)((double)a.budget_total * (double)a.hist[op] / (double)a.n_pool);
        s_sel[op] = 0;
    }
    if (tid == 0) lab_sums(a, norm, s_lab);
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
        dv[k] = alive[k] ? init_ds(a, norm, fv[k]) : 1.0f;
        if (alive[k] && (opv[k] < 0 || opv[k] >= a.n_ops || !isfinite(fv[k]))) alive[k] = false;
    }
    __syncthreads();
    float S = s_lab[0], Q = s_lab[1], Mf = s_lab[2];
    int picks = 0;
    for (int p = 0; p < a.budget_total; ++p) {
        const float r = __fdiv_rn(1.0f, __fadd_rn(Mf, 1.0f));
        Best b{0.f, 0.f, -1};
#pragma unroll
        for (int k = 0; k < kMaxPer; ++k) {
            if (!alive[k] || !((float)s_sel[opv[k]] < s_budget[opv[k]])) continue;
            const Best c{total_score(fv[k], dv[k], S, Q, Mf, r), fv[k], base + k};
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
    // the cluster wins while each thread scans <= 4 candidates per pick (measured: 3.0 us/pick at
    // 16,384 vs 6.8 cooperative); beyond that the 148-CTA cooperative grid's wider scan wins
    if (n_pool <= (int64_t)kMaxCluster * kCThreads * 4) {
        // cluster path: C CTAs (as many as useful, <= 8), each holding ceil(n_pool / C) candidates
        // in shared memory: the per-pick scan is spread wide, the exchange stays one cluster barrier
        const int C = (int)std::min<int64_t>(kMaxCluster, std::max<int64_t>(1, (n_pool + kCThreads - 1) / kCThreads));
        const int per = (int)((n_pool + C - 1) / C);
        SelArgs a{pool, ops, n_pool, lab, n_lab, n_ops, budget_total, per, mm, hist, nullptr, out, n_out};
        const int smem = ((per + kCThreads - 1) / kCThreads) * kCThreads * (4 + 4 + 2);
        if ((e = prepare_kernel(k_rdu_cluster, kPerCta * (4 + 4 + 2))) != cudaSuccess) return e;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(kCThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, k_rdu_cluster, a);
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }
    const int64_t per_block_max = (int64_t)kThreads * kMaxPer;
    int grid = (int)std::min<int64_t>(num_sms, (n_pool + kThreads - 1) / kThreads);
    if (grid < 1) grid = 1;
    const int64_t per = (n_pool + (int64_t)grid * kThreads - 1) / ((int64_t)grid * kThreads);
    if (per > kMaxPer || n_pool > per_block_max * num_sms) return cudaErrorInvalidValue;
    SelArgs a{pool, ops, n_pool, lab, n_lab, n_ops, budget_total, (int)per, mm, hist, keys, out, n_out};
    void* args[] = {&a};
    e = cudaLaunchCooperativeKernel((void*)k_rdu_select, dim3(grid), dim3(kThreads), args, 0, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace tcl
