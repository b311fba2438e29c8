// topk_eval.cu -- the Top-k score of PAPER.md Eq. 12 (§7.1.2), reading R22:
//   Top-k = sum_t minlat_t w_t / sum_t (min latency among task t's k best-predicted candidates) w_t
// Task t = one subgraph of one model: candidates off[t] .. off[t+1]-1 (CSR), true latencies, the
// cost model's predicted scores (larger = better; NaN = -inf; ties: lower index first, R15).
//
// k_task_topk: one CTA per task (grid-stride).  The task's (score, index) pairs become u64 keys
// (order-preserving score bits << 32 | ~index), are bitonic-sorted descending in shared memory
// (integer compare: exact and deterministic), and the latencies of the first min(k, T) sorted
// positions are min-reduced for every requested k.  Per task it writes w*minlat and w*pmin_k in
// fp64 (exact: a product of two fp32 values).  k_topk_reduce: one CTA sums the task columns in a
// fixed strided + tree order (deterministic) and writes score / num / den.
#include <algorithm>
#include <cmath>

#include "../kernels.h"

namespace tcl {

namespace teval {

constexpr int kThreads = 512;

__device__ __forceinline__ unsigned long long task_key(float s, uint32_t j) {
    if (s != s) s = -INFINITY;  // NaN ranks last (R15)
    uint32_t b = __float_as_uint(s);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((unsigned long long)b << 32) | (0xFFFFFFFFu - j);
}

__device__ __forceinline__ float block_min(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // red[] may still be read by the previous call
    if (lane == 0) red[warp] = v;
    __syncthreads();
    v = lane < kThreads / 32 ? red[lane] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(kThreads)
k_task_topk(const float* __restrict__ scores, const float* __restrict__ lat, const int64_t* __restrict__ off,
            const float* __restrict__ w, int64_t n_tasks, int cap, TopkEvalKs ks, double* __restrict__ cols,
            int* __restrict__ err) {
    extern __shared__ unsigned long long keys[];
    __shared__ float red[kThreads / 32];
    const int ncol = ks.n + 1;
    for (int64_t t = blockIdx.x; t < n_tasks; t += gridDim.x) {
        const int64_t o = off[t];
        const int64_t T = off[t + 1] - o;
        if (T < 1 || T > cap) {
            if (threadIdx.x == 0) {
                atomicOr(err, ERR_TASK);
                for (int c = 0; c < ncol; ++c) cols[(size_t)c * n_tasks + t] = NAN;
            }
            continue;
        }
        int P = 1;
        while (P < T) P <<= 1;
        float m = INFINITY;
        for (int j = threadIdx.x; j < P; j += kThreads) {
            keys[j] = j < T ? task_key(scores[o + j], (uint32_t)j) : 0ull;  // 0 sorts after every real key
            if (j < T) m = fminf(m, lat[o + j]);
        }
        __syncthreads();
        // bitonic sort, descending
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = threadIdx.x; i < (P >> 1); i += kThreads) {
                    const int lo = 2 * stride * (i / stride) + (i % stride);
                    const int hi = lo + stride;
                    const bool desc = (lo & size) == 0;
                    const unsigned long long a = keys[lo], b = keys[hi];
                    if (desc ? (a < b) : (a > b)) {
                        keys[lo] = b;
                        keys[hi] = a;
                    }
                }
                __syncthreads();
            }
        }
        const float wt = w[t];
        m = block_min(m, red);
        if (threadIdx.x == 0) cols[t] = (double)m * (double)wt;
        for (int c = 0; c < ks.n; ++c) {
            const int kk = (int)((int64_t)ks.k[c] < T ? (int64_t)ks.k[c] : T);
            float pm = INFINITY;
            for (int j = threadIdx.x; j < kk; j += kThreads)
                pm = fminf(pm, lat[o + (0xFFFFFFFFu - (uint32_t)(keys[j] & 0xFFFFFFFFull))]);
            pm = block_min(pm, red);
            if (threadIdx.x == 0) cols[(size_t)(c + 1) * n_tasks + t] = (double)pm * (double)wt;
        }
        __syncthreads();  // keys[] reused by the next task
    }
}

__global__ void __launch_bounds__(1024) k_topk_reduce(const double* __restrict__ cols, int64_t n_tasks, int ncol,
                                                      double* __restrict__ out) {
    __shared__ double red[1024];
    double num = 0.0;
    for (int c = 0; c < ncol; ++c) {
        double v = 0.0;
        for (int64_t t = threadIdx.x; t < n_tasks; t += 1024) v += cols[(size_t)c * n_tasks + t];
        red[threadIdx.x] = v;
        __syncthreads();
        for (int s = 512; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (c == 0) {
                num = red[0];
            } else {
                const int j = c - 1, nk = ncol - 1;
                out[j] = num / red[0];
                out[nk + j] = num;
                out[2 * nk + j] = red[0];
            }
        }
        __syncthreads();
    }
}

}  // namespace teval

cudaError_t launch_topk_eval(const float* scores, const float* lat, const int64_t* off, const float* w,
                             int64_t n_tasks, int max_task_len, const TopkEvalKs& ks, double* cols,
                             double* out, int* err, int num_sms, cudaStream_t s) {
    using namespace teval;
    int P = 1;
    while (P < max_task_len) P <<= 1;
    const size_t smem = (size_t)P * sizeof(unsigned long long);
    cudaError_t e = prepare_kernel(k_task_topk, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = (int)std::min<int64_t>(n_tasks, (int64_t)num_sms * 4);
    k_task_topk<<<grid, kThreads, smem, s>>>(scores, lat, off, w, n_tasks, max_task_len, ks, cols, err);
    k_topk_reduce<<<1, 1024, 0, s>>>(cols, n_tasks, ks.n + 1, out);
    return cudaGetLastError();
}

}  // namespace tcl
