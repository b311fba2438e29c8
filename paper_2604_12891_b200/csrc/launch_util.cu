// launch_util.cu -- per-device kernel preparation (dynamic shared-memory opt-in and occupancy).
//
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device-context setting, and
// tcl.h allows models on different devices (and one model per stream across host threads) in one
// process: the opt-in is therefore cached per (kernel, device) under a lock, never in a
// process-wide static of the launcher.
#include <map>
#include <mutex>
#include <tuple>

#include "kernels.h"

namespace tcl {

cudaError_t prepare_kernel_raw(const void* fn, int smem, int threads, int* blocks_per_sm) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> smem_set;            // (fn, device) -> opted-in bytes
    static std::map<std::tuple<const void*, int, int, int>, int> occ;      // (fn, device, smem, threads) -> CTAs/SM
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    const auto k2 = std::make_pair(fn, dev);
    auto it = smem_set.find(k2);
    if (it == smem_set.end() || it->second < smem) {
        if (smem > 48 * 1024 || it != smem_set.end()) {
            e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
        }
        smem_set[k2] = smem;
    }
    if (blocks_per_sm) {
        const auto k4 = std::make_tuple(fn, dev, smem, threads);
        auto jt = occ.find(k4);
        if (jt == occ.end()) {
            int b = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem);
            if (e != cudaSuccess || b < 1) b = 1;
            jt = occ.emplace(k4, b).first;
        }
        *blocks_per_sm = jt->second;
    }
    return cudaSuccess;
}

}  // namespace tcl
