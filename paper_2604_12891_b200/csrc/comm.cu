// comm.cu -- multi-GPU global top-k.
//
// Candidates are independent, so each rank scores a contiguous shard with no exchange; the only
// collective is one ncclAllGather of k packed 8-byte (score, index) keys per rank over NVLink 5 /
// NVSwitch (k*8 bytes: 512 B at k = 64, 8 KiB at k = 1024) enqueued on the scoring stream, then
// the identical merge kernel on every rank -> the same global top-k everywhere.  At these sizes the
// exchange is launch/latency-bound (µs), so NCCL's all-gather is the right tool; there is no
// compute to fuse it with (the merge consumes all G*k keys).
#include <nccl.h>

#include <string>

#include "../../include/tcl.h"
#include "internal.h"
#include "kernels.h"
#include "topk_key.h"

#include <algorithm>

using namespace tcl;

static tcl_status nccl_error(ncclResult_t r, const char* where) {
    return set_error(TCL_ENCCL, std::string(where) + ": " + ncclGetErrorString(r));
}

namespace tcl {
void comm_destroy(tcl_model* m) {
    if (m->comm) ncclCommDestroy((ncclComm_t)m->comm);
    m->comm = nullptr;
}
}  // namespace tcl

extern "C" {

tcl_status tcl_comm_unique_id(uint8_t id_out[128]) {
    if (!id_out) return set_error(TCL_EINVAL, "null pointer");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nccl_error(r, "ncclGetUniqueId");
    memcpy(id_out, &id, 128);
    return TCL_OK;
}

tcl_status tcl_comm_init(tcl_model* m, const uint8_t id[128], int32_t nranks, int32_t rank) {
    if (!m || !id || nranks < 1 || rank < 0 || rank >= nranks) return set_error(TCL_EINVAL, "bad argument");
    cudaError_t e = cudaSetDevice(m->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    comm_destroy(m);
    ncclUniqueId uid;
    memcpy(&uid, id, 128);
    ncclComm_t c;
    ncclResult_t r = ncclCommInitRank(&c, nranks, uid, rank);
    if (r != ncclSuccess) return nccl_error(r, "ncclCommInitRank");
    m->comm = c;
    m->nranks = nranks;
    m->rank = rank;
    if (m->keys_recv) cudaFree(m->keys_recv);
    e = cudaMalloc((void**)&m->keys_recv, (size_t)nranks * 4096 * sizeof(unsigned long long));
    if (e != cudaSuccess) return set_error(TCL_ENOMEM, "cudaMalloc(keys_recv)");
    return TCL_OK;
}

// scratch for a local top-k of n keys and a merge of `total` keys
static tcl_status ensure_comm_tmp(tcl_model* m, int64_t n, int64_t total, int k) {
    const size_t need = (size_t)k + topk_tmp_keys(std::max<int64_t>(std::max<int64_t>(n, total), 1), k) + k;
    if (need <= m->topk_tmp_cap) return TCL_OK;
    if (m->topk_tmp) cudaFree(m->topk_tmp);
    m->topk_tmp = nullptr;
    m->topk_tmp_cap = 0;
    ++m->ws_gen;   // graphs that baked in the old scratch are stale
    if (cudaMalloc((void**)&m->topk_tmp, need * sizeof(unsigned long long)) != cudaSuccess)
        return set_error(TCL_ENOMEM, "cudaMalloc(topk_tmp)");
    m->topk_tmp_cap = need;
    return TCL_OK;
}

static tcl_status check_local(tcl_model* m, const float* scores, int64_t n_local, int64_t index_base, int32_t k) {
    if (!m || n_local < 0 || k <= 0 || k > 4096 || index_base < 0) return set_error(TCL_EINVAL, "bad argument");
    if (n_local > 0 && !scores) return set_error(TCL_EINVAL, "null pointer");
    if (index_base + n_local > 0xFFFFFFFFll) return set_error(TCL_EINVAL, "global index must be < 2^32");
    return TCL_OK;
}

tcl_status tcl_topk_local_keys(tcl_model* m, const float* scores, int64_t n_local, int64_t index_base, int32_t k,
                               uint64_t* keys, void* stream) {
    tcl_status st = check_local(m, scores, n_local, index_base, k);
    if (st != TCL_OK) return st;
    if (!keys) return set_error(TCL_EINVAL, "null pointer");
    cudaError_t e = cudaSetDevice(m->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    if ((st = ensure_comm_tmp(m, n_local, 0, k)) != TCL_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    ProfScope ps(m, TCL_PROF_TOPK, s);
    m->launches += launch_topk_keys(scores, n_local, k, index_base, reinterpret_cast<unsigned long long*>(keys),
                                    m->topk_tmp, s);
    e = cudaGetLastError();
    return e == cudaSuccess ? TCL_OK : cuda_error(e, "tcl_topk_local_keys");
}

tcl_status tcl_topk_merge_keys(tcl_model* m, const uint64_t* keys, int64_t count, int32_t k, int64_t* idx, float* top,
                               void* stream) {
    if (!m || count < 0 || k <= 0 || k > 4096) return set_error(TCL_EINVAL, "bad argument");
    if (!idx || !top || (count > 0 && !keys)) return set_error(TCL_EINVAL, "null pointer");
    cudaError_t e = cudaSetDevice(m->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    tcl_status st = ensure_comm_tmp(m, 0, count, k);
    if (st != TCL_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    ProfScope ps(m, TCL_PROF_TOPK, s);
    m->launches += launch_topk_merge(reinterpret_cast<const unsigned long long*>(keys), count, k, idx, top,
                                     m->topk_tmp, s);
    e = cudaGetLastError();
    return e == cudaSuccess ? TCL_OK : cuda_error(e, "tcl_topk_merge_keys");
}

tcl_status tcl_topk_global(tcl_model* m, const float* scores, int64_t n_local, int64_t index_base,
                           int32_t k, int64_t* idx, float* top, void* stream) {
    tcl_status st = check_local(m, scores, n_local, index_base, k);
    if (st != TCL_OK) return st;
    if (!idx || !top) return set_error(TCL_EINVAL, "null pointer");
    if (!m->comm) return set_error(TCL_ESTATE, "tcl_comm_init has not been called");
    cudaStream_t s = (cudaStream_t)stream;
    // local best k (packed keys) -> all-gather of nranks * k keys over NVLink -> merge on every rank
    if ((st = tcl_topk_local_keys(m, scores, n_local, index_base, k, reinterpret_cast<uint64_t*>(m->keys_send), stream)) != TCL_OK)
        return st;
    {
        ProfScope ps(m, TCL_PROF_ALLGATHER, s);
        ncclResult_t r = ncclAllGather(m->keys_send, m->keys_recv, (size_t)k, ncclUint64, (ncclComm_t)m->comm, s);
        if (r != ncclSuccess) return nccl_error(r, "ncclAllGather");
        // errors NCCL raises asynchronously (a peer's failure, a network / NVLink fault) surface here
        ncclResult_t ar = ncclSuccess;
        r = ncclCommGetAsyncError((ncclComm_t)m->comm, &ar);
        if (r != ncclSuccess) return nccl_error(r, "ncclCommGetAsyncError");
        if (ar != ncclSuccess && ar != ncclInProgress) return nccl_error(ar, "ncclAllGather (asynchronous error)");
    }
    return tcl_topk_merge_keys(m, reinterpret_cast<const uint64_t*>(m->keys_recv), (int64_t)m->nranks * k, k, idx, top,
                               stream);
}

tcl_status tcl_shard_range(int64_t n_global, int32_t nranks, int32_t rank, int64_t* start, int64_t* count) {
    if (!start || !count || n_global < 0 || nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(TCL_EINVAL, "bad argument");
    const int64_t per = (n_global + nranks - 1) / nranks;
    const int64_t st = std::min<int64_t>(n_global, (int64_t)rank * per);
    *start = st;
    *count = std::max<int64_t>(0, std::min<int64_t>(n_global, st + per) - st);
    return TCL_OK;
}

uint64_t tcl_topk_key(float score, int64_t global_index) {
    return (uint64_t)topk_key(score, (uint32_t)global_index);
}

}  // extern "C"
