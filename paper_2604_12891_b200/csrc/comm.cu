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

tcl_status tcl_topk_global(tcl_model* m, const float* scores, int64_t n_local, int64_t index_base,
                           int32_t k, int64_t* idx, float* top, void* stream) {
    if (!m || n_local < 0 || k <= 0 || k > 4096 || index_base < 0) return set_error(TCL_EINVAL, "bad argument");
    if (!idx || !top || (n_local > 0 && !scores)) return set_error(TCL_EINVAL, "null pointer");
    if (!m->comm) return set_error(TCL_ESTATE, "tcl_comm_init has not been called");
    if (index_base + n_local > 0xFFFFFFFFll) return set_error(TCL_EINVAL, "global index must be < 2^32");
    cudaError_t e = cudaSetDevice(m->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    cudaStream_t s = (cudaStream_t)stream;
    // scratch: local tournament + merge over nranks*k keys
    const int64_t total = (int64_t)m->nranks * k;
    const size_t need = (size_t)k + topk_tmp_keys(std::max<int64_t>(std::max<int64_t>(n_local, total), 1), k) + k;
    if (need > m->topk_tmp_cap) {
        if (m->topk_tmp) cudaFree(m->topk_tmp);
        m->topk_tmp = nullptr;
        m->topk_tmp_cap = 0;
        ++m->ws_gen;   // graphs that baked in the old scratch are stale
        e = cudaMalloc((void**)&m->topk_tmp, need * sizeof(unsigned long long));
        if (e != cudaSuccess) return set_error(TCL_ENOMEM, "cudaMalloc(topk_tmp)");
        m->topk_tmp_cap = need;
    }
    {
        ProfScope ps(m, TCL_PROF_TOPK, s);
        m->launches += launch_topk_keys(scores, n_local, k, index_base, m->keys_send, m->topk_tmp, s);
    }
    {
        ProfScope ps(m, TCL_PROF_ALLGATHER, s);
        ncclResult_t r = ncclAllGather(m->keys_send, m->keys_recv, (size_t)k, ncclUint64,
                                       (ncclComm_t)m->comm, s);
        if (r != ncclSuccess) return nccl_error(r, "ncclAllGather");
    }
    {
        ProfScope ps(m, TCL_PROF_TOPK, s);
        m->launches += launch_topk_merge(m->keys_recv, total, k, idx, top, m->topk_tmp, s);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "tcl_topk_global");
    return TCL_OK;
}

}  // extern "C"
