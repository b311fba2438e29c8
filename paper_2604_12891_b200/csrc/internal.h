// internal.h -- the model object behind the opaque tcl_model handle (host side only).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (stage ranges in ProfScope)

#include <string>
#include <vector>

#include "../../include/tcl.h"

#define TCL_STR_(x) #x
#define TCL_STR(x) TCL_STR_(x)

namespace tcl {

constexpr int kXld = 32;  // packed feature row width (d_in <= 32, zero-padded -> 16-byte rows)

struct LayerPtrs {
    const float *ln_w, *ln_b, *W_in, *w_conv, *b_conv, *W_x, *W_dt, *b_dt, *A_log, *Dv, *W_out;
};

struct WeightPtrs {  // device pointers into the fp32 blob (canonical order, include/tcl.h)
    const float *enc_W1, *enc_b1, *enc_W2, *enc_b2, *enc_W3, *enc_b3;
    std::vector<LayerPtrs> layers;
    const float *lnf_w, *lnf_b;
    const float *dec_W1, *dec_b1, *dec_W2, *dec_b2, *dec_W3, *dec_b3;
};

// One Eq. 7 lateral site: V [a][ldv] (zero-padded input columns), c [a], Ua = diag(alpha) U
// [out][ad_ld] (zero-padded to a multiple of 16 columns).
struct AdapterSite {
    const float *V, *c, *Ua;
    int in, out, ldv;
};

// Training state (tcl_train_init): gradients, Adam moments, saved activations, backward scratch.
struct TrainState {
    int64_t cap_n = 0, rows = 0, nW = 0;
    int step = 0;
    float lr = 7e-4f, b1 = 0.9f, b2 = 0.999f, eps = 1e-8f, sigma = 1.0f;
    float *g = nullptr, *mA = nullptr, *vA = nullptr;                 // [nW]
    float *E1pre = nullptr, *E1 = nullptr, *E2pre = nullptr, *E2 = nullptr;
    std::vector<float*> Hin, Aln, XZ, U, DBC, Delta, S, G;             // per layer (Hin: n_layer + 1)
    float *pooled = nullptr, *d1pre = nullptr, *d1 = nullptr, *d2pre = nullptr, *d2 = nullptr, *scores = nullptr;
    float *dH = nullptr, *dA = nullptr, *dXZ = nullptr, *dU = nullptr, *dpre = nullptr, *dDpre = nullptr,
          *dDBC = nullptr, *dG = nullptr, *xhdy = nullptr, *dE1 = nullptr, *dE2 = nullptr;
    float *ds = nullptr, *dd1 = nullptr, *dd2 = nullptr, *dpooled = nullptr, *dAlog_part = nullptr,
          *dD_part = nullptr, *gloss = nullptr, *loss = nullptr;
    float* part = nullptr;
    size_t part_cap = 0;
    int* step_dev = nullptr;       // Adam step counter (device; graph replays advance it)
    float* corr_dev = nullptr;     // Adam bias corrections 1 - beta^t
    // CUDA graph of one step, replayed while the call signature is unchanged
    struct Key {
        const void *feats, *lens, *lat, *off, *loss;
        int64_t n, n_groups, ws_gen;
        int max_group, apply;
        bool operator==(const Key& o) const {
            return feats == o.feats && lens == o.lens && lat == o.lat && off == o.off && loss == o.loss && n == o.n &&
                   n_groups == o.n_groups && ws_gen == o.ws_gen && max_group == o.max_group && apply == o.apply;
        }
    } key{};
    cudaGraphExec_t graph = nullptr;
    int64_t graph_launches = 0;    // kernels per replay
    cudaStream_t gstream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    std::vector<void*> allocs;
};

// CUDA-graph cache of repeated calls (TCL_OPT_GRAPHS): a call is identified by its kind, every
// pointer and size it was given and the generation of the model's scratch buffers it bakes in.
struct GraphKey {
    int kind = -1;                 // 0 tcl_score, 1 tcl_score_mc, 2 tcl_topk
    const void* p[6] = {};
    int64_t v[6] = {};
    int64_t gen = 0;
    bool operator==(const GraphKey& o) const {
        if (kind != o.kind || gen != o.gen) return false;
        for (int i = 0; i < 6; ++i)
            if (p[i] != o.p[i] || v[i] != o.v[i]) return false;
        return true;
    }
};
struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;          // kernels per replay
    uint64_t stamp = 0;            // LRU
};

// One row GEMM of the fp32 path on the 3xTF32 tensor-core kernel (gemm_tf32.cu): W_hi / W_lo
// copies (split on the device from the fp32 weights) and their tensor maps.
struct Tf32W {
    const float* w = nullptr;      // the fp32 weight [n][k] it is split from
    float* hi = nullptr;
    float* lo = nullptr;
    CUtensorMap tm_hi, tm_lo;      // box {32, bn}
    int bn = 0, n = 0, k = 0;      // bn == 0: this GEMM stays on the SIMT kernel
};

struct Workspace {
    int64_t cap_n = 0, rows = 0;
    int32_t* cu = nullptr;        // [cap_n + 1]
    int32_t* row_cand = nullptr;  // [rows]
    float* X = nullptr;           // [rows][kXld]
    float* H = nullptr;           // [rows][dm]   residual stream
    float* A = nullptr;           // [rows][dm]   LN_l(H)
    float* XZ = nullptr;          // [rows][2 di] in_proj output
    float* U = nullptr;           // [rows][max(di, e1)]  conv output / encoder hidden 1
    float* Delta = nullptr;       // [rows][max(di, e2)]  softplus(dt) / encoder hidden 2
    float* G = nullptr;           // [rows][di]   gated scan output
    float* DBC = nullptr;         // [rows][ldbc] x_proj output
    float* m2 = nullptr;          // [cap_n] MC Welford M2
    float* pooled = nullptr;      // [cap_n][dm]  masked mean of LN_f(H)
    float* dh1 = nullptr;         // [cap_n][h1]  decoder hidden 1
    float* dh2 = nullptr;         // [cap_n][h2]  decoder hidden 2
    float* dsc = nullptr;         // [cap_n]      per-pass score (MC)
    int32_t* lens_mc = nullptr;   // [cap_n]      lengths of the batched MC passes (pass-major)
    int* scan_ctr = nullptr;      // [kMaxLayers] k_scan work-group counters, zeroed per forward
    // bf16 tensor-core path
    __nv_bfloat16* Xb = nullptr;   // [rows][kXld]  packed features
    __nv_bfloat16* XZb = nullptr;  // [rows][max(2 di, e1 + e2)]  in_proj output / encoder hidden
    __nv_bfloat16* Ab = nullptr;   // [rows][dm]    LN_l(H)
    __nv_bfloat16* Gb = nullptr;   // [rows][di]    gated scan output
    uint8_t* Pk = nullptr;         // [rows][pk_ld] mixer packet: u, Delta (fp16), B, C (fp32)
    int pk_ld = 0;                 // packet row bytes (4 di + 8 N)
    __nv_bfloat16* GZb = nullptr;  // [rows][di] SiLU(z), the scan's gate (in_proj epilogue)
    CUtensorMap tmGZs, tmUs;       // k_inconv stores: SiLU(z) -> GZb, u -> packet (box {64, 125})
    CUtensorMap tmXb, tmE1b, tmE2b, tmAb, tmGb;        // GEMM A operands (box {64, 128})
    CUtensorMap tmE1o, tmE2o, tmXZo;                   // GEMM bf16 outputs (box {64, 32}, TMA store)
    CUtensorMap tmHf, tmAo;                            // residual stream fp32 (box {32,32}), LN out (box {64,32})
    // KB + AC two-column model (fp32 path): the KB column's buffers and the lateral activations
    float* Hk = nullptr;          // [rows][dm]  KB residual stream
    float* E1k = nullptr;         // [rows][e1]  KB encoder hidden 1
    float* E2k = nullptr;         // [rows][e2]  KB encoder hidden 2
    float* Lat = nullptr;         // [rows][ad_ld] SiLU(V h^KB + c), columns >= a stay zero
    float* pooled_k = nullptr;    // [cap_n][dm]
    float* dh1k = nullptr;        // [cap_n][h1]
    CUtensorMap tmAbS2;                                // k_inconv A half-slices for 2-CTA cluster multicast (box {64, 64})
    CUtensorMap tmX32, tmE1f, tmE2f, tmA32, tmG32;     // fp32 path 3xTF32 A operands (box {32, 128})
    std::vector<void*> allocs;
};

tcl_status set_error(tcl_status st, const std::string& msg);
tcl_status cuda_error(cudaError_t e, const char* where);

}  // namespace tcl

struct tcl_model {
    tcl_dims dims{};
    int device = 0;
    int ldbc = 0;
    float* w_dev = nullptr;
    tcl::WeightPtrs wp{};
    float* W1p = nullptr;   // [e1][kXld]
    float* A2 = nullptr;    // [n_layer][di][N]  A * log2(e)
    float* invA = nullptr;  // [n_layer][di][N]  1 / A
    int* d_err = nullptr;
    tcl::Workspace ws;
    int64_t ws_gen = 0;     // bumped on every (re)allocation of model-owned scratch (graph keys)
    int use_graphs = 1;     // tcl_set_option(TCL_OPT_GRAPHS)
    int scan_mode = 0;      // tcl_set_option(TCL_OPT_SCAN): 0 auto, 1 sequential, 2 chunked across L
    // fp32 path: row GEMMs on the 3xTF32 tensor-core kernel: enc1, enc2, enc3, then (in, out) per layer
    std::vector<tcl::Tf32W> tfw;
    float* tf_split = nullptr;
    std::vector<tcl::GraphEntry> graphs;     // captured calls (LRU, <= kMaxGraphs)
    std::vector<tcl::GraphKey> seen;         // calls seen once (captured on their second occurrence)
    uint64_t graph_clock = 0;
    cudaStream_t cap_stream = nullptr;       // capture stream (the graphs are launched on the caller's)
    unsigned long long* topk_tmp = nullptr;
    size_t topk_tmp_cap = 0;
    // multi-GPU
    void* comm = nullptr;   // ncclComm_t
    int nranks = 1, rank = 0;
    unsigned long long* keys_send = nullptr;  // [4096]
    unsigned long long* keys_recv = nullptr;  // [nranks * 4096]
    // end-to-end host path staging
    int64_t stage_cap = 0;
    float* stage_feats = nullptr;
    int32_t* stage_lens = nullptr;
    float* stage_scores = nullptr;
    int64_t* stage_idx = nullptr;
    float* stage_top = nullptr;
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> chunk_events;
    int64_t launches = 0;
    cudaError_t fwd_err = cudaSuccess;   // a host-side launch refusal inside the fp32 forward (reported by forward_any)
    void* rdu_scratch = nullptr;
    size_t rdu_scratch_cap = 0;
    // KB + AC two-column model (tcl_model_create_kbac): this object holds the AC column
    tcl_model* kb = nullptr;      // the KB column (weights only; its workspace is unused)
    int ad_rank = 0, ad_ld = 0;
    float* ad_dev = nullptr;
    std::vector<tcl::AdapterSite> ad;   // enc1, enc2, enc3, layer 0..n_layer-1, dec1, dec2
    double* eval_cols = nullptr;
    tcl::TrainState* tr = nullptr;  // tcl_train_init   // tcl_topk_score per-task columns
    size_t eval_cols_cap = 0;
    // bf16 tensor-core path (precision == TCL_PREC_BF16_PROJ)
    int use_tc = 0, num_sms = 148, nxp = 0, rp = 0;
    std::vector<void*> bf_allocs;
    __nv_bfloat16 *W1b = nullptr, *W2b = nullptr, *W3b = nullptr;
    std::vector<__nv_bfloat16*> Winb, Woutb, Wdtb;
    std::vector<__half*> Wxh;            // x_proj weights in fp16 (k_xdt: fp16 operands, u is fp16)
    CUtensorMap tmW1, tmW2, tmW3;
    std::vector<CUtensorMap> tmWin, tmWout;   // W_in box {64, inconv_channels(di)}; W_out box {64, dm}
    // per-stage instrumentation (tcl_profile_enable)
    int prof_on = 0;
    struct ProfRec { int kind; cudaEvent_t a, b; };
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> prof_pool;
    double prof_ms[TCL_PROF_NKINDS] = {};
    int64_t prof_n[TCL_PROF_NKINDS] = {};
};

namespace tcl {
void comm_destroy(tcl_model* m);

// NVTX range names of the stage kinds (tcl.h TCL_PROF_*), for nsys / ncu --nvtx timelines
inline const char* prof_stage_name(int k) {
    static const char* const names[TCL_PROF_NKINDS] = {
        "tcl:pack", "tcl:encoder", "tcl:layernorm", "tcl:in_proj", "tcl:conv", "tcl:x_proj", "tcl:dt_proj",
        "tcl:scan", "tcl:out_proj", "tcl:head", "tcl:topk", "tcl:mixer", "tcl:allgather", "tcl:mc",
        "tcl:lateral", "tcl:xdt"};
    return (k >= 0 && k < TCL_PROF_NKINDS) ? names[k] : "tcl:?";
}

// Brackets the launches issued in its scope with an NVTX range (host side; a no-op without a tool
// attached) and, when profiling is on, with CUDA events.
struct ProfScope {
    tcl_model* m; int kind; cudaStream_t s; cudaEvent_t a = nullptr;
    static cudaEvent_t get(tcl_model* m) {
        if (!m->prof_pool.empty()) { cudaEvent_t e = m->prof_pool.back(); m->prof_pool.pop_back(); return e; }
        cudaEvent_t e; cudaEventCreate(&e); return e;
    }
    ProfScope(tcl_model* m_, int k, cudaStream_t s_) : m(m_), kind(k), s(s_) {
        nvtxRangePushA(prof_stage_name(k));
        if (m->prof_on) { a = get(m); cudaEventRecord(a, s); }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = get(m);
            cudaEventRecord(b, s);
            m->prof_recs.push_back({kind, a, b});
        }
        nvtxRangePop();
    }
};
}
