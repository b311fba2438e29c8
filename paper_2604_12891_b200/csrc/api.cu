// api.cu -- host side of libtcl.so: the C ABI declared in include/tcl.h.
//
// Responsibilities: dims validation, weight upload and preprocessing, a grow-on-demand workspace
// arena, the per-chunk launch sequence of the forward pass, MC-dropout passes
// (CS6), top-k (a11), the host->device pipelined end-to-end call, and sticky error reporting.
// Every arithmetic step of the path runs in the kernels under kernels/; this file only launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tcl.h"
#include "internal.h"
#include "kernels.h"

using namespace tcl;

namespace {
thread_local std::string g_last_error;
}

namespace tcl {
tcl_status set_error(tcl_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}
tcl_status cuda_error(cudaError_t e, const char* where) {
    return set_error(TCL_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
}  // namespace tcl

#define CUDA_TRY(call)                                                 \
    do {                                                               \
        cudaError_t _e = (call);                                       \
        if (_e != cudaSuccess) return tcl::cuda_error(_e, #call);      \
    } while (0)

// ------------------------------------------------------------------------------ dims / weights
static int64_t weights_count_of(const tcl_dims& d) {
    const int64_t dm = d.d_model, di = (int64_t)d.expand * d.d_model, N = d.d_state,
                  R = d.dt_rank;
    int64_t c = 0;
    c += (int64_t)d.enc_dims[0] * d.d_in + d.enc_dims[0];
    c += (int64_t)d.enc_dims[1] * d.enc_dims[0] + d.enc_dims[1];
    c += (int64_t)d.enc_dims[2] * d.enc_dims[1] + d.enc_dims[2];
    c += d.n_layer * (dm + dm + 2 * di * dm + di * d.d_conv + di + (R + 2 * N) * di + di * R + di +
                      di * N + di + dm * di);
    c += dm + dm;
    c += (int64_t)d.dec_dims[0] * dm + d.dec_dims[0];
    c += (int64_t)d.dec_dims[1] * d.dec_dims[0] + d.dec_dims[1];
    c += (int64_t)d.dec_dims[2] * d.dec_dims[1] + d.dec_dims[2];
    return c;
}

static tcl_status validate_dims(const tcl_dims* d) {
    if (!d) return set_error(TCL_EINVAL, "dims is NULL");
    const int di = d->expand * d->d_model;
    auto bad = [](const char* m) { return set_error(TCL_ESHAPE, m); };
    if (d->d_in < 1 || d->d_in > 32) return bad("d_in must be in [1, 32]");
    if (d->max_len < 1 || d->max_len > 256) return bad("max_len must be in [1, 256]");
    if (d->d_model < 32 || d->d_model > 256 || d->d_model % 32) return bad("d_model must be a multiple of 32 in [32, 256]");
    if (d->n_layer < 0 || d->n_layer > 64) return bad("n_layer must be in [0, 64]");
    if (d->d_state != 8 && d->d_state != 16) return bad("d_state must be 8 or 16");
    if (d->d_conv < 1 || d->d_conv > 8) return bad("d_conv must be in [1, 8]");
    if (d->expand < 1 || di > 512 || di % 32) return bad("d_inner = expand*d_model must be a multiple of 32 <= 512");
    if (d->dt_rank < 1 || d->dt_rank > 32 || d->dt_rank % 4) return bad("dt_rank must be a multiple of 4 in [4, 32]");
    if (d->enc_dims[2] != d->d_model) return bad("enc_dims[2] must equal d_model");
    for (int i = 0; i < 2; ++i)
        if (d->enc_dims[i] < 32 || d->enc_dims[i] > 512 || d->enc_dims[i] % 32) return bad("enc_dims[0..1] must be multiples of 32 in [32, 512]");
    if (d->dec_dims[2] != 1) return bad("dec_dims[2] must be 1");
    if (d->dec_dims[0] < 1 || d->dec_dims[0] > 256 || d->dec_dims[1] < 1 || d->dec_dims[1] > 256)
        return bad("dec_dims[0..1] must be in [1, 256]");
    if (!(d->ln_eps > 0.0f)) return bad("ln_eps must be > 0");
    if (!(d->dropout_p >= 0.0f && d->dropout_p < 1.0f)) return set_error(TCL_EINVAL, "dropout_p must be in [0, 1)");
    if (d->precision != TCL_PREC_FP32 && d->precision != TCL_PREC_BF16_PROJ) return bad("unknown precision");
    if (d->disc != TCL_DISC_ZOH && d->disc != TCL_DISC_EULER_B) return bad("unknown disc");
    return TCL_OK;
}

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

// ------------------------------------------------------------------------------ workspace
template <typename T>
static tcl_status dev_alloc(T** p, size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        *p = nullptr;
        return set_error(TCL_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    return TCL_OK;
}

static void free_workspace(tcl_model* m) {
    Workspace& w = m->ws;
    for (void* p : w.allocs) cudaFree(p);
    w = Workspace();
}

template <typename T>
static tcl_status ws_take(tcl_model* m, T** p, size_t count) {
    tcl_status st = dev_alloc(p, count);
    if (st == TCL_OK) m->ws.allocs.push_back(*p);
    return st;
}

// Ensure the workspace holds a chunk of `chunk_n` candidates.
static tcl_status ensure_workspace(tcl_model* m, int64_t chunk_n) {
    if (chunk_n <= m->ws.cap_n) return TCL_OK;
    free_workspace(m);
    const tcl_dims& d = m->dims;
    const int64_t rows = chunk_n * d.max_len;
    const int dm = d.d_model, di = d.expand * d.d_model;
    Workspace& w = m->ws;
    tcl_status st;
#define TAKE(p, cnt) if ((st = ws_take(m, &w.p, (size_t)(cnt))) != TCL_OK) { free_workspace(m); return st; }
    TAKE(cu, chunk_n + 1);
    TAKE(row_cand, rows);
    TAKE(X, rows * kXld);
    TAKE(H, rows * dm);
    TAKE(A, rows * dm);
    TAKE(XZ, rows * 2 * di);
    const int64_t udim = std::max<int64_t>(di, d.enc_dims[0]);
    const int64_t ddim = std::max<int64_t>(di, d.enc_dims[1]);
    TAKE(U, rows * udim);
    TAKE(Delta, rows * ddim);
    TAKE(G, rows * di);
    TAKE(DBC, rows * m->ldbc);
    TAKE(m2, chunk_n);
#undef TAKE
    w.cap_n = chunk_n;
    w.rows = rows;
    return TCL_OK;
}

static tcl_status ensure_topk_tmp(tcl_model* m, int64_t n, int k) {
    size_t need = (size_t)k + topk_tmp_keys(std::max<int64_t>(n, 1), k) + (size_t)k;
    if (need <= m->topk_tmp_cap) return TCL_OK;
    if (m->topk_tmp) cudaFree(m->topk_tmp);
    m->topk_tmp = nullptr;
    m->topk_tmp_cap = 0;
    tcl_status st = dev_alloc(&m->topk_tmp, need);
    if (st != TCL_OK) return st;
    m->topk_tmp_cap = need;
    return TCL_OK;
}

// ------------------------------------------------------------------------------ forward
// One chunk of candidates [0, n) (pointers already offset).  If mc_mean != nullptr the head
// accumulates Welford statistics for pass drop.pass instead of writing scores.
static void forward_chunk(tcl_model* m, const float* feats, const int32_t* lens, int64_t n,
                          float* scores, const DropoutCtx& drop, float* mc_mean, cudaStream_t s) {
    const tcl_dims& d = m->dims;
    Workspace& w = m->ws;
    const int L = d.max_len, dm = d.d_model, di = d.expand * d.d_model, N = d.d_state,
              R = d.dt_rank;
    const int e1 = d.enc_dims[0], e2 = d.enc_dims[1];
    const int max_rows = (int)(n * L);
    const int32_t* P = w.cu + n;  // device: number of packed rows
    int64_t& nl = m->launches;

    {
        ProfScope ps(m, TCL_PROF_PACK, s);
        launch_lens_prefix(lens, n, L, w.cu, m->d_err, s); ++nl;
        launch_pack(feats, lens, w.cu, n, L, d.d_in, kXld, w.X, nullptr, w.row_cand, s); ++nl;
    }

    auto gemm = [&](const float* X, int ldx, const float* W, int ldw, const float* b, float* Y,
                    int ldy, int K, int Nout, int epi, int site, int kind) {
        ProfScope ps(m, kind, s);
        GemmArgs g{};
        g.X = X; g.ldx = ldx; g.W = W; g.ldw = ldw; g.bias = b; g.Y = Y; g.ldy = ldy;
        g.K = K; g.N = Nout; g.max_rows = max_rows; g.p_rows = P; g.epi = epi;
        g.drop = drop; g.site = site; g.row_cand = w.row_cand; g.cu = w.cu;
        if (epi != EPI_SILU) g.drop.enabled = 0;
        launch_gemm_simt(g, s);
        ++nl;
    };
    // encoder: SiLU after linears 1 and 2 (R1), dropout sites 0, 1 (R17)
    float* E1 = w.U;      // aliases: encoder hidden states live in the mixer buffers
    float* E2 = w.Delta;
    gemm(w.X, kXld, m->W1p, kXld, m->wp.enc_b1, E1, e1, kXld, e1, EPI_SILU, 0, TCL_PROF_ENCODER);
    gemm(E1, e1, m->wp.enc_W2, e1, m->wp.enc_b2, E2, e2, e1, e2, EPI_SILU, 1, TCL_PROF_ENCODER);
    gemm(E2, e2, m->wp.enc_W3, e2, m->wp.enc_b3, w.H, dm, e2, dm, EPI_NONE, -1, TCL_PROF_ENCODER);

    for (int l = 0; l < d.n_layer; ++l) {
        const LayerPtrs& q = m->wp.layers[l];
        {
            ProfScope ps(m, TCL_PROF_LAYERNORM, s);
            launch_layernorm(w.H, dm, dm, q.ln_w, q.ln_b, d.ln_eps, w.A, nullptr, dm, max_rows, P, s); ++nl;
        }
        gemm(w.A, dm, q.W_in, dm, nullptr, w.XZ, 2 * di, dm, 2 * di, EPI_NONE, -1, TCL_PROF_IN_PROJ);
        {
            ProfScope ps(m, TCL_PROF_CONV, s);
            launch_conv_silu(w.XZ, 2 * di, q.w_conv, q.b_conv, di, d.d_conv, w.U, w.row_cand, w.cu,
                             max_rows, P, s); ++nl;
        }
        gemm(w.U, di, q.W_x, di, nullptr, w.DBC, m->ldbc, di, R + 2 * N, EPI_NONE, -1, TCL_PROF_X_PROJ);
        gemm(w.DBC, m->ldbc, q.W_dt, R, q.b_dt, w.Delta, di, R, di, EPI_SOFTPLUS, -1, TCL_PROF_DT_PROJ);
        ScanArgs sa{};
        sa.U = w.U; sa.Delta = w.Delta; sa.Z = w.XZ + di; sa.ldz = 2 * di;
        sa.BC = w.DBC; sa.ldbc = m->ldbc; sa.b_off = R; sa.c_off = R + N;
        sa.A2 = m->A2 + (size_t)l * di * N; sa.invA = m->invA + (size_t)l * di * N; sa.Dv = q.Dv;
        sa.G = w.G; sa.cu = w.cu; sa.lens = lens; sa.n = n; sa.di = di; sa.N = N; sa.disc = d.disc;
        sa.accurate = d.precision == TCL_PREC_FP32; sa.max_len = L;
        {
            ProfScope ps(m, TCL_PROF_SCAN, s);
            launch_scan(sa, s); ++nl;
        }
        gemm(w.G, di, q.W_out, di, nullptr, w.H, dm, di, dm, EPI_RESID, -1, TCL_PROF_OUT_PROJ);
    }

    HeadArgs h{};
    h.H = w.H; h.ldh = dm; h.dm = dm; h.lnf_w = m->wp.lnf_w; h.lnf_b = m->wp.lnf_b; h.eps = d.ln_eps;
    h.W1 = m->wp.dec_W1; h.b1 = m->wp.dec_b1; h.h1 = d.dec_dims[0];
    h.W2 = m->wp.dec_W2; h.b2 = m->wp.dec_b2; h.h2 = d.dec_dims[1];
    h.W3 = m->wp.dec_W3; h.b3 = m->wp.dec_b3;
    h.cu = w.cu; h.lens = lens; h.max_len = L; h.n = n; h.scores = scores; h.drop = drop;
    h.mean = mc_mean; h.m2 = w.m2;
    ProfScope ps(m, TCL_PROF_HEAD, s);
    launch_head(h, s); ++nl;
}

static int64_t chunk_cap(const tcl_model* m) {
    // bound the activation arena: <= 4M packed rows per chunk (>= 1 candidate)
    int64_t c = (int64_t)(4 << 20) / m->dims.max_len;
    return std::max<int64_t>(c, 1);
}

// ------------------------------------------------------------------------------ C ABI
extern "C" {

size_t tcl_weights_count(const tcl_dims* dims) {
    if (validate_dims(dims) != TCL_OK) return 0;
    return (size_t)weights_count_of(*dims);
}

const char* tcl_last_error(void) { return g_last_error.c_str(); }

const char* tcl_build_info(void) {
    return "libtcl: sm_100a (tcgen05/TMA) build, CUDA " TCL_STR(__CUDACC_VER_MAJOR__) "." TCL_STR(__CUDACC_VER_MINOR__);
}

tcl_status tcl_model_create(const float* weights_host, size_t n_floats, const tcl_dims* dims,
                            int cuda_device, tcl_model** out) {
    if (!weights_host || !out) return set_error(TCL_EINVAL, "null pointer");
    *out = nullptr;
    tcl_status st = validate_dims(dims);
    if (st != TCL_OK) return st;
    if ((int64_t)n_floats != weights_count_of(*dims))
        return set_error(TCL_ESHAPE, "n_floats does not match tcl_weights_count(dims)");
    CUDA_TRY(cudaSetDevice(cuda_device));
    tcl_model* m = new tcl_model();
    m->dims = *dims;
    m->device = cuda_device;
    const tcl_dims& d = m->dims;
    const int dm = d.d_model, di = d.expand * d.d_model, N = d.d_state, R = d.dt_rank;
    m->ldbc = round_up(R + 2 * N, 4);

    // fp32 blob on the device; pointers by canonical offsets (include/tcl.h)
    if ((st = dev_alloc(&m->w_dev, n_floats)) != TCL_OK) { delete m; return st; }
    cudaError_t e = cudaMemcpy(m->w_dev, weights_host, n_floats * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { tcl_model_destroy(m); return cuda_error(e, "cudaMemcpy(weights)"); }
    const float* p = m->w_dev;
    const float* hp = weights_host;
    WeightPtrs& wp = m->wp;
    std::vector<const float*> host_Alog;
#define TAKE(dst, cnt) do { wp.dst = p; p += (cnt); hp += (cnt); } while (0)
    TAKE(enc_W1, (size_t)d.enc_dims[0] * d.d_in); TAKE(enc_b1, d.enc_dims[0]);
    TAKE(enc_W2, (size_t)d.enc_dims[1] * d.enc_dims[0]); TAKE(enc_b2, d.enc_dims[1]);
    TAKE(enc_W3, (size_t)d.enc_dims[2] * d.enc_dims[1]); TAKE(enc_b3, d.enc_dims[2]);
    const float* host_W1 = weights_host;
    wp.layers.resize(d.n_layer);
    for (int l = 0; l < d.n_layer; ++l) {
        LayerPtrs& q = wp.layers[l];
#define TAKEL(dst, cnt) do { q.dst = p; p += (cnt); hp += (cnt); } while (0)
        TAKEL(ln_w, dm); TAKEL(ln_b, dm);
        TAKEL(W_in, (size_t)2 * di * dm);
        TAKEL(w_conv, (size_t)di * d.d_conv); TAKEL(b_conv, di);
        TAKEL(W_x, (size_t)(R + 2 * N) * di);
        TAKEL(W_dt, (size_t)di * R); TAKEL(b_dt, di);
        host_Alog.push_back(hp);
        TAKEL(A_log, (size_t)di * N); TAKEL(Dv, di);
        TAKEL(W_out, (size_t)dm * di);
#undef TAKEL
    }
    TAKE(lnf_w, dm); TAKE(lnf_b, dm);
    TAKE(dec_W1, (size_t)d.dec_dims[0] * dm); TAKE(dec_b1, d.dec_dims[0]);
    TAKE(dec_W2, (size_t)d.dec_dims[1] * d.dec_dims[0]); TAKE(dec_b2, d.dec_dims[1]);
    TAKE(dec_W3, (size_t)d.dec_dims[2] * d.dec_dims[1]); TAKE(dec_b3, d.dec_dims[2]);
#undef TAKE

    // Weight preprocessing (once per model): W1 zero-padded to kXld input columns; A = -exp(A_log)
    // pre-scaled by log2(e) for ex2, and 1/A for the ZOH input coefficient (reading R5, R8).
    {
        std::vector<float> w1p((size_t)d.enc_dims[0] * kXld, 0.0f);
        for (int o = 0; o < d.enc_dims[0]; ++o)
            for (int i = 0; i < d.d_in; ++i) w1p[(size_t)o * kXld + i] = host_W1[(size_t)o * d.d_in + i];
        if ((st = dev_alloc(&m->W1p, w1p.size())) != TCL_OK) { tcl_model_destroy(m); return st; }
        cudaMemcpy(m->W1p, w1p.data(), w1p.size() * sizeof(float), cudaMemcpyHostToDevice);
        std::vector<float> a2((size_t)std::max(1, d.n_layer) * di * N), ia(a2.size());
        for (int l = 0; l < d.n_layer; ++l)
            for (int j = 0; j < di * N; ++j) {
                double A = -std::exp((double)host_Alog[l][j]);
                a2[(size_t)l * di * N + j] = (float)(A * 1.4426950408889634);
                ia[(size_t)l * di * N + j] = (float)(1.0 / A);
            }
        if ((st = dev_alloc(&m->A2, a2.size())) != TCL_OK) { tcl_model_destroy(m); return st; }
        if ((st = dev_alloc(&m->invA, ia.size())) != TCL_OK) { tcl_model_destroy(m); return st; }
        cudaMemcpy(m->A2, a2.data(), a2.size() * sizeof(float), cudaMemcpyHostToDevice);
        cudaMemcpy(m->invA, ia.data(), ia.size() * sizeof(float), cudaMemcpyHostToDevice);
    }
    if ((st = dev_alloc(&m->d_err, 1)) != TCL_OK) { tcl_model_destroy(m); return st; }
    CUDA_TRY(cudaMemset(m->d_err, 0, sizeof(int)));
    if ((st = dev_alloc(&m->keys_send, 4096)) != TCL_OK) { tcl_model_destroy(m); return st; }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { tcl_model_destroy(m); return cuda_error(e, "model_create"); }
    *out = m;
    return TCL_OK;
}

tcl_status tcl_model_destroy(tcl_model* m) {
    if (!m) return TCL_OK;
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    free_workspace(m);
    comm_destroy(m);
    for (void* q : {(void*)m->w_dev, (void*)m->W1p, (void*)m->A2, (void*)m->invA, (void*)m->d_err,
                    (void*)m->topk_tmp, (void*)m->keys_send, (void*)m->keys_recv,
                    (void*)m->stage_feats, (void*)m->stage_lens, (void*)m->stage_scores,
                    (void*)m->stage_idx, (void*)m->stage_top})
        if (q) cudaFree(q);
    if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
    for (auto ev : m->chunk_events) cudaEventDestroy(ev);
    for (auto& r : m->prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto ev : m->prof_pool) cudaEventDestroy(ev);
    delete m;
    return TCL_OK;
}

tcl_status tcl_reserve(tcl_model* m, int64_t n_max, int32_t mc_passes_max) {
    if (!m || n_max < 0 || mc_passes_max < 0) return set_error(TCL_EINVAL, "bad argument");
    CUDA_TRY(cudaSetDevice(m->device));
    return ensure_workspace(m, std::min(n_max, chunk_cap(m)));
}

tcl_status tcl_score(tcl_model* m, const float* feats, const int32_t* lens, int64_t n, float* scores,
                     void* stream) {
    if (!m || n < 0) return set_error(TCL_EINVAL, "bad argument");
    if (n == 0) return TCL_OK;
    if (!feats || !lens || !scores) return set_error(TCL_EINVAL, "null pointer");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t cap = chunk_cap(m);
    tcl_status st = ensure_workspace(m, std::min(n, cap));
    if (st != TCL_OK) return st;
    DropoutCtx nodrop{};
    const size_t stride = (size_t)m->dims.max_len * m->dims.d_in;
    for (int64_t off = 0; off < n; off += cap) {
        const int64_t nc = std::min(cap, n - off);
        forward_chunk(m, feats + off * stride, lens + off, nc, scores + off, nodrop, nullptr, s);
    }
    CUDA_TRY(cudaGetLastError());
    return TCL_OK;
}

tcl_status tcl_score_mc(tcl_model* m, const float* feats, const int32_t* lens, int64_t n,
                        int32_t n_passes, uint64_t seed, int64_t index_base, float* mean,
                        float* var, void* stream) {
    if (!m || n < 0 || n_passes < 1 || index_base < 0) return set_error(TCL_EINVAL, "bad argument");
    if (n == 0) return TCL_OK;
    if (!feats || !lens || !mean || !var) return set_error(TCL_EINVAL, "null pointer");
    if (index_base + n > 0xFFFFFFFFll) return set_error(TCL_EINVAL, "index_base + n must be < 2^32");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t cap = chunk_cap(m);
    tcl_status st = ensure_workspace(m, std::min(n, cap));
    if (st != TCL_OK) return st;
    const double p = m->dims.dropout_p;
    DropoutCtx drop{};
    drop.seed = seed;
    drop.thr = (uint32_t)std::floor(p * 4294967296.0);
    drop.scale = (float)(1.0 / (1.0 - p));
    drop.enabled = 1;
    const size_t stride = (size_t)m->dims.max_len * m->dims.d_in;
    for (int64_t off = 0; off < n; off += cap) {
        const int64_t nc = std::min(cap, n - off);
        drop.index_base = index_base + off;
        for (int ps = 0; ps < n_passes; ++ps) {
            drop.pass = ps;
            forward_chunk(m, feats + off * stride, lens + off, nc, nullptr, drop, mean + off, s);
        }
        ProfScope ps(m, TCL_PROF_MC, s);
        launch_mc_finalize(m->ws.m2, nc, n_passes, var + off, s);
        ++m->launches;
    }
    CUDA_TRY(cudaGetLastError());
    return TCL_OK;
}

tcl_status tcl_topk(tcl_model* m, const float* scores, int64_t n, int32_t k, int64_t index_base,
                    int64_t* idx, float* top, void* stream) {
    if (!m || n < 0 || k <= 0 || k > 4096 || index_base < 0) return set_error(TCL_EINVAL, "bad argument");
    if (!idx || !top || (n > 0 && !scores)) return set_error(TCL_EINVAL, "null pointer");
    if (index_base + n > 0xFFFFFFFFll) return set_error(TCL_EINVAL, "index_base + n must be < 2^32");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = (cudaStream_t)stream;
    tcl_status st = ensure_topk_tmp(m, n, k);
    if (st != TCL_OK) return st;
    unsigned long long* keys = m->topk_tmp;                 // k keys
    unsigned long long* tmp = m->topk_tmp + k;
    ProfScope ps(m, TCL_PROF_TOPK, s);
    m->launches += launch_topk_keys(scores, n, k, index_base, keys, tmp, s);
    m->launches += launch_topk_merge(keys, k, k, idx, top, tmp, s);
    CUDA_TRY(cudaGetLastError());
    return TCL_OK;
}

tcl_status tcl_sync_error(tcl_model* m, void* stream) {
    if (!m) return set_error(TCL_EINVAL, "null model");
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    int flag = 0;
    CUDA_TRY(cudaMemcpy(&flag, m->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemset(m->d_err, 0, sizeof(int)));
    if (flag & ERR_LEN) return set_error(TCL_ELEN, "a candidate length outside [1, max_len] was seen");
    return TCL_OK;
}

int64_t tcl_launch_count(const tcl_model* m) { return m ? m->launches : 0; }

tcl_status tcl_profile_enable(tcl_model* m, int enable) {
    if (!m) return set_error(TCL_EINVAL, "null model");
    m->prof_on = enable ? 1 : 0;
    return TCL_OK;
}

tcl_status tcl_profile_read(tcl_model* m, double* ms_out, int64_t* launches_out, int reset) {
    if (!m || !ms_out || !launches_out) return set_error(TCL_EINVAL, "null pointer");
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaDeviceSynchronize());
    for (auto& r : m->prof_recs) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
        m->prof_ms[r.kind] += ms;
        m->prof_n[r.kind] += 1;
        m->prof_pool.push_back(r.a);
        m->prof_pool.push_back(r.b);
    }
    m->prof_recs.clear();
    for (int k = 0; k < TCL_PROF_NKINDS; ++k) { ms_out[k] = m->prof_ms[k]; launches_out[k] = m->prof_n[k]; }
    if (reset)
        for (int k = 0; k < TCL_PROF_NKINDS; ++k) { m->prof_ms[k] = 0; m->prof_n[k] = 0; }
    return TCL_OK;
}

const char* tcl_profile_name(int kind) {
    static const char* names[TCL_PROF_NKINDS] = {"pack", "encoder", "layernorm", "in_proj", "conv",
                                                 "x_proj", "dt_proj", "scan", "out_proj", "head",
                                                 "topk", "mixer", "allgather", "mc"};
    return (kind >= 0 && kind < TCL_PROF_NKINDS) ? names[kind] : "";
}

tcl_status tcl_score_host(tcl_model* m, const float* feats_h, const int32_t* lens_h, int64_t n,
                          int64_t index_base, float* scores_h, int32_t k, int64_t* idx_h, float* top_h,
                          void* stream) {
    if (!m || n < 0 || k < 0 || k > 4096 || index_base < 0) return set_error(TCL_EINVAL, "bad argument");
    if (n > 0 && (!feats_h || !lens_h || !scores_h)) return set_error(TCL_EINVAL, "null pointer");
    if (k > 0 && (!idx_h || !top_h)) return set_error(TCL_EINVAL, "null pointer");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = (cudaStream_t)stream;
    const tcl_dims& d = m->dims;
    const size_t stride = (size_t)d.max_len * d.d_in;
    if (n > m->stage_cap) {
        for (void* q : {(void*)m->stage_feats, (void*)m->stage_lens, (void*)m->stage_scores})
            if (q) cudaFree(q);
        m->stage_feats = nullptr; m->stage_lens = nullptr; m->stage_scores = nullptr; m->stage_cap = 0;
        tcl_status st;
        if ((st = dev_alloc(&m->stage_feats, (size_t)n * stride)) != TCL_OK) return st;
        if ((st = dev_alloc(&m->stage_lens, (size_t)n)) != TCL_OK) return st;
        if ((st = dev_alloc(&m->stage_scores, (size_t)n)) != TCL_OK) return st;
        m->stage_cap = n;
    }
    if (!m->stage_idx) {
        tcl_status st;
        if ((st = dev_alloc(&m->stage_idx, 4096)) != TCL_OK) return st;
        if ((st = dev_alloc(&m->stage_top, 4096)) != TCL_OK) return st;
    }
    if (!m->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
    // Pipeline: the copy stream uploads sub-chunk j+1 while the compute stream scores chunk j.
    const int64_t sub = std::max<int64_t>(1, std::min<int64_t>(chunk_cap(m), 8192));
    const int64_t nsub = (n + sub - 1) / sub;
    while ((int64_t)m->chunk_events.size() < nsub) {
        cudaEvent_t ev;
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        m->chunk_events.push_back(ev);
    }
    cudaEvent_t start_ev;
    CUDA_TRY(cudaEventCreateWithFlags(&start_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(start_ev, s));
    CUDA_TRY(cudaStreamWaitEvent(m->copy_stream, start_ev, 0));
    for (int64_t j = 0; j < nsub; ++j) {
        const int64_t off = j * sub, nc = std::min(sub, n - off);
        CUDA_TRY(cudaMemcpyAsync(m->stage_feats + off * stride, feats_h + off * stride,
                                 (size_t)nc * stride * sizeof(float), cudaMemcpyHostToDevice, m->copy_stream));
        CUDA_TRY(cudaMemcpyAsync(m->stage_lens + off, lens_h + off, (size_t)nc * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, m->copy_stream));
        CUDA_TRY(cudaEventRecord(m->chunk_events[j], m->copy_stream));
    }
    for (int64_t j = 0; j < nsub; ++j) {
        const int64_t off = j * sub, nc = std::min(sub, n - off);
        CUDA_TRY(cudaStreamWaitEvent(s, m->chunk_events[j], 0));
        tcl_status st = tcl_score(m, m->stage_feats + off * stride, m->stage_lens + off, nc,
                                  m->stage_scores + off, s);
        if (st != TCL_OK) { cudaEventDestroy(start_ev); return st; }
    }
    cudaEventDestroy(start_ev);
    if (k > 0) {
        tcl_status st = (m->comm && m->nranks > 1)
            ? tcl_topk_global(m, m->stage_scores, n, index_base, k, m->stage_idx, m->stage_top, s)
            : tcl_topk(m, m->stage_scores, n, k, index_base, m->stage_idx, m->stage_top, s);
        if (st != TCL_OK) return st;
        CUDA_TRY(cudaMemcpyAsync(idx_h, m->stage_idx, (size_t)k * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(top_h, m->stage_top, (size_t)k * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    if (n > 0)
        CUDA_TRY(cudaMemcpyAsync(scores_h, m->stage_scores, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, s));
    return tcl_sync_error(m, stream);
}

}  // extern "C"
