// api.cu -- host side of libtcl.so: the C ABI declared in include/tcl.h.
//
// Responsibilities: dims validation, weight upload and preprocessing, a grow-on-demand workspace
// arena, the per-chunk launch sequence of the forward pass, MC-dropout passes
// (CS6), top-k (a11), the host->device pipelined end-to-end call, and sticky error reporting.
// Every arithmetic step of the path runs in the kernels under kernels/; this file only launches.
#include <cuda_fp16.h>
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
#include "kernels_mixer.h"
#include "kernels_tc.h"

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
    if (d->dec_dims[0] < 4 || d->dec_dims[0] > 256 || d->dec_dims[1] < 4 || d->dec_dims[1] > 256 ||
        d->dec_dims[0] % 4 || d->dec_dims[1] % 4)
        return bad("dec_dims[0..1] must be multiples of 4 in [4, 256]");
    if (!(d->ln_eps > 0.0f)) return bad("ln_eps must be > 0");
    if (!(d->dropout_p >= 0.0f && d->dropout_p < 1.0f)) return set_error(TCL_EINVAL, "dropout_p must be in [0, 1)");
    if (d->precision != TCL_PREC_FP32 && d->precision != TCL_PREC_BF16_PROJ) return bad("unknown precision");
    if (d->disc != TCL_DISC_ZOH && d->disc != TCL_DISC_EULER_B) return bad("unknown disc");
    return TCL_OK;
}

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

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

static uint16_t f2bf(float f) {  // round to nearest even (weights are finite)
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// Upload a bf16 copy of W [rows][cols] into a zero-padded [rows_p][cols_p] device matrix.
static tcl_status upload_bf16(tcl_model* m, const float* W, int rows, int cols, int rows_p, int cols_p,
                              __nv_bfloat16** out) {
    std::vector<uint16_t> h((size_t)rows_p * cols_p, 0);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) h[(size_t)r * cols_p + c] = f2bf(W[(size_t)r * cols + c]);
    tcl_status st = dev_alloc(out, h.size());
    if (st != TCL_OK) return st;
    m->bf_allocs.push_back(*out);
    cudaError_t e = cudaMemcpy(*out, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? TCL_OK : cuda_error(e, "upload_bf16");
}

// Upload an fp16 copy of W [rows][cols] into a zero-padded [rows_p][cols_p] device matrix.
static tcl_status upload_f16(tcl_model* m, const float* W, int rows, int cols, int rows_p, int cols_p, __half** out) {
    std::vector<__half> h((size_t)rows_p * cols_p, __float2half(0.0f));
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) h[(size_t)r * cols_p + c] = __float2half_rn(W[(size_t)r * cols + c]);
    tcl_status st = dev_alloc(out, h.size());
    if (st != TCL_OK) return st;
    m->bf_allocs.push_back(*out);
    cudaError_t e = cudaMemcpy(*out, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? TCL_OK : cuda_error(e, "upload_f16");
}

// Host offsets of the canonical blob (include/tcl.h), for the bf16 copies.
struct HostW {
    const float *W1, *W2, *W3;
    std::vector<const float*> Win, Wx, Wdt, Wout;
};
static HostW host_offsets(const tcl_dims& d, const float* w) {
    const int dm = d.d_model, di = d.expand * d.d_model, N = d.d_state, R = d.dt_rank;
    HostW h;
    const float* p = w;
    h.W1 = p; p += (size_t)d.enc_dims[0] * d.d_in + d.enc_dims[0];
    h.W2 = p; p += (size_t)d.enc_dims[1] * d.enc_dims[0] + d.enc_dims[1];
    h.W3 = p; p += (size_t)d.enc_dims[2] * d.enc_dims[1] + d.enc_dims[2];
    for (int l = 0; l < d.n_layer; ++l) {
        p += 2 * dm;
        h.Win.push_back(p); p += (size_t)2 * di * dm;
        p += (size_t)di * d.d_conv + di;
        h.Wx.push_back(p); p += (size_t)(R + 2 * N) * di;
        h.Wdt.push_back(p); p += (size_t)di * R + di;
        p += (size_t)di * N + di;
        h.Wout.push_back(p); p += (size_t)dm * di;
    }
    return h;
}

static tcl_status validate_tc(const tcl_dims& d) {
    const int dm = d.d_model, di = d.expand * d.d_model;
    auto bad = [](const char* msg) { return set_error(TCL_ESHAPE, msg); };
    if (dm != 64 && dm != 128 && dm != 256) return bad("bf16 path: d_model must be 64, 128 or 256");
    if (di != 64 && di != 128 && di != 256) return bad("bf16 path: d_inner must be 64, 128 or 256");
    for (int i = 0; i < 2; ++i)
        if (d.enc_dims[i] > 256) return bad("bf16 path: enc_dims[0..1] must be <= 256");
    if (d.dt_rank > 32) return bad("bf16 path: dt_rank must be <= 32");
    if (d.d_conv != 4) return bad("bf16 path: d_conv must be 4");
    if (round_up(d.dt_rank + 2 * d.d_state, 8) > 64) return bad("bf16 path: dt_rank + 2 d_state must be <= 64");
    return TCL_OK;
}

static tcl_status setup_tc(tcl_model* m, const float* wh) {
    const tcl_dims& d = m->dims;
    tcl_status st = validate_tc(d);
    if (st != TCL_OK) return st;
    const int dm = d.d_model, di = d.expand * d.d_model, N = d.d_state, R = d.dt_rank;
    const int e1 = d.enc_dims[0], e2 = d.enc_dims[1];
    m->use_tc = 1;
    cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, m->device);
    m->nxp = round_up(R + 2 * N, 8);
    m->rp = R <= 16 ? 16 : 32;
    HostW h = host_offsets(d, wh);
    if ((st = upload_bf16(m, h.W1, e1, d.d_in, e1, kXld, &m->W1b)) != TCL_OK) return st;
    if ((st = upload_bf16(m, h.W2, e2, e1, e2, e1, &m->W2b)) != TCL_OK) return st;
    if ((st = upload_bf16(m, h.W3, dm, e2, dm, e2, &m->W3b)) != TCL_OK) return st;
    bool ok = make_tmap_bf16(&m->tmW1, m->W1b, kXld, e1, kXld * 2, 64, e1) &&
              make_tmap_bf16(&m->tmW2, m->W2b, e1, e2, (uint64_t)e1 * 2, 64, e2) &&
              make_tmap_bf16(&m->tmW3, m->W3b, e2, dm, (uint64_t)e2 * 2, 64, dm);
    for (int l = 0; l < d.n_layer && ok; ++l) {
        __nv_bfloat16 *win, *wout, *wdt;
        __half* wx;
        if ((st = upload_bf16(m, h.Win[l], 2 * di, dm, 2 * di, dm, &win)) != TCL_OK) return st;
        if ((st = upload_bf16(m, h.Wout[l], dm, di, dm, di, &wout)) != TCL_OK) return st;
        if ((st = upload_f16(m, h.Wx[l], R + 2 * N, di, m->nxp, di, &wx)) != TCL_OK) return st;
        if ((st = upload_bf16(m, h.Wdt[l], di, R, di, m->rp, &wdt)) != TCL_OK) return st;
        m->Winb.push_back(win); m->Woutb.push_back(wout); m->Wxh.push_back(wx); m->Wdtb.push_back(wdt);
        CUtensorMap a, b;
        ok = make_tmap_bf16(&a, win, dm, 2 * di, (uint64_t)dm * 2, 64, inconv_channels(di)) &&
             make_tmap_bf16(&b, wout, di, dm, (uint64_t)di * 2, 64, dm);
        m->tmWin.push_back(a);
        m->tmWout.push_back(b);
    }
    if (!ok) return set_error(TCL_ECUDA, "cuTensorMapEncodeTiled failed (weights)");
    return TCL_OK;
}

// ------------------------------------------------------------------------------ fp32 path: 3xTF32
// The fp32 path's row GEMMs (encoder linears, in_proj, out_proj) run on the tensor cores as 3xTF32
// (gemm_tf32.cu); a GEMM whose weight slice does not fit the kernel stays on the SIMT kernel (a
// per-model choice by dims, never by n: scores stay batch-invariant).  W_hi / W_lo are split on the
// device from the fp32 weights (at creation and after every Adam update).
static int tf32_pick_bn(int n, int k, bool full_row) {
    if (full_row) return tf32_gemm_supported(n, k) ? n : 0;
    for (int bn : {256, 128, 64, 32})
        if (bn <= n && n % bn == 0 && tf32_gemm_supported(bn, k)) return bn;
    return 0;
}

static void refresh_tf32(tcl_model* m, cudaStream_t s) {
    for (Tf32W& t : m->tfw)
        if (t.bn) launch_tf32_split(t.w, (int64_t)t.n * t.k, t.hi, t.lo, s);
}

static tcl_status setup_tf32(tcl_model* m) {
    const tcl_dims& d = m->dims;
    const int dm = d.d_model, di = d.expand * d.d_model, e1 = d.enc_dims[0], e2 = d.enc_dims[1];
    // full-row tiles (LayerNorm in the epilogue) for the GEMMs that write the residual stream: at
    // d_model <= 128 the row fits one 3xTF32 tile (forward_chunk fuses only where they exist)
    const bool fuse_ln = dm <= 128 && d.n_layer > 0;
    struct G { const float* w; int n, k; bool full; };
    std::vector<G> gs = {{m->W1p, e1, kXld, false}, {m->wp.enc_W2, e2, e1, false}, {m->wp.enc_W3, dm, e2, fuse_ln}};
    for (int l = 0; l < d.n_layer; ++l) {
        gs.push_back({m->wp.layers[l].W_in, 2 * di, dm, false});
        gs.push_back({m->wp.layers[l].W_out, dm, di, fuse_ln && l + 1 < d.n_layer});
    }
    size_t total = 0;
    for (const G& g : gs) total += 2 * (size_t)g.n * g.k;
    tcl_status st = dev_alloc(&m->tf_split, total);
    if (st != TCL_OK) return st;
    float* p = m->tf_split;
    for (const G& g : gs) {
        Tf32W t;
        t.w = g.w; t.n = g.n; t.k = g.k; t.hi = p; t.lo = p + (size_t)g.n * g.k;
        p += 2 * (size_t)g.n * g.k;
        t.bn = tf32_pick_bn(g.n, g.k, g.full);
        if (t.bn && !(make_tmap_f32_sw64(&t.tm_hi, t.hi, g.k, g.n, (uint64_t)g.k * 4, t.bn) &&
                      make_tmap_f32_sw64(&t.tm_lo, t.lo, g.k, g.n, (uint64_t)g.k * 4, t.bn)))
            return set_error(TCL_ECUDA, "cuTensorMapEncodeTiled failed (tf32 weights)");
        m->tfw.push_back(t);
    }
    refresh_tf32(m, 0);
    const cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? TCL_OK : cuda_error(e, "setup_tf32");
}

// ------------------------------------------------------------------------------ workspace

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
    TAKE(pooled, chunk_n * dm);
    TAKE(dh1, chunk_n * d.dec_dims[0]);
    TAKE(dh2, chunk_n * d.dec_dims[1]);
    TAKE(dsc, chunk_n);
    TAKE(lens_mc, chunk_n);
    TAKE(scan_ctr, 64);
    if (m->kb) {
        TAKE(Hk, rows * dm);
        TAKE(E1k, rows * d.enc_dims[0]);
        TAKE(E2k, rows * d.enc_dims[1]);
        TAKE(Lat, rows * m->ad_ld);
        TAKE(pooled_k, chunk_n * dm);
        TAKE(dh1k, chunk_n * d.dec_dims[0]);
        // columns a .. ad_ld of Lat are never written: zero them once (they meet zero weights)
        if (cudaMemset(w.Lat, 0, sizeof(float) * (size_t)(rows * m->ad_ld)) != cudaSuccess) {
            free_workspace(m);
            return set_error(TCL_ECUDA, "cudaMemset(Lat)");
        }
    }
    if (!m->use_tc) {   // 3xTF32 A operands of the fp32 path (box {32, 128})
        const int e1 = d.enc_dims[0], e2 = d.enc_dims[1];
        const bool ok = make_tmap_f32_sw64(&w.tmX32, w.X, kXld, rows, kXld * 4, 128) &&
                        make_tmap_f32_sw64(&w.tmE1f, w.U, e1, rows, (uint64_t)e1 * 4, 128) &&
                        make_tmap_f32_sw64(&w.tmE2f, w.Delta, e2, rows, (uint64_t)e2 * 4, 128) &&
                        make_tmap_f32_sw64(&w.tmA32, w.A, dm, rows, (uint64_t)dm * 4, 128) &&
                        make_tmap_f32_sw64(&w.tmG32, w.G, di, rows, (uint64_t)di * 4, 128);
        if (!ok) { free_workspace(m); return set_error(TCL_ECUDA, "cuTensorMapEncodeTiled failed (fp32 workspace)"); }
    }
    if (m->use_tc) {
        const int64_t xzw = std::max<int64_t>(2 * di, (int64_t)d.enc_dims[0] + d.enc_dims[1]);
        TAKE(Xb, rows * kXld);
        TAKE(XZb, rows * xzw);
        TAKE(Ab, rows * dm);
        TAKE(Gb, rows * di);
        w.pk_ld = mixer_packet_bytes(di, d.d_state);
        TAKE(Pk, rows * w.pk_ld);
        TAKE(GZb, rows * di);
        const int e1 = d.enc_dims[0], e2 = d.enc_dims[1];
        __nv_bfloat16* E1b = w.XZb;
        __nv_bfloat16* E2b = w.XZb + rows * e1;
        bool ok = make_tmap_bf16(&w.tmXb, w.Xb, kXld, rows, kXld * 2, 64, 128) &&
                  make_tmap_bf16(&w.tmE1b, E1b, e1, rows, (uint64_t)e1 * 2, 64, 128) &&
                  make_tmap_bf16(&w.tmE2b, E2b, e2, rows, (uint64_t)e2 * 2, 64, 128) &&
                  make_tmap_bf16(&w.tmAb, w.Ab, dm, rows, (uint64_t)dm * 2, 64, 128) &&
                  make_tmap_bf16(&w.tmGb, w.Gb, di, rows, (uint64_t)di * 2, 64, 128);
        // output maps (only used when the output tile is >= 64 columns wide)
        if (e1 >= 64) ok = ok && make_tmap_bf16(&w.tmE1o, E1b, e1, rows, (uint64_t)e1 * 2, 64, 32);
        if (e2 >= 64) ok = ok && make_tmap_bf16(&w.tmE2o, E2b, e2, rows, (uint64_t)e2 * 2, 64, 32);
        ok = ok && make_tmap_bf16(&w.tmXZo, w.XZb, 2 * di, rows, (uint64_t)2 * di * 2, 64, 32);
        // k_inconv stores: SiLU(z) -> GZb, u -> the packet's first di columns (2-byte elements)
        ok = ok && make_tmap_bf16(&w.tmGZs, w.GZb, di, rows, (uint64_t)di * 2, 64, 125) &&
             make_tmap_bf16(&w.tmUs, w.Pk, (uint64_t)w.pk_ld / 2, rows, (uint64_t)w.pk_ld, 64, 125);
        ok = ok && make_tmap_f32(&w.tmHf, w.H, dm, rows, (uint64_t)dm * 4, 32, 32);
        ok = ok && make_tmap_bf16(&w.tmAo, w.Ab, dm, rows, (uint64_t)dm * 2, 64, 32);
        if (inconv_split(di) == 2) ok = ok && make_tmap_bf16(&w.tmAbS2, w.Ab, dm, rows, (uint64_t)dm * 2, 64, 64);

        if (!ok) { free_workspace(m); return set_error(TCL_ECUDA, "cuTensorMapEncodeTiled failed (workspace)"); }
    }
#undef TAKE
    w.cap_n = chunk_n;
    w.rows = rows;
    ++m->ws_gen;   // captured graphs that baked in the old buffers are stale now
    return TCL_OK;
}

static tcl_status ensure_topk_tmp(tcl_model* m, int64_t n, int k) {
    size_t need = (size_t)k + topk_tmp_keys(std::max<int64_t>(n, 1), k) + (size_t)k;
    if (need <= m->topk_tmp_cap) return TCL_OK;
    ++m->ws_gen;
    if (m->topk_tmp) cudaFree(m->topk_tmp);
    m->topk_tmp = nullptr;
    m->topk_tmp_cap = 0;
    tcl_status st = dev_alloc(&m->topk_tmp, need);
    if (st != TCL_OK) return st;
    m->topk_tmp_cap = need;
    return TCL_OK;
}

// ------------------------------------------------------------------------------ head
// LN_f + masked mean (warp per candidate), then the decoder MLP (head.cu: one
// launch below 8,192 candidates; above, the pool kernel and three small fp32 GEMMs over the
// candidates); MC passes fold each pass' score into (mean, M2) with Welford's update (batched MC
// passes: the scores of all passes, then one reduction, launch_mc_reduce).
static void run_head(tcl_model* m, const int32_t* lens, int64_t n, float* scores, const DropoutCtx& drop,
                     float* mc_mean, cudaStream_t s, bool lnf_in_ab = false) {
    const tcl_dims& d = m->dims;
    Workspace& w = m->ws;
    const int dm = d.d_model, h1 = d.dec_dims[0], h2 = d.dec_dims[1];
    int64_t& nl = m->launches;
    ProfScope ps(m, TCL_PROF_HEAD, s);
    {   // the fused head: pool + decoder + score / Welford in one launch (bit-identical to the below)
        HeadArgs a{};
        a.H = w.H; a.ldh = dm;
        a.F = lnf_in_ab ? w.Ab : nullptr; a.ldf = dm;
        a.lnf_w = m->wp.lnf_w; a.lnf_b = m->wp.lnf_b; a.eps = d.ln_eps;
        a.cu = w.cu; a.lens = lens; a.max_len = d.max_len; a.n = n;
        a.dm = dm; a.h1 = h1; a.h2 = h2;
        a.W1 = m->wp.dec_W1; a.b1 = m->wp.dec_b1; a.W2 = m->wp.dec_W2; a.b2 = m->wp.dec_b2;
        a.W3 = m->wp.dec_W3; a.b3 = m->wp.dec_b3;
        a.drop = drop;
        a.scores = scores; a.mc_mean = mc_mean; a.m2 = w.m2; a.pooled = w.pooled;
        if (launch_head_fused(a, s)) {
            ++nl;
            return;
        }
    }
    if (lnf_in_ab)  // bf16 path: the last GEMM epilogue already wrote LN_f(H) (bf16) into Ab
        launch_pool_bf16(w.Ab, dm, dm, w.cu, lens, d.max_len, n, w.pooled, s);
    else
        launch_pool(w.H, dm, dm, m->wp.lnf_w, m->wp.lnf_b, d.ln_eps, w.cu, lens, d.max_len, n, w.pooled, s);
    ++nl;
    auto dec = [&](const float* X, int K, const float* W, const float* b, float* Y, int Nout, int epi, int site) {
        GemmArgs g{};
        g.X = X; g.ldx = K; g.W = W; g.ldw = K; g.bias = b; g.Y = Y; g.ldy = Nout; g.K = K; g.N = Nout;
        g.max_rows = (int)n; g.p_rows = nullptr; g.rows_const = (int)n; g.rows_are_cands = 1; g.epi = epi;
        g.drop = drop; g.site = site;
        if (epi != EPI_SILU) g.drop.enabled = 0;
        launch_gemm_simt(g, s);
        ++nl;
    };
    dec(w.pooled, dm, m->wp.dec_W1, m->wp.dec_b1, w.dh1, h1, EPI_SILU, 2);
    dec(w.dh1, h1, m->wp.dec_W2, m->wp.dec_b2, w.dh2, h2, EPI_SILU, 3);
    float* out = mc_mean ? w.dsc : scores;
    dec(w.dh2, h2, m->wp.dec_W3, m->wp.dec_b3, out, 1, EPI_NONE, -1);
    if (mc_mean) launch_welford(w.dsc, lens, d.max_len, n, drop.pass, mc_mean, w.m2, s);
    else launch_mask_invalid(lens, d.max_len, n, scores, s);
    ++nl;
}

// ------------------------------------------------------------------------------ forward
// fp32 launch helpers shared by the one-column and the KB + AC two-column forward.
struct F32Run {
    tcl_model* m;      // owner of the workspace (the AC column for KB + AC)
    int max_rows;
    const int32_t* P;  // device: packed row count
    DropoutCtx drop;
    cudaStream_t s;
    const int32_t* lens;
    int64_t n;
    // one-column forward at d_model 128: the LayerNorm that follows a GEMM writing the residual
    // stream (LN_0 after the encoder, LN_{l+1} after out_proj_l) runs in that GEMM's epilogue
    bool fuse_ln = false;
    const float* ln_g = nullptr;   // set by the caller of gemm(..., EPI_RESID_LN / EPI_LN, ...)
    const float* ln_b = nullptr;
    bool tf32 = false;             // one-column model: row GEMMs on the 3xTF32 tensor-core kernel

    // 3xTF32 row GEMM (gemm_tf32.cu).  epi 0: Y = acc; 1: Y = SiLU(acc + b) [+ dropout, site];
    // 3: Y (the residual stream, ldy = N) = [Y +] acc + b, then LN -> ws.A when lng != nullptr.
    void gemm_tf(const CUtensorMap& amap, const Tf32W& tw, const float* b, float* Y, int ldy, int epi, int site,
                 int kind, bool residual = false, const float* lng = nullptr, const float* lnb = nullptr) const {
        ProfScope ps(m, kind, s);
        Tf32GemmParams p{};
        p.n_tiles = tw.n / tw.bn; p.p_rows = P; p.epi = epi; p.bias = b;
        p.Y = Y; p.ldy = ldy; p.H = Y; p.ldh = ldy; p.residual = residual ? 1 : 0;
        p.out = lng ? m->ws.A : nullptr; p.ldo = tw.n; p.ln_g = lng; p.ln_b = lnb; p.eps = m->dims.ln_eps;
        p.drop = drop; p.site = site; p.row_cand = m->ws.row_cand; p.cu = m->ws.cu;
        if (epi != 1) p.drop.enabled = 0;
        const cudaError_t e = launch_gemm_tf32(amap, tw.tm_hi, tw.tm_lo, p, tw.bn, tw.k, m->num_sms, s);
        if (e != cudaSuccess && m->fwd_err == cudaSuccess) m->fwd_err = e;
        ++m->launches;
    }

    // Y = epi(X W^T [+ X2 W2^T] + b) over the packed rows (or over the n candidates: cands = true)
    void gemm(const float* X, int ldx, const float* W, int ldw, const float* b, float* Y, int ldy, int K,
              int Nout, int epi, int site, int kind, const float* X2 = nullptr, int ldx2 = 0,
              const float* W2 = nullptr, int K2 = 0, bool cands = false, bool dropout = true) const {
        ProfScope ps(m, kind, s);
        GemmArgs g{};
        if (epi == EPI_RESID_LN || epi == EPI_LN) {
            g.ln_g = ln_g; g.ln_b = ln_b; g.ln_eps = m->dims.ln_eps; g.Y2 = m->ws.A; g.ldy2 = Nout;
        }
        g.X = X; g.ldx = ldx; g.W = W; g.ldw = ldw; g.bias = b; g.Y = Y; g.ldy = ldy;
        g.K = K; g.N = Nout; g.epi = epi; g.drop = drop; g.site = site;
        if (cands) { g.max_rows = (int)n; g.rows_const = (int)n; g.rows_are_cands = 1; }
        else { g.max_rows = max_rows; g.p_rows = P; g.row_cand = m->ws.row_cand; g.cu = m->ws.cu; }
        g.X2 = X2; g.ldx2 = ldx2; g.W2 = W2; g.ldw2 = K2; g.K2 = K2;
        if (epi != EPI_SILU || !dropout) g.drop.enabled = 0;
        launch_gemm_simt(g, s);
        ++m->launches;
    }
    // Lat = SiLU(V hkb + c) for one Eq. 7 site (no dropout: the adapters' inner activation)
    void lateral(const AdapterSite& a, const float* hkb, int ldh, bool cands) const {
        gemm(hkb, ldh, a.V, a.ldv, a.c, m->ws.Lat, m->ad_ld, a.ldv, m->ad_rank, EPI_SILU, -1,
             TCL_PROF_LATERAL, nullptr, 0, nullptr, 0, cands, false);
    }
    // One Mamba block of column `col` on the residual stream H (pre-norm, in_proj, conv, x_proj,
    // dt_proj, scan, out_proj + residual); `site` adds the Eq. 7 lateral to out_proj's sums.
    void layer(const tcl_model* col, int l, float* H, const AdapterSite* site) const {
        const tcl_dims& d = m->dims;
        Workspace& w = m->ws;
        const int dm = d.d_model, di = d.expand * d.d_model, N = d.d_state, R = d.dt_rank;
        const LayerPtrs& q = col->wp.layers[l];
        if (!fuse_ln) {   // (fused: the previous GEMM's epilogue already wrote LN_l(H) into A)
            ProfScope ps(m, TCL_PROF_LAYERNORM, s);
            launch_layernorm(H, dm, dm, q.ln_w, q.ln_b, d.ln_eps, w.A, nullptr, dm, max_rows, P, s,
                             /*gemm_epilogue_order=*/true); ++m->launches;
        }
        const Tf32W* tw_in = (tf32 && !site) ? &m->tfw[3 + 2 * l] : nullptr;
        const Tf32W* tw_out = (tf32 && !site) ? &m->tfw[4 + 2 * l] : nullptr;
        if (tw_in && tw_in->bn) gemm_tf(w.tmA32, *tw_in, nullptr, w.XZ, 2 * di, 0, -1, TCL_PROF_IN_PROJ);
        else gemm(w.A, dm, q.W_in, dm, nullptr, w.XZ, 2 * di, dm, 2 * di, EPI_NONE, -1, TCL_PROF_IN_PROJ);
        if (mixer_f32_supported(di, N, R, d.d_conv)) {
            // conv + x_proj + dt_proj + scan in one kernel (mixer_f32.cu): the sequential scan, or the
            // warp-shuffle chunked scan across L (TCL_OPT_SCAN; chosen per model, never per n)
            ProfScope ps(m, TCL_PROF_MIXER, s);
            MixerF32Args a{};
            a.XZ = w.XZ; a.ldxz = 2 * di; a.G = w.G; a.ldg = di;
            a.A2 = col->A2 + (size_t)l * di * N; a.invA = col->invA + (size_t)l * di * N; a.Dv = q.Dv;
            a.w_conv = q.w_conv; a.b_conv = q.b_conv; a.W_x = q.W_x; a.W_dt = q.W_dt; a.b_dt = q.b_dt;
            a.cu = w.cu; a.n = n; a.DI = di; a.N = N; a.R = R; a.disc = d.disc; a.max_len = d.max_len;
            // auto = sequential: measured, the chunked scan's shuffle steps cost more than the
            // parallelism they buy at every BASELINE configuration
            if (m->scan_mode == 2) launch_mixer_lpar(a, s);
            else launch_mixer_f32(a, m->num_sms, s);   // errors surface through cudaGetLastError in forward_any
            ++m->launches;
        } else {
        {
            ProfScope ps(m, TCL_PROF_CONV, s);
            launch_conv_silu(w.XZ, 2 * di, q.w_conv, q.b_conv, di, d.d_conv, w.U, w.row_cand, w.cu,
                             max_rows, P, s); ++m->launches;
        }
        gemm(w.U, di, q.W_x, di, nullptr, w.DBC, m->ldbc, di, R + 2 * N, EPI_NONE, -1, TCL_PROF_X_PROJ);
        gemm(w.DBC, m->ldbc, q.W_dt, R, q.b_dt, w.Delta, di, R, di, EPI_SOFTPLUS, -1, TCL_PROF_DT_PROJ);
        ScanArgs sa{};
        sa.U = w.U; sa.Delta = w.Delta; sa.Z = w.XZ + di; sa.ldz = 2 * di;
        sa.BC = w.DBC; sa.ldbc = m->ldbc; sa.b_off = R; sa.c_off = R + N;
        sa.A2 = col->A2 + (size_t)l * di * N; sa.invA = col->invA + (size_t)l * di * N; sa.Dv = q.Dv;
        sa.G = w.G; sa.cu = w.cu; sa.lens = lens; sa.n = n; sa.di = di; sa.N = N; sa.disc = d.disc;
        sa.accurate = d.precision == TCL_PREC_FP32; sa.max_len = d.max_len;
        {
            ProfScope ps(m, TCL_PROF_SCAN, s);
            launch_scan(sa, s); ++m->launches;
        }
        }
        if (site) {
            gemm(w.G, di, q.W_out, di, nullptr, H, dm, di, dm, EPI_RESID, -1, TCL_PROF_OUT_PROJ, w.Lat, m->ad_ld,
                 site->Ua, m->ad_ld);
        } else if (tw_out && tw_out->bn) {   // out_proj + residual (+ the next LayerNorm) on 3xTF32
            const bool ln = fuse_ln && l + 1 < d.n_layer;
            gemm_tf(w.tmG32, *tw_out, nullptr, H, dm, 3, -1, TCL_PROF_OUT_PROJ, true,
                    ln ? col->wp.layers[l + 1].ln_w : nullptr, ln ? col->wp.layers[l + 1].ln_b : nullptr);
        } else if (fuse_ln && l + 1 < d.n_layer) {
            F32Run r2 = *this;
            r2.ln_g = col->wp.layers[l + 1].ln_w;
            r2.ln_b = col->wp.layers[l + 1].ln_b;
            r2.gemm(w.G, di, q.W_out, di, nullptr, H, dm, di, dm, EPI_RESID_LN, -1, TCL_PROF_OUT_PROJ);
        } else {
            gemm(w.G, di, q.W_out, di, nullptr, H, dm, di, dm, EPI_RESID, -1, TCL_PROF_OUT_PROJ);
        }
    }
};

// KB + AC two-column forward (§6 Eq. 7, reading R23), fp32 path.  Site by site the KB
// (frozen, deterministic) runs first; Lat = SiLU(V h^KB_{i-1} + c) is formed from the KB's input
// to that site and enters the AC's GEMM as a second K segment against diag(alpha) U (the lateral
// sum joins the same accumulators, before bias and activation).  MC dropout: AC column only.
static void forward_chunk_kbac(tcl_model* m, const float* feats, const int32_t* lens, int64_t n,
                               float* scores, const DropoutCtx& drop, float* mc_mean, cudaStream_t s,
                               int64_t n_src = 0) {
    const tcl_dims& d = m->dims;
    Workspace& w = m->ws;
    const tcl_model* kb = m->kb;
    const int L = d.max_len, dm = d.d_model;
    const int e1 = d.enc_dims[0], e2 = d.enc_dims[1], h1 = d.dec_dims[0], h2 = d.dec_dims[1];
    const int ld = m->ad_ld;
    F32Run r{m, (int)(n * L), w.cu + n, drop, s, lens, n};
    const std::vector<AdapterSite>& ad = m->ad;
    {
        ProfScope ps(m, TCL_PROF_PACK, s);
        launch_lens_prefix(lens, n, L, w.cu, m->d_err, s); ++m->launches;
        launch_pack(feats, lens, w.cu, n, L, d.d_in, kXld, w.X, nullptr, w.row_cand, s, n_src); ++m->launches;
    }
    float* E1 = w.U;
    float* E2 = w.Delta;
    // encoder layer 1: h^KB_0 = the features
    r.gemm(w.X, kXld, kb->W1p, kXld, kb->wp.enc_b1, w.E1k, e1, kXld, e1, EPI_SILU, 0, TCL_PROF_ENCODER, nullptr, 0,
           nullptr, 0, false, false);
    r.lateral(ad[0], w.X, kXld, false);
    r.gemm(w.X, kXld, m->W1p, kXld, m->wp.enc_b1, E1, e1, kXld, e1, EPI_SILU, 0, TCL_PROF_ENCODER, w.Lat, ld, ad[0].Ua, ld);
    // encoder layer 2
    r.lateral(ad[1], w.E1k, e1, false);
    r.gemm(w.E1k, e1, kb->wp.enc_W2, e1, kb->wp.enc_b2, w.E2k, e2, e1, e2, EPI_SILU, 1, TCL_PROF_ENCODER, nullptr, 0,
           nullptr, 0, false, false);
    r.gemm(E1, e1, m->wp.enc_W2, e1, m->wp.enc_b2, E2, e2, e1, e2, EPI_SILU, 1, TCL_PROF_ENCODER, w.Lat, ld, ad[1].Ua, ld);
    // encoder layer 3 (no activation, R1)
    r.lateral(ad[2], w.E2k, e2, false);
    r.gemm(w.E2k, e2, kb->wp.enc_W3, e2, kb->wp.enc_b3, w.Hk, dm, e2, dm, EPI_NONE, -1, TCL_PROF_ENCODER);
    r.gemm(E2, e2, m->wp.enc_W3, e2, m->wp.enc_b3, w.H, dm, e2, dm, EPI_NONE, -1, TCL_PROF_ENCODER, w.Lat, ld,
           ad[2].Ua, ld);
    // Mamba blocks: the lateral reads the KB's block input, so it is formed before the KB block runs
    DropoutCtx nodrop = drop;
    nodrop.enabled = 0;
    F32Run rk = r;
    rk.drop = nodrop;
    for (int l = 0; l < d.n_layer; ++l) {
        r.lateral(ad[3 + l], w.Hk, dm, false);
        rk.layer(kb, l, w.Hk, nullptr);
        r.layer(m, l, w.H, &ad[3 + l]);
    }
    // head: KB pooled + dec1 (its inputs to the AC's dec1 / dec2 laterals), then the AC decoder
    {
        ProfScope ps(m, TCL_PROF_HEAD, s);
        launch_pool(w.Hk, dm, dm, kb->wp.lnf_w, kb->wp.lnf_b, d.ln_eps, w.cu, lens, L, n, w.pooled_k, s);
        launch_pool(w.H, dm, dm, m->wp.lnf_w, m->wp.lnf_b, d.ln_eps, w.cu, lens, L, n, w.pooled, s);
        m->launches += 2;
    }
    r.gemm(w.pooled_k, dm, kb->wp.dec_W1, dm, kb->wp.dec_b1, w.dh1k, h1, dm, h1, EPI_SILU, 2, TCL_PROF_HEAD, nullptr,
           0, nullptr, 0, true, false);
    r.lateral(ad[3 + d.n_layer], w.pooled_k, dm, true);
    r.gemm(w.pooled, dm, m->wp.dec_W1, dm, m->wp.dec_b1, w.dh1, h1, dm, h1, EPI_SILU, 2, TCL_PROF_HEAD, w.Lat, ld,
           ad[3 + d.n_layer].Ua, ld, true);
    r.lateral(ad[4 + d.n_layer], w.dh1k, h1, true);
    r.gemm(w.dh1, h1, m->wp.dec_W2, h1, m->wp.dec_b2, w.dh2, h2, h1, h2, EPI_SILU, 3, TCL_PROF_HEAD, w.Lat, ld,
           ad[4 + d.n_layer].Ua, ld, true);
    float* out = mc_mean ? w.dsc : scores;
    r.gemm(w.dh2, h2, m->wp.dec_W3, h2, m->wp.dec_b3, out, 1, h2, 1, EPI_NONE, -1, TCL_PROF_HEAD, nullptr, 0, nullptr,
           0, true);
    if (mc_mean) launch_welford(w.dsc, lens, L, n, drop.pass, mc_mean, w.m2, s);
    else launch_mask_invalid(lens, L, n, scores, s);
    ++m->launches;
}

// One chunk of candidates [0, n) (pointers already offset).  If mc_mean != nullptr the head
// accumulates Welford statistics for pass drop.pass instead of writing scores.
static void forward_chunk(tcl_model* m, const float* feats, const int32_t* lens, int64_t n,
                          float* scores, const DropoutCtx& drop, float* mc_mean, cudaStream_t s,
                          int64_t n_src = 0) {
    const tcl_dims& d = m->dims;
    Workspace& w = m->ws;
    const int L = d.max_len, dm = d.d_model;
    const int e1 = d.enc_dims[0], e2 = d.enc_dims[1];
    F32Run r{m, (int)(n * L), w.cu + n, drop, s, lens, n};
    {
        ProfScope ps(m, TCL_PROF_PACK, s);
        launch_lens_prefix(lens, n, L, w.cu, m->d_err, s); ++m->launches;
        launch_pack(feats, lens, w.cu, n, L, d.d_in, kXld, w.X, nullptr, w.row_cand, s, n_src); ++m->launches;
    }
    // encoder: SiLU after linears 1 and 2 (R1), dropout sites 0, 1 (R17)
    float* E1 = w.U;      // aliases: encoder hidden states live in the mixer buffers
    float* E2 = w.Delta;
    r.tf32 = !m->tfw.empty();
    // LN_l fused into the GEMM that writes the residual stream: the SIMT kernels' LN epilogue
    // (d_model 128), or full-row 3xTF32 tiles for the encoder's linear 3 and every out_proj but the last
    bool tf_rows = r.tf32 && m->tfw[2].bn == dm;
    for (int l = 0; l + 1 < d.n_layer && tf_rows; ++l) tf_rows = m->tfw[4 + 2 * l].bn == dm;
    r.fuse_ln = d.n_layer > 0 && (dm == 128 || tf_rows);
    if (r.tf32 && m->tfw[0].bn) r.gemm_tf(w.tmX32, m->tfw[0], m->wp.enc_b1, E1, e1, 1, 0, TCL_PROF_ENCODER);
    else r.gemm(w.X, kXld, m->W1p, kXld, m->wp.enc_b1, E1, e1, kXld, e1, EPI_SILU, 0, TCL_PROF_ENCODER);
    if (r.tf32 && m->tfw[1].bn) r.gemm_tf(w.tmE1f, m->tfw[1], m->wp.enc_b2, E2, e2, 1, 1, TCL_PROF_ENCODER);
    else r.gemm(E1, e1, m->wp.enc_W2, e1, m->wp.enc_b2, E2, e2, e1, e2, EPI_SILU, 1, TCL_PROF_ENCODER);
    if (r.tf32 && m->tfw[2].bn) {   // linear 3 (+ LN_0 at d_model 128)
        r.gemm_tf(w.tmE2f, m->tfw[2], m->wp.enc_b3, w.H, dm, 3, -1, TCL_PROF_ENCODER, false,
                  r.fuse_ln ? m->wp.layers[0].ln_w : nullptr, r.fuse_ln ? m->wp.layers[0].ln_b : nullptr);
    } else if (r.fuse_ln) {
        F32Run r0 = r;
        r0.ln_g = m->wp.layers[0].ln_w;
        r0.ln_b = m->wp.layers[0].ln_b;
        r0.gemm(E2, e2, m->wp.enc_W3, e2, m->wp.enc_b3, w.H, dm, e2, dm, EPI_LN, -1, TCL_PROF_ENCODER);
    } else {
        r.gemm(E2, e2, m->wp.enc_W3, e2, m->wp.enc_b3, w.H, dm, e2, dm, EPI_NONE, -1, TCL_PROF_ENCODER);
    }
    for (int l = 0; l < d.n_layer; ++l) r.layer(m, l, w.H, nullptr);
    run_head(m, lens, n, scores, drop, mc_mean, s);
}

static bool debug_sync_on() {   // TCL_DEBUG_SYNC=1: synchronise and check after every launch (debugging)
    static const bool on = [] { const char* e = getenv("TCL_DEBUG_SYNC"); return e && e[0] == '1'; }();
    return on;
}

static tcl_status debug_sync(const char* where, cudaStream_t s) {
    if (!debug_sync_on()) return TCL_OK;
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, where);
    fprintf(stderr, "[tcl] %s ok\n", where);
    return TCL_OK;
}

// The bf16 projection path (precision == TCL_PREC_BF16_PROJ): tcgen05 GEMMs with fused
// epilogues for the encoder / in_proj / out_proj(+LN), one fused mixer kernel per layer.
static tcl_status forward_chunk_tc(tcl_model* m, const float* feats, const int32_t* lens, int64_t n,
                                   float* scores, const DropoutCtx& drop, float* mc_mean, cudaStream_t s,
                                   int64_t n_src = 0) {
    const tcl_dims& d = m->dims;
    Workspace& w = m->ws;
    const int L = d.max_len, dm = d.d_model, di = d.expand * d.d_model, N = d.d_state, R = d.dt_rank;
    const int e1 = d.enc_dims[0], e2 = d.enc_dims[1];
    const int32_t* P = w.cu + n;
    int64_t& nl = m->launches;
    const int64_t rows = w.rows;
    __nv_bfloat16* E1b = w.XZb;
    __nv_bfloat16* E2b = w.XZb + rows * e1;
    cudaError_t e;
    {
        ProfScope ps(m, TCL_PROF_PACK, s);
        launch_lens_prefix(lens, n, L, w.cu, m->d_err, s); ++nl;
        launch_pack(feats, lens, w.cu, n, L, d.d_in, kXld, nullptr, w.Xb, w.row_cand, s, n_src); ++nl;
    }
    if (debug_sync("pack", s) != TCL_OK) return TCL_ECUDA;
    auto base = [&]() {
        TcGemmParams p{};
        p.n_tiles = 1; p.p_rows = P; p.drop = drop; p.drop.enabled = 0; p.row_cand = w.row_cand; p.cu = w.cu;
        p.eps = d.ln_eps;
        return p;
    };
    auto kb_of = [](int K) { return (K + 63) / 64; };
    {
        ProfScope ps(m, TCL_PROF_ENCODER, s);
        if (enc12_supported(e1, e2, d.d_in)) {
            // linears 1 and 2 chained: E1 stays in shared memory (gemm_tc_enc.cu)
            EncParams ep{};
            ep.p_rows = P; ep.b1 = m->wp.enc_b1; ep.b2 = m->wp.enc_b2; ep.drop = drop;
            ep.row_cand = w.row_cand; ep.cu = w.cu;
            if ((e = launch_enc12(w.tmXb, m->tmW1, m->tmW2, w.tmE2o, ep, e1, e2, m->num_sms, s)) != cudaSuccess)
                return cuda_error(e, "enc12");
            ++nl;
            if (debug_sync("enc12", s) != TCL_OK) return TCL_ECUDA;
        } else {
        TcGemmParams p = base();
        p.epi = TC_EPI_BF16; p.bias = m->wp.enc_b1; p.act_silu = 1; p.out = E1b; p.ldo = e1;
        p.drop.enabled = drop.enabled; p.site = 0;
        if ((e = launch_gemm_tc(w.tmXb, m->tmW1, w.tmE1o, p, e1, 1, m->num_sms, s)) != cudaSuccess) return cuda_error(e, "enc1");
        ++nl;
        if (debug_sync("enc1", s) != TCL_OK) return TCL_ECUDA;
        p.bias = m->wp.enc_b2; p.out = E2b; p.ldo = e2; p.site = 1;
        if ((e = launch_gemm_tc(w.tmE1b, m->tmW2, w.tmE2o, p, e2, kb_of(e1), m->num_sms, s)) != cudaSuccess) return cuda_error(e, "enc2");
        ++nl;
        if (debug_sync("enc2", s) != TCL_OK) return TCL_ECUDA;
        }
        TcGemmParams q = base();
        q.epi = TC_EPI_RESID_LN; q.bias = m->wp.enc_b3; q.residual = 0; q.H = w.H; q.ldh = dm;
        q.out = (d.n_layer > 0 || dm >= 128) ? w.Ab : nullptr; q.ldo = dm;
        q.ln_g = d.n_layer > 0 ? m->wp.layers[0].ln_w : m->wp.lnf_w;
        q.ln_b = d.n_layer > 0 ? m->wp.layers[0].ln_b : m->wp.lnf_b;
        e = dm >= 128 ? launch_gemm_tc_ln(w.tmE2b, m->tmW3, w.tmHf, w.tmAo, q, dm, kb_of(e2), m->num_sms, s)
                      : launch_gemm_tc(w.tmE2b, m->tmW3, w.tmXZo, q, dm, kb_of(e2), m->num_sms, s);
        if (e != cudaSuccess) return cuda_error(e, "enc3");
        ++nl;
        if (debug_sync("enc3", s) != TCL_OK) return TCL_ECUDA;
    }
    CUDA_TRY(cudaMemsetAsync(w.scan_ctr, 0, sizeof(int) * (size_t)d.n_layer, s));   // k_scan work groups
    for (int l = 0; l < d.n_layer; ++l) {
        const LayerPtrs& q = m->wp.layers[l];
        {   // in_proj + SiLU(z) + conv + SiLU (inconv.cu): x never leaves the SM
            ProfScope ps(m, TCL_PROF_IN_PROJ, s);
            InConvParams a{};
            a.p_rows = P; a.row_cand = w.row_cand; a.w_conv = q.w_conv; a.b_conv = q.b_conv;
            a.DI = di; a.d_conv = d.d_conv;
            const CUtensorMap& amap = inconv_split(di) == 2 ? w.tmAbS2 : w.tmAb;
            if ((e = launch_inconv(amap, m->tmWin[l], w.tmGZs, w.tmUs, a, dm, m->num_sms, s)) != cudaSuccess)
                return cuda_error(e, "inconv");
            ++nl;
            if (debug_sync("inconv", s) != TCL_OK) return TCL_ECUDA;
        }
        {   // x_proj + dt_proj + softplus -> packet (mixer_split.cu)
            ProfScope ps(m, TCL_PROF_XDT, s);
            XdtArgs a{};
            a.Pk = w.Pk; a.pk_ld = w.pk_ld; a.b_dt = q.b_dt;
            a.Wx_h = m->Wxh[l]; a.Wdt_b = m->Wdtb[l];
            a.cu = w.cu; a.n = n; a.DI = di; a.N = N; a.R = R; a.RP = m->rp; a.max_len = L;
            if ((e = launch_xdt(a, m->num_sms, s)) != cudaSuccess) return cuda_error(e, "xdt");
            ++nl;
            if (debug_sync("xdt", s) != TCL_OK) return TCL_ECUDA;
        }
        {   // the selective scan + D skip + gate (SFU-bound)
            ProfScope ps(m, TCL_PROF_SCAN, s);
            ScanBf16Args a{};
            a.Pk = w.Pk; a.GZ = w.GZb; a.G = w.Gb;
            a.A2 = m->A2 + (size_t)l * di * N; a.invA = m->invA + (size_t)l * di * N; a.Dv = q.Dv;
            a.cu = w.cu; a.n = n; a.DI = di; a.N = N; a.disc = d.disc; a.work_counter = w.scan_ctr + l;
            if ((e = launch_scan_bf16(a, m->num_sms, s)) != cudaSuccess) return cuda_error(e, "scan");
            ++nl;
            if (debug_sync("scan", s) != TCL_OK) return TCL_ECUDA;
        }
        {
            ProfScope ps(m, TCL_PROF_OUT_PROJ, s);
            TcGemmParams p = base();
            p.epi = TC_EPI_RESID_LN; p.residual = 1; p.H = w.H; p.ldh = dm;
            const bool last = l + 1 == d.n_layer;
            // last layer (LN kernel): write only LN_f(H) (bf16, the head's input), not H itself
            p.out = (last && dm < 128) ? nullptr : w.Ab; p.ldo = dm;
            p.skip_h_store = last && dm >= 128;
            p.ln_g = last ? m->wp.lnf_w : m->wp.layers[l + 1].ln_w;
            p.ln_b = last ? m->wp.lnf_b : m->wp.layers[l + 1].ln_b;
            e = dm >= 128 ? launch_gemm_tc_ln(w.tmGb, m->tmWout[l], w.tmHf, w.tmAo, p, dm, kb_of(di), m->num_sms, s)
                          : launch_gemm_tc(w.tmGb, m->tmWout[l], w.tmXZo, p, dm, kb_of(di), m->num_sms, s);
            if (e != cudaSuccess) return cuda_error(e, "out_proj");
            ++nl;
            if (debug_sync("out_proj", s) != TCL_OK) return TCL_ECUDA;
        }
    }
    run_head(m, lens, n, scores, drop, mc_mean, s, /*lnf_in_ab=*/dm >= 128);
    return TCL_OK;
}

// n_src > 0: candidate i takes the features of candidate i mod n_src (batched MC passes).
static tcl_status forward_any(tcl_model* m, const float* feats, const int32_t* lens, int64_t n, float* scores,
                              const DropoutCtx& drop, float* mc_mean, cudaStream_t s, int64_t n_src = 0) {
    if (m->use_tc) {
        tcl_status st = forward_chunk_tc(m, feats, lens, n, scores, drop, mc_mean, s, n_src);
        if (st != TCL_OK) return st;
        return debug_sync("forward_chunk_tc", s);
    }
    m->fwd_err = cudaSuccess;
    if (m->kb) forward_chunk_kbac(m, feats, lens, n, scores, drop, mc_mean, s, n_src);
    else forward_chunk(m, feats, lens, n, scores, drop, mc_mean, s, n_src);
    if (m->fwd_err != cudaSuccess) return cuda_error(m->fwd_err, "forward_chunk: 3xTF32 GEMM launch refused");
    const cudaError_t e = cudaGetLastError();   // launch-configuration errors of the fp32 kernels
    if (e != cudaSuccess) return cuda_error(e, m->kb ? "forward_chunk_kbac" : "forward_chunk");
    return debug_sync(m->kb ? "forward_chunk_kbac" : "forward_chunk", s);
}

// ------------------------------------------------------------------------------ CUDA graphs
// A repeated call (same kind, pointers, sizes, seeds, scratch generation) is replayed from a
// CUDA graph: the first occurrence launches directly, the second is captured (on a private stream,
// thread-local capture mode) and launched on the caller's stream, later ones only replay.  The
// launch sequence of a call depends on nothing but its key, so a replay is bit-identical to the
// direct launches (tested).  Per-stage profiling and TCL_DEBUG_SYNC always launch directly.
static bool debug_sync_on();
constexpr size_t kMaxGraphs = 8, kMaxSeen = 16;

template <class F>
static tcl_status run_graphed(tcl_model* m, const GraphKey& key, cudaStream_t s, F&& enqueue) {
    if (!m->use_graphs || m->prof_on || debug_sync_on()) return enqueue(s);
    for (GraphEntry& g : m->graphs) {
        if (g.key == key) {
            g.stamp = ++m->graph_clock;
            CUDA_TRY(cudaGraphLaunch(g.exec, s));
            m->launches += g.launches;
            return TCL_OK;
        }
    }
    auto it = std::find(m->seen.begin(), m->seen.end(), key);
    if (it == m->seen.end()) {   // first occurrence: direct launches
        if (m->seen.size() >= kMaxSeen) m->seen.erase(m->seen.begin());
        m->seen.push_back(key);
        return enqueue(s);
    }
    m->seen.erase(it);
    if (!m->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&m->cap_stream, cudaStreamNonBlocking));
    const int64_t before = m->launches;
    CUDA_TRY(cudaStreamBeginCapture(m->cap_stream, cudaStreamCaptureModeThreadLocal));
    const tcl_status st = enqueue(m->cap_stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(m->cap_stream, &graph);
    const int64_t nl = m->launches - before;
    m->launches = before;
    if (st != TCL_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (ce != cudaSuccess) return cuda_error(ce, "graph capture");
    GraphEntry g;
    g.key = key;
    g.launches = nl;
    const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return cuda_error(ie, "graph instantiate");
    if (m->graphs.size() >= kMaxGraphs) {   // evict the least recently used
        auto lru = std::min_element(m->graphs.begin(), m->graphs.end(),
                                    [](const GraphEntry& a, const GraphEntry& b) { return a.stamp < b.stamp; });
        cudaGraphExecDestroy(lru->exec);
        m->graphs.erase(lru);
    }
    g.stamp = ++m->graph_clock;
    m->graphs.push_back(g);
    CUDA_TRY(cudaGraphLaunch(g.exec, s));
    m->launches += nl;
    return TCL_OK;
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
    if (d.precision == TCL_PREC_BF16_PROJ) {
        if ((st = setup_tc(m, weights_host)) != TCL_OK) { tcl_model_destroy(m); return st; }
    } else if ((st = setup_tf32(m)) != TCL_OK) {
        tcl_model_destroy(m);
        return st;
    }
    if ((st = dev_alloc(&m->d_err, 1)) != TCL_OK) { tcl_model_destroy(m); return st; }
    CUDA_TRY(cudaMemset(m->d_err, 0, sizeof(int)));
    if ((st = dev_alloc(&m->keys_send, 4096)) != TCL_OK) { tcl_model_destroy(m); return st; }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { tcl_model_destroy(m); return cuda_error(e, "model_create"); }
    *out = m;
    return TCL_OK;
}

static int64_t adapters_count_of(const tcl_dims& d, int a, std::vector<AdapterSite>* sites) {
    const int ins[3] = {d.d_in, d.enc_dims[0], d.enc_dims[1]};
    const int outs[3] = {d.enc_dims[0], d.enc_dims[1], d.d_model};
    int64_t c = 0;
    for (int s = 0; s < 5 + d.n_layer; ++s) {
        int in, out;
        if (s < 3) { in = ins[s]; out = outs[s]; }
        else if (s < 3 + d.n_layer) { in = out = d.d_model; }
        else if (s == 3 + d.n_layer) { in = d.d_model; out = d.dec_dims[0]; }
        else { in = d.dec_dims[0]; out = d.dec_dims[1]; }
        if (sites) sites->push_back(AdapterSite{nullptr, nullptr, nullptr, in, out, s == 0 ? kXld : in});
        c += (int64_t)a * in + a + (int64_t)out * a + out;
    }
    return c;
}

size_t tcl_adapters_count(const tcl_dims* dims, int32_t adapter_rank) {
    if (!dims || adapter_rank < 1) return 0;
    return (size_t)adapters_count_of(*dims, adapter_rank, nullptr);
}

tcl_status tcl_model_create_kbac(const float* kb_weights_host, const float* ac_weights_host, size_t n_floats,
                                 const float* adapters_host, size_t n_adapter_floats, int32_t adapter_rank,
                                 const tcl_dims* dims, int cuda_device, tcl_model** out) {
    if (!kb_weights_host || !ac_weights_host || !adapters_host || !out) return set_error(TCL_EINVAL, "null pointer");
    *out = nullptr;
    tcl_status st = validate_dims(dims);
    if (st != TCL_OK) return st;
    if (dims->precision != TCL_PREC_FP32) return set_error(TCL_ESHAPE, "KB+AC: only TCL_PREC_FP32 is supported");
    if (adapter_rank < 1 || adapter_rank > 64) return set_error(TCL_ESHAPE, "adapter_rank must be in [1, 64]");
    std::vector<AdapterSite> sites;
    if ((int64_t)n_adapter_floats != adapters_count_of(*dims, adapter_rank, &sites))
        return set_error(TCL_ESHAPE, "n_adapter_floats does not match tcl_adapters_count(dims, adapter_rank)");
    tcl_model *kb = nullptr, *m = nullptr;
    if ((st = tcl_model_create(kb_weights_host, n_floats, dims, cuda_device, &kb)) != TCL_OK) return st;
    if ((st = tcl_model_create(ac_weights_host, n_floats, dims, cuda_device, &m)) != TCL_OK) {
        tcl_model_destroy(kb);
        return st;
    }
    m->kb = kb;
    const int a = adapter_rank, ld = round_up(a, 16);
    m->ad_rank = a;
    m->ad_ld = ld;
    // device layout per site: V [a][ldv] (zero-padded), c [a], Ua = diag(alpha) U [out][ld] (zero-padded)
    std::vector<float> host;
    std::vector<size_t> offs;
    const float* p = adapters_host;
    for (AdapterSite& st_ : sites) {
        const float *V = p, *c = p + (size_t)a * st_.in, *U = c + a, *alpha = U + (size_t)st_.out * a;
        p = alpha + st_.out;
        offs.push_back(host.size());
        for (int j = 0; j < a; ++j)
            for (int i = 0; i < st_.ldv; ++i) host.push_back(i < st_.in ? V[(size_t)j * st_.in + i] : 0.0f);
        for (int j = 0; j < a; ++j) host.push_back(c[j]);
        for (int o = 0; o < st_.out; ++o)
            for (int j = 0; j < ld; ++j) host.push_back(j < a ? alpha[o] * U[(size_t)o * a + j] : 0.0f);
    }
    if ((st = dev_alloc(&m->ad_dev, host.size())) != TCL_OK) { tcl_model_destroy(m); return st; }
    cudaError_t e = cudaMemcpy(m->ad_dev, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { tcl_model_destroy(m); return cuda_error(e, "cudaMemcpy(adapters)"); }
    for (size_t k = 0; k < sites.size(); ++k) {
        AdapterSite& q = sites[k];
        q.V = m->ad_dev + offs[k];
        q.c = q.V + (size_t)a * q.ldv;
        q.Ua = q.c + a;
    }
    m->ad = sites;
    *out = m;
    return TCL_OK;
}

static void free_train(tcl_model* m);

tcl_status tcl_model_destroy(tcl_model* m) {
    if (!m) return TCL_OK;
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    free_workspace(m);
    comm_destroy(m);
    for (GraphEntry& g : m->graphs) cudaGraphExecDestroy(g.exec);
    if (m->cap_stream) cudaStreamDestroy(m->cap_stream);
    for (void* q : {(void*)m->w_dev, (void*)m->W1p, (void*)m->A2, (void*)m->invA, (void*)m->d_err,
                    (void*)m->topk_tmp, (void*)m->keys_send, (void*)m->keys_recv,
                    (void*)m->stage_feats, (void*)m->stage_lens, (void*)m->stage_scores,
                    (void*)m->stage_idx, (void*)m->stage_top})
        if (q) cudaFree(q);
    if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
    for (auto ev : m->chunk_events) cudaEventDestroy(ev);
    for (void* q : m->bf_allocs) cudaFree(q);
    if (m->rdu_scratch) cudaFree(m->rdu_scratch);
    if (m->eval_cols) cudaFree(m->eval_cols);
    if (m->ad_dev) cudaFree(m->ad_dev);
    if (m->tf_split) cudaFree(m->tf_split);
    free_train(m);
    if (m->kb) tcl_model_destroy(m->kb);
    for (auto& r : m->prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto ev : m->prof_pool) cudaEventDestroy(ev);
    delete m;
    return TCL_OK;
}

tcl_status tcl_reserve(tcl_model* m, int64_t n_max, int32_t mc_passes_max) {
    if (!m || n_max < 0 || mc_passes_max < 0) return set_error(TCL_EINVAL, "bad argument");
    CUDA_TRY(cudaSetDevice(m->device));
    const int64_t cap = chunk_cap(m);
    // tcl_score_mc batches its passes: min(n, cap / p) * p <= min(n * p, cap) virtual candidates
    // (n_max >= cap: the whole arena; otherwise n_max * p < 2^22 * 2^31 cannot overflow)
    if (n_max >= cap) return ensure_workspace(m, cap);
    return ensure_workspace(m, std::min(n_max * std::max<int64_t>(1, mc_passes_max), cap));
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
    GraphKey key;
    key.kind = 0;
    key.p[0] = feats; key.p[1] = lens; key.p[2] = scores;
    key.v[0] = n;
    key.gen = m->ws_gen;
    st = run_graphed(m, key, s, [&](cudaStream_t cs) -> tcl_status {
        DropoutCtx nodrop{};
        const size_t stride = (size_t)m->dims.max_len * m->dims.d_in;
        for (int64_t off = 0; off < n; off += cap) {
            const int64_t nc = std::min(cap, n - off);
            tcl_status st2 = forward_any(m, feats + off * stride, lens + off, nc, scores + off, nodrop, nullptr, cs);
            if (st2 != TCL_OK) return st2;
        }
        CUDA_TRY(cudaGetLastError());
        return TCL_OK;
    });
    return st;
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
    // the passes run batched: one forward over passes x nc virtual candidates per chunk of nc
    const int64_t cb = std::max<int64_t>(1, cap / n_passes);
    const bool batched = cb * n_passes <= cap;
    tcl_status st = ensure_workspace(m, batched ? std::min(n, cb) * n_passes : std::min(n, cap));
    if (st != TCL_OK) return st;
    GraphKey key;
    key.kind = 1;
    key.p[0] = feats; key.p[1] = lens; key.p[2] = mean; key.p[3] = var;
    key.v[0] = n; key.v[1] = n_passes; key.v[2] = (int64_t)seed; key.v[3] = index_base;
    key.gen = m->ws_gen;
    return run_graphed(m, key, s, [&](cudaStream_t cs) -> tcl_status {
        const double p = m->dims.dropout_p;
        DropoutCtx drop{};
        drop.seed = seed;
        drop.thr = (uint32_t)std::floor(p * 4294967296.0);
        drop.scale = (float)(1.0 / (1.0 - p));
        drop.enabled = 1;
        const size_t stride = (size_t)m->dims.max_len * m->dims.d_in;
        if (batched) {
            // virtual candidate v = ps * nc + i is candidate i of pass ps: replicated lengths, the
            // pack reads features i = v mod nc, the dropout counter takes (ps, i) from v (pass_n);
            // every kernel is batch-invariant, so each pass scores exactly as a launch of its own
            for (int64_t off = 0; off < n; off += cb) {
                const int64_t nc = std::min(cb, n - off);
                const int64_t nv = nc * n_passes;
                for (int ps = 0; ps < n_passes; ++ps)
                    CUDA_TRY(cudaMemcpyAsync(m->ws.lens_mc + ps * nc, lens + off, sizeof(int32_t) * (size_t)nc,
                                             cudaMemcpyDeviceToDevice, cs));
                drop.index_base = index_base + off;
                drop.pass = 0;
                drop.pass_n = (uint32_t)nc;
                tcl_status st2 = forward_any(m, feats + off * stride, m->ws.lens_mc, nv, m->ws.dsc, drop, nullptr, cs, nc);
                if (st2 != TCL_OK) return st2;
                ProfScope ps(m, TCL_PROF_MC, cs);
                launch_mc_reduce(m->ws.dsc, lens + off, m->dims.max_len, nc, n_passes, mean + off, var + off, cs);
                ++m->launches;
            }
            CUDA_TRY(cudaGetLastError());
            return TCL_OK;
        }
        for (int64_t off = 0; off < n; off += cap) {
            const int64_t nc = std::min(cap, n - off);
            drop.index_base = index_base + off;
            for (int ps = 0; ps < n_passes; ++ps) {
                drop.pass = ps;
                tcl_status st2 = forward_any(m, feats + off * stride, lens + off, nc, nullptr, drop, mean + off, cs);
                if (st2 != TCL_OK) return st2;
            }
            ProfScope ps(m, TCL_PROF_MC, cs);
            launch_mc_finalize(m->ws.m2, nc, n_passes, var + off, cs);
            ++m->launches;
        }
        CUDA_TRY(cudaGetLastError());
        return TCL_OK;
    });
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
    GraphKey key;
    key.kind = 2;
    key.p[0] = scores; key.p[1] = idx; key.p[2] = top;
    key.v[0] = n; key.v[1] = k; key.v[2] = index_base;
    key.gen = m->ws_gen;
    return run_graphed(m, key, s, [&](cudaStream_t cs) -> tcl_status {
        unsigned long long* keys = m->topk_tmp;                 // k keys
        unsigned long long* tmp = m->topk_tmp + k;
        ProfScope ps(m, TCL_PROF_TOPK, cs);
        m->launches += launch_topk_keys(scores, n, k, index_base, keys, tmp, cs);   // sorted best k, 0-padded
        m->launches += launch_topk_decode(keys, k, idx, top, cs);
        CUDA_TRY(cudaGetLastError());
        return TCL_OK;
    });
}

tcl_status tcl_topk_score(tcl_model* m, const float* scores, const float* lat, const int64_t* off, const float* w,
                          int64_t n_tasks, int32_t max_task_len, const int32_t* ks_host, int32_t n_k,
                          double* result, void* stream) {
    if (!m || n_tasks < 1 || n_k < 1 || n_k > 16 || max_task_len < 1) return set_error(TCL_EINVAL, "bad argument");
    if (max_task_len > 16384) return set_error(TCL_ESHAPE, "max_task_len > 16384");
    if (!scores || !lat || !off || !w || !ks_host || !result) return set_error(TCL_EINVAL, "null pointer");
    tcl::TopkEvalKs ks{};
    ks.n = n_k;
    for (int j = 0; j < n_k; ++j) {
        if (ks_host[j] < 1) return set_error(TCL_EINVAL, "k < 1");
        ks.k[j] = ks_host[j];
    }
    CUDA_TRY(cudaSetDevice(m->device));
    const size_t need = (size_t)(n_k + 1) * (size_t)n_tasks;
    if (need > m->eval_cols_cap) {
        if (m->eval_cols) cudaFree(m->eval_cols);
        m->eval_cols = nullptr;
        m->eval_cols_cap = 0;
        CUDA_TRY(cudaMalloc(&m->eval_cols, need * sizeof(double)));
        m->eval_cols_cap = need;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
    cudaError_t e = tcl::launch_topk_eval(scores, lat, off, w, n_tasks, max_task_len, ks, m->eval_cols, result,
                                          m->d_err, sms, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_error(e, "topk_score");
    m->launches += 2;
    return TCL_OK;
}

tcl_status tcl_rdu_select(tcl_model* m, const float* pool, const int32_t* ops, int64_t n_pool, const float* lab,
                          int64_t n_lab, int32_t n_ops, int32_t budget_total, int64_t* out, int32_t* n_out,
                          void* stream) {
    if (!m || n_pool < 0 || n_lab < 0 || budget_total < 0 || n_ops < 1 || n_ops > 256)
        return set_error(TCL_EINVAL, "bad argument");
    if (!out || !n_out || (n_pool > 0 && (!pool || !ops)) || (n_lab > 0 && !lab))
        return set_error(TCL_EINVAL, "null pointer");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (n_pool == 0 || budget_total == 0) {
        CUDA_TRY(cudaMemsetAsync(n_out, 0, sizeof(int32_t), s));
        return TCL_OK;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
    if (n_pool > (int64_t)4096 * sms) return set_error(TCL_ESHAPE, "n_pool exceeds 4096 * SM count");
    const size_t need = rdu_scratch_bytes(sms, n_ops);
    if (need > m->rdu_scratch_cap) {
        if (m->rdu_scratch) cudaFree(m->rdu_scratch);
        m->rdu_scratch = nullptr;
        m->rdu_scratch_cap = 0;
        CUDA_TRY(cudaMalloc(&m->rdu_scratch, need));
        m->rdu_scratch_cap = need;
    }
    cudaError_t e = launch_rdu_select(pool, ops, n_pool, lab, n_lab, n_ops, budget_total, out, n_out,
                                      m->rdu_scratch, sms, s);
    if (e != cudaSuccess) return cuda_error(e, "rdu_select");
    m->launches += 2;
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
    if (flag & ERR_TASK) return set_error(TCL_ESHAPE, "a task with 0 or more than max_task_len candidates was seen");
    return TCL_OK;
}

int64_t tcl_launch_count(const tcl_model* m) { return m ? m->launches : 0; }

tcl_status tcl_set_option(tcl_model* m, int32_t option, int64_t value) {
    if (!m) return set_error(TCL_EINVAL, "null model");
    if (option == TCL_OPT_GRAPHS) {
        if (value != 0 && value != 1) return set_error(TCL_EINVAL, "TCL_OPT_GRAPHS takes 0 or 1");
        m->use_graphs = (int)value;
        return TCL_OK;
    }
    if (option == TCL_OPT_SCAN) {
        if (value < 0 || value > 2) return set_error(TCL_EINVAL, "TCL_OPT_SCAN takes 0 (auto), 1 or 2");
        const tcl_dims& d = m->dims;
        const int di = d.expand * d.d_model;
        if (value == 2 && !mixer_lpar_supported(di, d.d_state, d.dt_rank, d.d_conv, d.max_len))
            return set_error(TCL_ESHAPE, "chunked scan: needs max_len <= 32, d_inner 64 or 128, d_conv 4");
        m->scan_mode = (int)value;
        for (tcl_model* q = m->kb; q; q = q->kb) q->scan_mode = (int)value;
        return TCL_OK;
    }
    return set_error(TCL_EINVAL, "unknown option");
}

tcl_status tcl_debug_read(tcl_model* m, const char* name, float* out, int64_t rows, int64_t cols) {
    if (!m || !name || !out || rows < 0 || cols < 1) return set_error(TCL_EINVAL, "bad argument");
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaDeviceSynchronize());
    const Workspace& w = m->ws;
    if (rows > w.rows) return set_error(TCL_EINVAL, "rows exceed the workspace");
    const std::string nm(name);
    if (m->use_tc && (nm == "XZ" || nm == "GZ" || nm == "U" || nm == "DELTA" || nm == "BC")) {
        // bf16 path: u, Delta (fp16), B, C (fp32) in the mixer packet rows; SiLU(z) (bf16) in GZb;
        // x in XZb as [P][di] (bf16) only without the fused inmix kernel (which keeps x on chip)
        const int di = m->dims.expand * m->dims.d_model, N = m->dims.d_state;
        if (nm == "XZ") return set_error(TCL_EINVAL, "bf16 path: x stays on chip (k_inconv)");
        const int want = nm == "XZ" ? 2 * di : (nm == "BC" ? 2 * N : di);
        if (cols != want) return set_error(TCL_EINVAL, "cols does not match the buffer");
        std::vector<uint8_t> pk((size_t)rows * w.pk_ld);
        CUDA_TRY(cudaMemcpy(pk.data(), w.Pk, pk.size(), cudaMemcpyDeviceToHost));
        std::vector<uint16_t> xb((size_t)rows * di), zb((size_t)rows * di);
        if (nm == "XZ") CUDA_TRY(cudaMemcpy(xb.data(), w.XZb, xb.size() * 2, cudaMemcpyDeviceToHost));
        if (nm == "XZ" || nm == "GZ") CUDA_TRY(cudaMemcpy(zb.data(), w.GZb, zb.size() * 2, cudaMemcpyDeviceToHost));
        auto bf = [](uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; };
        auto hf = [](uint16_t h) { __half_raw r; r.x = h; return __half2float(__half(r)); };
        for (int64_t r = 0; r < rows; ++r) {
            const uint8_t* row = pk.data() + (size_t)r * w.pk_ld;
            for (int c = 0; c < want; ++c) {
                float v;
                uint16_t h;
                if (nm == "XZ" && c < di) v = bf(xb[(size_t)r * di + c]);
                else if (nm == "XZ") v = bf(zb[(size_t)r * di + c - di]);
                else if (nm == "GZ") v = bf(zb[(size_t)r * di + c]);
                else if (nm == "U") { memcpy(&h, row + 2 * c, 2); v = hf(h); }
                else if (nm == "DELTA") { memcpy(&h, row + 2 * di + 2 * c, 2); v = hf(h); }
                else memcpy(&v, row + 4 * di + 4 * c, 4);
                out[(size_t)r * want + c] = v;
            }
        }
        return TCL_OK;
    }
    const void* src = nullptr;
    bool bf = false;
    if (nm == "H") src = w.H;
    else if (nm == "A") { src = m->use_tc ? (const void*)w.Ab : (const void*)w.A; bf = m->use_tc; }
    else if (nm == "XZ") { src = m->use_tc ? (const void*)w.XZb : (const void*)w.XZ; bf = m->use_tc; }
    else if (nm == "G") { src = m->use_tc ? (const void*)w.Gb : (const void*)w.G; bf = m->use_tc; }
    else if (nm == "U" && !m->use_tc) src = w.U;
    else if (nm == "DELTA" && !m->use_tc) src = w.Delta;
    if (!src) return set_error(TCL_EINVAL, "unknown buffer name");
    const size_t cnt = (size_t)rows * cols;
    if (!bf) {
        CUDA_TRY(cudaMemcpy(out, src, cnt * sizeof(float), cudaMemcpyDeviceToHost));
    } else {
        std::vector<uint16_t> h(cnt);
        CUDA_TRY(cudaMemcpy(h.data(), src, cnt * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < cnt; ++i) {
            uint32_t u = (uint32_t)h[i] << 16;
            memcpy(&out[i], &u, 4);
        }
    }
    return TCL_OK;
}

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
                                                 "topk", "mixer", "allgather", "mc", "lateral", "xdt"};
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
    // Host->device copies run ~3-4x faster than scoring per candidate, so the sub-chunks grow
    // geometrically (x4): only the first, small copy is exposed, and the scoring runs as few,
    // large launches (no per-launch ramp/tail of many small grids).
    const int64_t cap = std::max<int64_t>(1, chunk_cap(m));
    std::vector<int64_t> sub_off, sub_n;
    // (small batches are one launch sequence: splitting them costs more in launch-bound kernels
    // than the exposed copy of the whole batch)
    for (int64_t off = 0, sz = std::min<int64_t>(cap, n <= 16384 ? n : 4096); off < n;) {
        const int64_t nc = std::min(sz, n - off);
        sub_off.push_back(off);
        sub_n.push_back(nc);
        off += nc;
        sz = std::min<int64_t>(cap, sz * 4);
    }
    const int64_t nsub = (int64_t)sub_off.size();
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
        const int64_t off = sub_off[j], nc = sub_n[j];
        CUDA_TRY(cudaMemcpyAsync(m->stage_feats + off * stride, feats_h + off * stride,
                                 (size_t)nc * stride * sizeof(float), cudaMemcpyHostToDevice, m->copy_stream));
        CUDA_TRY(cudaMemcpyAsync(m->stage_lens + off, lens_h + off, (size_t)nc * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, m->copy_stream));
        CUDA_TRY(cudaEventRecord(m->chunk_events[j], m->copy_stream));
    }
    for (int64_t j = 0; j < nsub; ++j) {
        const int64_t off = sub_off[j], nc = sub_n[j];
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

// ------------------------------------------------------------------------------ training
// SURVEY §8(f) NEXT #3 (reading R24): one LambdaRank (Eq. 6) training step of the fp32 model --
// forward with saved activations, loss + score gradient, backward of every layer, Adam (§7.1.3).

static void free_train(tcl_model* m) {
    if (!m->tr) return;
    if (m->tr->graph) cudaGraphExecDestroy(m->tr->graph);
    if (m->tr->gstream) cudaStreamDestroy(m->tr->gstream);
    if (m->tr->ev_in) cudaEventDestroy(m->tr->ev_in);
    if (m->tr->ev_out) cudaEventDestroy(m->tr->ev_out);
    for (void* p : m->tr->allocs) cudaFree(p);
    delete m->tr;
    m->tr = nullptr;
}

tcl_status tcl_train_init(tcl_model* m, int64_t n_max, float lr, float beta1, float beta2, float eps,
                          float sigma_rank) {
    if (!m || n_max < 1 || !(lr > 0.f) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) ||
        !(eps > 0.f) || !(sigma_rank > 0.f))
        return set_error(TCL_EINVAL, "bad argument");
    if (m->use_tc || m->kb) return set_error(TCL_ESHAPE, "training: TCL_PREC_FP32 one-column models only");
    if (n_max > chunk_cap(m)) return set_error(TCL_ESHAPE, "training: n_max exceeds one chunk");
    CUDA_TRY(cudaSetDevice(m->device));
    free_train(m);
    tcl_status st = ensure_workspace(m, n_max);
    if (st != TCL_OK) return st;
    const tcl_dims& d = m->dims;
    const int64_t rows = n_max * d.max_len;
    const int dm = d.d_model, di = d.expand * d.d_model, N = d.d_state;
    const int e1 = d.enc_dims[0], e2 = d.enc_dims[1], h1 = d.dec_dims[0], h2 = d.dec_dims[1];
    TrainState* t = new TrainState();
    m->tr = t;
    t->cap_n = n_max;
    t->rows = rows;
    t->nW = weights_count_of(d);
    t->lr = lr; t->b1 = beta1; t->b2 = beta2; t->eps = eps; t->sigma = sigma_rank;
    auto take = [&](float** p, int64_t cnt) -> tcl_status {
        tcl_status s2 = dev_alloc(p, (size_t)std::max<int64_t>(cnt, 1));
        if (s2 == TCL_OK) t->allocs.push_back(*p);
        return s2;
    };
#define TT(p, cnt) if ((st = take(&t->p, (cnt))) != TCL_OK) { free_train(m); return st; }
    TT(g, t->nW); TT(mA, t->nW); TT(vA, t->nW);
    TT(E1pre, rows * e1); TT(E1, rows * e1); TT(E2pre, rows * e2); TT(E2, rows * e2);
    for (int l = 0; l <= d.n_layer; ++l) {
        float* p = nullptr;
        if ((st = take(&p, rows * dm)) != TCL_OK) { free_train(m); return st; }
        t->Hin.push_back(p);
        if (l == d.n_layer) break;
        const int64_t sizes[7] = {rows * dm, rows * 2 * di, rows * di, rows * m->ldbc, rows * di, rows * di * N, rows * di};
        std::vector<float*>* lists[7] = {&t->Aln, &t->XZ, &t->U, &t->DBC, &t->Delta, &t->S, &t->G};
        for (int k = 0; k < 7; ++k) {
            if ((st = take(&p, sizes[k])) != TCL_OK) { free_train(m); return st; }
            lists[k]->push_back(p);
        }
    }
    TT(pooled, n_max * dm); TT(d1pre, n_max * h1); TT(d1, n_max * h1); TT(d2pre, n_max * h2); TT(d2, n_max * h2);
    TT(scores, n_max);
    TT(dH, rows * dm); TT(dA, rows * dm); TT(dXZ, rows * 2 * di); TT(dU, rows * di); TT(dpre, rows * di);
    TT(dDpre, rows * di); TT(dDBC, rows * m->ldbc); TT(dG, rows * di); TT(xhdy, rows * dm);
    TT(dE1, rows * e1); TT(dE2, rows * e2);
    TT(ds, n_max); TT(dd1, n_max * h1); TT(dd2, n_max * h2); TT(dpooled, n_max * dm);
    TT(dAlog_part, n_max * di * N); TT(dD_part, n_max * di); TT(gloss, n_max); TT(loss, 1);
    t->part_cap = (size_t)8 << 20;
    TT(part, (int64_t)t->part_cap);
    TT(corr_dev, 2);
    {
        int* p = nullptr;
        if ((st = dev_alloc(&p, 1)) != TCL_OK) { free_train(m); return st; }
        t->allocs.push_back(p);
        t->step_dev = p;
    }
#undef TT
    CUDA_TRY(cudaMemset(t->step_dev, 0, sizeof(int)));
    CUDA_TRY(cudaStreamCreateWithFlags(&t->gstream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&t->ev_in, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&t->ev_out, cudaEventDisableTiming));
    CUDA_TRY(cudaMemset(t->mA, 0, sizeof(float) * t->nW));
    CUDA_TRY(cudaMemset(t->vA, 0, sizeof(float) * t->nW));
    CUDA_TRY(cudaMemset(t->dDBC, 0, sizeof(float) * rows * m->ldbc));
    return TCL_OK;
}

// Enqueue one training step on stream s (validated arguments).
static tcl_status train_enqueue(tcl_model* m, const float* feats, const int32_t* lens, int64_t n, const float* latency,
                                const int64_t* group_offsets, int64_t n_groups, int32_t max_group,
                                int32_t apply_update, float* loss_dev, cudaStream_t s) {
    TrainState& t = *m->tr;
    const tcl_dims& d = m->dims;
    Workspace& w = m->ws;
    const int L = d.max_len, dm = d.d_model, di = d.expand * d.d_model, N = d.d_state, R = d.dt_rank;
    const int e1 = d.enc_dims[0], e2 = d.enc_dims[1], h1 = d.dec_dims[0], h2 = d.dec_dims[1];
    const int max_rows = (int)(n * L);
    const int32_t* P = w.cu + n;
    DropoutCtx nodrop{};
    F32Run r{m, max_rows, P, nodrop, s, lens, n};
    int64_t& nl = m->launches;
    auto G_ = [&](const float* p) { return t.g + (p - m->w_dev); };   // gradient slot of a weight
    auto wg = [&](const float* dY, int lddy, const float* X, int ldx, int Nout, int K, float* out, bool cands) {
        launch_wgrad(dY, lddy, X, ldx, Nout, K, cands ? nullptr : P, cands ? (int)n : max_rows, t.part, t.part_cap,
                     out, K, s);
        nl += 2;
    };
    auto cs = [&](const float* dY, int lddy, int Ncol, float* out, bool cands) {
        launch_colsum(dY, lddy, Ncol, cands ? nullptr : P, cands ? (int)n : max_rows, t.part, t.part_cap, out, s);
        nl += 2;
    };
    // ---- forward, saving activations
    {
        ProfScope ps(m, TCL_PROF_PACK, s);
        launch_lens_prefix(lens, n, L, w.cu, m->d_err, s); ++nl;
        launch_pack(feats, lens, w.cu, n, L, d.d_in, kXld, w.X, nullptr, w.row_cand, s); ++nl;
    }
    auto fgemm = [&](const float* X, int ldx, const float* W, const float* b, float* Y, int K, int Nout, int epi,
                     float* Ypre, bool cands) {
        GemmArgs g{};
        g.X = X; g.ldx = ldx; g.W = W; g.ldw = ldx == kXld && W == m->W1p ? kXld : K; g.bias = b; g.Y = Y; g.ldy = Nout;
        g.K = K; g.N = Nout; g.epi = epi; g.Ypre = Ypre;
        if (cands) { g.max_rows = (int)n; g.rows_const = (int)n; g.rows_are_cands = 1; }
        else { g.max_rows = max_rows; g.p_rows = P; g.row_cand = w.row_cand; g.cu = w.cu; }
        launch_gemm_simt(g, s);
        ++nl;
    };
    fgemm(w.X, kXld, m->W1p, m->wp.enc_b1, t.E1, kXld, e1, EPI_SILU, t.E1pre, false);
    fgemm(t.E1, e1, m->wp.enc_W2, m->wp.enc_b2, t.E2, e1, e2, EPI_SILU, t.E2pre, false);
    fgemm(t.E2, e2, m->wp.enc_W3, m->wp.enc_b3, t.Hin[0], e2, dm, EPI_NONE, nullptr, false);
    for (int l = 0; l < d.n_layer; ++l) {
        const LayerPtrs& q = m->wp.layers[l];
        launch_layernorm(t.Hin[l], dm, dm, q.ln_w, q.ln_b, d.ln_eps, t.Aln[l], nullptr, dm, max_rows, P, s); ++nl;
        fgemm(t.Aln[l], dm, q.W_in, nullptr, t.XZ[l], dm, 2 * di, EPI_NONE, nullptr, false);
        launch_conv_silu(t.XZ[l], 2 * di, q.w_conv, q.b_conv, di, d.d_conv, t.U[l], w.row_cand, w.cu, max_rows, P, s); ++nl;
        {
            GemmArgs g{};
            g.X = t.U[l]; g.ldx = di; g.W = q.W_x; g.ldw = di; g.Y = t.DBC[l]; g.ldy = m->ldbc; g.K = di; g.N = R + 2 * N;
            g.epi = EPI_NONE; g.max_rows = max_rows; g.p_rows = P;
            launch_gemm_simt(g, s); ++nl;
            GemmArgs h{};
            h.X = t.DBC[l]; h.ldx = m->ldbc; h.W = q.W_dt; h.ldw = R; h.bias = q.b_dt; h.Y = t.Delta[l]; h.ldy = di;
            h.K = R; h.N = di; h.epi = EPI_SOFTPLUS; h.max_rows = max_rows; h.p_rows = P;
            launch_gemm_simt(h, s); ++nl;
        }
        ScanArgs sa{};
        sa.U = t.U[l]; sa.Delta = t.Delta[l]; sa.Z = t.XZ[l] + di; sa.ldz = 2 * di;
        sa.BC = t.DBC[l]; sa.ldbc = m->ldbc; sa.b_off = R; sa.c_off = R + N;
        sa.A2 = m->A2 + (size_t)l * di * N; sa.invA = m->invA + (size_t)l * di * N; sa.Dv = q.Dv;
        sa.G = t.G[l]; sa.cu = w.cu; sa.lens = lens; sa.n = n; sa.di = di; sa.N = N; sa.disc = d.disc;
        sa.accurate = 1; sa.max_len = L; sa.S_out = t.S[l];
        launch_scan(sa, s); ++nl;
        CUDA_TRY(cudaMemcpyAsync(t.Hin[l + 1], t.Hin[l], sizeof(float) * (size_t)max_rows * dm, cudaMemcpyDeviceToDevice, s));
        GemmArgs g{};
        g.X = t.G[l]; g.ldx = di; g.W = q.W_out; g.ldw = di; g.Y = t.Hin[l + 1]; g.ldy = dm; g.K = di; g.N = dm;
        g.epi = EPI_RESID; g.max_rows = max_rows; g.p_rows = P;
        launch_gemm_simt(g, s); ++nl;
    }
    float* Hf = t.Hin[d.n_layer];
    launch_pool(Hf, dm, dm, m->wp.lnf_w, m->wp.lnf_b, d.ln_eps, w.cu, lens, L, n, t.pooled, s); ++nl;
    fgemm(t.pooled, dm, m->wp.dec_W1, m->wp.dec_b1, t.d1, dm, h1, EPI_SILU, t.d1pre, true);
    fgemm(t.d1, h1, m->wp.dec_W2, m->wp.dec_b2, t.d2, h1, h2, EPI_SILU, t.d2pre, true);
    fgemm(t.d2, h2, m->wp.dec_W3, m->wp.dec_b3, t.scores, h2, 1, EPI_NONE, nullptr, true);
    // ---- LambdaRank loss and dL/ds (Eq. 6)
    cudaError_t e = launch_lambdarank(t.scores, latency, group_offsets, n_groups, max_group, n, t.sigma, t.ds,
                                      t.gloss, t.loss, m->d_err, s);
    if (e != cudaSuccess) return cuda_error(e, "lambdarank");
    nl += 2;
    if (loss_dev) CUDA_TRY(cudaMemcpyAsync(loss_dev, t.loss, sizeof(float), cudaMemcpyDeviceToDevice, s));
    // ---- backward: decoder
    auto bgemm = [&](const float* X, int ldx, const float* W, int ldw, float* Y, int ldy, int K, int Nout, int epi,
                     bool cands) {   // Y (=|+=) X W   (W stored [K][Nout])
        GemmArgs g{};
        g.X = X; g.ldx = ldx; g.W = W; g.ldw = ldw; g.wT = 1; g.Y = Y; g.ldy = ldy; g.K = K; g.N = Nout; g.epi = epi;
        if (cands) { g.max_rows = (int)n; g.rows_const = (int)n; g.rows_are_cands = 1; }
        else { g.max_rows = max_rows; g.p_rows = P; }
        launch_gemm_simt(g, s);
        ++nl;
    };
    wg(t.ds, 1, t.d2, h2, 1, h2, G_(m->wp.dec_W3), true);
    cs(t.ds, 1, 1, G_(m->wp.dec_b3), true);
    launch_dec_out_bwd(t.ds, m->wp.dec_W3, t.d2pre, h2, n, t.dd2, s); ++nl;
    wg(t.dd2, h2, t.d1, h1, h2, h1, G_(m->wp.dec_W2), true);
    cs(t.dd2, h2, h2, G_(m->wp.dec_b2), true);
    bgemm(t.dd2, h2, m->wp.dec_W2, h1, t.dd1, h1, h2, h1, EPI_NONE, true);
    launch_silu_bwd(t.dd1, h1, t.d1pre, h1, t.dd1, h1, h1, nullptr, (int)n, s); ++nl;
    wg(t.dd1, h1, t.pooled, dm, h1, dm, G_(m->wp.dec_W1), true);
    cs(t.dd1, h1, h1, G_(m->wp.dec_b1), true);
    bgemm(t.dd1, h1, m->wp.dec_W1, dm, t.dpooled, dm, h1, dm, EPI_NONE, true);
    // final norm + masked mean
    launch_ln_bwd(Hf, dm, m->wp.lnf_w, d.ln_eps, nullptr, t.dpooled, w.row_cand, lens, t.dA, t.dH, 0, t.xhdy, max_rows,
                  P, s); ++nl;
    cs(t.xhdy, dm, dm, G_(m->wp.lnf_w), false);
    cs(t.dA, dm, dm, G_(m->wp.lnf_b), false);
    // Mamba blocks, last to first
    for (int l = d.n_layer - 1; l >= 0; --l) {
        const LayerPtrs& q = m->wp.layers[l];
        bgemm(t.dH, dm, q.W_out, di, t.dG, di, dm, di, EPI_NONE, false);
        wg(t.dH, dm, t.G[l], di, dm, di, G_(q.W_out), false);
        ScanBwdArgs b{};
        b.U = t.U[l]; b.Delta = t.Delta[l]; b.Z = t.XZ[l] + di; b.ldz = 2 * di;
        b.BC = t.DBC[l]; b.ldbc = m->ldbc; b.b_off = R; b.c_off = R + N;
        b.A_log = q.A_log; b.Dv = q.Dv; b.S = t.S[l]; b.dG = t.dG;
        b.dZ = t.dXZ + di; b.lddz = 2 * di; b.dU = t.dU; b.dDpre = t.dDpre; b.dBC = t.dDBC;
        b.dAlog_part = t.dAlog_part; b.dD_part = t.dD_part; b.cu = w.cu; b.lens = lens;
        b.n = n; b.di = di; b.N = N; b.disc = d.disc; b.max_len = L;
        launch_scan_bwd(b, s); ++nl;
        cs(t.dAlog_part, di * N, di * N, G_(q.A_log), true);
        cs(t.dD_part, di, di, G_(q.Dv), true);
        // dt_proj (softplus folded into dDpre)
        bgemm(t.dDpre, di, q.W_dt, R, t.dDBC, m->ldbc, di, R, EPI_NONE, false);
        wg(t.dDpre, di, t.DBC[l], m->ldbc, di, R, G_(q.W_dt), false);
        cs(t.dDpre, di, di, G_(q.b_dt), false);
        // x_proj: du += d[dt_r|B|C] W_x
        bgemm(t.dDBC, m->ldbc, q.W_x, di, t.dU, di, R + 2 * N, di, EPI_RESID, false);
        wg(t.dDBC, m->ldbc, t.U[l], di, R + 2 * N, di, G_(q.W_x), false);
        // causal conv + SiLU -> dx (x part of d[x|z])
        launch_conv_bwd(t.XZ[l], 2 * di, q.w_conv, q.b_conv, di, d.d_conv, t.dU, t.dpre, t.dXZ, 2 * di, w.row_cand,
                        w.cu, lens, P, max_rows, t.part, t.part_cap, G_(q.w_conv), G_(q.b_conv), s);
        nl += 4;
        // in_proj
        bgemm(t.dXZ, 2 * di, q.W_in, dm, t.dA, dm, 2 * di, dm, EPI_NONE, false);
        wg(t.dXZ, 2 * di, t.Aln[l], dm, 2 * di, dm, G_(q.W_in), false);
        // pre-norm, residual: dH += LN'(dA)
        launch_ln_bwd(t.Hin[l], dm, q.ln_w, d.ln_eps, t.dA, nullptr, w.row_cand, lens, nullptr, t.dH, 1, t.xhdy,
                      max_rows, P, s); ++nl;
        cs(t.xhdy, dm, dm, G_(q.ln_w), false);
        cs(t.dA, dm, dm, G_(q.ln_b), false);
    }
    // encoder
    wg(t.dH, dm, t.E2, e2, dm, e2, G_(m->wp.enc_W3), false);
    cs(t.dH, dm, dm, G_(m->wp.enc_b3), false);
    bgemm(t.dH, dm, m->wp.enc_W3, e2, t.dE2, e2, dm, e2, EPI_NONE, false);
    launch_silu_bwd(t.dE2, e2, t.E2pre, e2, t.dE2, e2, e2, P, max_rows, s); ++nl;
    wg(t.dE2, e2, t.E1, e1, e2, e1, G_(m->wp.enc_W2), false);
    cs(t.dE2, e2, e2, G_(m->wp.enc_b2), false);
    bgemm(t.dE2, e2, m->wp.enc_W2, e1, t.dE1, e1, e2, e1, EPI_NONE, false);
    launch_silu_bwd(t.dE1, e1, t.E1pre, e1, t.dE1, e1, e1, P, max_rows, s); ++nl;
    wg(t.dE1, e1, w.X, kXld, e1, d.d_in, G_(m->wp.enc_W1), false);
    cs(t.dE1, e1, e1, G_(m->wp.enc_b1), false);
    // ---- Adam, then the derived copies the forward reads (padded W1, A * log2 e, 1 / A)
    if (apply_update) {
        launch_adam(m->w_dev, t.g, t.mA, t.vA, t.nW, t.lr, t.b1, t.b2, t.eps, t.step_dev, t.corr_dev, s); nl += 2;
        launch_refresh_w1(m->wp.enc_W1, e1, d.d_in, kXld, m->W1p, s); ++nl;
        refresh_tf32(m, s);   // the 3xTF32 copies the scoring path reads
        for (const Tf32W& t : m->tfw) nl += t.bn ? 1 : 0;
        for (int l = 0; l < d.n_layer; ++l) {
            launch_refresh_a(m->wp.layers[l].A_log, di * N, m->A2 + (size_t)l * di * N, m->invA + (size_t)l * di * N, s);
            ++nl;
        }
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "train_step");
    return TCL_OK;
}

// One training step.  The ~110 launches of a step are captured once into a CUDA graph and
// replayed while the call signature (pointers, sizes, flags) and the workspace are unchanged; the
// graph runs on a private stream ordered after / before the caller's stream by events.
// tcl_set_option(TCL_OPT_GRAPHS, 0) (or per-stage profiling) launches directly.
tcl_status tcl_train_step(tcl_model* m, const float* feats, const int32_t* lens, int64_t n, const float* latency,
                          const int64_t* group_offsets, int64_t n_groups, int32_t max_group, int32_t apply_update,
                          float* loss_dev, void* stream) {
    if (!m || !m->tr) return set_error(TCL_ESTATE, "tcl_train_init was not called");
    TrainState& t = *m->tr;
    if (n < 2 || n > t.cap_n || n_groups < 1 || n_groups > n || max_group < 2 || max_group > 4096)
        return set_error(TCL_EINVAL, "bad argument (2 <= n <= n_max, 1 <= n_groups <= n, 2 <= max_group <= 4096)");
    if (!feats || !lens || !latency || !group_offsets) return set_error(TCL_EINVAL, "null pointer");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (apply_update) t.step += 1;
    if (!m->use_graphs || m->prof_on)
        return train_enqueue(m, feats, lens, n, latency, group_offsets, n_groups, max_group, apply_update, loss_dev, s);
    // the graph bakes in workspace pointers (cu, X, row_cand): a workspace reallocation by a
    // scoring call between steps (ws_gen) forces a re-capture
    const TrainState::Key key{feats, lens, latency, group_offsets, loss_dev, n, n_groups, m->ws_gen, max_group,
                              apply_update ? 1 : 0};
    if (!t.graph || !(t.key == key)) {
        if (t.graph) { cudaGraphExecDestroy(t.graph); t.graph = nullptr; }
        const int64_t before = m->launches;
        CUDA_TRY(cudaStreamBeginCapture(t.gstream, cudaStreamCaptureModeThreadLocal));
        tcl_status st = train_enqueue(m, feats, lens, n, latency, group_offsets, n_groups, max_group, apply_update,
                                      loss_dev, t.gstream);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(t.gstream, &g);
        t.graph_launches = m->launches - before;   // kernels per replay
        m->launches = before;                      // counted per replay below
        if (st != TCL_OK) { if (g) cudaGraphDestroy(g); return st; }
        if (e != cudaSuccess) return cuda_error(e, "train graph capture");
        e = cudaGraphInstantiate(&t.graph, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) { t.graph = nullptr; return cuda_error(e, "train graph instantiate"); }
        t.key = key;
    }
    CUDA_TRY(cudaEventRecord(t.ev_in, s));
    CUDA_TRY(cudaStreamWaitEvent(t.gstream, t.ev_in, 0));
    CUDA_TRY(cudaGraphLaunch(t.graph, t.gstream));
    CUDA_TRY(cudaEventRecord(t.ev_out, t.gstream));
    CUDA_TRY(cudaStreamWaitEvent(s, t.ev_out, 0));
    m->launches += t.graph_launches;
    return TCL_OK;
}

tcl_status tcl_train_read(tcl_model* m, int32_t what, float* host, int64_t count) {
    if (!m || !host || count < 0) return set_error(TCL_EINVAL, "bad argument");
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaDeviceSynchronize());
    const float* src = nullptr;
    int64_t avail = 0;
    const int64_t nW = weights_count_of(m->dims);
    if (what == 0) { src = m->w_dev; avail = nW; }
    else if (!m->tr) return set_error(TCL_ESTATE, "tcl_train_init was not called");
    else if (what == 1) { src = m->tr->g; avail = nW; }
    else if (what == 2) { src = m->tr->ds; avail = m->tr->cap_n; }
    else if (what == 3) { src = m->tr->scores; avail = m->tr->cap_n; }
    else return set_error(TCL_EINVAL, "what must be 0 (weights), 1 (gradients), 2 (dL/dscore), 3 (scores)");
    if (count > avail) return set_error(TCL_ESHAPE, "count exceeds the buffer");
    CUDA_TRY(cudaMemcpy(host, src, sizeof(float) * count, cudaMemcpyDeviceToHost));
    return TCL_OK;
}
