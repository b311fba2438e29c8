// kernels.h -- internal launchers of libtcl (not part of the C ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tcl {

// Opt a kernel in to `smem` bytes of dynamic shared memory on the CURRENT device (cached per
// device) and, if blocks_per_sm != nullptr, return its occupancy at `threads` threads per CTA.
cudaError_t prepare_kernel_raw(const void* fn, int smem, int threads, int* blocks_per_sm);
template <typename K>
inline cudaError_t prepare_kernel(K* kern, int smem, int threads = 0, int* blocks_per_sm = nullptr) {
    return prepare_kernel_raw(reinterpret_cast<const void*>(kern), smem, threads, blocks_per_sm);
}

// Device error bits (sticky, tcl_sync_error).
enum : int { ERR_LEN = 1, ERR_TASK = 2 };

// ---- pack ------------------------------------------------------------------
// cu[n+1] exclusive prefix of the valid lengths (invalid lengths count as 0 rows and raise
// ERR_LEN); cu[n] = P.  n <= 1<<20 per launch.
void launch_lens_prefix(const int32_t* lens, int64_t n, int32_t max_len, int32_t* cu, int* err,
                        cudaStream_t s);
// Gather the real rows of feats [n][L][d_in] into X [P][ldx] (columns d_in..ldx-1 zeroed) and
// write row_cand[P].  If x_bf16 != nullptr, also writes a bf16 copy [P][ldx].  Candidate i reads
// the features of candidate i mod n_src (batched MC passes: n = passes * n_src; n_src = n otherwise).
void launch_pack(const float* feats, const int32_t* lens, const int32_t* cu, int64_t n, int L,
                 int d_in, int ldx, float* X, void* x_bf16, int32_t* row_cand, cudaStream_t s,
                 int64_t n_src = 0);

// ---- SIMT fp32 GEMM with fused epilogues ------------------------------------------------------
enum Epi : int { EPI_NONE = 0, EPI_SILU = 1, EPI_SOFTPLUS = 2, EPI_RESID = 3,
                 // N == 128 only (one CTA column owns whole rows): Y (+)= acc + b, then Y2 = LN(Y) (next pre-norm)
                 EPI_RESID_LN = 4, EPI_LN = 5 };
struct GemmArgs {
    const float* X; int ldx;        // [M][K]
    const float* W; int ldw;        // [N][K] (PyTorch [out][in])
    const float* bias;              // [N] or nullptr
    float* Y; int ldy;              // [M][N]
    int K, N;
    int max_rows;                   // grid extent (rows)
    const int32_t* p_rows;          // device: actual row count (cu[n]); rows >= *p_rows skipped
    int rows_const;                 // row count when p_rows == nullptr
    int rows_are_cands;             // decoder: row = candidate, token 0 (dropout sites 2, 3)
    int epi;
    // dropout (EPI_SILU only): per-row candidate and token
    DropoutCtx drop; int site;
    const int32_t* row_cand; const int32_t* cu;
    // optional second operand pair accumulated into the same sums (KB+AC lateral term of Eq. 7):
    // Y = epi(X W^T + X2 W2^T + b), X2 [M][ldx2], W2 [N][ldw2], K2 columns; K % 16 == 0 when K2 > 0
    const float* X2; int ldx2; const float* W2; int ldw2; int K2;
    // training: wT != 0 reads W transposed (element (j, k) at W[k * ldw + j], i.e. Y = X W);
    // Ypre != nullptr also stores the pre-activation (before the epilogue) at Ypre[m * ldy + j]
    int wT; float* Ypre;
    // EPI_RESID_LN / EPI_LN: the LayerNorm that follows (affine, biased variance), output Y2
    const float* ln_g; const float* ln_b; float ln_eps; float* Y2; int ldy2;
};
void launch_gemm_simt(const GemmArgs& a, cudaStream_t s);

// ---- LayerNorm rows (fp32 in, fp32 out and/or bf16 out) ---------------------------------------
void launch_layernorm(const float* H, int ldh, int dm, const float* g, const float* b, float eps,
                      float* Y, void* Ybf16, int ldy, int max_rows, const int32_t* p_rows,
                      cudaStream_t s,
                      bool gemm_epilogue_order = false);

// ---- causal depthwise conv + SiLU (a5) --------------------------------------------------------
// X [P][ldx] (x part = first di columns) -> U [P][di]
void launch_conv_silu(const float* X, int ldx, const float* w, const float* b, int di, int dc,
                      float* U, const int32_t* row_cand, const int32_t* cu, int max_rows,
                      const int32_t* p_rows, cudaStream_t s);

// ---- selective scan + D skip + gate (a7) ------------------------------------------------------
struct ScanArgs {
    const float* U;      // [P][di]
    const float* Delta;  // [P][di]
    const float* Z; int ldz;  // z at Z[row*ldz + d]
    const float* BC; int ldbc; int b_off, c_off;  // B at BC[row*ldbc + b_off + n]
    const float* A2;     // [di][N]  A * log2(e)
    const float* invA;   // [di][N]  1 / A
    const float* Dv;     // [di]
    float* G;            // [P][di]  y * SiLU(z)
    const int32_t* cu; const int32_t* lens;
    int64_t n; int di, N, disc, accurate, max_len;
    float* S_out;        // training: states after step t at S_out[(row * di + d) * N + n] (or nullptr)
};
void launch_scan(const ScanArgs& a, cudaStream_t s);

// ---- fp32 path: conv + x_proj + dt_proj + scan fused in one persistent kernel (mixer_f32.cu) -----
struct MixerF32Args {
    const float* XZ; int ldxz;   // in_proj output [P][2 di] fp32: x = cols [0, di), z = [di, 2 di)
    float* G; int ldg;           // gated output [P][di]
    const float* A2;             // [di][N]  A * log2(e)
    const float* invA;           // [di][N]  1 / A
    const float* Dv;             // [di]
    const float* w_conv;         // [di][d_conv]
    const float* b_conv;         // [di]
    const float* W_x;            // [R + 2N][di]
    const float* W_dt;           // [di][R]
    const float* b_dt;           // [di]
    const int32_t* cu;           // [n + 1] packed row offsets (device)
    int64_t n;
    int DI, N, R, disc;
    int max_len;                 // L (the L-parallel variant needs L <= 32)
};
bool mixer_f32_supported(int di, int N, int R, int d_conv);
cudaError_t launch_mixer_f32(const MixerF32Args& a, int num_sms, cudaStream_t s);
// L-parallel variant (one CTA per candidate, warp-shuffle chunked scan across L) for short sequences
bool mixer_lpar_supported(int di, int N, int R, int d_conv, int max_len);
cudaError_t launch_mixer_lpar(const MixerF32Args& a, cudaStream_t s);

// ---- fused head (head.cu): pool + decoder + score / Welford in one launch ---------------------
struct HeadArgs {
    const float* H; int ldh;              // fp32 path: residual stream (LN_f applied here)
    const __nv_bfloat16* F; int ldf;      // bf16 path: LN_f(H) rows (nullptr on the fp32 path)
    const float* lnf_w; const float* lnf_b; float eps;
    const int32_t* cu; const int32_t* lens; int max_len; int64_t n;
    int dm, h1, h2;
    const float *W1, *b1, *W2, *b2, *W3, *b3;
    float* pooled;                        // [n][dm] scratch of the two-launch form (large n)
    DropoutCtx drop;                      // sites 2, 3 (MC); drop.pass = the Welford pass
    float* scores;                        // deterministic mode (NaN for invalid lengths)
    float* mc_mean; float* m2;            // MC mode (mc_mean != nullptr)
};
// false: dims not covered (decoder widths other than [dm/2, dm/4, 1]); the caller falls back.
// One launch for n < 8192; larger batches return false (the five-launch head is faster there).
bool launch_head_fused(const HeadArgs& a, cudaStream_t s);

// ---- head: LN_f + masked mean pool (warp per candidate) -> pooled [n][dm] -----------------------
void launch_pool(const float* H, int ldh, int dm, const float* lnf_w, const float* lnf_b, float eps,
                 const int32_t* cu, const int32_t* lens, int max_len, int64_t n, float* pooled,
                 cudaStream_t s);
// Masked mean of already-normalised bf16 rows F = LN_f(H) (bf16 path: written by the last
// out_proj epilogue) -> pooled [n][dm] fp32.
void launch_pool_bf16(const void* F, int ldf, int dm, const int32_t* cu, const int32_t* lens, int max_len,
                      int64_t n, float* pooled, cudaStream_t s);
// MC: Welford update of (mean, m2) with this pass' scores; invalid lengths -> NaN.
void launch_welford(const float* score, const int32_t* lens, int max_len, int64_t n, int pass,
                    float* mean, float* m2, cudaStream_t s);
// Scores of invalid candidates -> NaN (reading R16).
void launch_mask_invalid(const int32_t* lens, int max_len, int64_t n, float* scores, cudaStream_t s);

// ---- head: LN_f, masked mean, decoder (a9) ----------------------------------------------------
void launch_mc_finalize(const float* m2, int64_t n, int passes, float* var, cudaStream_t s);
// Batched MC passes: score [passes][n] -> Welford over the passes in order 0..passes-1 (the
// arithmetic of k_welford, pass by pass) -> mean [n], var = M2 / passes [n] (NaN: invalid length).
void launch_mc_reduce(const float* score, const int32_t* lens, int max_len, int64_t n, int passes, float* mean,
                      float* var, cudaStream_t s);

// ---- top-k ------------------------------------------------------------------------------------
// Local top-k keys: k keys (descending, sentinel 0 padded) of scores[0..n) with index_base.
// tmp must hold >= 2 * ceil(n / kTopkChunk) * k + 2 * kTopkChunk keys.
constexpr int kTopkChunk = 8192;
size_t topk_tmp_keys(int64_t n, int k);
// Both return the number of kernels launched.
int launch_topk_keys(const float* scores, int64_t n, int k, int64_t index_base,
                     unsigned long long* out_keys, unsigned long long* tmp, cudaStream_t s);
// Top-k of `count` keys -> decoded (idx, score) [k].  tmp: k + topk_tmp_keys(count, k) keys.
// decode k keys that are already the sorted top-k (0-padded) into (index, score)
int launch_topk_decode(const unsigned long long* keys, int k, int64_t* idx, float* score, cudaStream_t s);
int launch_topk_merge(const unsigned long long* keys, int64_t count, int k, int64_t* idx,
                      float* score, unsigned long long* tmp, cudaStream_t s);

// ---- RDU acquisition (Alg. 1, Eqs. 1-3) -------------------------------
// ---- training (train.cu) -------------------------------------------------
struct ScanBwdArgs {
    const float* U; const float* Delta; const float* Z; int ldz;
    const float* BC; int ldbc; int b_off, c_off;
    const float* A_log; const float* Dv;
    const float* S;      // saved states [P][di][N]
    const float* dG;     // [P][di]
    float* dZ; int lddz; // gate gradient (z part of d[x|z])
    float* dU;           // [P][di] scan-input gradient
    float* dDpre;        // [P][di] gradient of the softplus input
    float* dBC;          // B / C gradients at dBC[row * ldbc + b_off / c_off + n]
    float* dAlog_part;   // [n][di][N]
    float* dD_part;      // [n][di]
    const int32_t* cu; const int32_t* lens;
    int64_t n; int di, N, disc, max_len;
};
void launch_wgrad(const float* dY, int lddy, const float* X, int ldx, int Nout, int K, const int32_t* p_rows,
                  int max_rows, float* part, size_t part_cap, float* out, int ldo, cudaStream_t s);
void launch_colsum(const float* dY, int lddy, int Ncol, const int32_t* p_rows, int max_rows, float* part,
                   size_t part_cap, float* out, cudaStream_t s);
void launch_silu_bwd(const float* dPost, int ldp, const float* pre, int ldpre, float* dPre, int ldo, int Ncol,
                     const int32_t* p_rows, int max_rows, cudaStream_t s);
void launch_dec_out_bwd(const float* ds, const float* W3, const float* pre2, int h2, int64_t n, float* dpre2,
                        cudaStream_t s);
void launch_ln_bwd(const float* H, int dm, const float* g, float eps, const float* dY, const float* dpooled,
                   const int32_t* row_cand, const int32_t* lens, float* dYout, float* dH, int accumulate,
                   float* xhdy, int max_rows, const int32_t* p_rows, cudaStream_t s);
void launch_conv_bwd(const float* X, int ldx, const float* w, const float* b, int di, int dc, const float* dU,
                     float* dpre, float* dX, int lddx, const int32_t* row_cand, const int32_t* cu,
                     const int32_t* lens, const int32_t* p_rows, int max_rows, float* part, size_t part_cap,
                     float* dw, float* db, cudaStream_t s);
void launch_scan_bwd(const ScanBwdArgs& a, cudaStream_t s);
// LambdaRank loss + dL/ds over CSR groups (reading R24).  dscores [n_total] is zeroed first; a
// group with no member or more than max_group members, or outside [0, n_total), contributes 0
// and sets ERR_TASK in *err.
cudaError_t launch_lambdarank(const float* scores, const float* lat, const int64_t* off, int64_t n_groups,
                              int max_group, int64_t n_total, float sigma, float* dscores, float* gloss, float* loss,
                              int* err, cudaStream_t s);
void launch_adam(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
                 int* step_dev, float* corr_dev, cudaStream_t s);
void launch_refresh_w1(const float* W1, int e1, int d_in, int ldp, float* W1p, cudaStream_t s);
void launch_refresh_a(const float* alog, int diN, float* A2, float* invA, cudaStream_t s);

// Top-k score (Eq. 12): up to 16 k values per call.
struct TopkEvalKs { int n; int k[16]; };
cudaError_t launch_topk_eval(const float* scores, const float* lat, const int64_t* off, const float* w,
                             int64_t n_tasks, int max_task_len, const TopkEvalKs& ks, double* cols,
                             double* out, int* err, int num_sms, cudaStream_t s);
size_t rdu_scratch_bytes(int grid_max, int n_ops);
cudaError_t launch_rdu_select(const float* pool, const int32_t* ops, int64_t n_pool, const float* lab,
                              int64_t n_lab, int n_ops, int budget_total, int64_t* out, int32_t* n_out,
                              void* scratch, int num_sms, cudaStream_t s);

}  // namespace tcl
