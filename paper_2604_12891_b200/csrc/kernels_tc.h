// kernels_tc.h -- launchers of the tcgen05 / TMA kernels (bf16 projection path).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tcl {

enum TcEpi : int { TC_EPI_BF16 = 0, TC_EPI_RESID_LN = 1 };

struct TcGemmParams {
    int n_tiles;                 // N / BN (each CTA owns one N tile for the whole launch)
    const int32_t* p_rows;       // device: number of valid rows (packed tokens)
    int epi;
    // TC_EPI_BF16: out[row][n] = bf16(dropout(act(acc + bias)))
    const float* bias;           // [N] or nullptr
    int act_silu;
    __nv_bfloat16* out; int ldo; // bf16 output (EPI_BF16) / LayerNorm output (EPI_RESID_LN)
    // TC_EPI_RESID_LN: H = (residual ? H : 0) + acc (+ bias); out = bf16(LN(H) * g + b)
    float* H; int ldh; int residual;
    int skip_h_store;            // RESID_LN (gemm_tc_ln): do not write H back (last layer: only LN_f(H) is consumed)
    const float* ln_g; const float* ln_b; float eps;
    DropoutCtx drop; int site; const int32_t* row_cand; const int32_t* cu;
};

// Encoder linears 1 + 2 chained in one kernel (gemm_tc_enc.cu): E2 = SiLU(SiLU(X W1^T + b1) W2^T + b2)
struct EncParams {
    const int32_t* p_rows;       // device: number of packed rows
    const float* b1; const float* b2;
    DropoutCtx drop;             // sites 0 (E1) and 1 (E2) when enabled
    const int32_t* row_cand; const int32_t* cu;
};
bool enc12_supported(int e1, int e2, int d_in);
// X: [rows][32] bf16 (box {64, 128}); W1: [e1][32] (box {64, e1}); W2: [e2][e1] (box {64, e2});
// E2: bf16 output map (box {64, 32}).
cudaError_t launch_enc12(const CUtensorMap& x, const CUtensorMap& w1, const CUtensorMap& w2, const CUtensorMap& e2,
                         const EncParams& p, int e1n, int e2n, int num_sms, cudaStream_t s);

// 2-D bf16 tensor map, 128B swizzle, box {box_inner (<= 64), box_outer (<= 256)}.
bool make_tmap_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                    uint32_t box_inner, uint32_t box_outer);
// 2-D fp32 tensor map, 128B swizzle, box {box_inner (<= 32), box_outer}.
bool make_tmap_f32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                   uint32_t box_inner, uint32_t box_outer);
// fp32 map with box {16, box_outer} (64-byte rows) and 64-byte swizzle: the 3xTF32 GEMM's operands
bool make_tmap_f32_sw64(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                        uint32_t box_outer);
// Residual + LayerNorm GEMM (gemm_tc_ln.cu): bn = d_model in {128, 256}; H: fp32 map of the
// residual stream (box {32, 32}); O: bf16 map of the LayerNorm output (box {64, 32}).
cudaError_t launch_gemm_tc_ln(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& h,
                              const CUtensorMap& o, const TcGemmParams& p, int bn, int kb, int num_sms,
                              cudaStream_t s);
// A: [rows][K] (box {64, 128}); B: [N][K] weights (box {64, bn}); kb = ceil(K / 64).
// C: bf16 output map (box {64, 32}, 128B swizzle) used for TMA stores when BN >= 128 and the
// epilogue writes bf16 (ignored otherwise).
cudaError_t launch_gemm_tc(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                           const TcGemmParams& p, int bn, int kb, int num_sms, cudaStream_t s);

// ---- fp32 path on the tensor cores: 3xTF32 GEMM (gemm_tf32.cu) -------------------------------
struct Tf32GemmParams {
    int n_tiles;                 // N / BN
    const int32_t* p_rows;       // device: number of valid rows
    int epi;                     // 0: Y = acc; 1: Y = SiLU(acc + b) [+ dropout]; 3: H = [H +] acc + b [, out = LN(H)]
    const float* bias;           // [N] or nullptr
    float* Y; int ldy;           // epi 0 / 1 output (fp32)
    float* H; int ldh; int residual;
    float* out; int ldo;         // epi 3: LayerNorm output (fp32) or nullptr (needs n_tiles == 1)
    const float* ln_g; const float* ln_b; float eps;
    DropoutCtx drop; int site; const int32_t* row_cand; const int32_t* cu;
};
// bn in {32, 64, 128, 256}; k <= 256 (K-blocks of 32 fp32); both weight halves resident.
bool tf32_gemm_supported(int bn, int k);
// A: fp32 [rows][K] map (box {32, 128}, 128B swizzle); B / Blo: W_hi / W_lo [N][K] (box {32, bn}).
cudaError_t launch_gemm_tf32(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& blo,
                             const Tf32GemmParams& p, int bn, int k, int num_sms, cudaStream_t s);
// hi = w with the low 13 mantissa bits cleared, lo = tf32_rna(w - hi), element-wise (n floats).
void launch_tf32_split(const float* w, int64_t n, float* hi, float* lo, cudaStream_t s);

}  // namespace tcl
