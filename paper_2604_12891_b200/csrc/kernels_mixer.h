// kernels_mixer.h -- launchers of the bf16-path mixer kernels (mixer_split.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tcl {

// ---- split mixer (mixer_split.cu): k_mixprep (conv + x_proj + dt_proj) then k_scan (recurrence).
// Mixer packet, one row of mixer_packet_bytes(DI, N) = 4 DI + 8 N bytes per packed token:
//   [ u fp16 x DI | Delta fp16 x DI | B fp32 x N, C fp32 x N ]; the gate SiLU(z) is a separate
//   [P][DI] bf16 array (in_proj epilogue).
int mixer_packet_bytes(int di, int N);

struct MixPrepArgs {
    const __nv_bfloat16* X;              // in_proj x part [P][DI] (bf16, rows contiguous)
    uint8_t* Pk; int pk_ld;              // mixer packet [P][pk_ld bytes]: writes u, Delta, B, C
    const float* w_conv;                 // [DI][d_conv]
    const float* b_conv;                 // [DI]
    const float* b_dt;                   // [DI]
    const __nv_bfloat16* Wx_b;           // [NXP][DI] x_proj weights, rows >= R + 2N zero
    const __nv_bfloat16* Wdt_b;          // [DI][RP]  dt_proj weights, cols >= R zero
    const int32_t* cu; const int32_t* row_cand;
    int64_t n;
    int DI, N, R, RP, d_conv, max_len;
};
cudaError_t launch_mixprep(const MixPrepArgs& a, int num_sms, cudaStream_t s);

struct ScanBf16Args {
    const uint8_t* Pk;                   // mixer packet [P][4 DI + 8 N bytes]
    const __nv_bfloat16* GZ;             // SiLU(z) [P][DI] (in_proj epilogue)
    __nv_bfloat16* G;                    // gated output [P][DI]
    const float* A2;                     // [DI][N]  A * log2(e)
    const float* invA;                   // [DI][N]  1 / A   (ZOH)
    const float* Dv;                     // [DI]
    const int32_t* cu;
    int64_t n;
    int DI, N, disc;
};
cudaError_t launch_scan_bf16(const ScanBf16Args& a, int num_sms, cudaStream_t s);

}  // namespace tcl
