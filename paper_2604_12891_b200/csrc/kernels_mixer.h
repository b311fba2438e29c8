// kernels_mixer.h -- launcher of the fused mixer kernel (bf16 path).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tcl {

struct MixerArgs {
    const __nv_bfloat16* XZ; int ldxz;   // in_proj output [P][2 di]: x = cols [0, di), z = [di, 2 di)
    __nv_bfloat16* G; int ldg;           // gated output [P][di]
    const float* A2;                     // [di][N]  A * log2(e)
    const float* invA;                   // [di][N]  1 / A
    const float* Dv;                     // [di]
    const float* w_conv;                 // [di][d_conv]
    const float* b_conv;                 // [di]
    const float* b_dt;                   // [di]
    const __nv_bfloat16* Wx_b;           // [NXP][di] x_proj weights, rows >= R + 2N zero
    const __nv_bfloat16* Wdt_b;          // [di][RP]  dt_proj weights, cols >= R zero
    const int32_t* cu; const int32_t* lens;
    int64_t n;
    int DI, N, R, RP, d_conv, disc, max_len;
};

cudaError_t launch_mixer_fused(const MixerArgs& a, int num_sms, cudaStream_t s);

// ---- split mixer (mixer_split.cu): k_mixprep (conv + x_proj + dt_proj) then k_scan (recurrence).
// Mixer packet, one row of mixer_packet_bytes(DI, N) = 6 DI + 8 N bytes per packed token:
//   [ u fp16 x DI | Delta fp16 x DI | B fp32 x N, C fp32 x N | SiLU(z) bf16 x DI ]
int mixer_packet_bytes(int di, int N);
inline int mixer_packet_gz_offset(int di, int N) { return 4 * di + 8 * N; }

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
    const uint8_t* Pk;                   // mixer packet [P][6 DI + 8 N bytes] (all four parts)
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
