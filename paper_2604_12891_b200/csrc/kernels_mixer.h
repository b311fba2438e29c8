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

}  // namespace tcl
