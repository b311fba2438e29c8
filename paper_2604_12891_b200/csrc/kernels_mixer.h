// kernels_mixer.h -- launchers of the bf16-path mixer kernels (inconv.cu, mixer_split.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tcl {

// ---- the bf16 path's Mamba block: k_inconv (in_proj + SiLU(z) + conv + SiLU), k_xdt (x_proj +
// dt_proj + softplus), k_scan (recurrence), then out_proj.  They meet in the mixer packet, one row
// of mixer_packet_bytes(DI, N) = 4 DI + 8 N bytes per packed token:
//   [ u fp16 x DI | Delta fp16 x DI | B fp32 x N, C fp32 x N ]; the gate SiLU(z) is a separate
//   [P][DI] bf16 array (k_inconv).
int mixer_packet_bytes(int di, int N);

// ---- in_proj + SiLU(z) + conv + SiLU in one tcgen05 kernel (inconv.cu): writes SiLU(z) into GZ and u
// (fp16) into the packet's first DI columns, both by TMA stores from shared staging tiles.
struct InConvParams {
    const int32_t* p_rows;               // device: number of packed rows P
    const int32_t* row_cand;             // [P] candidate of each row (conv taps stay inside it)
    const float* w_conv;                 // [DI][4]
    const float* b_conv;                 // [DI]
    int DI, d_conv;
};
int inconv_split(int di);      // CTAs per row tile (2 at DI = 256: a cluster pair splits the channels)
int inconv_channels(int di);   // channels per CTA (the W_in map's box rows)
// a: LN_l(H) bf16 [rows][dm] (box {64, 128}, or {64, 64} when inconv_split == 2); w: W_in bf16
// [2 DI][dm] (box {64, inconv_channels}); gz: SiLU(z) bf16 [rows][DI] (box {64, 125}); u: the packet
// as 2-byte elements [rows][pk_ld / 2] (box {64, 125}).  All 128B-swizzled.
cudaError_t launch_inconv(const CUtensorMap& a, const CUtensorMap& w, const CUtensorMap& gz, const CUtensorMap& u,
                          const InConvParams& p, int dm, int num_sms, cudaStream_t s);

// ---- x_proj + dt_proj + softplus (mixer_split.cu, k_xdt): reads u (fp16) from the packet, writes
// Delta (fp16) and B, C (fp32) into it.
struct XdtArgs {
    uint8_t* Pk; int pk_ld;              // mixer packet [P][pk_ld bytes]
    const float* b_dt;                   // [DI]
    const __half* Wx_h;                  // [NXP][DI] x_proj weights in fp16, rows >= R + 2N zero
    const __nv_bfloat16* Wdt_b;          // [DI][RP]  dt_proj weights, cols >= R zero
    const int32_t* cu;
    int64_t n;
    int DI, N, R, RP, max_len;
};
cudaError_t launch_xdt(const XdtArgs& a, int num_sms, cudaStream_t s);

struct ScanBf16Args {
    const uint8_t* Pk;                   // mixer packet [P][4 DI + 8 N bytes]
    const __nv_bfloat16* GZ;             // SiLU(z) [P][DI] (k_inconv)
    __nv_bfloat16* G;                    // gated output [P][DI]
    const float* A2;                     // [DI][N]  A * log2(e)
    const float* invA;                   // [DI][N]  1 / A   (ZOH)
    const float* Dv;                     // [DI]
    const int32_t* cu;
    int64_t n;
    int DI, N, disc;
    int* work_counter;                   // zeroed before the launch: candidate groups are claimed from it
    int group;                           // candidates per claimed group; 0 = static partition (set by the launcher)
};
cudaError_t launch_scan_bf16(const ScanBf16Args& a, int num_sms, cudaStream_t s);

}  // namespace tcl
