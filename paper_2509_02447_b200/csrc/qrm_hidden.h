// Host/device parameter blocks of the learned (conv) extractor kernels.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "qrm_types.h"

namespace qrm {

constexpr int kHiddenLayers = 9;
constexpr int kHiddenC = 64;
constexpr int kHiddenBlocksPerTile = 32;  // 128-pixel output blocks of a 64x64 tile

struct HiddenLayerParams {
    const __nv_bfloat16* w_swizzled;  // [9][64][64] pre-swizzled smem image of the layer
    const float* bias;                // [64] folded BN bias
    __nv_bfloat16* act_out;           // [T][64][64][64] (null for the last layer)
    float* pool_out;                  // [T][32][64] per-block channel sums (last layer)
    int64_t tiles;
    int last;
    // Last layer of the pair kernel with the linear layer fused: pool_out[t][b][o]
    // receives block b's share of logit o, sum_c wl[o][c] * partial_b[c], instead
    // of the channel partials (hidden_sign_kernel adds the 32 shares in order).
    int32_t fuse_linear;
    const float* wl;  // [nbits][nbits]
    int32_t nbits;
};

struct Conv0Params {
    WindowSource src;
    int64_t tiles;
    int32_t K;
    const float* w0;  // [64 co][32 k] folded, tf32, 128B-swizzled smem image (k = tap*3 + ci, zero k >= 27)
    const float* b0;  // [64]
    __nv_bfloat16* act_out;
};

struct HeadParams {
    const float* pool;  // [T][32][64]
    const float* wl;    // [nbits][nbits]
    const float* bl;    // [nbits]
    int64_t tiles;
    int32_t nbits, kbits, tau_msg, tau_raw, fuse_t1;
    uint64_t key_cw, key_msg;
    const RsTables* rs;
    float* logits;  // nullable [T][nbits]
    qrm_record* out;
    int32_t* pending_count;
    PendingEntry* pending;
};

cudaError_t launch_hidden_prep(uint64_t seed, int nbits, __nv_bfloat16* w_sw, float* bias, float* w0, float* wl,
                               float* bl, cudaStream_t st);
cudaError_t launch_conv0(const Conv0Params& p, const CUtensorMap& tmap_out, int sm_count, cudaStream_t st);
// tmap: 4-D load map of the input activations; tmap_out: 2-D store map of the
// output activations ({64 ch, T*4096 px}, box {64, 32}, 128B swizzle).
cudaError_t launch_conv64(const CUtensorMap& tmap, const CUtensorMap& tmap_out, const HiddenLayerParams& p,
                          int sm_count, cudaStream_t st);
// Same layer on CTA pairs (cluster of 2, cta_group::2 MMAs, M = 256).
cudaError_t launch_conv64_pair(const CUtensorMap& tmap, const CUtensorMap& tmap_out, const HiddenLayerParams& p,
                               int sm_count, cudaStream_t st);
cudaError_t launch_hidden_head(const HeadParams& p, cudaStream_t st);
// Logits from the last layer's per-block shares (pool = [T][32][64]) -> hard bits -> RS -> records.
cudaError_t launch_hidden_sign(const HeadParams& p, cudaStream_t st);

}  // namespace qrm
