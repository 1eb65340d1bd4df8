// Tile-window addressing shared by the decode and completion kernels.
#pragma once

#include "qrm_device.cuh"
#include "qrm_types.h"

namespace qrm {

// Base of image `img`'s l x l window. Direct: the tile origin comes from the
// counter RNG (select_tile on the 256x256 working image, tiling.cpp:23-47)
// plus the centre-crop offset (transforms.cpp:24-38); rows are `pitch` apart.
// Staged: windows were packed contiguously, 3 l^2 bytes each.
__device__ __forceinline__ const uint8_t* window_base(const WindowSource& s, int64_t img, int K) {
    if (!s.direct) return s.base + img * static_cast<int64_t>(K);
    int tx, ty;
    select_tile(kWorkingSize, kWorkingSize, s.l, s.strategy, s.tile_seed, s.first_draw + static_cast<uint64_t>(img),
                tx, ty);
    return s.base + img * s.image_stride + static_cast<int64_t>(s.y_off + ty) * s.pitch +
           static_cast<int64_t>(s.x_off + tx) * 3;
}

// Exact reference hard bit of a zero integer correlation. The reference sums
// double(float(v/127.5 - 1)) * P sequentially (stego.cpp:60-64) and tests
// soft > 0 (stego.cpp:12). Every term is a multiple of 2^-31 (the float ulp at
// |d| >= 1/255) and |sum| < 2^16, so every partial sum is exact in double and
// the reference's result is the exact sum of L(v) P with the integer
// L(v) = float(v/127.5 - 1) * 2^31, in any order. For a tied bit the exact
// integer correlation sum (2v - 255) P is 0, so
//   255 * sum L(v) P = sum E(v) P,   E(v) = 255 L(v) - (2v - 255) 2^31,
// and E(v) is 255 * 2^31 times float's rounding error of (2v - 255)/255:
// |E| <= 255 * 64, so the dot product fits int32 and has the reference's sign.
//
// tie_dot_partial: thread t of nt takes 16-byte chunks t, t + nt, ... of the
// window and of the pattern row, loading 8 chunks before using any. The E
// table is 256 int32 in shared memory: a bank-replicated copy (32 KB) made the
// lookups conflict-free but cost more to fill (1.9 us per CTA) than the
// conflicts of a 1 KB table cost in lookups.
constexpr int kTieLutWords = 256;

// float(v/127.5 - 1) equals (2v - 255) / 255.f (IEEE single division) for all
// 256 v, and the single division is far cheaper than the double one.
__device__ __forceinline__ int32_t tie_residual(int v) {
    const float d = __fdiv_rn(static_cast<float>(2 * v - 255), 255.0f);
    const long long L = static_cast<long long>(d * 2147483648.0f);  // exact: |d| >= 1/255 > 2^-8
    return static_cast<int32_t>(255ll * L - static_cast<long long>(2 * v - 255) * 2147483648ll);
}

__device__ __forceinline__ void tie_lut_fill(int32_t* elut, int tid, int nthreads) {
    for (int v = tid; v < kTieLutWords; v += nthreads) elut[v] = tie_residual(v);
}

__device__ __forceinline__ int32_t tie_dot_partial(const WindowSource& s, int64_t img, int K, const int8_t* pat,
                                                   const int32_t* elut, int t, int nt) {
    const uint8_t* wb = window_base(s, img, K);
    const int row_bytes = 3 * s.l;
    const int pitch = s.direct ? s.pitch : row_bytes;
    int32_t acc = 0;
    const bool vec = ((reinterpret_cast<uintptr_t>(wb) | reinterpret_cast<uintptr_t>(pat) |
                       static_cast<uintptr_t>(pitch) | static_cast<uintptr_t>(row_bytes)) & 15) == 0;
    if (vec) {
        constexpr int U = 8;
        const int per_row = row_bytes / 16, nchunks = K / 16;
        for (int c0 = t; c0 < nchunks; c0 += U * nt) {
            uint4 v[U], q[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + u * nt;
                const bool ok = c < nchunks;
                const int cc = ok ? c : 0;
                const int r = cc / per_row;
                v[u] = __ldg(reinterpret_cast<const uint4*>(wb + static_cast<int64_t>(r) * pitch) + (cc - r * per_row));
                q[u] = ok ? __ldg(reinterpret_cast<const uint4*>(pat) + cc) : make_uint4(0, 0, 0, 0);  // P = 0: no term
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t vw[4] = {v[u].x, v[u].y, v[u].z, v[u].w}, qw[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int32_t e = elut[(vw[w] >> (8 * k)) & 0xFF];
                        const int32_t pv = static_cast<int8_t>((qw[w] >> (8 * k)) & 0xFF);  // +1, -1 (0: padding)
                        acc += e * pv;
                    }
            }
        }
    } else {
        for (int px = t; px < K; px += nt) {
            const int trow = px / row_bytes;
            const int32_t e = elut[wb[static_cast<int64_t>(trow) * pitch + (px - trow * row_bytes)]];
            acc += e * static_cast<int32_t>(pat[px]);
        }
    }
    return acc;
}

// The same with the whole warp: the reference's hard bit.
__device__ __forceinline__ bool tie_bit_exact(const WindowSource& s, int64_t img, int K, const int8_t* pat,
                                              const int32_t* elut, int lane) {
    int32_t acc = tie_dot_partial(s, img, K, pat, elut, lane, 32);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    return acc > 0;
}

}  // namespace qrm
