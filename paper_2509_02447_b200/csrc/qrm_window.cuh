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

}  // namespace qrm
