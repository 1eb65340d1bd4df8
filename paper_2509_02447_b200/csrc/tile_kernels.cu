// Tile extraction and normalisation into bf16 NHWC tiles (north-star item 1):
// preprocess (transforms.cpp:42-47; a centre crop at >= 256 px) -> select_tile
// (tiling.cpp:23-47) -> extract_tile (tiling.cpp:62-77) -> normalize
// (image.cpp:32-38: float(v / 127.5 - 1)), emitted as bf16 (round to nearest
// even) for a learned decoder's first layer.
//
// tile_bf16_kernel: persistent CTAs; one elected thread streams each tile's
// 64 rows x 192 B window into shared memory with a single 3-D TMA box
// (images viewed as [count][rows][row bytes], the box placed at the tile's
// origin), double buffered so the next window lands while this one is
// converted. All threads then map bytes through a 256-entry bf16 table and
// write the tile's contiguous 24 KB (or 32 KB padded to 4 channels) with 16-B
// stores. HBM-bound: 12,288 B read + 24,576 B written per tile.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "qrm_device.cuh"
#include "qrm_types.h"
#include "qrm_window.cuh"

namespace qrm {

constexpr int kTbThreads = 256;
constexpr int kTbRow = 192;             // 64 px x 3 B
constexpr int kTbWin = 64 * kTbRow;     // 12,288 B

__global__ void __launch_bounds__(kTbThreads) tile_bf16_kernel(const __grid_constant__ CUtensorMap tmap,
                                                               const __grid_constant__ TileBf16Params p) {
    __shared__ __align__(128) uint8_t win[2][kTbWin];
    __shared__ uint16_t lut[256];
    __shared__ __align__(8) uint64_t full[2];
    const int tid = threadIdx.x;
    for (int v = tid; v < 256; v += kTbThreads) {
        const float f = __double2float_rn(__dsub_rn(__ddiv_rn(static_cast<double>(v), 127.5), 1.0));
        lut[v] = __bfloat16_as_ushort(__float2bfloat16_rn(f));
    }
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    griddep_launch_dependents();  // the next launch's prologue and first loads may overlap this one
    auto issue = [&](int64_t t, int buf) {
        int x0 = 0, y0 = 0;
        if (p.src.direct) {
            int tx, ty;
            select_tile(kWorkingSize, kWorkingSize, p.src.l, p.src.strategy, p.src.tile_seed,
                        p.src.first_draw + static_cast<uint64_t>(t), tx, ty);
            x0 = (p.src.x_off + tx) * 3;
            y0 = p.src.y_off + ty;
        }
        mbar_arrive_expect_tx(&full[buf], kTbWin);
        tma_load_3d(smem_u32(win[buf]), &tmap, x0, y0, static_cast<int>(t), &full[buf]);
    };
    int64_t t = blockIdx.x;
    if (tid == 0 && t < p.count) issue(t, 0);
    for (int i = 0; t < p.count; t += gridDim.x, ++i) {
        const int buf = i & 1;
        // the other buffer was fully consumed before the previous iteration's barrier
        if (tid == 0 && t + gridDim.x < p.count) issue(t + gridDim.x, buf ^ 1);
        mbar_wait(&full[buf], (i >> 1) & 1);
        if (i == 0) griddep_wait();  // the previous launch is done with the output
        const uint8_t* w = win[buf];
        if (p.channels == 4) {
            // 2 pixels (6 bytes -> 16 B) per 16-B store; 2048 stores per tile
            uint4* dst = reinterpret_cast<uint4*>(p.out + t * (64 * 64 * 4));
            for (int j = tid; j < 64 * 64 / 2; j += kTbThreads) {
                const uint8_t* s = w + j * 6;
                dst[j] = make_uint4(lut[s[0]] | (static_cast<uint32_t>(lut[s[1]]) << 16), lut[s[2]],
                                    lut[s[3]] | (static_cast<uint32_t>(lut[s[4]]) << 16), lut[s[5]]);
            }
        } else {
            // 8 bytes -> one 16-B store; 1536 stores per tile
            uint4* dst = reinterpret_cast<uint4*>(p.out + t * (64 * 64 * 3));
            for (int j = tid; j < kTbWin / 8; j += kTbThreads) {
                const uint8_t* s = w + j * 8;
                dst[j] = make_uint4(lut[s[0]] | (static_cast<uint32_t>(lut[s[1]]) << 16),
                                    lut[s[2]] | (static_cast<uint32_t>(lut[s[3]]) << 16),
                                    lut[s[4]] | (static_cast<uint32_t>(lut[s[5]]) << 16),
                                    lut[s[6]] | (static_cast<uint32_t>(lut[s[7]]) << 16));
            }
        }
        __syncthreads();  // every thread is done with win[buf] before it is refilled
    }
}

// fetch_windows_tma_kernel — the host pipeline's transfer stage with TMA: one
// 3-D box (64 rows x 192 B) per image read straight from mapped pinned host
// memory into shared memory, then one bulk copy of the 12 KB window to its
// slot in HBM. One thread per CTA drives kFtBuf windows in flight.
constexpr int kFtBuf = 3;
__global__ void __launch_bounds__(32) fetch_windows_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                               const __grid_constant__ WindowSource src, int64_t count,
                                                               uint8_t* __restrict__ out) {
    __shared__ __align__(128) uint8_t win[kFtBuf][kTbWin];
    __shared__ __align__(8) uint64_t full[kFtBuf];
    if (threadIdx.x != 0) return;
    for (int b = 0; b < kFtBuf; ++b) mbar_init(&full[b], 1);
    mbar_fence_init();
    auto issue = [&](int64_t t, int b) {
        int tx, ty;
        select_tile(kWorkingSize, kWorkingSize, src.l, src.strategy, src.tile_seed,
                    src.first_draw + static_cast<uint64_t>(t), tx, ty);
        mbar_arrive_expect_tx(&full[b], kTbWin);
        tma_load_3d(smem_u32(win[b]), &tmap, (src.x_off + tx) * 3, src.y_off + ty, static_cast<int>(t), &full[b]);
    };
    const int64_t g = gridDim.x;
    for (int b = 0; b < kFtBuf && blockIdx.x + b * g < count; ++b) issue(blockIdx.x + b * g, b);
    int i = 0;
    for (int64_t t = blockIdx.x; t < count; t += g, ++i) {
        const int b = i % kFtBuf;
        mbar_wait(&full[b], (i / kFtBuf) & 1);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + t * kTbWin),
                     "r"(smem_u32(win[b])), "r"(kTbWin)
                     : "memory");
        bulk_commit();
        const int64_t tn = t + kFtBuf * g;
        if (tn < count) {
            bulk_wait_read<0>();  // the store has read win[b]
            issue(tn, b);
        }
    }
    bulk_wait<0>();
}

cudaError_t launch_fetch_windows_tma(const CUtensorMap& tmap, const WindowSource& src, int64_t count, uint8_t* out,
                                     int sm_count, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    // one CTA (one thread, 3 windows in flight) per SM already fills the link
    // (1, 2, 4 or 8 per SM measured the same); the decode kernel keeps the SMs
    int64_t grid = sm_count > 0 ? sm_count : 148;
    if (grid > count) grid = count;
    fetch_windows_tma_kernel<<<static_cast<unsigned>(grid), 32, 0, st>>>(tmap, src, count, out);
    return cudaGetLastError();
}

cudaError_t launch_tile_bf16(const CUtensorMap& tmap, const TileBf16Params& p, int sm_count, cudaStream_t st) {
    if (p.count <= 0) return cudaSuccess;
    int64_t grid = static_cast<int64_t>(sm_count > 0 ? sm_count : 148) * 8;
    if (grid > p.count) grid = p.count;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kTbThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // programmatic dependent launch
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, tile_bf16_kernel, tmap, p);
}

}  // namespace qrm
