// Learned tile extractor: a HiDDeN / Stable-Signature-style conv stack
// (north-star item 2) as implicit-GEMM tcgen05 kernels, sm_100a.
//
// Model contract (oracle/hidden_oracle.c): 9 x [conv3x3 (pad 1) -> BN(eval)
// -> ReLU] at 64x64 (3->64, 7 x 64->64, 64->n_bits), AdaptiveAvgPool(1),
// Linear(n_bits, n_bits), bit = logit > 0. BN is folded into the conv
// weights/bias on the device; weights are bf16, accumulation fp32 in TMEM,
// activations bf16 NHWC.
//
// conv64_kernel — one 3x3 64->64 layer. A CTA is persistent over 128-pixel
// output blocks (2 image rows). Per block: one 4-D TMA brings the 4 input rows
// it needs (32 KB, rows outside the image zero-filled by TMA) into a
// 128B-swizzled buffer whose 128-byte rows are pixels (64 bf16 channels). Each
// of the 9 taps is then a *shifted view* of that buffer (descriptor start at
// pixel 64(1+dy)+dx, base-offset set for the swizzle phase); the two pixels
// per row whose horizontal neighbour falls outside the image are excluded
// with tcgen05.mma's disable-output-lane mask. The 9 taps x 4 K-steps = 36
// MMAs (M=128, N=64, K=16) accumulate into one of two TMEM buffers while 4
// epilogue warps drain the other (bias + ReLU -> bf16 NHWC, or, for the last
// layer, the per-block channel sums of the average pool). All 9 taps of folded
// weights (72 KB) stay resident in shared memory.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "qrm_device.cuh"
#include "qrm_hidden.h"
#include "qrm_rs.cuh"
#include "qrm_types.h"
#include "qrm_window.cuh"

namespace qrm {

constexpr int kHC = 64;                    // channels
constexpr int kHSide = 64;                 // tile side (l)
constexpr int kHPix = kHSide * kHSide;     // 4096 pixels per tile
constexpr int kHM = 128;                   // pixels per output block (2 rows)
constexpr int kHBlocks = kHPix / kHM;      // 32 blocks per tile
constexpr int kHWBytes = 9 * kHC * kHC * 2;  // 73,728 B of bf16 weights per layer
constexpr int kHABytes = 4 * kHSide * kHC * 2;  // 32 KB: 4 input rows
constexpr int kHAStages = 2;
constexpr int kHThreads = 192;             // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue

struct HiddenSmem {
    uint64_t w_full;
    uint64_t a_full[kHAStages], a_empty[kHAStages];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
    float bias[kHC];
    float pool[4][kHC];  // per-epilogue-warp channel sums (last layer)
};
// layout: [W 72 KB][A0 32 KB][A1 32 KB][HiddenSmem] (+1 KB align slack, views may
// read <= 128 B outside an A buffer; those rows are masked lanes)
constexpr size_t kHSmemBytes = 1024 + kHWBytes + kHAStages * kHABytes + 1024;

__global__ void __launch_bounds__(kHThreads, 1)
    conv64_kernel(const __grid_constant__ CUtensorMap tmap_in, const __grid_constant__ HiddenLayerParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_s = smem_u32(base);
    const uint32_t a_s0 = w_s + kHWBytes;
    HiddenSmem& sm = *reinterpret_cast<HiddenSmem*>(base + kHWBytes + kHAStages * kHABytes + 128);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nblocks = p.tiles * kHBlocks;

    if (warp == 1) tmem_alloc<128>(&sm.tmem_base);
    if (tid == 0) {
        mbar_init(&sm.w_full, 1);
        for (int s = 0; s < kHAStages; ++s) {
            mbar_init(&sm.a_full[s], 1);
            mbar_init(&sm.a_empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&sm.acc_full[a], 1);
            mbar_init(&sm.acc_empty[a], 4);
        }
        mbar_fence_init();
    }
    if (tid < kHC) sm.bias[tid] = p.bias[tid];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ---------------------------------------------------------- TMA ----
        if (lane == 0) {
            mbar_arrive_expect_tx(&sm.w_full, kHWBytes);
            bulk_load(w_s, p.w_swizzled, kHWBytes, &sm.w_full);
            int i = 0;
            for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
                const int s = i % kHAStages;
                mbar_wait(&sm.a_empty[s], ((i / kHAStages) & 1) ^ 1);
                const int tile = static_cast<int>(b / kHBlocks);
                const int y0 = static_cast<int>(b % kHBlocks) * 2;
                mbar_arrive_expect_tx(&sm.a_full[s], kHABytes);
                tma_load_4d(a_s0 + s * kHABytes, &tmap_in, 0, 0, y0 - 1, tile, &sm.a_full[s]);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA ----
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16_f32(kHM, kHC);
            mbar_wait(&sm.w_full, 0);
            int i = 0;
            for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
                const int s = i % kHAStages, a = i & 1;
                mbar_wait(&sm.a_full[s], (i / kHAStages) & 1);
                mbar_wait(&sm.acc_empty[a], ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + a * kHC;
                const uint32_t as = a_s0 + s * kHABytes;
                const int ntaps = (p.dbg & 1) ? 1 : 9;
                for (int t = 0; t < ntaps; ++t) {
                    // centre tap first: it initialises every lane (no mask)
                    const int tap = t == 0 ? 4 : (t <= 4 ? t - 1 : t);
                    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
                    const uint32_t a_view = as + static_cast<uint32_t>((64 * (1 + dy) + dx) * 128);
                    // lanes whose horizontal neighbour is outside the image
                    uint32_t m0 = dx < 0 ? 1u : 0u, m1 = dx > 0 ? 0x80000000u : 0u;
                    if (p.dbg & 4) m0 = m1 = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        // A view starting mid swizzle-atom: the base-offset field stays 0
                        // (measured: the XOR pattern is taken from the absolute address bits,
                        // which TMA wrote with; setting (start>>7)&7 double-applies it).
                        const uint64_t da = sw128_kmajor_desc(a_view + 32 * k);
                        const uint64_t db = sw128_kmajor_desc(w_s + tap * (kHC * 128) + 32 * k);
                        umma_bf16_masked(d, da, db, idesc, (t | k) != 0, m0, m1, m0, m1);
                    }
                }
                umma_commit(&sm.a_empty[s]);
                umma_commit(&sm.acc_full[a]);
            }
        }
        __syncwarp();
    } else {
        // ----------------------------------------------------- epilogue ----
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int i = 0;
        for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
            const int a = i & 1;
            mbar_wait(&sm.acc_full[a], (i >> 1) & 1);
            tc_fence_after();
            uint32_t acc[kHC];
#pragma unroll
            for (int c = 0; c < kHC / 16; ++c) {
                uint32_t r16[16];
                tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + a * kHC + c * 16, r16);
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[c * 16 + j] = r16[j];
            }
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.acc_empty[a]);
            const int64_t tile = b / kHBlocks;
            const int pix = static_cast<int>(b % kHBlocks) * kHM + q * 32 + lane;
            float v[kHC];
#pragma unroll
            for (int c = 0; c < kHC; ++c) v[c] = fmaxf(__uint_as_float(acc[c]) + sm.bias[c], 0.0f);
            if (!p.last) {
                uint4* dst = reinterpret_cast<uint4*>(p.act_out + (tile * kHPix + pix) * kHC);
#pragma unroll
                for (int c = 0; c < kHC; c += 8) {
                    uint4 o;
                    __nv_bfloat162 h0 = __floats2bfloat162_rn(v[c], v[c + 1]);
                    __nv_bfloat162 h1 = __floats2bfloat162_rn(v[c + 2], v[c + 3]);
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(v[c + 4], v[c + 5]);
                    __nv_bfloat162 h3 = __floats2bfloat162_rn(v[c + 6], v[c + 7]);
                    o.x = *reinterpret_cast<uint32_t*>(&h0);
                    o.y = *reinterpret_cast<uint32_t*>(&h1);
                    o.z = *reinterpret_cast<uint32_t*>(&h2);
                    o.w = *reinterpret_cast<uint32_t*>(&h3);
                    dst[c / 8] = o;
                }
            } else {
                // Average pool, part 1: channel sums over this warp's 32 pixels by
                // recursive halving (each step a lane keeps half the channels).
#pragma unroll
                for (int o = 16, n = kHC / 2; o >= 1; o >>= 1, n >>= 1) {
                    const bool upper = (lane & o) != 0;
#pragma unroll
                    for (int c = 0; c < n; ++c) {
                        const float send = upper ? v[c] : v[c + n];
                        const float keep = upper ? v[c + n] : v[c];
                        v[c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
                // Step o kept the upper half iff lane bit log2(o) is set, adding
                // 2*o to the channel base: lane L now holds channels 2L, 2L+1.
                sm.pool[q][2 * lane] = v[0];
                sm.pool[q][2 * lane + 1] = v[1];
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (q == 0 && lane < kHC / 2) {
                    // part 2: fixed-order sum of the 4 warps -> per-block partial
                    for (int c2 = lane * 2; c2 < lane * 2 + 2; ++c2)
                        p.pool_out[(tile * kHBlocks + b % kHBlocks) * kHC + c2] =
                            ((sm.pool[0][c2] + sm.pool[1][c2]) + sm.pool[2][c2]) + sm.pool[3][c2];
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

// First layer (3 -> 64, K = 27): on CUDA cores (0.6% of the stack's FLOPs).
// One thread per pixel; the normalised input window comes straight from the
// image (same tile selection as the correlation decoder).
__global__ void __launch_bounds__(128) conv0_kernel(const __grid_constant__ Conv0Params p) {
    __shared__ float w[27 * kHC];
    __shared__ float bsh[kHC];
    for (int i = threadIdx.x; i < 27 * kHC; i += blockDim.x) w[i] = p.w0[i];
    if (threadIdx.x < kHC) bsh[threadIdx.x] = p.b0[threadIdx.x];
    __syncthreads();
    const int64_t tile = blockIdx.x / kHBlocks;
    if (tile >= p.tiles) return;
    const int pix = static_cast<int>(blockIdx.x % kHBlocks) * kHM + threadIdx.x;
    const int py = pix / kHSide, px = pix % kHSide;
    const uint8_t* wb = window_base(p.src, tile, p.K);
    const int pitch = p.src.direct ? p.src.pitch : 3 * kHSide;
    float x[27];
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const int sy = py + t / 3 - 1, sx = px + t % 3 - 1;
        const bool in = sy >= 0 && sy < kHSide && sx >= 0 && sx < kHSide;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // float(v/127.5 - 1) exactly as normalize (image.cpp:36)
            x[t * 3 + c] = in ? __double2float_rn(__dsub_rn(
                                    __ddiv_rn(static_cast<double>(wb[static_cast<int64_t>(sy) * pitch + sx * 3 + c]),
                                              127.5),
                                    1.0))
                              : 0.0f;
        }
    }
    __nv_bfloat16* dst = p.act_out + (tile * kHPix + pix) * kHC;
#pragma unroll
    for (int c0 = 0; c0 < kHC; c0 += 8) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = bsh[c0 + j];
#pragma unroll
            for (int k = 0; k < 27; ++k) s = fmaf(x[k], w[k * kHC + c0 + j], s);
            o[j] = fmaxf(s, 0.0f);
        }
        uint4 u;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(o[0], o[1]), h1 = __floats2bfloat162_rn(o[2], o[3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(o[4], o[5]), h3 = __floats2bfloat162_rn(o[6], o[7]);
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2);
        u.w = *reinterpret_cast<uint32_t*>(&h3);
        reinterpret_cast<uint4*>(dst)[c0 / 8] = u;
    }
}

// Head: pooled = sum of the 32 block partials (fixed order) / 4096 -> Linear ->
// hard bits -> (t = 1) RS + verify -> record. One warp per tile.
__global__ void __launch_bounds__(256) hidden_head_kernel(const __grid_constant__ HeadParams p) {
    __shared__ RsSmem T;
    __shared__ float pooled[8][kHC];
    rs_stage_tables(T, p.rs, threadIdx.x, blockDim.x);
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = static_cast<int64_t>(blockIdx.x) * 8 + w;
    if (tile >= p.tiles) return;
    const float* pp = p.pool + tile * kHBlocks * kHC;
    for (int c = lane; c < kHC; c += 32) {
        float s = 0.0f;
        for (int b = 0; b < kHBlocks; ++b) s += pp[b * kHC + c];
        pooled[w][c] = s * (1.0f / kHPix);
    }
    __syncwarp();
    const int nb = p.nbits;
    uint64_t raw = 0;
    for (int o0 = 0; o0 < nb; o0 += 32) {
        const int o = o0 + lane;
        float lg = 0.0f;
        if (o < nb) {
            lg = p.bl[o];
            for (int i = 0; i < nb; ++i) lg = fmaf(p.wl[o * nb + i], pooled[w][i], lg);
            if (p.logits) p.logits[tile * nb + o] = lg;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, o < nb && lg > 0.0f);
        raw |= static_cast<uint64_t>(__brev(bal)) << 32 >> o0;  // bit o -> word bit 63 - o
    }
    raw >>= (64 - nb);
    if (lane == 0) {
        qrm_record rec;
        if (p.fuse_t1) {
            uint64_t cw = 0;
            const int nerr = rs_t1_packed(T, raw, cw);
            make_record(rec, raw, nerr, cw, nb, p.kbits, p.key_cw, p.key_msg, p.tau_msg, p.tau_raw, 0);
        } else {
            rec.raw = raw;
            rec.msg = 0;
            rec.status = kRecPending;
            rec.errors = rec.matches = rec.verified = rec.ties = 0;
            const int slot = atomicAdd(p.pending_count, 1);
            p.pending[slot] = PendingEntry{tile, 0};
        }
        store_record(p.out + tile, rec);
    }
}

// Weight preparation: generate (oracle/hidden_oracle.c formulas), fold BN,
// write layer j >= 1 as the pre-swizzled bf16 smem image [tap][co][ci].
__device__ __forceinline__ void hidden_bn(uint64_t seed, int j, int c, float& g, float& be, float& m, float& v) {
    const uint64_t st = 0x4d00 + static_cast<uint64_t>(j);
    g = static_cast<float>(0.75 + 0.5 * rng_unit(seed, st, static_cast<uint64_t>(c)));
    be = static_cast<float>(0.1 * (2.0 * rng_unit(seed, st, 1000 + static_cast<uint64_t>(c)) - 1.0));
    m = static_cast<float>(0.05 * (2.0 * rng_unit(seed, st, 2000 + static_cast<uint64_t>(c)) - 1.0));
    v = static_cast<float>(0.75 + 0.5 * rng_unit(seed, st, 3000 + static_cast<uint64_t>(c)));
}

__device__ __forceinline__ float hidden_weight(uint64_t seed, int j, int co, int tap, int ci) {
    const int cin = j == 0 ? 3 : kHC;
    const double u = rng_unit(seed, 0x4c00 + static_cast<uint64_t>(j), static_cast<uint64_t>((co * 9 + tap) * cin + ci));
    return static_cast<float>((2.0 * u - 1.0) * sqrt(6.0 / (9.0 * cin)));
}

__global__ void hidden_prep_kernel(uint64_t seed, int nbits, __nv_bfloat16* w_sw, float* bias, float* w0, float* wl,
                                   float* bl) {
    // grid.x = layer (0..8), + one extra block for the linear head
    const int j = blockIdx.x;
    if (j == 9) {
        for (int i = threadIdx.x; i < nbits * nbits; i += blockDim.x) {
            const double u = rng_unit(seed, 0x4e00, static_cast<uint64_t>(i));
            wl[i] = static_cast<float>((2.0 * u - 1.0) * sqrt(6.0 / nbits));
        }
        for (int o = threadIdx.x; o < nbits; o += blockDim.x)
            bl[o] = static_cast<float>(0.1 * (2.0 * rng_unit(seed, 0x4e00, 1000000 + static_cast<uint64_t>(o)) - 1.0));
        return;
    }
    const int cout = j == 8 ? nbits : kHC;
    __shared__ float scale[kHC];
    for (int c = threadIdx.x; c < kHC; c += blockDim.x) {
        if (c < cout) {
            float g, be, m, v;
            hidden_bn(seed, j, c, g, be, m, v);
            const float s = g / sqrtf(v + 1e-5f);
            scale[c] = s;
            bias[j * kHC + c] = be - m * s;
        } else {
            scale[c] = 0.0f;
            bias[j * kHC + c] = 0.0f;
        }
    }
    __syncthreads();
    if (j == 0) {
        for (int i = threadIdx.x; i < 27 * kHC; i += blockDim.x) {
            const int k = i / kHC, co = i % kHC;
            w0[i] = hidden_weight(seed, 0, co, k / 3, k % 3) * scale[co];
        }
        return;
    }
    __nv_bfloat16* out = w_sw + static_cast<int64_t>(j - 1) * (9 * kHC * kHC);
    for (int i = threadIdx.x; i < 9 * kHC * kHC; i += blockDim.x) {
        const int tap = i / (kHC * kHC), co = (i / kHC) % kHC, ci = i % kHC;
        const float val = co < cout ? hidden_weight(seed, j, co, tap, ci) * scale[co] : 0.0f;
        // smem image of a 128B-swizzled K-major [64 rows][64 bf16] tile per tap
        const int chunk = ci / 8, within = ci % 8;
        const int off = tap * (kHC * kHC) + co * kHC + ((chunk ^ (co & 7)) * 8) + within;
        out[off] = __float2bfloat16_rn(val);
    }
}

// ---------------------------------------------------------------- launch --
cudaError_t launch_hidden_prep(uint64_t seed, int nbits, __nv_bfloat16* w_sw, float* bias, float* w0, float* wl,
                               float* bl, cudaStream_t st) {
    hidden_prep_kernel<<<10, 256, 0, st>>>(seed, nbits, w_sw, bias, w0, wl, bl);
    return cudaGetLastError();
}

cudaError_t launch_conv0(const Conv0Params& p, cudaStream_t st) {
    conv0_kernel<<<static_cast<unsigned>(p.tiles * kHBlocks), 128, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_conv64(const CUtensorMap& tmap, const HiddenLayerParams& p, int sm_count, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(conv64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kHSmemBytes));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int64_t nblocks = p.tiles * kHBlocks;
    int64_t grid = sm_count > 0 ? sm_count : 148;
    if (grid > nblocks) grid = nblocks;
    conv64_kernel<<<static_cast<unsigned>(grid), kHThreads, kHSmemBytes, st>>>(tmap, p);
    return cudaGetLastError();
}

cudaError_t launch_hidden_head(const HeadParams& p, cudaStream_t st) {
    hidden_head_kernel<<<static_cast<unsigned>((p.tiles + 7) / 8), 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace qrm
