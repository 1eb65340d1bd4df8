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
// pixel 64(1+dy)+dx, base-offset field 0: the swizzle XOR is taken from the
// absolute address bits); the two pixels per row whose horizontal neighbour
// falls outside the image are excluded with tcgen05.mma's disable-output-lane
// mask. The 9 taps x 4 K-steps = 36 MMAs (M=128, N=64, K=16) accumulate into
// one of two TMEM buffers while 4 epilogue warps drain the other: bias + ReLU
// -> bf16 rows written 128B-swizzled (bank-conflict free) into a 4 KB staging
// slab per warp and stored by one TMA tensor store per warp (32 contiguous
// NHWC pixels), or, for the last layer, the per-block channel sums of the
// average pool. All 9 taps of folded weights (72 KB) stay resident in shared
// memory; the A ring is 4 stages deep.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "qrm_device.cuh"
#include "qrm_hidden.h"
#include "qrm_launch.h"
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
constexpr int kHAStages = 4;
constexpr int kHThreads = 320;             // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int kHAcc = 4;                   // TMEM accumulator buffers (64 columns each)

struct HiddenSmem {
    uint64_t w_full;
    uint64_t a_full[kHAStages], a_empty[kHAStages];
    uint64_t acc_full[kHAcc], acc_empty[kHAcc];
    uint32_t tmem_base;
    float pool[4][kHC];  // per-epilogue-warp channel sums (last layer)
};
constexpr int kHOBytes = 4 * 32 * kHC * 2;  // 16 KB: output staging, 4 KB per epilogue warp
// layout: [W 72 KB][A0..A3 4 x 32 KB][O 16 KB][128 B][HiddenSmem] (+1 KB align
// slack; views may read <= 128 B outside an A buffer; those rows are masked lanes)
constexpr size_t kHSmemBytes = 1024 + kHWBytes + kHAStages * kHABytes + kHOBytes + 128 + sizeof(HiddenSmem);
static_assert(kHSmemBytes <= 232448, "conv64 shared memory exceeds 227 KB");

// Epilogue of one 128-pixel block. Eight epilogue warps: warp w reads TMEM
// lane quarter q = w % 4 (32 pixels, one per lane) and channel half h (32 of the
// 64 accumulator columns), so a block's 32 KB of TMEM is drained by twice as
// many warps. Bias + ReLU, then either bf16 NHWC rows -> the quarter's 128B-
// swizzled 4 KB slab (each half writes its four 16-B chunks of every row) ->
// one TMA store per quarter, or (last layer) the block's per-channel sums for
// the average pool. Named barriers 1..4 pair the two warps of a quarter.
constexpr int kHEpiWarps = 8;
constexpr int kHCh = kHC / 2;  // channels per epilogue warp

__device__ __forceinline__ void quarter_sync(int q) {
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
}

// kSlabs staging buffers of 16 KB rotate per block, so a quarter's TMA store
// may still be reading slab i while block i+1 writes slab i+1.
template <int kSlabs>
__device__ __forceinline__ void conv_epilogue(const HiddenLayerParams& p, const CUtensorMap* tmap_out,
                                              const uint32_t (&acc)[kHCh], const float* s_bias, float (*pool)[kHC],
                                              uint32_t o_s, int q, int h, int lane, int64_t tile, int blk, int iter,
                                              const float* wl_s = nullptr, float* part_s = nullptr) {
    const int pix = blk * kHM + q * 32 + lane;
    float v[kHCh];
#pragma unroll
    for (int c = 0; c < kHCh; ++c) v[c] = fmaxf(__uint_as_float(acc[c]) + s_bias[h * kHCh + c], 0.0f);
    if (!p.last) {
        // 16-B chunk c of row r at chunk c ^ (r & 7): conflict-free STS.128
        const uint32_t slab = o_s + (iter % kSlabs) * kHOBytes + q * 4096;
        if (h == 0 && lane == 0) bulk_wait_read<kSlabs - 1>();  // the store that used this slab has read it
        quarter_sync(q);
        const uint32_t row = slab + lane * 128;
#pragma unroll
        for (int c = 0; c < kHCh; c += 8) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(v[c], v[c + 1]);
            __nv_bfloat162 h1 = __floats2bfloat162_rn(v[c + 2], v[c + 3]);
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[c + 4], v[c + 5]);
            __nv_bfloat162 h3 = __floats2bfloat162_rn(v[c + 6], v[c + 7]);
            const int chunk = h * 4 + (c >> 3);
            st_shared_v4(row + (((chunk ^ lane) & 7) << 4),
                         make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                                    *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3)));
        }
        fence_proxy_async_smem();
        quarter_sync(q);
        if (h == 0 && lane == 0) {
            tma_store_2d(tmap_out, slab, 0, static_cast<int>(tile * kHPix + pix - lane));
            bulk_commit();
        }
    } else {
        // Average pool, part 1: channel sums over this warp's 32 pixels by
        // recursive halving; step o keeps the upper half iff lane bit o is set,
        // so lane L ends with channel h*32 + L.
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int c = 0; c < o; ++c) {
                const float send = upper ? v[c] : v[c + o];
                const float keep = upper ? v[c + o] : v[c];
                v[c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        pool[q][h * kHCh + lane] = v[0];
        asm volatile("bar.sync 5, 256;" ::: "memory");
        const int c2 = h * kHCh + lane;
        if (p.fuse_linear) {
            // linear layer fused: part = the block's channel sums (fixed order);
            // the block's share of logit o, sum_c wl[o][c] part[c], as four
            // 16-channel dot products (thread t: o = t % 64, channels 16 (t / 64)
            // + 0..15; wl_s is [c][o], so a warp's lanes read consecutive o)
            // added in fixed order. hidden_sign_kernel adds the 32 shares.
            if (q == 0) part_s[c2] = ((pool[0][c2] + pool[1][c2]) + pool[2][c2]) + pool[3][c2];
            asm volatile("bar.sync 5, 256;" ::: "memory");
            const int t = (q + 4 * h + 2) % 8 * 32 + lane;  // 0..255 over the 8 epilogue warps
            const int o = t & (kHC - 1), g = t >> 6;
            float s = 0.0f;
#pragma unroll
            for (int c = 16 * g; c < 16 * g + 16; ++c) s = fmaf(wl_s[c * kHC + o], part_s[c], s);
            part_s[kHC + g * kHC + o] = s;
            asm volatile("bar.sync 5, 256;" ::: "memory");
            if (g == 0 && o < p.nbits) {
                const float* sh = part_s + kHC;
                p.pool_out[(tile * kHBlocks + blk) * kHC + o] = ((sh[o] + sh[kHC + o]) + sh[2 * kHC + o]) + sh[3 * kHC + o];
            }
        } else {
            // part 2: fixed-order sum of the 4 quarters -> per-block partial
            if (q == 0)
                p.pool_out[(tile * kHBlocks + blk) * kHC + c2] = ((pool[0][c2] + pool[1][c2]) + pool[2][c2]) + pool[3][c2];
            asm volatile("bar.sync 5, 256;" ::: "memory");
        }
    }
}

// This warp's 32 accumulator columns of TMEM buffer `a` (lane quarter q).
__device__ __forceinline__ void load_acc_half(uint32_t tmem, int q, int h, int a, uint32_t (&acc)[kHCh]) {
#pragma unroll
    for (int c = 0; c < kHCh / 16; ++c) {
        uint32_t r16[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + a * kHC + h * kHCh + c * 16, r16);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c * 16 + j] = r16[j];
    }
    tmem_ld_wait();
}

__global__ void __launch_bounds__(kHThreads, 1)
    conv64_kernel(const __grid_constant__ CUtensorMap tmap_in, const __grid_constant__ CUtensorMap tmap_out,
                  const __grid_constant__ HiddenLayerParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ float s_bias[kHC];  // static: read with LDS broadcasts in the epilogue
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_s = smem_u32(base);
    const uint32_t a_s0 = w_s + kHWBytes;
    const uint32_t o_s = a_s0 + kHAStages * kHABytes;
    HiddenSmem& sm = *reinterpret_cast<HiddenSmem*>(base + kHWBytes + kHAStages * kHABytes + kHOBytes + 128);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nblocks = p.tiles * kHBlocks;

    if (warp == 1) tmem_alloc<kHAcc * kHC>(&sm.tmem_base);
    if (tid == 0) {
        mbar_init(&sm.w_full, 1);
        for (int s = 0; s < kHAStages; ++s) {
            mbar_init(&sm.a_full[s], 1);
            mbar_init(&sm.a_empty[s], 1);
        }
        for (int a = 0; a < kHAcc; ++a) {
            mbar_init(&sm.acc_full[a], 1);
            mbar_init(&sm.acc_empty[a], kHEpiWarps);
        }
        mbar_fence_init();
    }
    if (tid < kHC) s_bias[tid] = p.bias[tid];
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
        // The whole warp runs the loop (uniform control flow); one elected lane
        // issues. Descriptors are a per-block base plus compile-time offsets.
        const uint32_t idesc = idesc_bf16_f32(kHM, kHC);
        const uint64_t db0 = sw128_kmajor_desc(w_s);
        mbar_wait(&sm.w_full, 0);
        int i = 0;
        for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
            const int s = i % kHAStages, a = i % kHAcc;
            mbar_wait(&sm.a_full[s], (i / kHAStages) & 1);
            mbar_wait(&sm.acc_empty[a], ((i / kHAcc) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + a * kHC;
            const uint64_t da0 = sw128_kmajor_desc(a_s0 + s * kHABytes);
            if (elect_one()) {
#pragma unroll
                for (int t = 0; t < 9; ++t) {
                    // centre tap first: it initialises every lane (no mask)
                    const int tap = t == 0 ? 4 : (t <= 4 ? t - 1 : t);
                    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
                    // A view: pixel row 64(1+dy)+dx of the 4-row buffer. It may start mid
                    // swizzle-atom; the base-offset field stays 0 (measured: the XOR
                    // pattern is taken from the absolute address bits TMA wrote with).
                    const int view = (64 * (1 + dy) + dx) * 128;
                    // lanes whose horizontal neighbour is outside the image
                    const uint32_t m0 = dx < 0 ? 1u : 0u, m1 = dx > 0 ? 0x80000000u : 0u;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t da = da0 + static_cast<uint64_t>(static_cast<int64_t>((view + 32 * k) >> 4));
                        const uint64_t db = db0 + static_cast<uint64_t>((tap * (kHC * 128) + 32 * k) >> 4);
                        umma_bf16_masked(d, da, db, idesc, (t | k) != 0, m0, m1, m0, m1);
                    }
                }
                umma_commit(&sm.a_empty[s]);
                umma_commit(&sm.acc_full[a]);
            }
            __syncwarp();
        }
    } else {
        // ----------------------------------------------------- epilogue ----
        const int q = warp & 3, h = (warp - 2) >> 2;  // TMEM lane quarter, channel half
        int i = 0;
        for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, ++i) {
            const int a = i % kHAcc;
            mbar_wait(&sm.acc_full[a], (i / kHAcc) & 1);
            tc_fence_after();
            uint32_t acc[kHCh];
            load_acc_half(tmem, q, h, a, acc);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.acc_empty[a]);
            conv_epilogue<1>(p, &tmap_out, acc, s_bias, sm.pool, o_s, q, h, lane, b / kHBlocks,
                                 static_cast<int>(b % kHBlocks), i);
        }
        if (!p.last && h == 0 && lane == 0) bulk_wait<0>();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kHAcc * kHC>(tmem);
    }
}


// conv64_pair_kernel — the same layer on CTA pairs (cluster of 2, cta_group::2).
// A pair-block is 256 output pixels = 4 image rows of one tile: CTA r holds
// rows y0+2r, y0+2r+1 (its own 4-row TMA window, as conv64_kernel) and half of
// the folded weights (output channels 32r..32r+31, 36 KB). The even CTA issues
// M=256 x N=64 x K=16 MMAs that read A rows 0-127 / 128-255 and the two weight
// halves from the two CTAs' smem, and each CTA's TMEM receives its 128 rows x
// 64 channels. Per-CTA operand traffic per MMA falls from 4 KB A + 2 KB B to
// 4 KB A + 1 KB B, and the freed weight smem buys a 5th A stage.
//   full[s]     (even CTA)  2 arrivals (+tx): both CTAs' TMA windows landed
//   empty[s]    (each CTA)  multicast commit of the pair's MMAs
//   acc_full[a] (each CTA)  multicast commit
//   acc_empty[a](even CTA)  16 arrivals: the 8 epilogue warps of both CTAs
constexpr int kPWBytes = kHWBytes / 2;  // 36 KB: 9 taps x 32 co x 64 ci
constexpr int kPAStages = 4;
constexpr int kPSlabs = 2;  // output staging slabs (16 KB each)
struct PairSmem {
    uint64_t w_full;
    uint64_t a_full[kPAStages], a_empty[kPAStages];
    uint64_t acc_full[kHAcc], acc_empty[kHAcc];
    uint32_t tmem_base;
    float pool[4][kHC];
    float part[5 * kHC];  // fused linear: the block's channel sums, then 4 partial dot products
    float wl[kHC * kHC];  // fused linear: wl[o][c] at c * 64 + o (conflict-free across o)
};
constexpr size_t kPSmemBytes = 1024 + kPWBytes + kPAStages * kHABytes + kPSlabs * kHOBytes + 128 + sizeof(PairSmem);
static_assert(kPSmemBytes <= 232448, "conv64 pair shared memory exceeds 227 KB");
constexpr int kPairBlocks = kHBlocks / 2;  // 16 pair-blocks (4 rows) per tile

__global__ void __launch_bounds__(kHThreads, 1)
    conv64_pair_kernel(const __grid_constant__ CUtensorMap tmap_in, const __grid_constant__ CUtensorMap tmap_out,
                       const __grid_constant__ HiddenLayerParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ float s_bias[kHC];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t w_s = smem_u32(base);
    const uint32_t a_s0 = w_s + kPWBytes;
    const uint32_t o_s = a_s0 + kPAStages * kHABytes;
    PairSmem& sm = *reinterpret_cast<PairSmem*>(base + kPWBytes + kPAStages * kHABytes + kPSlabs * kHOBytes + 128);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_ctarank();  // 0 = even CTA (MMA issuer), 1 = odd
    const int64_t npb = p.tiles * kPairBlocks;
    const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (warp == 1) tmem_alloc_pair<kHAcc * kHC>(&sm.tmem_base);
    if (tid == 0) {
        mbar_init(&sm.w_full, 1);
        for (int s = 0; s < kPAStages; ++s) {
            mbar_init(&sm.a_full[s], 2);
            mbar_init(&sm.a_empty[s], 1);
        }
        for (int a = 0; a < kHAcc; ++a) {
            mbar_init(&sm.acc_full[a], 1);
            mbar_init(&sm.acc_empty[a], 2 * kHEpiWarps);
        }
        mbar_fence_init();
    }
    if (tid < kHC) s_bias[tid] = p.bias[tid];
    if (p.fuse_linear)
        for (int x = tid; x < kHC * kHC; x += kHThreads) {  // zero-padded to 64 x 64
            const int o = x % kHC, c = x / kHC;
            sm.wl[x] = (o < p.nbits && c < p.nbits) ? p.wl[o * p.nbits + c] : 0.0f;
        }
    tc_fence_before();
    cluster_sync_all();  // barriers initialised in both CTAs before any remote arrive
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    // Barrier phase 2 ("both weight halves resident"): the TMA warp arrives at
    // once and waits only after its loop; the MMA warp waits before its first MMA.
    if (warp == 0) {
        // ---------------------------------------------------------- TMA ----
        cluster_arrive();
        if (lane == 0) {
            // this CTA's weight half: output channels 32r..32r+31 of every tap
            mbar_arrive_expect_tx(&sm.w_full, kPWBytes);
            for (int t = 0; t < 9; ++t)
                bulk_load(w_s + t * 4096, p.w_swizzled + (t * kHC + 32 * rank) * kHC, 4096, &sm.w_full);
            int i = 0;
            for (int64_t b = pair; b < npb; b += npairs, ++i) {
                const int s = i % kPAStages;
                mbar_wait(&sm.a_empty[s], ((i / kPAStages) & 1) ^ 1);
                const int tile = static_cast<int>(b / kPairBlocks);
                const int y0 = static_cast<int>(b % kPairBlocks) * 4 + 2 * static_cast<int>(rank);
                const uint32_t full0 = map_to_rank(smem_u32(&sm.a_full[s]), 0);
                mbar_arrive_expect_tx_cluster(full0, kHABytes);
                tma_load_4d_pair(a_s0 + s * kHABytes, &tmap_in, 0, 0, y0 - 1, tile, full0);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA ----
        mbar_wait(&sm.w_full, 0);
        cluster_sync_all();  // both weight halves resident
        if (rank == 0) {
            const uint32_t idesc = idesc_bf16_f32(2 * kHM, kHC);
            const uint64_t db0 = sw128_kmajor_desc(w_s);
            int i = 0;
            for (int64_t b = pair; b < npb; b += npairs, ++i) {
                const int s = i % kPAStages, a = i % kHAcc;
                mbar_wait(&sm.a_full[s], (i / kPAStages) & 1);
                mbar_wait(&sm.acc_empty[a], ((i / kHAcc) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + a * kHC;
                const uint64_t da0 = sw128_kmajor_desc(a_s0 + s * kHABytes);
                if (elect_one()) {
#pragma unroll
                    for (int t = 0; t < 9; ++t) {
                        const int tap = t == 0 ? 4 : (t <= 4 ? t - 1 : t);  // centre tap first (no mask)
                        const int dy = tap / 3 - 1, dx = tap % 3 - 1;
                        const int view = (64 * (1 + dy) + dx) * 128;
                        const uint32_t m0 = dx < 0 ? 1u : 0u, m1 = dx > 0 ? 0x80000000u : 0u;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint64_t da = da0 + static_cast<uint64_t>(static_cast<int64_t>((view + 32 * k) >> 4));
                            const uint64_t db = db0 + static_cast<uint64_t>((tap * 4096 + 32 * k) >> 4);
                            umma_bf16_pair_masked(d, da, db, idesc, (t | k) != 0, m0, m1);
                        }
                    }
                    umma_commit_pair_mc(&sm.a_empty[s], 0x3);
                    umma_commit_pair_mc(&sm.acc_full[a], 0x3);
                }
                __syncwarp();
            }
        }
    } else {
        // ----------------------------------------------------- epilogue ----
        cluster_sync_all();
        const int q = warp & 3, h = (warp - 2) >> 2;
        uint32_t empty0[kHAcc];
#pragma unroll
        for (int a = 0; a < kHAcc; ++a) empty0[a] = map_to_rank(smem_u32(&sm.acc_empty[a]), 0);
        int i = 0;
        for (int64_t b = pair; b < npb; b += npairs, ++i) {
            const int a = i % kHAcc;
            mbar_wait(&sm.acc_full[a], (i / kHAcc) & 1);
            tc_fence_after();
            uint32_t acc[kHCh];
            load_acc_half(tmem, q, h, a, acc);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(empty0[a]);
            conv_epilogue<kPSlabs>(p, &tmap_out, acc, s_bias, sm.pool, o_s, q, h, lane, b / kPairBlocks,
                                   static_cast<int>(b % kPairBlocks) * 2 + static_cast<int>(rank), i, sm.wl, sm.part);
        }
        if (!p.last && h == 0 && lane == 0) bulk_wait<0>();
    }
    __syncwarp();
    if (warp == 0) cluster_wait();  // the TMA warp's wait of barrier phase 2
    tc_fence_before();
    cluster_sync_all();  // both CTAs done with TMEM and with each other's smem
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<kHAcc * kHC>(tmem);
    }
}

// First layer (3 -> 64, K = 27) as one tcgen05 kind::tf32 GEMM per 128-pixel
// block: D[128 px][64 co] = A[128 px][32] . W0[64 co][32]^T, K = 27 taps x
// channels zero-padded to 32 (fp32 rows of exactly 128 B, one 128B-swizzle
// atom row). Persistent CTAs (several per SM) set up once — normalisation
// table (float(v/127.5 - 1), image.cpp:36, rounded to tf32), folded weights,
// TMEM — then loop over blocks: stage the block's 4 input rows (u8), build
// each pixel's im2col row, one thread issues the 4 MMAs (K = 8 each), and the
// epilogue (bias + ReLU -> bf16, 128B-swizzled per-warp slab, one TMA store per
// warp) drains TMEM. The A tile doubles as the output staging slab.
constexpr int kC0Threads = 128;
constexpr int kC0K = 32;  // padded K (fp32 elements per A/B row)

__global__ void __launch_bounds__(kC0Threads) conv0_kernel(const __grid_constant__ CUtensorMap tmap_out,
                                                           const __grid_constant__ Conv0Params p) {
    __shared__ __align__(1024) uint8_t a_tile[kHM * kC0K * 4];  // 16 KB A (im2col, fp32/tf32)
    __shared__ __align__(1024) uint8_t o_tile[kHM * kHC * 2];   // 16 KB output staging (4 KB per warp)
    __shared__ __align__(1024) uint8_t b_tile[kHC * kC0K * 4];  // 8 KB W0 (pre-swizzled)
    __shared__ float lut[256];
    __shared__ float bsh[kHC];
    __shared__ __align__(16) uint8_t rows[4][3 * kHSide];
    // the block's 4 input rows normalised, channel-planar, x + 1 (columns -1 and
    // 64 stay 0: the zero padding), so each im2col tap is one conflict-free LDS
    __shared__ float rowf[4][3][kHSide + 4];
    __shared__ uint64_t done;
    __shared__ uint32_t tmem_slot;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nblocks = p.tiles * kHBlocks;
    if (warp == 0) tmem_alloc<kHC>(&tmem_slot);
    if (tid == 0) {
        mbar_init(&done, 1);
        mbar_fence_init();
    }
    // normalisation table, exactly float(v/127.5 - 1.0) then tf32-rounded
    for (int v = tid; v < 256; v += kC0Threads) {
        const float f = __double2float_rn(static_cast<double>(v) / 127.5 - 1.0);
        uint32_t t;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(f));
        lut[v] = __uint_as_float(t);
    }
    if (tid < kHC) bsh[tid] = p.b0[tid];
    for (int i = tid; i < 4 * 3 * (kHSide + 4); i += kC0Threads) (&rowf[0][0][0])[i] = 0.0f;
    {
        const uint4* src = reinterpret_cast<const uint4*>(p.w0);
        uint4* dst = reinterpret_cast<uint4*>(b_tile);
#pragma unroll
        for (int i = 0; i < (kHC * kC0K * 4) / 16 / kC0Threads; ++i)
            dst[tid + i * kC0Threads] = __ldg(src + tid + i * kC0Threads);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t idesc = idesc_tf32_f32(kHM, kHC);
    const uint64_t da = sw128_kmajor_desc(smem_u32(a_tile)), db = sw128_kmajor_desc(smem_u32(b_tile));
    const int pitch = p.src.direct ? p.src.pitch : 3 * kHSide;
    constexpr int kRow16 = 3 * kHSide / 16;  // 12 16-B chunks per input row; threads < 48 move one each

    // Software pipeline: the 4 input rows of block b+grid are fetched into
    // registers while block b is computed, so the DRAM latency overlaps.
    auto fetch = [&](int64_t b, uint4& v) -> bool {
        if (tid >= 4 * kRow16 || b >= nblocks) return false;
        const int64_t tile = b / kHBlocks;
        const int sy = static_cast<int>(b % kHBlocks) * 2 - 1 + tid / kRow16;
        if (sy < 0 || sy >= kHSide) return false;  // zero-padded by the im2col below
        v = __ldg(reinterpret_cast<const uint4*>(window_base(p.src, tile, p.K) + static_cast<int64_t>(sy) * pitch) +
                  tid % kRow16);
        return true;
    };
    uint4 pre = make_uint4(0, 0, 0, 0);
    bool have = fetch(blockIdx.x, pre);
    uint32_t phase = 0;

    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, phase ^= 1) {
        const int64_t tile = b / kHBlocks;
        const int blk = static_cast<int>(b % kHBlocks);
        const int y0 = blk * 2;
        if (have) reinterpret_cast<uint4*>(rows[tid / kRow16])[tid % kRow16] = pre;
        __syncthreads();
        have = fetch(b + gridDim.x, pre);
        // normalise each input byte once (768 table lookups per block instead of
        // 27 per pixel); zero padding is in the normalised domain: rows outside
        // the tile contribute 0.0, not lut[0] = -1
#pragma unroll
        for (int j = 0; j < 4 * 3 * kHSide / kC0Threads; ++j) {
            const int i = tid + j * kC0Threads;
            const int r = i / (3 * kHSide), byte = i - r * (3 * kHSide);
            const int sy = y0 - 1 + r;
            rowf[r][byte % 3][byte / 3 + 1] = (sy >= 0 && sy < kHSide) ? lut[rows[r][byte]] : 0.0f;
        }
        __syncthreads();

        // im2col row of pixel (y0 + tid/64, tid%64): k = tap*3 + c, tap = 3(dy+1) + (dx+1)
        {
            const int ry = 1 + (tid >> 6), px = tid & 63;
            float x[kC0K];
#pragma unroll
            for (int t = 0; t < 9; ++t)
#pragma unroll
                for (int c = 0; c < 3; ++c) x[t * 3 + c] = rowf[ry + t / 3 - 1][c][px + t % 3];
#pragma unroll
            for (int k = 27; k < kC0K; ++k) x[k] = 0.0f;
            const uint32_t row = smem_u32(a_tile) + tid * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                st_shared_v4(row + (((c ^ tid) & 7) << 4),
                             make_uint4(__float_as_uint(x[4 * c]), __float_as_uint(x[4 * c + 1]),
                                        __float_as_uint(x[4 * c + 2]), __float_as_uint(x[4 * c + 3])));
        }
        fence_proxy_async_smem();  // generic-proxy writes of A -> visible to the tensor core
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < kC0K / 8; ++k) umma_tf32(tmem, da + 2 * k, db + 2 * k, idesc, k != 0);
            umma_commit(&done);
        }
        mbar_wait(&done, phase);
        tc_fence_after();
        uint32_t acc[kHC];
#pragma unroll
        for (int c = 0; c < kHC / 16; ++c) {
            uint32_t r16[16];
            tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 16, r16);
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[c * 16 + j] = r16[j];
        }
        tmem_ld_wait();
        tc_fence_before();
        // this warp's previous output store must have read its slab (issued a block ago)
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        const uint32_t slab = smem_u32(o_tile) + warp * 4096;
        const uint32_t row = slab + lane * 128;
#pragma unroll
        for (int c = 0; c < kHC; c += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = fmaxf(__uint_as_float(acc[c + j]) + bsh[c + j], 0.0f);
            __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]);
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[4], v[5]), h3 = __floats2bfloat162_rn(v[6], v[7]);
            st_shared_v4(row + ((((c >> 3) ^ lane) & 7) << 4),
                         make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                                    *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3)));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(&tmap_out, slab, 0, static_cast<int>(tile * kHPix + blk * kHM + warp * 32));
            bulk_commit();
        }
    }
    if (lane == 0) bulk_wait<0>();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<kHC>(tmem);
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

// Sign: logit o = bl[o] + (sum of the 32 blocks' shares, in block order) / 4096
// -> hard bits -> (t = 1) RS + verify -> record. One warp per tile.
__global__ void __launch_bounds__(256) hidden_sign_kernel(const __grid_constant__ HeadParams p) {
    __shared__ RsSmem T;
    rs_stage_tables(T, p.rs, threadIdx.x, blockDim.x);
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = static_cast<int64_t>(blockIdx.x) * 8 + w;
    if (tile >= p.tiles) return;
    const int nb = p.nbits;
    uint64_t raw = 0;
    for (int o0 = 0; o0 < nb; o0 += 32) {
        const int o = o0 + lane;
        float lg = 0.0f;
        if (o < nb) {
            const float* sh = p.pool + tile * kHBlocks * kHC + o;
            float s = 0.0f;
#pragma unroll 8
            for (int b = 0; b < kHBlocks; ++b) s += sh[b * kHC];
            lg = fmaf(s, 1.0f / kHPix, p.bl[o]);
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
        // smem image of the 128B-swizzled K-major [64 co][32 k] fp32 (tf32-rounded) B tile
        for (int i = threadIdx.x; i < kHC * kC0K; i += blockDim.x) {
            const int co = i / kC0K, k = i % kC0K;
            const float val = k < 27 ? hidden_weight(seed, 0, co, k / 3, k % 3) * scale[co] : 0.0f;
            uint32_t t;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(val));
            w0[co * kC0K + (((k / 4) ^ (co & 7)) * 4) + (k % 4)] = __uint_as_float(t);
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

cudaError_t launch_conv0(const Conv0Params& p, const CUtensorMap& tmap_out, int sm_count, cudaStream_t st) {
    int64_t grid = static_cast<int64_t>(sm_count > 0 ? sm_count : 148) * 4;  // 4 resident per SM (118 regs x 128 thr)
    if (grid > p.tiles * kHBlocks) grid = p.tiles * kHBlocks;
    conv0_kernel<<<static_cast<unsigned>(grid), kC0Threads, 0, st>>>(tmap_out, p);
    return cudaGetLastError();
}

cudaError_t launch_conv64(const CUtensorMap& tmap, const CUtensorMap& tmap_out, const HiddenLayerParams& p,
                          int sm_count, cudaStream_t st) {
    static PerDeviceOnce once;  // function attributes are per device context
    const cudaError_t e = once.run([] {
        return cudaFuncSetAttribute(conv64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kHSmemBytes));
    });
    if (e != cudaSuccess) return e;
    const int64_t nblocks = p.tiles * kHBlocks;
    int64_t grid = sm_count > 0 ? sm_count : 148;
    if (grid > nblocks) grid = nblocks;
    conv64_kernel<<<static_cast<unsigned>(grid), kHThreads, kHSmemBytes, st>>>(tmap, tmap_out, p);
    return cudaGetLastError();
}


cudaError_t launch_conv64_pair(const CUtensorMap& tmap, const CUtensorMap& tmap_out, const HiddenLayerParams& p,
                               int sm_count, cudaStream_t st) {
    static PerDeviceOnce once;  // function attributes are per device context
    const cudaError_t e = once.run([] {
        return cudaFuncSetAttribute(conv64_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kPSmemBytes));
    });
    if (e != cudaSuccess) return e;
    const int64_t npb = p.tiles * kPairBlocks;
    int64_t pairs = (sm_count > 0 ? sm_count : 148) / 2;
    if (pairs > npb) pairs = npb;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
    cfg.blockDim = dim3(kHThreads);
    cfg.dynamicSmemBytes = kPSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, conv64_pair_kernel, tmap, tmap_out, p);
}

cudaError_t launch_hidden_sign(const HeadParams& p, cudaStream_t st) {
    hidden_sign_kernel<<<static_cast<unsigned>((p.tiles + 7) / 8), 256, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_hidden_head(const HeadParams& p, cudaStream_t st) {
    hidden_head_kernel<<<static_cast<unsigned>((p.tiles + 7) / 8), 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace qrm
