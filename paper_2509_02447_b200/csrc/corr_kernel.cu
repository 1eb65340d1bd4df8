// Tile decode for the spread-spectrum watermark, sm_100a.
//
// Reference path (per image): preprocess (transforms.cpp:42-47) -> select_tile
// (tiling.cpp:23-47) -> extract_tile (tiling.cpp:62-77) ->
// SpreadSpectrumCodec::extract (stego.cpp:53-67) -> harden (stego.cpp:10-14)
// -> bw_decode (rs.cpp:188) -> verify (detect.cpp:180-195).
//
// B200 restatement. The correlation is a GEMM D[img][bit] = sum_px A[img][px]
// * P[bit][px] with A = the raw u8 tile window and P = the +-1 planes as s8.
// Since normalize is v/127.5 - 1 and P is +-1, the reference's sign test on
// sum_px float(v/127.5-1) P is the sign of the EXACT integer
//   S = sum_px (2v - 255) P = 2 D - 255 colsum(P)
// except when S == 0, where the reference's double rounding decides; those
// (image, bit) pairs are re-evaluated exactly (tie_bit_exact, qrm_window.cuh; for codes
// the epilogue cannot finish, by detect_finish_kernel), so hard bits are
// bit-exact.
//
// corr_detect_kernel: one CTA = 128 images (UMMA M) x 64 bit columns (N) x a
// K range. Warps 0-3 stream 128-byte K chunks of the 128 tile windows
// (cp.async, 16 B per thread, straight into the 128B-swizzled K-major operand
// layout) and of the pattern matrix into a 4-stage smem ring. Warp 4 issues tcgen05.mma kind::i8
// (u8 x s8 -> s32, accumulators in TMEM). With few images the K range is split
// over a cluster of 2 or 4 CTAs that reduce through DSMEM. The epilogue (one
// image per thread = one TMEM lane) reads 64 columns with tcgen05.ld, forms S,
// hardens, packs the raw word and — t = 1 codes without ties — runs the RS
// decoder and verify in registers, so one launch produces final records.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "qrm_device.cuh"
#include "qrm_launch.h"
#include "qrm_rs.cuh"
#include "qrm_types.h"
#include "qrm_window.cuh"

namespace qrm {

constexpr int kCorrM = 128;
constexpr int kCorrN = 64;
constexpr int kCorrKC = 128;  // bytes of K per stage
// A 4-stage ring, with the end-of-kernel buffers (split-K partials, tie list)
// aliased into it, keeps a CTA at ~99 KB of smem, so two fit on an SM. The
// grid still places one CTA per SM (the occupancy query's cluster waves); the
// other half of each SM takes the next batch's CTAs (programmatic dependent
// launch), which stream while this batch's CTAs run their tails. Measured per
// 4096-image step, back to back: 6 stages (one CTA per SM) 18.5 us; 4 stages
// 13.0 us; 3 stages (three CTAs per SM) 13.5 us but the host pipeline's
// transfer kernel then ran erratically beside the decode grids (configs[4]
// 0.5-3.1 M img/s vs 3.6); two CTAs per SM from one batch (66 clusters)
// 19.2 us. An isolated launch is slower (27.5 vs 26.6 us at 6 stages).
constexpr int kCorrStages = 4;
constexpr int kCorrABytes = kCorrM * kCorrKC;  // 16 KiB
constexpr int kCorrBBytes = kCorrN * kCorrKC;  // 8 KiB
constexpr int kCorrStageBytes = kCorrABytes + kCorrBBytes;
constexpr int kCorrProducers = 128;
constexpr int kCorrThreads = 160;
constexpr int kRedStride = kCorrN + 4;  // int32 words per reduction row (padded: conflict-free v4 access)

struct CorrSmem {
    uint64_t full[kCorrStages];
    uint64_t empty[kCorrStages];
    uint64_t accum_full;
    uint32_t tmem_base;
    alignas(16) int32_t thr[kCorrN];  // 255 * colsum(P_i): bit i = 2 D_i > thr_i
    RsSmem rs;
    int nties;  // t = 1 codes: this CTA's images with tied bits (TieList)
};
// Once every MMA of the cluster is done the rings are idle, and the end-of-
// kernel buffers live there: the split-K partials pushed by the cluster,
// red[rank][row within my 128/S rows][kRedStride] (ring offset 0), then the
// tie list.
struct TieEntry {
    int64_t image;
    uint64_t tie_mask, raw;
};
struct TieList {
    TieEntry ties[kCorrM];
    int32_t elut[kTieLutWords];  // tie residual table (qrm_window.cuh)
    int32_t red[kCorrThreads / 32];  // per-warp partial dot products
};
constexpr int kRedBytes = kCorrM * kRedStride * 4;
static_assert(kRedBytes + sizeof(TieList) <= kCorrStages * kCorrStageBytes, "end-of-kernel buffers exceed the ring");

constexpr size_t kCorrSmemBytes = 1024 /*align slack*/ + kCorrStages * kCorrStageBytes + sizeof(CorrSmem);

// Epilogue, part 1: columns [c0, c0 + NC) of one image. S_i = 2 D_i - 255
// colsum_i; bit i = S_i > 0 (harden), tie i = S_i == 0, as 64-bit column masks
// (bit i = column i); soft values for those columns when asked.
template <int NC>
__device__ __forceinline__ void image_columns(const DetectParams& p, const CorrSmem& sm, int64_t img, int c0,
                                              const uint32_t (&acc)[NC], uint64_t& pos, uint64_t& zer) {
    const int nb = p.nbits;
    pos = 0;
    zer = 0;
    const int4* thr4 = reinterpret_cast<const int4*>(sm.thr + c0);
#pragma unroll
    for (int q = 0; q < NC / 4; ++q) {
        const int4 t = thr4[q];
        const int tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = 4 * q + u;
            const int s2 = 2 * static_cast<int>(acc[i]) - tv[u];
            pos |= static_cast<uint64_t>(s2 > 0) << i;
            zer |= static_cast<uint64_t>(s2 == 0) << i;
        }
    }
    pos <<= c0;
    zer <<= c0;
    if (p.soft) {
        const double inv = 1.0 / (255.0 * static_cast<double>(p.K));
#pragma unroll
        for (int i = 0; i < NC; ++i)  // constant indices keep acc[] in registers
            if (c0 + i < nb)
                p.soft[img * nb + c0 + i] = static_cast<double>(2 * static_cast<int>(acc[i]) - sm.thr[c0 + i]) * inv;
    }
}

// Epilogue, part 2: pack MSB-first; t = 1 code without ties: RS-correct +
// verify in registers and write the record. Tied images go to the CTA's tie
// list (finish_ties); codes the epilogue cannot finish, to the pending list.
__device__ __forceinline__ void finish_masks(const DetectParams& p, CorrSmem& sm, TieList& tl, int64_t img,
                                             uint64_t pos, uint64_t zer) {
    const int nb = p.nbits;
    const uint64_t nmask = nb >= 64 ? ~0ull : ((1ull << nb) - 1);
    const uint64_t tmask = zer & nmask;
    const uint64_t raw = __brevll(pos) >> (64 - nb);
    if (p.raw_out) p.raw_out[img] = raw;
    qrm_record rec;
    if (tmask == 0 && p.fuse_t1) {
        uint64_t cw = 0;
        const int nerr = rs_t1_packed(sm.rs, raw, cw);
        make_record(rec, raw, nerr, cw, nb, p.kbits, p.key_cw, p.key_msg, p.tau_msg, p.tau_raw, 0);
    } else if (p.fuse_t1) {
        // tied bits: resolved by the whole CTA after the epilogue (finish_ties)
        const int slot = atomicAdd(&sm.nties, 1);
        tl.ties[slot] = TieEntry{img, tmask, raw};
        return;
    } else {
        rec.raw = raw;
        rec.msg = 0;
        rec.status = kRecPending;
        rec.errors = 0;
        rec.matches = 0;
        rec.verified = 0;
        rec.ties = static_cast<uint8_t>(__popcll(tmask));
        const int slot = atomicAdd(p.pending_count, 1);
        p.pending[slot] = PendingEntry{img, tmask};
    }
    store_record(p.out + img, rec);
}

// t = 1 codes: the CTA's images with tied bits (collected by finish_image).
// Each tied bit is one exact dot product over the window, computed by the
// whole CTA (every thread's chunk loads in flight at once), then thread 0
// runs RS + verify + the record.
__device__ __noinline__ void finish_ties(const DetectParams& p, CorrSmem& sm, TieList& tl, int warp, int lane) {
    tie_lut_fill(tl.elut, threadIdx.x, kCorrThreads);
    __syncthreads();
    griddep_wait();  // the previous grid is done with the records
    const int nb = p.nbits;
    const int nties = sm.nties;
    for (int e = 0; e < nties; ++e) {  // CTA-uniform
        const TieEntry te = tl.ties[e];
        uint64_t raw = te.raw;
        for (uint64_t m = te.tie_mask; m; m &= m - 1) {  // CTA-uniform
            const int b = __ffsll(static_cast<long long>(m)) - 1;
            int32_t part = tie_dot_partial(p.src, te.image, p.K, p.patterns + static_cast<int64_t>(b) * p.K_pad,
                                           tl.elut, threadIdx.x, kCorrThreads);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (lane == 0) tl.red[warp] = part;
            __syncthreads();
            int32_t tot = 0;
#pragma unroll
            for (int w = 0; w < kCorrThreads / 32; ++w) tot += tl.red[w];
            __syncthreads();  // tl.red is reused by the next bit
            if (tot > 0) raw |= 1ull << (nb - 1 - b);
        }
        if (threadIdx.x == 0) {
            if (p.raw_out) p.raw_out[te.image] = raw;
            uint64_t cw = 0;
            const int nerr = rs_t1_packed(sm.rs, raw, cw);
            qrm_record rec;
            make_record(rec, raw, nerr, cw, nb, p.kbits, p.key_cw, p.key_msg, p.tau_msg, p.tau_raw,
                        __popcll(te.tie_mask));
            store_record(p.out + te.image, rec);
        }
    }
}

// Launched as clusters of S = 1, 2 or 4 CTAs along K (split-K): CTA r of a
// cluster accumulates K chunks [r K/S, (r+1) K/S) of the same 128 images in its
// own TMEM, pushes the partial rows owned by each peer into the peer's shared
// memory (DSMEM), and after one cluster barrier each CTA finishes 128/S images.
__global__ void __launch_bounds__(kCorrThreads, 1) corr_detect_kernel(const __grid_constant__ DetectParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    CorrSmem& sm = *reinterpret_cast<CorrSmem*>(ring + kCorrStages * kCorrStageBytes);
    int32_t* red = reinterpret_cast<int32_t*>(ring);
    TieList& tl = *reinterpret_cast<TieList*>(ring + kRedBytes);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const uint32_t S = cluster_nctarank();  // 1 without a cluster launch
    const uint32_t rank = cluster_ctarank();
    const int tile_m = p.tile_m;  // images in this tile (<= 128): tiles are balanced over the SMs
    const int64_t m0 = static_cast<int64_t>(blockIdx.x / S) * tile_m;
    const int kc_total = p.K_pad / kCorrKC;
    const int kc_begin = static_cast<int>(static_cast<int64_t>(kc_total) * rank / S);
    const int kchunks = static_cast<int>(static_cast<int64_t>(kc_total) * (rank + 1) / S) - kc_begin;

    if (warp == 4) tmem_alloc<kCorrN>(&sm.tmem_base);
    if (tid == 0) {
        for (int s = 0; s < kCorrStages; ++s) {
            mbar_init(&sm.full[s], kCorrProducers + 1);  // + thread 0's expect_tx arrival for the pattern bulk copy
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.accum_full, 1);
        mbar_fence_init();
        sm.nties = 0;
    }
    griddep_launch_dependents();  // the completion kernel may launch; it waits for this grid
    if (tid < kCorrN) sm.thr[tid] = 255 * __ldg(p.colsum + tid);
    if (p.fuse_t1) rs_stage_tables(sm.rs, p.rs, tid, kCorrThreads);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const int rows_per = kCorrM / static_cast<int>(S);

    if (warp < 4) {
        // ------------------------------------------------------ producer --
        const int c = tid & 7;    // 16-byte chunk within the 128-byte K chunk
        const int rb = tid >> 3;  // rows rb + 16 j
        const uint8_t* wb[8];
        bool valid[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t img = m0 + rb + 16 * j;
            valid[j] = rb + 16 * j < tile_m && img < p.count;
            wb[j] = valid[j] ? window_base(p.src, img, p.K) : nullptr;
        }
        const int row_bytes = 3 * p.src.l;
        const int pitch = p.src.direct ? p.src.pitch : row_bytes;
        const uint32_t ring_u32 = smem_u32(ring);
        if (p.wait_inputs) griddep_wait();  // the preceding kernel may have written the windows
        // K offset of this thread's 16 B, as (tile row, column) — stepped, no division per stage.
        int kbyte = kc_begin * kCorrKC + c * 16;
        int trow = kbyte / row_bytes;
        int tcol = kbyte - trow * row_bytes;
        // (L2 prefetch of tile rows ahead of the ring — bulk or per line — was
        // measured slower at every batch size: 4096 imgs 26.2 -> 30.2/36.7 us.)
        for (int it = 0; it < kchunks; ++it) {
            const int s = it % kCorrStages;
            mbar_wait(&sm.empty[s], ((it / kCorrStages) & 1) ^ 1);
            const uint32_t a_s = ring_u32 + s * kCorrStageBytes;
            const uint32_t b_s = a_s + kCorrABytes;
            if (tid == 0) {  // the stage's pattern operand: one bulk copy of its pre-swizzled smem image
                mbar_arrive_expect_tx(&sm.full[s], kCorrBBytes);
                bulk_load(b_s, p.patterns_sw + static_cast<int64_t>(kc_begin + it) * kCorrBBytes, kCorrBBytes,
                          &sm.full[s]);
            }
            if (kbyte < p.K) {
                const int64_t off = static_cast<int64_t>(trow) * pitch + tcol;
                // .L2::64B: fill only the 64-B sector pairs the 192-B row covers (the
                // default 128-B fill over-reads 1.33x: ncu 68.0 -> 51.2 MB per 50.3 MB)
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (valid[j]) cp_async16_l2_64(a_s + sw128_offset(rb + 16 * j, c), wb[j] + off);
            }
            // Never block on the copies: the barrier phase completes when every
            // producer's copies for this stage have landed.
            cp_async_mbar_arrive(&sm.full[s]);
            kbyte += kCorrKC;
            tcol += kCorrKC;
            while (tcol >= row_bytes) {
                tcol -= row_bytes;
                ++trow;
            }
        }
        cp_async_wait<0>();

        // ------------------------------------------------------ epilogue --
        mbar_wait(&sm.accum_full, 0);
        tc_fence_after();
        uint32_t acc[kCorrN];
#pragma unroll
        for (int q = 0; q < kCorrN / 16; ++q) {
            uint32_t r16[16];
            tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + q * 16, r16);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[q * 16 + i] = r16[i];
        }
        tmem_ld_wait();
        tc_fence_before();

        const int row = warp * 32 + lane;
        if (S == 1) {
            griddep_wait();  // the previous completion kernel is done with records / the pending list
            const int64_t img = m0 + row;
            if (row < tile_m && img < p.count) {
                uint64_t pos, zer;
                image_columns<kCorrN>(p, sm, img, 0, acc, pos, zer);
                finish_masks(p, sm, tl, img, pos, zer);
            }
        } else {
            // push this partial row to its owner CTA: slot `rank`, local row
            const uint32_t owner = static_cast<uint32_t>(row / rows_per);
            const uint32_t local = static_cast<uint32_t>(row % rows_per);
            // the owner's ring takes the partials: wait until every MMA of the
            // cluster is done (each CTA's producers passed its accum_full)
            cluster_arrive();
            cluster_wait();
            const uint32_t dst = map_to_rank(smem_u32(&red[(rank * rows_per + local) * kRedStride]), owner);
#pragma unroll
            for (int q = 0; q < kCorrN / 4; ++q)
                st_cluster_v4(dst + 16 * q, acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
        }
    } else if (warp == 4) {
        // ------------------------------------------------------ MMA issuer --
        if (lane == 0) {
            const uint32_t idesc = idesc_i8_u8s8(kCorrM, kCorrN);
            const uint32_t ring_u32 = smem_u32(ring);
            for (int it = 0; it < kchunks; ++it) {
                const int s = it % kCorrStages;
                mbar_wait(&sm.full[s], (it / kCorrStages) & 1);
                // The stage's bytes are in smem (written through the generic
                // proxy by cp.async); order them before the async-proxy MMA reads.
                fence_proxy_async_smem();
                tc_fence_after();
                const uint32_t a_s = ring_u32 + s * kCorrStageBytes;
                const uint64_t da = sw128_kmajor_desc(a_s);
                const uint64_t db = sw128_kmajor_desc(a_s + kCorrABytes);
#pragma unroll
                for (int k = 0; k < kCorrKC / 32; ++k)  // K = 32 bytes per kind::i8 MMA
                    umma_i8(tmem, da + 2 * k, db + 2 * k, idesc, (it | k) != 0);
                umma_commit(&sm.empty[s]);
            }
            umma_commit(&sm.accum_full);
        }
        __syncwarp();
        if (S > 1) {  // the producers' "all MMAs done" cluster barrier phase
            cluster_arrive();
            cluster_wait();
        }
    }
    if (S > 1) {
        cluster_sync_all();  // every partial row has landed in its owner's smem
        // All producer threads reduce: S images' worth of threads per image row
        // would idle, so each of the 128/rows_per threads of an image sums a
        // column slice over the S partials and the slices' masks are OR-ed
        // across the group (consecutive lanes) before one lane finishes it.
        if (tid < kCorrProducers) {
            griddep_wait();  // the previous completion kernel is done with records / the pending list
            const int per = kCorrProducers / rows_per;  // S threads per image (rows_per = 128 / S)
            const int r = tid / per, part = tid % per;
            const int row = static_cast<int>(rank) * rows_per + r;
            const int64_t img = m0 + row;
            uint64_t pos = 0, zer = 0;
            auto slice = [&](auto nc_tag) {
                constexpr int NC = decltype(nc_tag)::value;
                const int c0 = part * NC;
                uint32_t acc[NC];
#pragma unroll
                for (int i = 0; i < NC; ++i) acc[i] = 0;
                for (uint32_t s = 0; s < S; ++s) {
                    const int4* src = reinterpret_cast<const int4*>(&red[(s * rows_per + r) * kRedStride + c0]);
#pragma unroll
                    for (int q = 0; q < NC / 4; ++q) {
                        const int4 v = src[q];
                        acc[4 * q] += v.x;
                        acc[4 * q + 1] += v.y;
                        acc[4 * q + 2] += v.z;
                        acc[4 * q + 3] += v.w;
                    }
                }
                if (row < tile_m && img < p.count) image_columns<NC>(p, sm, img, c0, acc, pos, zer);
            };
            if (per == 8) slice(std::integral_constant<int, kCorrN / 8>{});       // S = 8 (forced)
            else if (per == 4) slice(std::integral_constant<int, kCorrN / 4>{});  // S = 4
            else slice(std::integral_constant<int, kCorrN / 2>{});                // S = 2
            for (int o = 1; o < per; o <<= 1) {  // the group's lanes are consecutive
                pos |= __shfl_xor_sync(0xffffffffu, pos, o);
                zer |= __shfl_xor_sync(0xffffffffu, zer, o);
            }
            if (part == 0 && row < tile_m && img < p.count) finish_masks(p, sm, tl, img, pos, zer);
        }
    }
    __syncthreads();
    if (sm.nties > 0) finish_ties(p, sm, tl, warp, lane);  // rare: exact zero correlations
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc<kCorrN>(tmem);
    }
}

static cudaLaunchConfig_t corr_config(unsigned grid, unsigned S, cudaStream_t st, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kCorrThreads);
    cfg.dynamicSmemBytes = kCorrSmemBytes;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch: the prologue and streaming may overlap the
    // previous kernel; the epilogue griddep_wait()s before writing outputs
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cfg;
}

// Co-resident clusters of size S (one CTA per SM; clusters must fit a GPC),
// cached per device.
static int max_active_clusters(unsigned S, int sms) {
    static std::atomic<int> table[kMaxDevices][9];
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int>* cache = table[dev < kMaxDevices ? dev : 0];
    if (cache[S].load() == 0) {
        cudaLaunchAttribute attr[2];
        cudaLaunchConfig_t cfg = corr_config(S * 64, S, nullptr, attr);
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, corr_detect_kernel, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = sms / static_cast<int>(S);
        }
        cache[S].store(n);
    }
    return cache[S].load();
}

cudaError_t launch_corr_detect(const DetectParams& p_in, int sm_count, cudaStream_t st) {
    // function attributes belong to each device's context: set once per device
    static PerDeviceOnce once;
    cudaError_t e = once.run([] {
        cudaError_t r = cudaFuncSetAttribute(corr_detect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kCorrSmemBytes));
        if (r != cudaSuccess) return r;
        cudaFuncSetAttribute(corr_detect_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaGetLastError();
        return cudaSuccess;
    });
    if (e != cudaSuccess) return e;
    const int64_t tiles128 = (p_in.count + kCorrM - 1) / kCorrM;
    if (tiles128 == 0) return cudaSuccess;
    // Split K over a cluster when there are too few 128-image tiles to give
    // every SM a CTA (waves of co-resident clusters from the occupancy query).
    const int sms = sm_count > 0 ? sm_count : 148;
    unsigned S = 1;
    while (S < 4 && tiles128 * S * 2 <= sms && (p_in.K_pad / kCorrKC) >= static_cast<int>(8 * S * 2)) S *= 2;
    if (p_in.ksplit == 1 || p_in.ksplit == 2 || p_in.ksplit == 4 || p_in.ksplit == 8)
        S = static_cast<unsigned>(p_in.ksplit);  // forced (context's QRM_CORR_KSPLIT)
    // Balance: whole waves of co-resident clusters, each tile <= 128 images.
    const int64_t per_wave = max_active_clusters(S, sms);
    const int64_t waves = (tiles128 + per_wave - 1) / per_wave;
    int64_t tiles = waves * per_wave;
    int64_t tile_m = (p_in.count + tiles - 1) / tiles;
    if (tile_m < 16) tile_m = 16;  // never split a tile into slivers
    tiles = (p_in.count + tile_m - 1) / tile_m;
    DetectParams p = p_in;
    p.tile_m = static_cast<int32_t>(tile_m);
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = corr_config(static_cast<unsigned>(tiles) * S, S, st, attr);
    return cudaLaunchKernelEx(&cfg, corr_detect_kernel, p);
}

// The pattern operand per 128-byte K chunk as the exact shared-memory image the
// MMA reads (64 rows x 128 B, 128B-swizzled K-major): chunk kc at
// out + kc * 8 KB, so a stage fetches it with one bulk copy instead of 512
// 16-byte cp.async.
__global__ void swizzle_patterns_kernel(const int8_t* __restrict__ pat, int K_pad, int8_t* __restrict__ out) {
    const int64_t total = static_cast<int64_t>(K_pad / kCorrKC) * kCorrN * (kCorrKC / 16);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % (kCorrKC / 16));
        const int n = static_cast<int>((i / (kCorrKC / 16)) % kCorrN);
        const int64_t kc = i / (kCorrKC / 16) / kCorrN;
        const uint4 v = *reinterpret_cast<const uint4*>(pat + static_cast<int64_t>(n) * K_pad + kc * kCorrKC + c * 16);
        *reinterpret_cast<uint4*>(out + kc * kCorrBBytes + sw128_offset(n, c)) = v;
    }
}

cudaError_t launch_swizzle_patterns(const int8_t* pat, int K_pad, int8_t* out, cudaStream_t st) {
    swizzle_patterns_kernel<<<148, 256, 0, st>>>(pat, K_pad, out);
    return cudaGetLastError();
}

size_t corr_smem_bytes() { return kCorrSmemBytes; }

}  // namespace qrm
