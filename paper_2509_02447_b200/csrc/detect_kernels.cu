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
// (image, bit) pairs are re-evaluated with the reference's exact sequential
// double summation by detect_finish_kernel, so hard bits are bit-exact.
//
// corr_detect_kernel: one CTA = 128 images (UMMA M) x 64 bit columns (N) x
// the whole K = 3 l^2. Warps 0-3 stream 128-byte K chunks of the 128 tile
// windows (cp.async, 16 B per thread, written straight into the 128B-swizzled
// K-major operand layout) and of the pattern matrix into a 6-stage smem ring;
// warp 4 issues tcgen05.mma kind::i8 (u8 x s8 -> s32, accumulators in TMEM).
// The epilogue (warps 0-3, one image per thread = one TMEM lane) reads 64
// columns with tcgen05.ld, forms S, hardens, packs the raw word and — for
// t = 1 codes without ties — runs the RS decoder and verify in registers, so
// one launch produces final records.
#include <cuda_runtime.h>

#include "qrm_device.cuh"
#include "qrm_rs.cuh"
#include "qrm_types.h"

namespace qrm {

constexpr int kCorrM = 128;
constexpr int kCorrN = 64;
constexpr int kCorrKC = 128;  // bytes of K per stage
constexpr int kCorrStages = 6;
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
    int32_t colsum[kCorrN];
    RsSmem rs;
    // Split-K partials from the cluster: [rank][row within my 128/S rows][kRedStride]
    alignas(16) int32_t red[kCorrM * kRedStride];
};

constexpr size_t kCorrSmemBytes = 1024 /*align slack*/ + kCorrStages * kCorrStageBytes + sizeof(CorrSmem);

// Epilogue for one image (one TMEM lane): S = 2 D - 255 colsum, harden, pack,
// and — t = 1 code, no exact-zero correlation — RS-correct + verify in place.
__device__ __forceinline__ void finish_image(const DetectParams& p, const CorrSmem& sm, int64_t img,
                                             const uint32_t (&acc)[kCorrN]) {
    const int nb = p.nbits;
    uint64_t raw = 0, tmask = 0;
    const double inv = 1.0 / (255.0 * static_cast<double>(p.K));
#pragma unroll
    for (int i = 0; i < kCorrN; ++i) {
        if (i < nb) {
            const int S = 2 * static_cast<int>(acc[i]) - 255 * sm.colsum[i];
            raw |= static_cast<uint64_t>(S > 0) << (nb - 1 - i);
            tmask |= static_cast<uint64_t>(S == 0) << i;
            if (p.soft) p.soft[img * nb + i] = static_cast<double>(S) * inv;
        }
    }
    if (p.raw_out) p.raw_out[img] = raw;
    qrm_record rec;
    if (tmask == 0 && p.fuse_t1) {
        uint64_t cw = 0;
        const int nerr = rs_t1_packed(sm.rs, raw, cw);
        make_record(rec, raw, nerr, cw, nb, p.kbits, p.key_cw, p.key_msg, p.tau_msg, p.tau_raw, 0);
    } else {
        rec.raw = raw;
        rec.msg = 0;
        rec.status = kRecPending;
        rec.errors = 0;
        rec.matches = 0;
        rec.verified = 0;
        rec.ties = static_cast<uint8_t>(__popcll(tmask));
        rec.reserved[0] = rec.reserved[1] = rec.reserved[2] = 0;
        const int slot = atomicAdd(p.pending_count, 1);
        p.pending[slot] = PendingEntry{img, tmask};
    }
    store_record(p.out + img, rec);
}

// Diagnostics: per-CTA phase timestamps (thread 0), only when requested.
__device__ __forceinline__ void dbg_mark(const DetectParams& p, int phase, int tid) {
    if (p.dbg_times && tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.dbg_times[static_cast<int64_t>(blockIdx.x) * 8 + phase] = t;
    }
}

__device__ __forceinline__ const uint8_t* window_base(const WindowSource& s, int64_t img, int K) {
    if (!s.direct) return s.base + img * static_cast<int64_t>(K);
    int tx, ty;
    select_tile(kWorkingSize, kWorkingSize, s.l, s.strategy, s.tile_seed, s.first_draw + static_cast<uint64_t>(img),
                tx, ty);
    return s.base + img * s.image_stride + static_cast<int64_t>(s.y_off + ty) * s.pitch +
           static_cast<int64_t>(s.x_off + tx) * 3;
}

// Launched as clusters of S = 1, 2 or 4 CTAs along K (split-K): CTA r of a
// cluster accumulates K chunks [r K/S, (r+1) K/S) of the same 128 images in its
// own TMEM, pushes the partial rows owned by each peer into the peer's shared
// memory (DSMEM), and after one cluster barrier each CTA finishes 128/S images.
__global__ void __launch_bounds__(kCorrThreads, 1) corr_detect_kernel(const __grid_constant__ DetectParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    CorrSmem& sm = *reinterpret_cast<CorrSmem*>(ring + kCorrStages * kCorrStageBytes);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    dbg_mark(p, 0, tid);
    const uint32_t S = cluster_nctarank();  // 1 without a cluster launch
    const uint32_t rank = cluster_ctarank();
    const int64_t m0 = static_cast<int64_t>(blockIdx.x / S) * kCorrM;
    const int kc_total = p.K_pad / kCorrKC;
    const int kc_begin = static_cast<int>(static_cast<int64_t>(kc_total) * rank / S);
    const int kchunks = static_cast<int>(static_cast<int64_t>(kc_total) * (rank + 1) / S) - kc_begin;

    if (warp == 4) tmem_alloc<kCorrN>(&sm.tmem_base);
    if (tid == 0) {
        for (int s = 0; s < kCorrStages; ++s) {
            mbar_init(&sm.full[s], kCorrProducers);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.accum_full, 1);
        mbar_fence_init();
    }
    for (int i = tid; i < kCorrN; i += kCorrThreads) sm.colsum[i] = p.colsum[i];
    if (p.fuse_t1) rs_stage_tables(sm.rs, p.rs, tid, kCorrThreads);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const int rows_per = kCorrM / static_cast<int>(S);
    dbg_mark(p, 1, tid);

    if (warp < 4) {
        // ------------------------------------------------------ producer --
        const int c = tid & 7;       // 16-byte chunk within the 128-byte K chunk
        const int rb = tid >> 3;     // rows rb + 16 j
        const uint8_t* wb[8];
        bool valid[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t img = m0 + rb + 16 * j;
            valid[j] = img < p.count;
            wb[j] = valid[j] ? window_base(p.src, img, p.K) : nullptr;
        }
        const int row_bytes = 3 * p.src.l;
        const int pitch = p.src.direct ? p.src.pitch : row_bytes;
        const uint32_t ring_u32 = smem_u32(ring);
        for (int it = 0; it < kchunks; ++it) {
            const int s = it % kCorrStages;
            mbar_wait(&sm.empty[s], ((it / kCorrStages) & 1) ^ 1);
            const uint32_t a_s = ring_u32 + s * kCorrStageBytes;
            const uint32_t b_s = a_s + kCorrABytes;
            const int kbyte = (kc_begin + it) * kCorrKC + c * 16;
            if (kbyte < p.K) {
                const int trow = kbyte / row_bytes;
                const int64_t off = static_cast<int64_t>(trow) * pitch + (kbyte - trow * row_bytes);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (valid[j]) cp_async16(a_s + sw128_offset(rb + 16 * j, c), wb[j] + off);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = rb + 16 * j;
                cp_async16(b_s + sw128_offset(n, c), p.patterns + static_cast<int64_t>(n) * p.K_pad + kbyte);
            }
            // Never block on the copies: the barrier phase completes when every
            // producer's copies for this stage have landed. (A wait_group +
            // proxy fence here drains ALL in-flight copies and serialises the
            // ring to one stage — measured 18% of HBM bandwidth.)
            cp_async_mbar_arrive(&sm.full[s]);
        }
        cp_async_wait<0>();

        // ------------------------------------------------------ epilogue --
        dbg_mark(p, 2, tid);
        mbar_wait(&sm.accum_full, 0);
        dbg_mark(p, 3, tid);
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
        dbg_mark(p, 4, tid);

        const int row = warp * 32 + lane;
        if (S == 1) {
            const int64_t img = m0 + row;
            if (img < p.count) finish_image(p, sm, img, acc);
            dbg_mark(p, 5, tid);
        } else {
            // push this partial row to its owner CTA: slot `rank`, local row
            const uint32_t owner = static_cast<uint32_t>(row / rows_per);
            const uint32_t local = static_cast<uint32_t>(row % rows_per);
            const uint32_t dst = map_to_rank(
                smem_u32(&sm.red[(rank * rows_per + local) * kRedStride]), owner);
#pragma unroll
            for (int q = 0; q < kCorrN / 4; ++q)
                st_cluster_v4(dst + 16 * q, acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
            dbg_mark(p, 5, tid);
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
                if (!(p.exp_flags & 1)) fence_proxy_async_smem();
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
    }
    if (S > 1) {
        cluster_sync_all();  // every partial row has landed in its owner's smem
        dbg_mark(p, 6, tid);
        if (tid < rows_per) {
            uint32_t acc[kCorrN];
#pragma unroll
            for (int i = 0; i < kCorrN; ++i) acc[i] = 0;
            for (uint32_t s = 0; s < S; ++s) {
                const int4* src = reinterpret_cast<const int4*>(&sm.red[(s * rows_per + tid) * kRedStride]);
#pragma unroll
                for (int q = 0; q < kCorrN / 4; ++q) {
                    const int4 v = src[q];
                    acc[4 * q] += v.x;
                    acc[4 * q + 1] += v.y;
                    acc[4 * q + 2] += v.z;
                    acc[4 * q + 3] += v.w;
                }
            }
            const int64_t img = m0 + static_cast<int64_t>(rank) * rows_per + tid;
            if (img < p.count) finish_image(p, sm, img, acc);
        }
    }
    dbg_mark(p, 7, tid);
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc<kCorrN>(tmem);
    }
}

// Exact reference hard bit for a zero integer correlation: the reference sums
// double(float(v/127.5 - 1)) * P sequentially over px (stego.cpp:60-64) and
// tests soft > 0 (stego.cpp:12); replay that exact summation order.
__device__ __forceinline__ bool reference_tie_bit(const WindowSource& s, int64_t img, int K, const int8_t* pat) {
    const uint8_t* wb = window_base(s, img, K);
    const int row_bytes = 3 * s.l;
    const int pitch = s.direct ? s.pitch : row_bytes;
    double acc = 0.0;
    for (int px = 0; px < K; ++px) {
        const int trow = px / row_bytes;
        const uint8_t v = wb[static_cast<int64_t>(trow) * pitch + (px - trow * row_bytes)];
        const double d = static_cast<double>(__double2float_rn(__dsub_rn(__ddiv_rn(static_cast<double>(v), 127.5), 1.0)));
        acc = pat[px] > 0 ? __dadd_rn(acc, d) : __dsub_rn(acc, d);
    }
    return acc * (1.0 / static_cast<double>(K)) > 0.0;
}

// Completes pending records: resolves exact-zero correlations bit-exactly,
// then RS-corrects (t = 1 closed form or warp Berlekamp-Massey) and verifies.
// One warp per pending image; lane b re-evaluates tied bit b.
template <int TMAX>
__global__ void __launch_bounds__(256) detect_finish_kernel(const __grid_constant__ DetectParams p) {
    __shared__ RsSmem T;
    rs_stage_tables(T, p.rs, threadIdx.x, blockDim.x);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int npend = *p.pending_count;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); e < npend;
         e += warps) {
        const PendingEntry pe = p.pending[e];
        uint64_t raw = p.out[pe.image].raw;
        const int nb = p.nbits;
        for (int b0 = 0; b0 < nb; b0 += 32) {
            const int b = b0 + lane;
            uint64_t setbit = 0;
            if (b < nb && ((pe.tie_mask >> b) & 1)) {
                const bool bit = reference_tie_bit(p.src, pe.image, p.K, p.patterns + static_cast<int64_t>(b) * p.K_pad);
                setbit = static_cast<uint64_t>(bit) << (nb - 1 - b);
            }
            // OR-reduce the resolved bits (tied bits were 0 in raw)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) setbit |= __shfl_xor_sync(0xffffffffu, setbit, o);
            raw |= setbit;
        }
        if (p.raw_out && lane == 0) p.raw_out[pe.image] = raw;
        int nerr;
        uint64_t cw = 0;
        if (T.t == 1 && T.r <= 3) {
            nerr = rs_t1_packed(T, raw, cw);
        } else {
            uint32_t sym[1];
            const int i = lane;
            sym[0] = i < T.n ? static_cast<uint32_t>((raw >> (T.m * (T.n - 1 - i))) & ((1u << T.m) - 1)) : 0u;
            nerr = rs_warp_bm<TMAX, 1>(T, sym, lane);
            uint64_t part = 0;
            if (nerr >= 0 && i < T.n) part = static_cast<uint64_t>(sym[0]) << (T.m * (T.n - 1 - i));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part |= __shfl_xor_sync(0xffffffffu, part, o);
            cw = part;
        }
        if (lane == 0) {
            qrm_record rec;
            make_record(rec, raw, nerr, cw, nb, p.kbits, p.key_cw, p.key_msg, p.tau_msg, p.tau_raw,
                        __popcll(pe.tie_mask));
            store_record(p.out + pe.image, rec);
        }
    }
}

// One output sample of the preprocess geometry: pixel (ox, oy) of the
// (virtual) resized image, channel c — a direct read, or resize_bilinear
// (image.cpp:57-85) evaluated in double with no FMA contraction.
__device__ __forceinline__ uint8_t sample_pixel(const GatherDesc& d, int ox, int oy, int c) {
    if (!d.upscale) return d.img[(static_cast<int64_t>(oy) * d.w + ox) * 3 + c];
    const double sx = __ddiv_rn(static_cast<double>(d.w), static_cast<double>(d.sw));
    const double sy = __ddiv_rn(static_cast<double>(d.h), static_cast<double>(d.sh));
    const double fy = __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(oy), 0.5), sy), 0.5);
    const double y0d = floor(fy);
    const double wy = __dsub_rn(fy, y0d);
    const int y0 = min(max(static_cast<int>(y0d), 0), d.h - 1);
    const int y1 = min(max(static_cast<int>(y0d) + 1, 0), d.h - 1);
    const double fx = __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(ox), 0.5), sx), 0.5);
    const double x0d = floor(fx);
    const double wx = __dsub_rn(fx, x0d);
    const int x0 = min(max(static_cast<int>(x0d), 0), d.w - 1);
    const int x1 = min(max(static_cast<int>(x0d) + 1, 0), d.w - 1);
    auto at = [&](int x, int y) { return static_cast<double>(d.img[(static_cast<int64_t>(y) * d.w + x) * 3 + c]); };
    const double omx = __dsub_rn(1.0, wx), omy = __dsub_rn(1.0, wy);
    const double top = __dadd_rn(__dmul_rn(at(x0, y0), omx), __dmul_rn(at(x1, y0), wx));
    const double bot = __dadd_rn(__dmul_rn(at(x0, y1), omx), __dmul_rn(at(x1, y1), wx));
    double q = floor(__dadd_rn(__dadd_rn(__dmul_rn(top, omy), __dmul_rn(bot, wy)), 0.5));
    q = fmin(fmax(q, 0.0), 255.0);
    return static_cast<uint8_t>(q);
}

// Stages one l x l window per image into a contiguous [count][3 l^2] buffer:
// the path for ragged batches, unaligned windows and inputs below the working
// size, whose preprocess is a bilinear upscale (image.cpp:57-85 composed with
// the centre crop, transforms.cpp:49-84) evaluated only on the window.
__global__ void gather_windows_kernel(const GatherDesc* __restrict__ descs, int64_t count, int l,
                                      uint8_t* __restrict__ out) {
    const int K = 3 * l * l;
    for (int64_t img = blockIdx.y; img < count; img += gridDim.y) {
        const GatherDesc d = descs[img];
        uint8_t* dst = out + img * static_cast<int64_t>(K);
        for (int px = blockIdx.x * blockDim.x + threadIdx.x; px < K; px += gridDim.x * blockDim.x) {
            const int c = px % 3, xy = px / 3;
            dst[px] = sample_pixel(d, d.tx + xy % l + d.x_off, d.ty + xy / l + d.y_off, c);
        }
    }
}

// Rectangular out_w x out_h window of one image (resize / crop / preprocess
// host utilities), optionally normalised to float(v/127.5 - 1) (image.cpp:36).
__global__ void resample_kernel(const GatherDesc d, int out_w, int out_h, int normalize, void* __restrict__ out) {
    const int64_t n = static_cast<int64_t>(out_w) * out_h * 3;
    for (int64_t px = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; px < n;
         px += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(px % 3);
        const int64_t xy = px / 3;
        const uint8_t v = sample_pixel(d, static_cast<int>(xy % out_w) + d.x_off, static_cast<int>(xy / out_w) + d.y_off, c);
        if (normalize)
            static_cast<float*>(out)[px] = __double2float_rn(__dsub_rn(__ddiv_rn(static_cast<double>(v), 127.5), 1.0));
        else
            static_cast<uint8_t*>(out)[px] = v;
    }
}

// ---------------------------------------------------------------- launch --
static inline bool ok(cudaError_t e) { return e == cudaSuccess; }

cudaError_t launch_corr_detect(const DetectParams& p, int sm_count, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(corr_detect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kCorrSmemBytes));
        if (!ok(e)) return e;
        configured = true;
    }
    const int64_t tiles = (p.count + kCorrM - 1) / kCorrM;
    if (tiles == 0) return cudaSuccess;
    // Split K over a cluster when there are too few 128-image tiles to give
    // every SM a CTA (one CTA per SM: the 6-stage ring uses ~180 KB of smem).
    const int sms = sm_count > 0 ? sm_count : 148;
    unsigned S = 1;
    while (S < 4 && tiles * S * 2 <= sms && (p.K_pad / kCorrKC) >= static_cast<int>(8 * S * 2)) S *= 2;
    if (const char* env = getenv("QRM_CORR_KSPLIT")) {  // experiment hook
        const int v = atoi(env);
        if (v == 1 || v == 2 || v == 4 || v == 8) S = static_cast<unsigned>(v);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(tiles) * S);
    cfg.blockDim = dim3(kCorrThreads);
    cfg.dynamicSmemBytes = kCorrSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, corr_detect_kernel, p);
}

cudaError_t launch_detect_finish(const DetectParams& p, int tmax, int sm_count, cudaStream_t st) {
    const int blocks = sm_count > 0 ? sm_count : 148;
    if (tmax <= 1) detect_finish_kernel<1><<<blocks, 256, 0, st>>>(p);
    else if (tmax <= 2) detect_finish_kernel<2><<<blocks, 256, 0, st>>>(p);
    else if (tmax <= 4) detect_finish_kernel<4><<<blocks, 256, 0, st>>>(p);
    else detect_finish_kernel<8><<<blocks, 256, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_gather_windows(const GatherDesc* descs, int64_t count, int l, uint8_t* out, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const int K = 3 * l * l;
    dim3 grid(static_cast<unsigned>((K + 255) / 256), static_cast<unsigned>(count < 65535 ? count : 65535));
    gather_windows_kernel<<<grid, 256, 0, st>>>(descs, count, l, out);
    return cudaGetLastError();
}

cudaError_t launch_resample(const GatherDesc& d, int out_w, int out_h, int normalize, void* out, cudaStream_t st) {
    const int64_t n = static_cast<int64_t>(out_w) * out_h * 3;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    resample_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(d, out_w, out_h, normalize, out);
    return cudaGetLastError();
}

size_t corr_smem_bytes() { return kCorrSmemBytes; }

}  // namespace qrm
