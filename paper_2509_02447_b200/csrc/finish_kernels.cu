// Completion and staging kernels of the detection path (sm_100a):
//  * detect_finish_kernel — exact tie resolution (tie_bit_exact, qrm_window.cuh) + general-t RS + verify for
//    the records the decode kernel (corr_kernel.cu) left pending;
//  * gather_windows_kernel / resample_kernel — the preprocess geometry
//    (bilinear upscale, centre crop, transforms.cpp:24-84) evaluated only on
//    the pixels that are used.
#include <cuda_runtime.h>

#include "qrm_device.cuh"
#include "qrm_rs.cuh"
#include "qrm_types.h"
#include "qrm_window.cuh"

namespace qrm {

// Completes pending records: resolves exact-zero correlations bit-exactly,
// then RS-corrects (t = 1 closed form or warp Berlekamp-Massey) and verifies.
// One warp per pending image; lane b re-evaluates tied bit b.
template <int TMAX>
__global__ void __launch_bounds__(256) detect_finish_kernel(const __grid_constant__ DetectParams p) {
    __shared__ RsSmem T;
    __shared__ int32_t elut[kTieLutWords];  // tie_bit_exact's residual table (qrm_window.cuh)
    __shared__ int npend_s;
    griddep_wait();               // the decode grid's records and pending list are complete
    griddep_launch_dependents();  // the next decode may start its prologue
    if (threadIdx.x == 0) npend_s = *reinterpret_cast<volatile int32_t*>(p.pending_count);
    __syncthreads();
    const int npend = npend_s;
    if (npend > 0) {  // nothing to do: skip the staging
        rs_stage_tables(T, p.rs, threadIdx.x, blockDim.x);
        tie_lut_fill(elut, threadIdx.x, blockDim.x);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); e < npend;
         e += warps) {
        const PendingEntry pe = p.pending[e];
        uint64_t raw = p.out[pe.image].raw;
        const int nb = p.nbits;
        // each tied bit by the whole warp (exact int64 dot product; tied bits are 0 in raw)
        for (uint64_t m = pe.tie_mask; m; m &= m - 1) {
            const int b = __ffsll(static_cast<long long>(m)) - 1;
            if (tie_bit_exact(p.src, pe.image, p.K, p.patterns + static_cast<int64_t>(b) * p.K_pad, elut, lane))
                raw |= 1ull << (nb - 1 - b);
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
    // The last block to finish re-arms the pending counter for the next
    // launch (pending_count[1] is the block ticket), so no memset is needed.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int ticket = atomicAdd(p.pending_count + 1, 1);
        if (ticket == static_cast<int>(gridDim.x) - 1) {
            p.pending_count[0] = 0;
            p.pending_count[1] = 0;
            __threadfence();
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


// Host-buffer path, transfer stage: copy each image's l x l window from
// mapped (zero-copy) pinned host memory into contiguous device windows. Only
// the window crosses PCIe (3 l^2 of the 3 w h bytes). Plain 16-B loads, NB per
// thread in flight before any store, keep enough reads outstanding to fill the
// link (measured ~48 GB/s of the ~55 GB/s copy-engine rate, round-1 PCIe probe in profiles/r1_pcie_probe.log).
template <int NB>
__global__ void __launch_bounds__(256) fetch_windows_kernel(const WindowSource src, int64_t count, int K,
                                                            uint8_t* __restrict__ out) {
    const int row16 = (3 * src.l) / 16;  // 16-B chunks per window row
    const int per_img = src.l * row16;
    const int64_t total = count * per_img;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; base < total;
         base += stride * NB) {
        uint4 v[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int64_t i = base + j * stride;
            if (i < total) {
                const int64_t img = i / per_img;
                const int rem = static_cast<int>(i - img * per_img);
                const int r = rem / row16, c = rem - r * row16;
                v[j] = __ldg(reinterpret_cast<const uint4*>(window_base(src, img, K) +
                                                            static_cast<int64_t>(r) * src.pitch) + c);
            }
        }
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int64_t i = base + j * stride;
            if (i < total) reinterpret_cast<uint4*>(out)[i] = v[j];  // windows packed contiguously
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


cudaError_t launch_fetch_windows(const WindowSource& src, int64_t count, int K, uint8_t* out, int sm_count,
                                 cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    const int64_t chunks = count * (K / 16);
    int64_t grid = (chunks + 256 * 4 - 1) / (256 * 4);
    const int64_t cap = 2 * (sm_count > 0 ? sm_count : 148);  // leave the SMs' smem to the decode kernel
    if (grid > cap) grid = cap;
    fetch_windows_kernel<4><<<static_cast<unsigned>(grid), 256, 0, st>>>(src, count, K, out);
    return cudaGetLastError();
}

cudaError_t launch_detect_finish(const DetectParams& p, int tmax, int sm_count, cudaStream_t st) {
    // Programmatic dependent launch: the completion kernel's launch overlaps the
    // decode kernel's tail; it griddep_wait()s before reading the decode's output.
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sm_count > 0 ? sm_count : 148);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (tmax <= 1) return cudaLaunchKernelEx(&cfg, detect_finish_kernel<1>, p);
    if (tmax <= 2) return cudaLaunchKernelEx(&cfg, detect_finish_kernel<2>, p);
    if (tmax <= 4) return cudaLaunchKernelEx(&cfg, detect_finish_kernel<4>, p);
    return cudaLaunchKernelEx(&cfg, detect_finish_kernel<8>, p);
}

cudaError_t launch_gather_windows(const GatherDesc* descs, int64_t count, int l, uint8_t* out, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const int K = 3 * l * l;
    dim3 grid(static_cast<unsigned>((K + 255) / 256), static_cast<unsigned>(count < 65535 ? count : 65535));
    gather_windows_kernel<<<grid, 256, 0, st>>>(descs, count, l, out);
    return cudaGetLastError();
}

// SyntheticStageLoad on the device: holds the stream for `ns` nanoseconds (one
// warp, global timer), the stage-stream analogue of the reference's
// synthetic_wait sleep (detect.cpp:243-245).
__global__ void stage_load_kernel(long long ns) {
    if (threadIdx.x != 0) return;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(2000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (static_cast<long long>(t - t0) < ns);
}

cudaError_t launch_stage_load(long long ns, cudaStream_t st) {
    if (ns <= 0) return cudaSuccess;
    stage_load_kernel<<<1, 32, 0, st>>>(ns);
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


}  // namespace qrm
