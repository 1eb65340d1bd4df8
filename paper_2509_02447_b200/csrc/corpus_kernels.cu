// Device-side construction of the codec state and of synthetic inputs.
//
//  * pattern planes P_i[px] = (rng_word(seed, i, px) & 1) ? +1 : -1
//    (SpreadSpectrumCodec ctor, stego.cpp:16-27), stored as the s8 B operand
//    [64][K_pad] of the correlation GEMM, plus colsum_i = sum_px P_i[px];
//  * the benchmark corpus (cmd_bench recipe, cli.cpp:404-411):
//    synthetic_image (image.cpp:157-189) -> normalize (image.cpp:32-38) ->
//    embed_image_grid (stego.cpp:77-92) -> denormalize (image.cpp:49-55).
//    Double/float arithmetic uses explicit _rn intrinsics so no FMA
//    contraction changes a rounding relative to the reference's x86 build.
#include <cuda_runtime.h>

#include "qrm_device.cuh"
#include "qrm_types.h"

namespace qrm {

__global__ void build_patterns_kernel(uint64_t seed, int nbits, int K, int K_pad, int8_t* __restrict__ pat,
                                      int32_t* __restrict__ colsum) {
    const int row = blockIdx.y;  // 0..63
    int local = 0;
    for (int px = blockIdx.x * blockDim.x + threadIdx.x; px < K_pad; px += gridDim.x * blockDim.x) {
        int8_t v = 0;
        if (row < nbits && px < K) v = (rng_word(seed, static_cast<uint64_t>(row), static_cast<uint64_t>(px)) & 1) ? 1 : -1;
        pat[static_cast<int64_t>(row) * K_pad + px] = v;
        local += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local != 0) atomicAdd(colsum + row, local);
}

// delta[px] = sum_i (2 b_i - 1) P_i[px] (SpreadSpectrumCodec::residual, stego.cpp:29-38).
__global__ void residual_kernel(uint64_t seed, int nbits, int K, uint64_t codeword, float* __restrict__ delta) {
    for (int px = blockIdx.x * blockDim.x + threadIdx.x; px < K; px += gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (int i = 0; i < nbits; ++i) {
            const float sign = ((codeword >> (nbits - 1 - i)) & 1) ? 1.0f : -1.0f;
            const float p = (rng_word(seed, static_cast<uint64_t>(i), static_cast<uint64_t>(px)) & 1) ? 1.0f : -1.0f;
            acc = __fadd_rn(acc, __fmul_rn(sign, p));
        }
        delta[px] = acc;
    }
}

__device__ __forceinline__ uint8_t quantize_u8(double v) {  // image.cpp:42-45
    double q = floor(__dadd_rn(v, 0.5));
    q = fmin(fmax(q, 0.0), 255.0);
    return static_cast<uint8_t>(q);
}

__device__ __forceinline__ float normalize_u8(uint8_t v) {  // image.cpp:36
    return __double2float_rn(__dsub_rn(__ddiv_rn(static_cast<double>(v), 127.5), 1.0));
}

struct CorpusParams {
    uint64_t first_seed;
    int64_t count;
    int32_t w, h, l, embed;
    float alpha;
    const float* delta;  // [3 l^2] when embed
    uint8_t* out;
};

// grid: (row blocks, images); one thread per pixel (3 channels).
__global__ void __launch_bounds__(256) corpus_kernel(const __grid_constant__ CorpusParams p) {
    __shared__ double coef[3][3][4];  // amp, fx, fy, phase
    constexpr double kTau = 6.283185307179586;
    for (int64_t img = blockIdx.y; img < p.count; img += gridDim.y) {
        const uint64_t seed = p.first_seed + static_cast<uint64_t>(img);
        __syncthreads();
        if (threadIdx.x < 36) {
            // CounterRng(seed, 0x514e) draws in order (c, i, {amp, fx, fy, phase}).
            const int q = threadIdx.x, c = q / 12, i = (q / 4) % 3, f = q % 4;
            const double u = rng_unit(seed, 0x514e, static_cast<uint64_t>(q));
            double v;
            if (f == 0) v = __dadd_rn(10.0, __dmul_rn(14.0, u));
            else if (f == 3) v = __dmul_rn(kTau, u);
            else v = __dadd_rn(1.0, floor(__dmul_rn(u, 4.0)));
            coef[c][i][f] = v;
        }
        __syncthreads();
        const int w = p.w, h = p.h;
        const int64_t npx = static_cast<int64_t>(w) * h;
        uint8_t* dst = p.out + img * npx * 3;
        const int hm1 = h - 1 > 1 ? h - 1 : 1;
        const int hh = h > 1 ? h : 1;
        for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < npx;
             q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int y = static_cast<int>(q / w), x = static_cast<int>(q % w);
            const double gradient =
                __dadd_rn(118.0, __dmul_rn(90.0, __dsub_rn(__ddiv_rn(__dsub_rn(__dsub_rn(static_cast<double>(h), 1.0),
                                                                             static_cast<double>(y)),
                                                                   static_cast<double>(hm1)),
                                                          0.5)));
            const double ta = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, static_cast<double>(y)), static_cast<double>(hh)));
            const double tex = __dmul_rn(34.0, fmax(0.0, ta));
            const bool in_cell = p.embed && (x / p.l + 1) * p.l <= w && (y / p.l + 1) * p.l <= h;
            const int cpx = ((y % p.l) * p.l + (x % p.l)) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double v = gradient;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const double arg = __dadd_rn(
                        __dmul_rn(kTau, __dadd_rn(__ddiv_rn(__dmul_rn(coef[c][i][1], static_cast<double>(x)),
                                                            static_cast<double>(w)),
                                                  __ddiv_rn(__dmul_rn(coef[c][i][2], static_cast<double>(y)),
                                                            static_cast<double>(h)))),
                        coef[c][i][3]);
                    v = __dadd_rn(v, __dmul_rn(coef[c][i][0], cos(arg)));
                }
                const double u = rng_unit(seed, 0x7e30 + c, static_cast<uint64_t>(q));
                v = __dadd_rn(v, __dmul_rn(tex, __dsub_rn(__dmul_rn(2.0, u), 1.0)));
                uint8_t b = quantize_u8(v);
                if (p.embed) {
                    float f = normalize_u8(b);
                    if (in_cell) {
                        f = __fadd_rn(f, __fmul_rn(p.alpha, p.delta[cpx + c]));
                        f = fminf(fmaxf(f, -1.0f), 1.0f);
                    }
                    b = quantize_u8(__dmul_rn(__dadd_rn(static_cast<double>(f), 1.0), 127.5));
                }
                dst[q * 3 + c] = b;
            }
        }
    }
}

// SpreadSpectrumCodec::extract (stego.cpp:53-67) on an arbitrary normalised
// float tile: one thread per bit replays the reference's sequential double
// summation in pixel order (patterns regenerated from the counter RNG), so the
// soft values are bit-identical to the reference's.
__global__ void extract_float_kernel(uint64_t seed, int nbits, int K, const float* __restrict__ tile,
                                     double* __restrict__ soft) {
    const int bit = blockIdx.x * blockDim.x + threadIdx.x;
    if (bit >= nbits) return;
    double acc = 0.0;
    for (int px = 0; px < K; ++px) {
        const double d = static_cast<double>(tile[px]);
        acc = (rng_word(seed, static_cast<uint64_t>(bit), static_cast<uint64_t>(px)) & 1) ? __dadd_rn(acc, d)
                                                                                         : __dsub_rn(acc, d);
    }
    soft[bit] = __dmul_rn(acc, 1.0 / static_cast<double>(K));
}

cudaError_t launch_extract_float(uint64_t seed, int nbits, int K, const float* tile, double* soft, cudaStream_t st) {
    extract_float_kernel<<<(nbits + 63) / 64, 64, 0, st>>>(seed, nbits, K, tile, soft);
    return cudaGetLastError();
}

cudaError_t launch_build_patterns(uint64_t seed, int nbits, int K, int K_pad, int8_t* pat, int32_t* colsum,
                                  cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(colsum, 0, sizeof(int32_t) * kMaxNBits, st);
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>((K_pad + 1023) / 1024), kMaxNBits);
    build_patterns_kernel<<<grid, 256, 0, st>>>(seed, nbits, K, K_pad, pat, colsum);
    return cudaGetLastError();
}

cudaError_t launch_residual(uint64_t seed, int nbits, int K, uint64_t codeword, float* delta, cudaStream_t st) {
    residual_kernel<<<static_cast<unsigned>((K + 255) / 256), 256, 0, st>>>(seed, nbits, K, codeword, delta);
    return cudaGetLastError();
}

cudaError_t launch_corpus(uint64_t first_seed, int64_t count, int w, int h, int l, int embed, float alpha,
                          const float* delta, uint8_t* out, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    CorpusParams p{first_seed, count, w, h, l, embed, alpha, delta, out};
    const int64_t npx = static_cast<int64_t>(w) * h;
    unsigned gx = static_cast<unsigned>((npx + 255) / 256);
    if (gx > 64) gx = 64;
    const unsigned gy = static_cast<unsigned>(count < 65535 ? count : 65535);
    corpus_kernel<<<dim3(gx, gy), 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace qrm
