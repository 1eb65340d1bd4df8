// Robustness attacks on the device: apply_attack
// (transforms.cpp:289-362) over a batch of same-size byte images, bit-exact
// with the reference. Every double operation the reference performs is
// replayed in the same order with explicitly rounded intrinsics (no FMA
// contraction); transcendental constants (the Gaussian weights exp(-1/2),
// exp(-1), the DCT cosines) are evaluated on the host with the same libm calls
// the reference makes and passed in, so device libm never enters the result.
//
//   brightness / contrast / saturation / sharpness / blur / overlay_text:
//     attack_pixel_kernel, one thread per output byte;
//   contrast pivot: luma_mean_kernel, one thread per image summing in the
//     reference's pixel order (mean_luma, transforms.cpp:123-130);
//   jpeg_approx: jpeg_block_kernel, one thread per (image, channel, 8x8 block)
//     (jpeg_approx_attack, transforms.cpp:224-278);
//   centercrop / resizeto / crop / resize / normalize: the resample geometry
//     (resize_bilinear image.cpp:57-85, center_crop image.cpp:87-105).
#include <cuda_runtime.h>

#include "qrm_types.h"

namespace qrm {

namespace {

__device__ __forceinline__ uint8_t quantize_d(double v) {  // image.cpp:42-45
    double q = floor(__dadd_rn(v, 0.5));
    q = fmin(fmax(q, 0.0), 255.0);
    return static_cast<uint8_t>(q);
}

// x * v + (1 - x) * pivot (transforms.cpp:133-135)
__device__ __forceinline__ double lever_d(double x, double v, double pivot) {
    return __dadd_rn(__dmul_rn(x, v), __dmul_rn(__dsub_rn(1.0, x), pivot));
}

// 0.299 r + 0.587 g + 0.114 b, left to right
__device__ __forceinline__ double luma_d(const uint8_t* p) {
    return __dadd_rn(__dadd_rn(__dmul_rn(0.299, static_cast<double>(p[0])), __dmul_rn(0.587, static_cast<double>(p[1]))),
                     __dmul_rn(0.114, static_cast<double>(p[2])));
}

// gaussian3x3 (transforms.cpp:137-160) at one sample, quantized
__device__ __forceinline__ uint8_t gauss_at(const uint8_t* img, int w, int h, int x, int y, int c, double kC,
                                            double kE, double kD, double kSum) {
    double acc = 0.0;
    for (int dy = -1; dy <= 1; ++dy) {
        const int sy = min(max(y + dy, 0), h - 1);
        for (int dx = -1; dx <= 1; ++dx) {
            const int sx = min(max(x + dx, 0), w - 1);
            const double wgt = (dx == 0 && dy == 0) ? kC : (dx != 0 && dy != 0) ? kD : kE;
            acc = __dadd_rn(acc, __dmul_rn(wgt, static_cast<double>(img[(static_cast<int64_t>(sy) * w + sx) * 3 + c])));
        }
    }
    return quantize_d(__ddiv_rn(acc, kSum));
}

// "QRMARK" in the reference's 5x7 font (transforms.cpp:162-176), scaled x3 at (8, 8)
__constant__ uint8_t c_glyphs[6][7] = {
    {0b01110, 0b10001, 0b10001, 0b10001, 0b10101, 0b10010, 0b01101},  // Q
    {0b11110, 0b10001, 0b10001, 0b11110, 0b10100, 0b10010, 0b10001},  // R
    {0b10001, 0b11011, 0b10101, 0b10101, 0b10001, 0b10001, 0b10001},  // M
    {0b01110, 0b10001, 0b10001, 0b11111, 0b10001, 0b10001, 0b10001},  // A
    {0b11110, 0b10001, 0b10001, 0b11110, 0b10100, 0b10010, 0b10001},  // R
    {0b10001, 0b10010, 0b10100, 0b11000, 0b10100, 0b10010, 0b10001},  // K
};

__device__ __forceinline__ bool stamped(int x, int y) {  // overlay_text_stamp (transforms.cpp:178-205)
    constexpr int kScale = 3, kOx = 8, kOy = 8;
    const int gy = (y - kOy) / kScale;
    if (y < kOy || gy >= 7) return false;
    const int rel = x - kOx;
    if (rel < 0) return false;
    const int ch = rel / (6 * kScale), gx = (rel % (6 * kScale)) / kScale;
    if (ch >= 6 || gx >= 5) return false;
    return (c_glyphs[ch][gy] >> (4 - gx)) & 1;
}

}  // namespace

__global__ void luma_mean_kernel(AttackParams p) {
    const int64_t img = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (img >= p.count) return;
    const uint8_t* src = p.in + img * p.in_stride;
    double acc = 0.0;
    for (int y = 0; y < p.h; ++y)
        for (int x = 0; x < p.w; ++x) acc = __dadd_rn(acc, luma_d(src + (static_cast<int64_t>(y) * p.w + x) * 3));
    p.pivot[img] = __ddiv_rn(acc, __dmul_rn(static_cast<double>(p.w), static_cast<double>(p.h)));
}

__global__ void attack_pixel_kernel(AttackParams p) {
    const int64_t per = static_cast<int64_t>(p.w) * p.h * 3;
    const int64_t total = per * p.count;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t img = i / per;
        const int s = static_cast<int>(i - img * per);
        const int c = s % 3, xy = s / 3, x = xy % p.w, y = xy / p.w;
        const uint8_t* src = p.in + img * p.in_stride;
        const double v = static_cast<double>(src[s]);
        uint8_t o;
        switch (p.op) {
            case QRM_ATTACK_BRIGHTNESS: o = quantize_d(__dmul_rn(v, p.param)); break;
            case QRM_ATTACK_CONTRAST: o = quantize_d(lever_d(p.param, v, p.pivot[img])); break;
            case QRM_ATTACK_SATURATION: o = quantize_d(lever_d(p.param, v, luma_d(src + (s - c)))); break;
            case QRM_ATTACK_SHARPNESS:
                o = quantize_d(lever_d(p.param, v,
                                       static_cast<double>(gauss_at(src, p.w, p.h, x, y, c, p.kC, p.kE, p.kD, p.kSum))));
                break;
            case QRM_ATTACK_BLUR: o = gauss_at(src, p.w, p.h, x, y, c, p.kC, p.kE, p.kD, p.kSum); break;
            case QRM_ATTACK_OVERLAY_TEXT: o = stamped(x, y) ? uint8_t{255} : src[s]; break;
            default: o = src[s];
        }
        p.out[img * p.out_stride + s] = o;
    }
}

// dct8 (transforms.cpp:210-222) with host cosines C[u][i] = cos((2i+1) u pi / 16).
__device__ __forceinline__ void dct8_d(const double (&in)[8], double (&out)[8], bool inverse, const double* C,
                                       double c0) {
    if (!inverse) {
        for (int u = 0; u < 8; ++u) {
            const double cu = u == 0 ? c0 : 0.5;
            double acc = 0.0;
            for (int i = 0; i < 8; ++i) acc = __dadd_rn(acc, __dmul_rn(in[i], C[u * 8 + i]));
            out[u] = __dmul_rn(cu, acc);
        }
    } else {
        for (int i = 0; i < 8; ++i) {
            double acc = 0.0;
            for (int u = 0; u < 8; ++u) {
                const double cu = u == 0 ? c0 : 0.5;
                acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(cu, in[u]), C[u * 8 + i]));
            }
            out[i] = acc;
        }
    }
}

__global__ void jpeg_block_kernel(AttackParams p) {
    __shared__ double C[64], Q[64];
    if (threadIdx.x < 64) {
        C[threadIdx.x] = p.jpeg_cos[threadIdx.x];
        Q[threadIdx.x] = p.jpeg_quant[threadIdx.x];
    }
    __syncthreads();
    const int bw = (p.w + 7) / 8, bh = (p.h + 7) / 8;
    const int64_t per = static_cast<int64_t>(bw) * bh * 3;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= per * p.count) return;
    const int64_t img = t / per;
    int r = static_cast<int>(t - img * per);
    const int c = r % 3;
    r /= 3;
    const int bx = (r % bw) * 8, by = (r / bw) * 8;
    const uint8_t* src = p.in + img * p.in_stride;
    double block[8][8], tmp[8][8];
    for (int y = 0; y < 8; ++y)
        for (int x = 0; x < 8; ++x) {
            const int sx = min(bx + x, p.w - 1), sy = min(by + y, p.h - 1);
            block[y][x] = __dsub_rn(static_cast<double>(src[(static_cast<int64_t>(sy) * p.w + sx) * 3 + c]), 128.0);
        }
    for (int y = 0; y < 8; ++y) dct8_d(block[y], tmp[y], false, C, p.dct_c0);
    for (int x = 0; x < 8; ++x) {
        double col[8], res[8];
        for (int y = 0; y < 8; ++y) col[y] = tmp[y][x];
        dct8_d(col, res, false, C, p.dct_c0);
        for (int y = 0; y < 8; ++y) {
            const double q = Q[y * 8 + x];
            tmp[y][x] = __dmul_rn(round(__ddiv_rn(res[y], q)), q);
        }
    }
    for (int x = 0; x < 8; ++x) {
        double col[8], res[8];
        for (int y = 0; y < 8; ++y) col[y] = tmp[y][x];
        dct8_d(col, res, true, C, p.dct_c0);
        for (int y = 0; y < 8; ++y) tmp[y][x] = res[y];
    }
    uint8_t* dst = p.out + img * p.out_stride;
    for (int y = 0; y < 8; ++y) {
        double row[8];
        dct8_d(tmp[y], row, true, C, p.dct_c0);
        for (int x = 0; x < 8; ++x) {
            if (bx + x >= p.w || by + y >= p.h) continue;
            dst[(static_cast<int64_t>(by + y) * p.w + bx + x) * 3 + c] = quantize_d(__dadd_rn(row[x], 128.0));
        }
    }
}

// Geometry ops: output pixel (x, y) = pixel (x + x_off, y + y_off) of the
// image resized to sw x sh (resize = 0: the image itself); u8 or normalised.
__global__ void attack_resample_kernel(AttackParams p) {
    const int64_t per = static_cast<int64_t>(p.ow) * p.oh * 3;
    const int64_t total = per * p.count;
    const double sx = __ddiv_rn(static_cast<double>(p.w), static_cast<double>(p.sw));
    const double sy = __ddiv_rn(static_cast<double>(p.h), static_cast<double>(p.sh));
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t img = i / per;
        const int s = static_cast<int>(i - img * per);
        const int c = s % 3, xy = s / 3;
        const int ox = xy % p.ow + p.x_off, oy = xy / p.ow + p.y_off;
        const uint8_t* src = p.in + img * p.in_stride;
        uint8_t v;
        if (!p.resize) {
            v = src[(static_cast<int64_t>(oy) * p.w + ox) * 3 + c];
        } else {  // resize_bilinear (image.cpp:57-85), no FMA contraction
            const double fy = __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(oy), 0.5), sy), 0.5);
            const double y0d = floor(fy), wy = __dsub_rn(fy, y0d);
            const int y0 = min(max(static_cast<int>(y0d), 0), p.h - 1), y1 = min(max(static_cast<int>(y0d) + 1, 0), p.h - 1);
            const double fx = __dsub_rn(__dmul_rn(__dadd_rn(static_cast<double>(ox), 0.5), sx), 0.5);
            const double x0d = floor(fx), wx = __dsub_rn(fx, x0d);
            const int x0 = min(max(static_cast<int>(x0d), 0), p.w - 1), x1 = min(max(static_cast<int>(x0d) + 1, 0), p.w - 1);
            auto at = [&](int x, int y) { return static_cast<double>(src[(static_cast<int64_t>(y) * p.w + x) * 3 + c]); };
            const double omx = __dsub_rn(1.0, wx), omy = __dsub_rn(1.0, wy);
            const double top = __dadd_rn(__dmul_rn(at(x0, y0), omx), __dmul_rn(at(x1, y0), wx));
            const double bot = __dadd_rn(__dmul_rn(at(x0, y1), omx), __dmul_rn(at(x1, y1), wx));
            v = quantize_d(__dadd_rn(__dmul_rn(top, omy), __dmul_rn(bot, wy)));
        }
        if (p.normalize)  // normalize (image.cpp:32-38)
            reinterpret_cast<float*>(p.out + img * p.out_stride)[s] =
                __double2float_rn(__dsub_rn(__ddiv_rn(static_cast<double>(v), 127.5), 1.0));
        else
            p.out[img * p.out_stride + s] = v;
    }
}

static unsigned grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    if (g > 148 * 64) g = 148 * 64;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

cudaError_t launch_attack_pixels(const AttackParams& p, cudaStream_t st) {
    if (p.op == QRM_ATTACK_CONTRAST) {
        luma_mean_kernel<<<grid_for(p.count, 128), 128, 0, st>>>(p);
        if (cudaError_t e = cudaGetLastError()) return e;
    }
    attack_pixel_kernel<<<grid_for(static_cast<int64_t>(p.w) * p.h * 3 * p.count, 256), 256, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_attack_jpeg(const AttackParams& p, cudaStream_t st) {
    const int64_t work = static_cast<int64_t>((p.w + 7) / 8) * ((p.h + 7) / 8) * 3 * p.count;
    jpeg_block_kernel<<<static_cast<unsigned>((work + 127) / 128), 128, 0, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_attack_resample(const AttackParams& p, cudaStream_t st) {
    attack_resample_kernel<<<grid_for(static_cast<int64_t>(p.ow) * p.oh * 3 * p.count, 256), 256, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace qrm
