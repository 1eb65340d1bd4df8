/*
 * hidden_oracle.c — fp32 CPU oracle for the learned ("HiDDeN / Stable
 * Signature") tile extractor (TEST INFRASTRUCTURE ONLY).
 *
 * PARITY UNPINNED BY THE REFERENCE: /root/reference has no conv extractor;
 * it deliberately replaces the CNN with a spread-spectrum correlation
 * (stego.cpp:53-67; WatermarkCodec, stego.hpp:32-40, is the plug-in
 * point for a learned extractor). The architecture below is the decoder of
 * HiDDeN (the Stable Signature extractor) as SURVEY.md 8(d)
 * specifies it, and is this repository's contract:
 *
 *   x0 = float(v/127.5 - 1) on the l x l x 3 tile (image.cpp:36), HWC
 *   layers j = 0..8: y = conv3x3(x, W_j) (pad 1, stride 1, no bias)
 *                    y = (y - mean_j) / sqrt(var_j + 1e-5) * gamma_j + beta_j   (BN, eval)
 *                    x = relu(y)
 *     cin_j = 3 (j = 0) else 64; cout_j = 64 (j < 8), n_bits (j = 8)
 *   pooled_c = mean over the l*l pixels of x_c          (AdaptiveAvgPool2d(1))
 *   logits = Wl pooled + bl                              (Linear n_bits -> n_bits)
 *   bit_i  = logits_i > 0
 *
 * Random-init parameters are pure functions of (seed, layer, index) through
 * the reference's counter RNG (rng.hpp:25-39), so the GPU and this oracle
 * build identical fp32 tensors independently:
 *   W_j[co][tap][ci] = (2u - 1) * sqrt(6 / (9 cin)),  u = rng_unit(seed, 0x4c00 + j, (co*9 + tap)*cin + ci)
 *   gamma = 0.75 + 0.5 u(0x4d00+j, c); beta = 0.1 (2u - 1) (ctr 1000 + c);
 *   mean = 0.05 (2u - 1) (ctr 2000 + c); var = 0.75 + 0.5 u (ctr 3000 + c)
 *   Wl[o][i] = (2u - 1) * sqrt(6 / n_bits), u = rng_unit(seed, 0x4e00, o*n_bits + i); bl_o = 0.1 (2u - 1) (ctr 1e6 + o)
 * Accumulation is in double (the oracle is the fp32 model evaluated exactly
 * enough to be the reference for the bf16 tensor-core path).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

uint64_t orc_rng_word(uint64_t seed, uint64_t stream, uint64_t ctr);
double orc_rng_unit(uint64_t seed, uint64_t stream, uint64_t ctr);

enum { HID_LAYERS = 9, HID_C = 64 };

static int cin_of(int j) { return j == 0 ? 3 : HID_C; }
static int cout_of(int j, int nbits) { return j == HID_LAYERS - 1 ? nbits : HID_C; }

/* Parameter generators (exported: tests compare them with the GPU's and torch). */
ORC_API float orc_hidden_weight(uint64_t seed, int j, int co, int tap, int ci) {
    const int cin = cin_of(j);
    const double u = orc_rng_unit(seed, 0x4c00 + (uint64_t)j, (uint64_t)((co * 9 + tap) * cin + ci));
    return (float)((2.0 * u - 1.0) * sqrt(6.0 / (9.0 * cin)));
}

ORC_API void orc_hidden_bn(uint64_t seed, int j, int c, float* gamma, float* beta, float* mean, float* var) {
    const uint64_t st = 0x4d00 + (uint64_t)j;
    *gamma = (float)(0.75 + 0.5 * orc_rng_unit(seed, st, (uint64_t)c));
    *beta = (float)(0.1 * (2.0 * orc_rng_unit(seed, st, 1000 + (uint64_t)c) - 1.0));
    *mean = (float)(0.05 * (2.0 * orc_rng_unit(seed, st, 2000 + (uint64_t)c) - 1.0));
    *var = (float)(0.75 + 0.5 * orc_rng_unit(seed, st, 3000 + (uint64_t)c));
}

ORC_API float orc_hidden_linear_w(uint64_t seed, int nbits, int o, int i) {
    const double u = orc_rng_unit(seed, 0x4e00, (uint64_t)(o * nbits + i));
    return (float)((2.0 * u - 1.0) * sqrt(6.0 / nbits));
}

ORC_API float orc_hidden_linear_b(uint64_t seed, int o) {
    return (float)(0.1 * (2.0 * orc_rng_unit(seed, 0x4e00, 1000000 + (uint64_t)o) - 1.0));
}

static void forward_impl(uint64_t seed, int nbits, int l, const uint8_t* tile, double* logits, double* pooled_out,
                         int stop_after, float* act_out);

/* One tile (u8 l x l x 3, HWC) -> logits[nbits] and (optional) pooled[nbits]. */
ORC_API void orc_hidden_forward(uint64_t seed, int nbits, int l, const uint8_t* tile, double* logits, double* pooled_out) {
    forward_impl(seed, nbits, l, tile, logits, pooled_out, -1, NULL);
}

/* Activations (HWC, l*l*cout floats) after layer `stop_after` (diagnostics). */
ORC_API void orc_hidden_activation(uint64_t seed, int nbits, int l, const uint8_t* tile, int stop_after, float* act_out) {
    forward_impl(seed, nbits, l, tile, NULL, NULL, stop_after, act_out);
}

static void forward_impl(uint64_t seed, int nbits, int l, const uint8_t* tile, double* logits, double* pooled_out,
                         int stop_after, float* act_out) {
    const int P = l * l;
    float* x = malloc(sizeof(float) * (size_t)P * HID_C);
    float* y = malloc(sizeof(float) * (size_t)P * HID_C);
    float* w = malloc(sizeof(float) * (size_t)HID_C * 9 * HID_C);
    for (int i = 0; i < P * 3; ++i) x[i] = (float)(tile[i] / 127.5 - 1.0);
    for (int j = 0; j < HID_LAYERS; ++j) {
        const int cin = cin_of(j), cout = cout_of(j, nbits);
        for (int co = 0; co < cout; ++co)
            for (int t = 0; t < 9; ++t)
                for (int ci = 0; ci < cin; ++ci) w[(co * 9 + t) * cin + ci] = orc_hidden_weight(seed, j, co, t, ci);
        for (int py = 0; py < l; ++py)
            for (int px = 0; px < l; ++px)
                for (int co = 0; co < cout; ++co) {
                    double acc = 0.0;
                    for (int ky = 0; ky < 3; ++ky) {
                        const int sy = py + ky - 1;
                        if (sy < 0 || sy >= l) continue;
                        for (int kx = 0; kx < 3; ++kx) {
                            const int sx = px + kx - 1;
                            if (sx < 0 || sx >= l) continue;
                            const float* xi = x + ((size_t)sy * l + sx) * cin;
                            const float* wi = w + (co * 9 + ky * 3 + kx) * cin;
                            for (int ci = 0; ci < cin; ++ci) acc += (double)xi[ci] * wi[ci];
                        }
                    }
                    float g, b, m, v;
                    orc_hidden_bn(seed, j, co, &g, &b, &m, &v);
                    double z = (acc - m) / sqrt((double)v + 1e-5) * g + b;
                    y[((size_t)py * l + px) * cout + co] = (float)(z > 0.0 ? z : 0.0);
                }
        float* tmp = x;
        x = y;
        y = tmp;
        if (j == stop_after) {
            memcpy(act_out, x, sizeof(float) * (size_t)P * cout);
            free(x);
            free(y);
            free(w);
            return;
        }
    }
    double pooled[256];
    for (int c = 0; c < nbits; ++c) {
        double s = 0.0;
        for (int p = 0; p < P; ++p) s += x[(size_t)p * nbits + c];
        pooled[c] = s / P;
        if (pooled_out) pooled_out[c] = pooled[c];
    }
    for (int o = 0; o < nbits; ++o) {
        double s = orc_hidden_linear_b(seed, o);
        for (int i = 0; i < nbits; ++i) s += (double)orc_hidden_linear_w(seed, nbits, o, i) * pooled[i];
        logits[o] = s;
    }
    free(x);
    free(y);
    free(w);
}
