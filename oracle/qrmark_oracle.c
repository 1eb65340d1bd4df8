/*
 * qrmark_oracle.c — CPU restatement of the QRMark tile-detection path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity oracle: it is compiled by
 * oracle/Makefile into oracle/_build/liboracle.so and may be loaded only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu-baseline leg. The
 * product (paper_2509_02447_b200/) never links or calls it.
 *
 * Every function restates the reference algorithm it cites
 * (/root/reference/proj/..., file:line). Parity of this restatement is pinned
 * against the compiled reference (oracle/_ref/libqrmark_ref.so) and against the
 * golden fixtures in tests/golden/ (generated from oracle/_ref by
 * tests/golden/make_golden.py).
 *
 * Conventions: bit vectors are one byte per bit (BitVec, rs.hpp:16); packed
 * words are MSB-first (bit 0 of the vector = most significant bit).
 * Return codes: 0 ok, 1 InvalidInput, 2 DivisionByZero, 3 InfeasibleConfig.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_DIVZERO = 2, ORC_INFEASIBLE = 3 };

/* ------------------------------------------------------------------ rng ---
 * include/qrmark/rng.hpp:13-39 */
static const uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

ORC_API uint64_t orc_mix64(uint64_t x) { /* rng.hpp:15-22 */
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

ORC_API uint64_t orc_rng_word(uint64_t seed, uint64_t stream, uint64_t ctr) { /* rng.hpp:25-28 */
    uint64_t key = orc_mix64(seed + kGolden * (stream + 1));
    return orc_mix64(key ^ (ctr * 0xd6e8feb86659fd93ULL) ^ (ctr >> 32));
}

ORC_API uint64_t orc_rng_below(uint64_t seed, uint64_t stream, uint64_t ctr, uint64_t bound) { /* rng.hpp:31-34 */
    unsigned __int128 wide = (unsigned __int128)orc_rng_word(seed, stream, ctr) * bound;
    return (uint64_t)(wide >> 64);
}

ORC_API double orc_rng_unit(uint64_t seed, uint64_t stream, uint64_t ctr) { /* rng.hpp:37-39 */
    return (double)(orc_rng_word(seed, stream, ctr) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------- gf ---
 * src/gf.cpp:7-55: log/antilog tables over alpha = 2. GF(16) poly 0x13,
 * GF(256) poly 0x11D. */
typedef struct {
    int m, q;
    uint16_t exp[255];
    uint16_t log[256];
} field_t;

static field_t g_f16, g_f256;
static int g_fields_ready = 0;

static void field_build(field_t* f, int m, uint32_t poly) { /* gf.cpp:7-18 */
    f->m = m;
    f->q = 1 << m;
    memset(f->log, 0, sizeof f->log);
    uint32_t v = 1;
    for (int i = 0; i < f->q - 1; ++i) {
        f->exp[i] = (uint16_t)v;
        f->log[v] = (uint16_t)i;
        v <<= 1;
        if (v & (1u << m)) v ^= poly;
    }
}

static const field_t* field_of(int m) {
    if (!g_fields_ready) {
        field_build(&g_f16, 4, 0x13);
        field_build(&g_f256, 8, 0x11d);
        g_fields_ready = 1;
    }
    return m == 4 ? &g_f16 : (m == 8 ? &g_f256 : NULL);
}

static uint16_t gmul(const field_t* f, uint16_t a, uint16_t b) { /* gf.cpp:30-37 */
    if (a == 0 || b == 0) return 0;
    int s = f->log[a] + f->log[b];
    if (s >= f->q - 1) s -= f->q - 1;
    return f->exp[s];
}

static uint16_t ginv(const field_t* f, uint16_t a) { /* gf.cpp:39-43 (a != 0) */
    return f->exp[(f->q - 1 - f->log[a]) % (f->q - 1)];
}

ORC_API int orc_gf_mul(int m, int a, int b) { return gmul(field_of(m), (uint16_t)a, (uint16_t)b); }
ORC_API int orc_gf_inv(int m, int a) { return a ? ginv(field_of(m), (uint16_t)a) : -1; }

/* ------------------------------------------------------------------- rs ---
 * src/rs.cpp. Code: X_i = alpha^i (rs.cpp:52-63), t = (n-k)/2. */
#define ORC_MAXN 255

static int code_check(int m, int n, int k) { /* CodeParams::make, rs.cpp:52-56 */
    const field_t* f = field_of(m);
    if (!f) return ORC_INVALID;
    if (n > f->q - 1) return ORC_INVALID;
    if (k <= 0 || k >= n) return ORC_INVALID;
    return ORC_OK;
}

static void bits_to_syms(const uint8_t* bits, int nsym, int m, uint16_t* out) { /* rs.cpp:8-17 */
    for (int s = 0; s < nsym; ++s) {
        uint16_t v = 0;
        for (int b = 0; b < m; ++b) v = (uint16_t)((v << 1) | (bits[s * m + b] & 1));
        out[s] = v;
    }
}

static void syms_to_bits(const uint16_t* syms, int nsym, int m, uint8_t* out) { /* rs.cpp:19-25 */
    for (int s = 0; s < nsym; ++s)
        for (int b = 0; b < m; ++b) out[s * m + b] = (syms[s] >> (m - 1 - b)) & 1;
}

/* Polynomial helpers, coefficients lowest degree first; returns degree (-1 = 0). */
static int poly_deg(const uint16_t* c, int len) {
    int d = len - 1;
    while (d >= 0 && c[d] == 0) --d;
    return d;
}

static uint16_t poly_eval(const field_t* f, const uint16_t* c, int deg, uint16_t x) { /* gf.cpp:70-77 */
    uint16_t acc = 0;
    for (int i = deg; i >= 0; --i) acc = gmul(f, acc, x) ^ c[i];
    return acc;
}

/* rs_encode (rs.cpp:78-91): P = lagrange_interpolate over (X_i, msg_i), i < k
 * (gf.cpp:126-146), then C_i = P(X_i). */
ORC_API int orc_rs_encode(int m, int n, int k, const uint8_t* msg_bits, uint8_t* cw_bits) {
    int rc = code_check(m, n, k);
    if (rc) return rc;
    const field_t* f = field_of(m);
    uint16_t X[ORC_MAXN], y[ORC_MAXN], P[ORC_MAXN], basis[ORC_MAXN + 1], tmp[ORC_MAXN + 1], cw[ORC_MAXN];
    for (int i = 0; i < n; ++i) X[i] = f->exp[i % (f->q - 1)];
    bits_to_syms(msg_bits, k, m, y);
    memset(P, 0, sizeof P);
    for (int i = 0; i < k; ++i) {
        memset(basis, 0, sizeof basis);
        basis[0] = 1;
        int bl = 1;
        uint16_t denom = 1;
        for (int j = 0; j < k; ++j) {
            if (j == i) continue;
            /* basis *= (x + X_j) */
            memset(tmp, 0, sizeof tmp);
            for (int a = 0; a < bl; ++a) {
                tmp[a] ^= gmul(f, basis[a], X[j]);
                tmp[a + 1] ^= basis[a];
            }
            ++bl;
            memcpy(basis, tmp, sizeof(uint16_t) * bl);
            denom = gmul(f, denom, X[i] ^ X[j]);
        }
        uint16_t s = gmul(f, y[i], ginv(f, denom));
        for (int a = 0; a < bl; ++a) P[a] ^= gmul(f, basis[a], s);
    }
    int pd = poly_deg(P, k);
    for (int i = 0; i < n; ++i) cw[i] = poly_eval(f, P, pd, X[i]);
    syms_to_bits(cw, n, m, cw_bits);
    return ORC_OK;
}

/* solve_linear (rs.cpp:97-128): Gauss-Jordan with first-nonzero pivoting,
 * free variables 0. Returns 1 when consistent. a is rows x cols row-major. */
static int solve_linear(const field_t* f, uint16_t* a, uint16_t* b, int rows, int cols, uint16_t* x) {
    int pivot_col[ORC_MAXN];
    int row = 0;
    for (int col = 0; col < cols && row < rows; ++col) {
        int piv = row;
        while (piv < rows && a[piv * cols + col] == 0) ++piv;
        if (piv == rows) continue;
        if (piv != row) {
            for (int j = 0; j < cols; ++j) {
                uint16_t t = a[piv * cols + j];
                a[piv * cols + j] = a[row * cols + j];
                a[row * cols + j] = t;
            }
            uint16_t t = b[piv];
            b[piv] = b[row];
            b[row] = t;
        }
        uint16_t inv = ginv(f, a[row * cols + col]);
        for (int j = col; j < cols; ++j) a[row * cols + j] = gmul(f, a[row * cols + j], inv);
        b[row] = gmul(f, b[row], inv);
        for (int r = 0; r < rows; ++r) {
            if (r == row || a[r * cols + col] == 0) continue;
            uint16_t fac = a[r * cols + col];
            for (int j = col; j < cols; ++j) a[r * cols + j] ^= gmul(f, fac, a[row * cols + j]);
            b[r] ^= gmul(f, fac, b[row]);
        }
        pivot_col[row] = col;
        ++row;
    }
    for (int r = row; r < rows; ++r)
        if (b[r] != 0) return 0;
    for (int j = 0; j < cols; ++j) x[j] = 0;
    for (int r = 0; r < row; ++r) x[pivot_col[r]] = b[r];
    return 1;
}

/* bw_attempt (rs.cpp:131-184). Returns errors (>=0) on success, -1 on reject. */
static int bw_attempt(const field_t* f, const uint16_t* R, const uint16_t* X, int n, int k, int t, int tp,
                      uint16_t* cw_out) {
    int nq = tp, nn = tp + k, cols = nq + nn;
    uint16_t* a = calloc((size_t)n * cols, sizeof(uint16_t));
    uint16_t b[ORC_MAXN], sol[2 * ORC_MAXN];
    for (int i = 0; i < n; ++i) {
        uint16_t xp = 1;
        for (int j = 0; j < nq; ++j) {
            a[i * cols + j] = gmul(f, R[i], xp);
            xp = gmul(f, xp, X[i]);
        }
        b[i] = gmul(f, R[i], xp);
        xp = 1;
        for (int j = 0; j < nn; ++j) {
            a[i * cols + nq + j] = xp;
            xp = gmul(f, xp, X[i]);
        }
    }
    int ok = solve_linear(f, a, b, n, cols, sol);
    free(a);
    if (!ok) return -1;
    uint16_t Q[ORC_MAXN + 1], N[2 * ORC_MAXN], quot[2 * ORC_MAXN], rem[2 * ORC_MAXN];
    for (int j = 0; j < nq; ++j) Q[j] = sol[j];
    Q[nq] = 1;
    int qd = nq; /* leading coefficient pinned to 1 */
    for (int j = 0; j < nn; ++j) N[j] = sol[nq + j];
    int nd = poly_deg(N, nn);
    if (nd >= qd + k) return -1; /* rs.cpp:166 */
    /* Poly::divmod (gf.cpp:105-124) */
    int pd;
    if (nd < qd) {
        if (nd >= 0) return -1; /* remainder = N != 0 */
        pd = -1;
        memset(quot, 0, sizeof quot);
    } else {
        memcpy(rem, N, sizeof(uint16_t) * (nd + 1));
        memset(quot, 0, sizeof(uint16_t) * (nd - qd + 1));
        uint16_t lead_inv = ginv(f, Q[qd]);
        for (int d = nd; d >= qd; --d) {
            uint16_t c = rem[d];
            if (c == 0) continue;
            uint16_t q = gmul(f, c, lead_inv);
            quot[d - qd] = q;
            for (int i = 0; i <= qd; ++i) rem[d - qd + i] ^= gmul(f, q, Q[i]);
        }
        if (poly_deg(rem, nd + 1) >= 0) return -1; /* rs.cpp:168 */
        pd = poly_deg(quot, nd - qd + 1);
    }
    if (pd >= k) return -1; /* rs.cpp:169 */
    int errors = 0;
    for (int i = 0; i < n; ++i) {
        cw_out[i] = pd >= 0 ? poly_eval(f, quot, pd, X[i]) : 0;
        if (cw_out[i] != R[i]) ++errors;
    }
    if (errors > t) return -1; /* rs.cpp:177 */
    return errors;
}

/* bw_decode (rs.cpp:188-196): ladder t' = t .. 0. Returns 1 decoded, 0 failure,
 * negative error code on a contract violation. */
ORC_API int orc_bw_decode(int m, int n, int k, const uint8_t* bits, uint8_t* msg_out, uint8_t* cw_out,
                          int* errors) {
    int rc = code_check(m, n, k);
    if (rc) return -rc;
    const field_t* f = field_of(m);
    int t = (n - k) / 2;
    uint16_t X[ORC_MAXN], R[ORC_MAXN], C[ORC_MAXN];
    for (int i = 0; i < n; ++i) X[i] = f->exp[i % (f->q - 1)];
    bits_to_syms(bits, n, m, R);
    for (int tp = t; tp >= 0; --tp) {
        int e = bw_attempt(f, R, X, n, k, t, tp, C);
        if (e >= 0) {
            uint8_t cwb[ORC_MAXN * 8];
            syms_to_bits(C, n, m, cwb);
            if (cw_out) memcpy(cw_out, cwb, (size_t)n * m);
            if (msg_out) memcpy(msg_out, cwb, (size_t)k * m);
            *errors = e;
            return 1;
        }
    }
    *errors = 0;
    return 0;
}

/* Packed-word convenience (n*m <= 64): nerr = errors or -1 on failure. */
ORC_API void orc_bw_decode_packed(int m, int n, int k, const uint64_t* words, int64_t count, uint64_t* cw_out,
                                  int8_t* nerr_out) {
    const int nb = n * m;
    uint8_t bits[64], cw[64];
    for (int64_t i = 0; i < count; ++i) {
        for (int b = 0; b < nb; ++b) bits[b] = (words[i] >> (nb - 1 - b)) & 1;
        int e = 0;
        int ok = orc_bw_decode(m, n, k, bits, NULL, cw, &e);
        if (ok == 1) {
            uint64_t w = 0;
            for (int b = 0; b < nb; ++b) w = (w << 1) | cw[b];
            cw_out[i] = w;
            nerr_out[i] = (int8_t)e;
        } else {
            cw_out[i] = 0;
            nerr_out[i] = -1;
        }
    }
}

/* ------------------------------------------------------------ verify ------
 * verify_threshold (detect.cpp:31-66). */
ORC_API int orc_verify_threshold(int n_bits, double fpr) {
    if (n_bits <= 0 || fpr <= 0.0 || fpr >= 1.0) return -1;
    if (n_bits <= 64) {
        long double bound = (long double)fpr * powl(2.0L, (long double)n_bits);
        unsigned __int128 binom = 1, tail = 0;
        int tau = n_bits + 1;
        for (int j = n_bits; j >= 0; --j) {
            tail += binom;
            if ((long double)tail <= bound) tau = j;
            else break;
            if (j > 0) binom = binom * (unsigned)j / (unsigned)(n_bits - j + 1);
        }
        return tau;
    }
    long double log2v = logl(2.0L), tail = 0.0L;
    int tau = n_bits + 1;
    for (int j = n_bits; j >= 0; --j) {
        long double lt = lgammal(n_bits + 1.0L) - lgammal(j + 1.0L) - lgammal(n_bits - j + 1.0L) - n_bits * log2v;
        tail += expl(lt);
        if (tail <= (long double)fpr) tau = j;
        else break;
    }
    return tau;
}

/* ------------------------------------------------------------ imaging -----
 * image.cpp / transforms.cpp. Images are interleaved HWC u8 (image.hpp:28-30). */
static uint8_t quantize(double v) { /* image.cpp:42-45 */
    double q = floor(v + 0.5);
    if (q < 0.0) q = 0.0;
    if (q > 255.0) q = 255.0;
    return (uint8_t)q;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* resize_bilinear (image.cpp:57-85). */
ORC_API int orc_resize_bilinear(const uint8_t* img, int w, int h, int ow, int oh, uint8_t* out) {
    if (ow <= 0 || oh <= 0) return ORC_INVALID;
    if (ow == w && oh == h) {
        memcpy(out, img, (size_t)w * h * 3);
        return ORC_OK;
    }
    const double sx = (double)w / ow, sy = (double)h / oh;
    for (int oy = 0; oy < oh; ++oy) {
        double fy = (oy + 0.5) * sy - 0.5, y0d = floor(fy), wy = fy - y0d;
        int y0 = clampi((int)y0d, 0, h - 1), y1 = clampi((int)y0d + 1, 0, h - 1);
        for (int ox = 0; ox < ow; ++ox) {
            double fx = (ox + 0.5) * sx - 0.5, x0d = floor(fx), wx = fx - x0d;
            int x0 = clampi((int)x0d, 0, w - 1), x1 = clampi((int)x0d + 1, 0, w - 1);
            for (int c = 0; c < 3; ++c) {
                double top = img[((size_t)y0 * w + x0) * 3 + c] * (1.0 - wx) + img[((size_t)y0 * w + x1) * 3 + c] * wx;
                double bot = img[((size_t)y1 * w + x0) * 3 + c] * (1.0 - wx) + img[((size_t)y1 * w + x1) * 3 + c] * wx;
                out[((size_t)oy * ow + ox) * 3 + c] = quantize(top * (1.0 - wy) + bot * wy);
            }
        }
    }
    return ORC_OK;
}

/* preprocess_geometry (transforms.cpp:24-38), working size 256 (transforms.hpp:11). */
ORC_API void orc_preprocess_geometry(int w, int h, int* upscale, int* sw, int* sh, int* xoff, int* yoff) {
    const int W = 256;
    int mn = w < h ? w : h;
    if (mn < W) {
        double s = (double)W / mn;
        long a = lround(w * s), b = lround(h * s);
        *upscale = 1;
        *sw = (int)a > W ? (int)a : W;
        *sh = (int)b > W ? (int)b : W;
    } else {
        *upscale = 0;
        *sw = w;
        *sh = h;
    }
    *xoff = (*sw - W) / 2;
    *yoff = (*sh - W) / 2;
}

/* normalize sample (image.cpp:36). */
static float norm_sample(uint8_t v) { return (float)(v / 127.5 - 1.0); }

/* The staged preprocess (transforms.cpp:42-47) restated as: optional
 * upscale, centre crop, normalise. out: 256*256*3 floats. */
ORC_API int orc_preprocess(const uint8_t* img, int w, int h, float* out) {
    if (w <= 0 || h <= 0) return ORC_INVALID;
    int up, sw, sh, xo, yo;
    orc_preprocess_geometry(w, h, &up, &sw, &sh, &xo, &yo);
    const uint8_t* src = img;
    uint8_t* staged = NULL;
    if (up) {
        staged = malloc((size_t)sw * sh * 3);
        orc_resize_bilinear(img, w, h, sw, sh, staged);
        src = staged;
    }
    for (int y = 0; y < 256; ++y)
        for (int x = 0; x < 256; ++x)
            for (int c = 0; c < 3; ++c)
                out[((size_t)y * 256 + x) * 3 + c] = norm_sample(src[((size_t)(y + yo) * sw + (x + xo)) * 3 + c]);
    free(staged);
    return ORC_OK;
}

/* ------------------------------------------------------------ tiling ------
 * select_tile (tiling.cpp:23-47). strategy: 0 random, 1 random_grid, 2 fixed. */
ORC_API int orc_select_tile(int w, int h, int l, int strategy, uint64_t seed, uint64_t draw, int* x, int* y) {
    int mn = w < h ? w : h;
    if (l <= 0 || l > mn) return ORC_INVALID;
    if (strategy == 2) {
        *x = 0;
        *y = 0;
    } else if (strategy == 0) {
        uint64_t nx = (uint64_t)(w - l) + 1, ny = (uint64_t)(h - l) + 1;
        *x = (int)orc_rng_below(seed, 2 * draw, 0, nx);
        *y = (int)orc_rng_below(seed, 2 * draw + 1, 0, ny);
    } else if (strategy == 1) {
        uint64_t cols = (uint64_t)(w / l), rows = (uint64_t)(h / l);
        uint64_t cell = orc_rng_below(seed, draw, 0, cols * rows);
        *x = (int)(cell % cols) * l;
        *y = (int)(cell / cols) * l;
    } else {
        return ORC_INVALID;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------- stego ------
 * Patterns P_i[px] = (rng_word(seed, i, px) & 1) ? +1 : -1 (stego.cpp:16-27). */
ORC_API void orc_pattern(uint64_t key_seed, int bit, int l, int8_t* out) {
    size_t S = (size_t)l * l * 3;
    for (size_t px = 0; px < S; ++px) out[px] = (orc_rng_word(key_seed, (uint64_t)bit, px) & 1) ? 1 : -1;
}

/* SpreadSpectrumCodec::extract (stego.cpp:53-67): soft_i = sum_px
 * double(tile[px]) * P_i[px] * (1/(3l^2)), summed sequentially in px order. */
ORC_API void orc_extract(uint64_t key_seed, int n_bits, int l, const float* tile, double* soft) {
    size_t S = (size_t)l * l * 3;
    int8_t* p = malloc(S);
    const double inv_n = 1.0 / (double)S;
    for (int i = 0; i < n_bits; ++i) {
        orc_pattern(key_seed, i, l, p);
        double acc = 0.0;
        for (size_t px = 0; px < S; ++px) acc += (double)tile[px] * p[px];
        soft[i] = acc * inv_n;
    }
    free(p);
}

/* The exact integer correlation S_i = sum_px (2 v_px - 255) * P_i[px] of a u8
 * tile (the quantity the GPU computes; soft_i ~= S_i / (255 * 3l^2)). */
ORC_API void orc_extract_exact(uint64_t key_seed, int n_bits, int l, const uint8_t* tile_u8, int64_t* S_out) {
    size_t S = (size_t)l * l * 3;
    int8_t* p = malloc(S);
    for (int i = 0; i < n_bits; ++i) {
        orc_pattern(key_seed, i, l, p);
        int64_t acc = 0;
        for (size_t px = 0; px < S; ++px) acc += (int64_t)(2 * (int)tile_u8[px] - 255) * p[px];
        S_out[i] = acc;
    }
    free(p);
}

/* synthetic_image (image.cpp:157-189). */
ORC_API void orc_synthetic_image(uint64_t seed, int w, int h, uint8_t* out) {
    const double kTau = 6.283185307179586;
    double amp[3][3], fx[3][3], fy[3][3], ph[3][3];
    uint64_t ctr = 0;
    for (int c = 0; c < 3; ++c)
        for (int i = 0; i < 3; ++i) {
            amp[c][i] = 10.0 + 14.0 * orc_rng_unit(seed, 0x514e, ctr++);
            fx[c][i] = 1.0 + floor(orc_rng_unit(seed, 0x514e, ctr++) * 4.0);
            fy[c][i] = 1.0 + floor(orc_rng_unit(seed, 0x514e, ctr++) * 4.0);
            ph[c][i] = kTau * orc_rng_unit(seed, 0x514e, ctr++);
        }
    int hm1 = h - 1 > 1 ? h - 1 : 1, hh = h > 1 ? h : 1;
    for (int y = 0; y < h; ++y) {
        double gradient = 118.0 + 90.0 * ((h - 1.0 - y) / hm1 - 0.5);
        double ta = 1.0 - 2.0 * y / hh;
        double texture_amp = 34.0 * (ta > 0.0 ? ta : 0.0);
        for (int x = 0; x < w; ++x) {
            uint64_t nc = (uint64_t)y * w + x;
            for (int c = 0; c < 3; ++c) {
                double v = gradient;
                for (int i = 0; i < 3; ++i)
                    v += amp[c][i] * cos(kTau * (fx[c][i] * x / w + fy[c][i] * y / h) + ph[c][i]);
                v += texture_amp * (2.0 * orc_rng_unit(seed, 0x7e30 + c, nc) - 1.0);
                out[((size_t)y * w + x) * 3 + c] = quantize(v);
            }
        }
    }
}

/* default_message (cli.cpp:47-51). */
ORC_API void orc_default_message(uint64_t key_seed, int n_bits, uint8_t* out) {
    for (int i = 0; i < n_bits; ++i) out[i] = orc_rng_word(key_seed, 0x6d73, i) & 1;
}

/* cmd_bench corpus (cli.cpp:404-411): normalize (image.cpp:32-38) ->
 * embed_image_grid (stego.cpp:77-92, residual stego.cpp:29-38) ->
 * denormalize (image.cpp:49-55). img is modified in place. */
ORC_API void orc_embed_grid_u8(uint8_t* img, int w, int h, uint64_t key_seed, double alpha, int l,
                               const uint8_t* cw_bits, int n_bits) {
    size_t S = (size_t)l * l * 3;
    float* delta = calloc(S, sizeof(float));
    int8_t* p = malloc(S);
    for (int i = 0; i < n_bits; ++i) {
        orc_pattern(key_seed, i, l, p);
        float sign = cw_bits[i] ? 1.0f : -1.0f;
        for (size_t px = 0; px < S; ++px) delta[px] += sign * p[px];
    }
    const float a = (float)alpha;
    const size_t total = (size_t)w * h * 3;
    float* norm = malloc(sizeof(float) * total);
    for (size_t i = 0; i < total; ++i) norm[i] = norm_sample(img[i]);
    for (int cy = 0; cy + l <= h; cy += l)
        for (int cx = 0; cx + l <= w; cx += l) {
            size_t px = 0;
            for (int y = 0; y < l; ++y)
                for (int x = 0; x < l; ++x)
                    for (int c = 0; c < 3; ++c, ++px) {
                        size_t idx = ((size_t)(cy + y) * w + (cx + x)) * 3 + c;
                        float v = norm[idx] + a * delta[px];
                        norm[idx] = v < -1.0f ? -1.0f : (v > 1.0f ? 1.0f : v);
                    }
        }
    for (size_t i = 0; i < total; ++i) img[i] = quantize(((double)norm[i] + 1.0) * 127.5);
    free(norm);
    free(p);
    free(delta);
}

/* ------------------------------------------------------------- detect -----
 * DetectionContext::detect_one (detect.cpp:164-198) with the cache disabled
 * (the codebook is transparent). */
typedef struct {
    int m, n, k;
    int tile_size, strategy;
    uint64_t tile_seed, key_seed;
    double alpha;
    const uint8_t* key_message; /* k*m bits */
    double fpr;
} orc_cfg;

typedef struct {
    uint64_t raw;      /* packed MSB-first (n*m <= 64) */
    uint64_t msg;      /* corrected message, packed MSB-first */
    int32_t decoded;   /* 1 decoded, 0 failure */
    int32_t errors;    /* errors_corrected */
    int32_t matches;   /* raw vs key codeword (bit_acc numerator) */
    int32_t verified;
    double bit_acc;
} orc_record;

static uint64_t pack_bits(const uint8_t* b, int n) {
    uint64_t w = 0;
    for (int i = 0; i < n; ++i) w = (w << 1) | (b[i] & 1);
    return w;
}

ORC_API int orc_detect_one(const uint8_t* img, int w, int h, uint64_t draw, const orc_cfg* cfg, orc_record* rec) {
    const int nb = cfg->n * cfg->m, kb = cfg->k * cfg->m;
    if (nb > 64) return ORC_INVALID;
    float* pre = malloc(sizeof(float) * 256 * 256 * 3);
    int rc = orc_preprocess(img, w, h, pre);
    if (rc) {
        free(pre);
        return rc;
    }
    int tx, ty;
    rc = orc_select_tile(256, 256, cfg->tile_size, cfg->strategy, cfg->tile_seed, draw, &tx, &ty);
    if (rc) {
        free(pre);
        return rc;
    }
    const int l = cfg->tile_size;
    float* tile = malloc(sizeof(float) * l * l * 3);
    for (int y = 0; y < l; ++y)
        for (int x = 0; x < l; ++x)
            for (int c = 0; c < 3; ++c)
                tile[((size_t)y * l + x) * 3 + c] = pre[((size_t)(ty + y) * 256 + (tx + x)) * 3 + c];
    double soft[64];
    orc_extract(cfg->key_seed, nb, l, tile, soft);
    uint8_t raw[64], key_cw[64], msg[64];
    for (int i = 0; i < nb; ++i) raw[i] = soft[i] > 0.0 ? 1 : 0; /* harden, stego.cpp:10-14 */
    orc_rs_encode(cfg->m, cfg->n, cfg->k, cfg->key_message, key_cw);
    int e = 0;
    int ok = orc_bw_decode(cfg->m, cfg->n, cfg->k, raw, msg, NULL, &e);
    int matches = 0;
    for (int i = 0; i < nb; ++i) matches += raw[i] == key_cw[i];
    rec->raw = pack_bits(raw, nb);
    rec->matches = matches;
    rec->bit_acc = (double)matches / (double)nb; /* bit_accuracy, rs.cpp:215-221 */
    if (ok == 1) {
        int mm = 0;
        for (int i = 0; i < kb; ++i) mm += msg[i] == cfg->key_message[i];
        rec->decoded = 1;
        rec->msg = pack_bits(msg, kb);
        rec->errors = e;
        rec->verified = mm >= orc_verify_threshold(kb, cfg->fpr);
    } else {
        rec->decoded = 0;
        rec->msg = 0;
        rec->errors = 0;
        rec->verified = matches >= orc_verify_threshold(nb, cfg->fpr);
    }
    free(tile);
    free(pre);
    return ORC_OK;
}

/* -------------------------------------------------------------- sched -----
 * allocate_streams (sched.cpp:50-114). Reference quirk kept visible: the
 * uniform mini-batch is static_cast<int>(floor(m_cap / sum u)), undefined for
 * values >= 2^31 (x86 yields INT_MIN -> InfeasibleConfig); the oracle reports
 * ORC_INFEASIBLE in that regime, mirroring the compiled reference. */
static double stage_time(const double* t, double b0, int k, int s, int m) { /* sched.cpp:27-30 */
    return t[k] * ((double)m / b0) / (double)s;
}

static int mem_ok(int K, const int* s, const int* m, const double* u, double cap) { /* sched.cpp:32-38 */
    double total = 0.0;
    for (int k = 0; k < K; ++k) total += (double)s[k] * (double)m[k] * u[k];
    return total <= cap;
}

static double bottleneck_of(int K, const double* t, double b0, const int* s, const int* m) {
    double worst = 0.0;
    for (int k = 0; k < K; ++k) {
        double v = stage_time(t, b0, k, s[k], m[k]);
        if (v > worst) worst = v;
    }
    return worst;
}

ORC_API int orc_allocate_streams(int K, const double* t, const double* u, double b0, int B, int P, double m_cap,
                                 double eps, int stall_cap, int* s_out, int* m_out, double* bottleneck_out) {
    if (K <= 0 || b0 < 1.0) return ORC_INVALID;
    for (int k = 0; k < K; ++k)
        if (t[k] <= 0.0 || u[k] < 0.0) return ORC_INVALID;
    if (P < K || B < 1) return ORC_INVALID;
    int s[64], m[64];
    double per_unit = 0.0;
    for (int k = 0; k < K; ++k) per_unit += u[k];
    int uniform = B;
    if (per_unit > 0.0) {
        double q = floor(m_cap / per_unit);
        int qi = (q >= 2147483648.0 || q < -2147483648.0) ? (int)0x80000000u : (int)q;
        if (qi < uniform) uniform = qi;
    }
    if (uniform < 1) return ORC_INFEASIBLE;
    for (int k = 0; k < K; ++k) {
        s[k] = 1;
        m[k] = uniform;
    }
    double bn = bottleneck_of(K, t, b0, s, m);
    int stall = 0;
    while (stall < stall_cap) {
        double gain = 0.0;
        int best = -1;
        for (int k = 0; k < K; ++k) {
            s[k] += 1;
            int tot = 0;
            for (int j = 0; j < K; ++j) tot += s[j];
            if (tot <= P && mem_ok(K, s, m, u, m_cap)) {
                double d = bn - bottleneck_of(K, t, b0, s, m);
                if (d > gain) {
                    gain = d;
                    best = k;
                }
            }
            s[k] -= 1;
        }
        if (gain > eps && best >= 0) {
            s[best] += 1;
            bn = bottleneck_of(K, t, b0, s, m);
            stall = 0;
        } else {
            ++stall;
        }
    }
    int total = 0;
    for (int k = 0; k < K; ++k) total += s[k];
    int m_unit = B / total > 1 ? B / total : 1;
    for (int k = 0; k < K; ++k) {
        if (stage_time(t, b0, k, s[k], m[k]) < bn / 2.0) {
            int doubled = 2 * m[k] < m_unit ? 2 * m[k] : m_unit;
            int saved = m[k];
            m[k] = doubled;
            if (!mem_ok(K, s, m, u, m_cap)) m[k] = saved;
        }
    }
    for (int k = 0; k < K; ++k) {
        s_out[k] = s[k];
        m_out[k] = m[k];
    }
    *bottleneck_out = bottleneck_of(K, t, b0, s, m);
    return ORC_OK;
}

/* lpt_schedule (sched.cpp:177-235) with shard_task (sched.cpp:161-173). */
typedef struct {
    int id, units;
    double lat, mem;
} orc_task;

static int pool_less(const orc_task* a, const orc_task* b) { /* (latency asc, id desc) */
    if (a->lat != b->lat) return a->lat < b->lat;
    return a->id > b->id;
}

ORC_API int orc_lpt_schedule(int ntasks, const int* ids, const double* lat, const double* mem, const int* units,
                             int S, double lambda, double m_cap, int b_min, int B, int cap, int* p_stream,
                             int* p_id, int* p_units, double* p_lat, double* p_mem, int* p_mb, int* n_pieces,
                             double* loads, int* m_unit_out) {
    if (S < 1 || b_min < 1) return ORC_INVALID;
    for (int i = 0; i < ntasks; ++i)
        if (lat[i] <= 0.0 || units[i] < 1) return ORC_INVALID;
    int maxpool = ntasks + 1;
    orc_task* pool = malloc(sizeof(orc_task) * (size_t)(maxpool > 0 ? maxpool : 1));
    int np = 0;
    for (int i = 0; i < ntasks; ++i) {
        orc_task t = {ids[i], units[i], lat[i], mem[i]};
        int pos = np; /* insertion sort keeps the pool ascending under pool_less */
        while (pos > 0 && pool_less(&t, &pool[pos - 1])) {
            pool[pos] = pool[pos - 1];
            --pos;
        }
        pool[pos] = t;
        ++np;
    }
    /* placed pieces, kept per stream in placement order */
    int total_units = 0;
    for (int i = 0; i < ntasks; ++i) total_units += units[i];
    int maxp = total_units + ntasks + 1;
    int* ps = malloc(sizeof(int) * maxp);
    orc_task* pt = malloc(sizeof(orc_task) * maxp);
    int placed = 0;
    for (int st = 0; st < S; ++st) loads[st] = 0.0;
    double placed_mem = 0.0;
    int rc = ORC_OK;
    while (np > 0) {
        orc_task task = pool[--np];
        int target = 0;
        for (int p = 1; p < S; ++p)
            if (loads[p] < loads[target]) target = p;
        double min_load = loads[target];
        int balanced = isinf(lambda) || loads[target] + task.lat <= (1.0 + lambda) * min_load;
        int fits = placed_mem + task.mem <= m_cap;
        if (balanced && fits) {
            ps[placed] = target;
            pt[placed++] = task;
            loads[target] += task.lat;
            placed_mem += task.mem;
            continue;
        }
        orc_task head = task, rest;
        int has_rest = 0;
        if (task.units > b_min) {
            double frac = (double)b_min / task.units;
            head.units = b_min;
            head.lat = task.lat * frac;
            head.mem = task.mem * frac;
            rest = task;
            rest.units = task.units - b_min;
            rest.lat = task.lat - head.lat;
            rest.mem = task.mem - head.mem;
            has_rest = 1;
        }
        if (placed_mem + head.mem > m_cap) {
            rc = ORC_INFEASIBLE;
            break;
        }
        ps[placed] = target;
        pt[placed++] = head;
        loads[target] += head.lat;
        placed_mem += head.mem;
        if (has_rest) { /* std::lower_bound: first position not less than rest */
            int pos = 0;
            while (pos < np && pool_less(&pool[pos], &rest)) ++pos;
            memmove(&pool[pos + 1], &pool[pos], sizeof(orc_task) * (size_t)(np - pos));
            pool[pos] = rest;
            ++np;
        }
    }
    if (rc == ORC_OK) {
        int m_unit = placed ? B / placed : b_min;
        if (m_unit < b_min) m_unit = b_min;
        int c = 0;
        for (int st = 0; st < S; ++st)
            for (int i = 0; i < placed; ++i)
                if (ps[i] == st) {
                    if (c < cap) {
                        p_stream[c] = st;
                        p_id[c] = pt[i].id;
                        p_units[c] = pt[i].units;
                        p_lat[c] = pt[i].lat;
                        p_mem[c] = pt[i].mem;
                        p_mb[c] = m_unit;
                    }
                    ++c;
                }
        *n_pieces = c;
        *m_unit_out = m_unit;
    }
    free(pool);
    free(ps);
    free(pt);
    return rc;
}
