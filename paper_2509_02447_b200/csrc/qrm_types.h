// Internal host/device types of the B200 detection path (not part of the ABI).
#pragma once

#include <cstdint>

#include "qrmark_gpu.h"

namespace qrm {

constexpr int kWorkingSize = 256;  // transforms.hpp:11
constexpr int kMaxNBits = 64;      // codeword bits handled by the fused detect path
constexpr uint8_t kRecPending = 0xFF;

// GF(2^m) tables + GRS parity structure of an (n, k) evaluation code with
// X_i = alpha^i (rs.cpp:52-63). Lives in device global memory; kernels stage
// it into shared memory.
struct alignas(16) RsTables {
    int32_t m, n, k, t, r, q1;  // r = n - k, q1 = 2^m - 1
    int32_t packed_ok;          // n*m <= 64
    int32_t nmask;              // r*m syndrome-bit masks (packed words)
    uint8_t exp2[512];          // alpha^i for i in [0, 2*q1), no modulo needed
    uint8_t log[256];           // log_alpha(v), v in [1, q1]
    uint8_t logv[256];          // log of the GRS column multipliers v_i = 1/prod_{l!=i}(X_i - X_l)
    uint64_t synd_mask[64];     // packed-word syndrome bits: S_j bit e = parity(word & synd_mask[j*m+e])
};

// Device codebook (row f1): open-addressing memo word -> (codeword, errors)
// for the general-t packed decoder. keys[i] == kCodebookEmpty: free slot.
constexpr uint64_t kCodebookEmpty = ~0ull;     // never a packed word (n*m < 64 required)
constexpr uint64_t kCodebookBusy = ~0ull - 1;  // claimed, value being written
constexpr int kCodebookProbes = 8;
struct CodebookTable {
    uint64_t* keys;  // nullptr: no table
    uint64_t* vals;
    int8_t* nerr;
    uint64_t mask;   // slots - 1 (power of two)
};

// One pending detection (tie resolution and/or general-t RS correction).
struct PendingEntry {
    int64_t image;
    uint64_t tie_mask;  // bit i set: correlation of pattern i was exactly zero
};

// Window addressing of the decode kernels. direct != 0: the tile window is
// read straight from the raw image (uniform batch, crop offset + per-image
// tile origin from the counter RNG). direct == 0: windows were staged
// contiguously (3 l^2 bytes each) by the gather kernel.
struct WindowSource {
    const uint8_t* base;
    int64_t image_stride;
    int32_t pitch;      // bytes per image row (direct) / 3l (staged)
    int32_t x_off;      // centre-crop offset, pixels (direct only)
    int32_t y_off;
    int32_t direct;
    int32_t strategy;
    int32_t l;
    uint64_t tile_seed;
    uint64_t first_draw;
};

struct GatherDesc {
    const uint8_t* img;  // image base (device or mapped host)
    int32_t w, h;        // source size
    int32_t upscale;
    int32_t sw, sh;      // virtual resized size
    int32_t x_off, y_off;
    int32_t tx, ty;      // tile origin in the 256 x 256 working image
};

struct DetectParams {
    WindowSource src;
    int64_t count;
    int32_t K;          // 3 l^2 correlation length
    int32_t K_pad;      // rounded up to the 128-byte pipeline chunk
    int32_t nbits;      // n*m
    int32_t kbits;      // k*m
    int32_t tau_msg, tau_raw;
    int32_t fuse_t1;    // epilogue may run the t=1 RS decoder itself
    int32_t tile_m;     // images per decode tile (<= 128 TMEM lanes); set by the launcher
    int32_t wait_inputs;  // 1: the windows may be written by the preceding kernel on the stream, so the
                          // producers griddep_wait() before their first load (no overlap with that kernel)
    int32_t ksplit;       // launcher: forced split-K cluster size (0: automatic)
    uint64_t key_cw, key_msg;
    const int8_t* patterns;   // [64][K_pad] s8, rows >= nbits zero
    const int8_t* patterns_sw;  // the same, per 128-byte K chunk: [K_pad/128][64 x 128 B SW128 smem image]
    const int32_t* colsum;    // [64] sum_px P_i[px]
    const RsTables* rs;
    qrm_record* out;
    double* soft;             // nullable, [count][nbits]
    uint64_t* raw_out;        // nullable, [count]
    int32_t* pending_count;
    PendingEntry* pending;    // capacity = count
};


// apply_attack (transforms.cpp:289-362) over a batch of same-size byte images.
struct AttackParams {
    const uint8_t* in;
    int64_t in_stride;
    int32_t w, h;
    uint8_t* out;  // u8 (or float for normalize)
    int64_t out_stride;
    int32_t ow, oh;
    int64_t count;
    int32_t op;
    double param;
    // geometry: output (x, y) = pixel (x + x_off, y + y_off) of the image resized to sw x sh
    int32_t resize, sw, sh, x_off, y_off, normalize;
    double* pivot;  // [count] mean luma (contrast)
    double kC, kE, kD, kSum;  // gaussian3x3 weights (host exp)
    const double* jpeg_cos;   // [8][8] host cos((2i+1) u pi / 16)
    const double* jpeg_quant; // [64]
    double dct_c0;            // sqrt(0.125)
};


// Tile extraction + normalisation into bf16 NHWC (north-star item 1).
struct TileBf16Params {
    WindowSource src;  // tile origins (direct) or contiguous staged windows
    int64_t count;
    int32_t K;         // 3 l^2
    int32_t channels;  // 3 or 4 output channels (4: zero-padded, 8-byte pixels)
    uint16_t* out;     // [count][l][l][channels] bf16
};

}  // namespace qrm
