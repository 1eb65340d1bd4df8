// Reed-Solomon decoding on the device, bit-exact with the reference's
// Berlekamp-Welch decoder (rs.cpp:131-196).
//
// The reference code is the evaluation code C = {(P(X_0..X_{n-1})) : deg P < k}
// with X_i = alpha^i (rs.cpp:52-63, 78-91) — a generalized RS code whose parity
// checks are S_j = sum_i v_i r_i X_i^j, j < n-k, v_i = 1/prod_{l!=i}(X_i - X_l).
// bw_decode returns the unique codeword within distance t (its ladder plus the
// `errors > t` check, rs.cpp:177/192-195, make it a bounded-distance decoder)
// or nullopt. Both decoders below implement exactly that contract:
//   * rs_t1_packed  — t = 1 codes, one codeword per thread, syndromes as
//     GF(2)-linear parities of the packed word (popc), closed-form locator.
//   * rs_seg_bm     — any t, one codeword per segment of W lanes (32/W codewords
//     per warp): lane-parallel syndromes (ballots of GF(2)-linear parities for
//     packed words, xor butterflies for symbol words), Berlekamp-Massey,
//     lane-parallel Chien search over the n valid locators only, Forney, then a
//     full n-k syndrome recheck.
// A success is reported only for a codeword c with all n-k checks zero and
// d(r, c) <= t, which is the unique BDD output; errors_corrected = d(r, c).
#pragma once

#include "qrm_device.cuh"
#include "qrm_types.h"

namespace qrm {

// Shared-memory copy of the tables a decoder needs.
// Same layout as the global image, so staging is a flat 16-byte-vector copy.
using RsSmem = RsTables;
static_assert(sizeof(RsTables) % 16 == 0, "RsTables must be copyable as uint4");

__device__ __forceinline__ void rs_stage_tables(RsSmem& s, const RsTables* g, int tid, int nthreads) {
    const uint4* src = reinterpret_cast<const uint4*>(g);
    uint4* dst = reinterpret_cast<uint4*>(&s);
    for (int i = tid; i < static_cast<int>(sizeof(RsTables) / 16); i += nthreads) dst[i] = __ldg(src + i);
}

__device__ __forceinline__ uint32_t gf_mul(const RsSmem& T, uint32_t a, uint32_t b) {
    return (a && b) ? T.exp2[T.log[a] + T.log[b]] : 0u;
}

__device__ __forceinline__ uint32_t gf_div(const RsSmem& T, uint32_t a, uint32_t b) {  // b != 0
    return a ? T.exp2[T.log[a] + T.q1 - T.log[b]] : 0u;
}

// Compile-time form of rs_t1_packed for the batched RS kernels: MB syndrome
// bits per symbol (4, or 8 for any m <= 8: masks above m are zero) and R = n-k
// checks, with the R*MB syndrome masks held in registers (mk) and only the
// log/antilog tables read from shared memory. Same result as rs_t1_packed.
template <int MB, int R>
__device__ __forceinline__ int rs_t1_fixed(const RsSmem& T, const uint64_t (&mk)[R * MB], uint64_t word,
                                           uint64_t& cw) {
    uint32_t S[R];
    uint32_t any = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        uint32_t s = 0;
#pragma unroll
        for (int e = 0; e < MB; ++e) {
            // parity of a 64-bit word = parity of its two halves XORed (one POPC)
            const uint64_t x = word & mk[j * MB + e];
            s |= static_cast<uint32_t>(__popc(static_cast<uint32_t>(x) ^ static_cast<uint32_t>(x >> 32)) & 1) << e;
        }
        S[j] = s;
        any |= s;
    }
    cw = word;
    if (!any) return 0;
    if (S[0] == 0 || S[1] == 0) return -1;
    const int q1 = T.q1;
    const int l0 = T.log[S[0]];
    int pos = static_cast<int>(T.log[S[1]]) - l0;
    if (pos < 0) pos += q1;
    if (pos >= T.n) return -1;
    if (R > 2) {
        if (S[R - 1] == 0) return -1;
        int want = l0 + 2 * pos;  // < 3 q1
        if (want >= q1) want -= q1;
        if (want >= q1) want -= q1;
        if (static_cast<int>(T.log[S[R - 1]]) != want) return -1;
    }
    int le = l0 - static_cast<int>(T.logv[pos]);
    if (le < 0) le += q1;
    cw = word ^ (static_cast<uint64_t>(T.exp2[le]) << (T.m * (T.n - 1 - pos)));
    return 1;
}

// t = 1 bounded-distance decode of a packed word (n*m <= 64, n-k in {2,3}).
// Returns errors_corrected (0/1) and the corrected codeword, or -1.
__device__ __forceinline__ int rs_t1_packed(const RsSmem& T, uint64_t word, uint64_t& cw) {
    const int m = T.m, r = T.r, q1 = T.q1;
    uint32_t S[4] = {0, 0, 0, 0};
    uint32_t any = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        if (j < r) {
            uint32_t s = 0;
            if (m == 4) {
#pragma unroll
                for (int e = 0; e < 4; ++e) s |= static_cast<uint32_t>(__popcll(word & T.synd_mask[j * 4 + e]) & 1) << e;
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) s |= static_cast<uint32_t>(__popcll(word & T.synd_mask[j * 8 + e]) & 1) << e;
            }
            S[j] = s;
            any |= s;
        }
    }
    if (!any) {
        cw = word;
        return 0;
    }
    if (S[0] == 0 || S[1] == 0) return -1;  // a single error has S_j = e v_i X_i^j != 0
    const int l0 = T.log[S[0]];
    int pos = static_cast<int>(T.log[S[1]]) - l0;
    if (pos < 0) pos += q1;  // X = S_1/S_0 = alpha^pos
    if (pos >= T.n) return -1;  // not a valid locator
    if (r > 2) {                // the extra check of odd n-k (gf16-15-12 has n-k = 3 > 2t)
        if (S[2] == 0) return -1;
        int want = l0 + 2 * pos;
        want %= q1;
        if (static_cast<int>(T.log[S[2]]) != want) return -1;
    }
    int le = l0 - static_cast<int>(T.logv[pos]);
    if (le < 0) le += q1;
    const uint64_t e = T.exp2[le];
    cw = word ^ (e << (m * (T.n - 1 - pos)));
    return 1;
}

// Record assembly shared by the fused epilogue and the finish kernel
// (detect.cpp:180-195): bit_acc numerator, verified against tau.
__device__ __forceinline__ void make_record(qrm_record& rec, uint64_t raw, int nerr, uint64_t cw, int nbits,
                                            int kbits, uint64_t key_cw, uint64_t key_msg, int tau_msg,
                                            int tau_raw, int ties) {
    const uint64_t nmask = nbits == 64 ? ~0ull : ((1ull << nbits) - 1);
    const uint64_t kmask = kbits == 64 ? ~0ull : ((1ull << kbits) - 1);
    const int matches = nbits - __popcll((raw ^ key_cw) & nmask);
    rec.raw = raw;
    rec.matches = static_cast<uint8_t>(matches);
    rec.ties = static_cast<uint8_t>(ties);
    rec.reserved[0] = rec.reserved[1] = rec.reserved[2] = 0;
    if (nerr >= 0) {
        const uint64_t msg = (cw >> (nbits - kbits)) & kmask;  // systematic prefix (rs.cpp:181)
        rec.msg = msg;
        rec.status = QRM_REC_DECODED;
        rec.errors = static_cast<uint8_t>(nerr);
        rec.verified = (kbits - __popcll((msg ^ key_msg) & kmask)) >= tau_msg;
    } else {
        rec.msg = 0;
        rec.status = QRM_REC_FAILED;
        rec.errors = 0;
        rec.verified = matches >= tau_raw;
    }
}

// 24-byte record as three 8-byte stores (the struct's byte fields would
// otherwise be written one ST.U8 at a time).
__device__ __forceinline__ void store_record(qrm_record* dst, const qrm_record& r) {
    const uint64_t info = static_cast<uint64_t>(r.status) | (static_cast<uint64_t>(r.errors) << 8) |
                          (static_cast<uint64_t>(r.matches) << 16) | (static_cast<uint64_t>(r.verified) << 24) |
                          (static_cast<uint64_t>(r.ties) << 32);
    uint64_t* o = reinterpret_cast<uint64_t*>(dst);
    o[0] = r.raw;
    o[1] = r.msg;
    o[2] = info;
}

// ------------------------------------------------- segmented warps ----
// A codeword occupies a segment of W lanes (W a power of two; W >= n for
// codes of up to 32 symbols, W = 32 with P symbols per lane beyond that), so
// a warp decodes 32/W codewords at once: lane sl = lane % W owns positions
// i = sl + W p. Every cross-lane step (ballots, xor butterflies) is executed
// by the whole warp with no early exits — segments that need less work carry
// neutral values through it.

// This lane's segment's bits of a warp ballot.
template <int W>
__device__ __forceinline__ uint32_t seg_ballot(bool pred, int lane) {
    const uint32_t b = __ballot_sync(0xffffffffu, pred);
    if constexpr (W == 32) return b;
    else return (b >> (lane & ~(W - 1))) & ((1u << W) - 1);
}

// Syndrome bits of packed words (n*m <= 64) as GF(2)-linear parities: lane sl
// computes bits sl, sl + W, ... (masks mk[q] = synd_mask[q W + sl]) and one
// ballot per W bits gives the segment all r*m bits (bit j*m + e = bit e of S_j).
template <int W>
__device__ __forceinline__ uint64_t seg_syndrome_bits(uint64_t w, const uint64_t (&mk)[64 / W], int nm, int lane) {
    uint64_t sb = 0;
#pragma unroll
    for (int q = 0; q < 64 / W; ++q) {
        if (q * W < nm) {  // warp-uniform
            const uint64_t x = w & mk[q];
            const bool bit = __popc(static_cast<uint32_t>(x) ^ static_cast<uint32_t>(x >> 32)) & 1;
            sb |= static_cast<uint64_t>(seg_ballot<W>(bit, lane)) << (q * W);
        }
    }
    return sb;
}

// Syndromes of symbol words: each lane folds its positions (log domain, X_i^j
// stepped incrementally), then one xor butterfly of width W per check:
// S_j = xor_i r_i v_i X_i^j for j < n-k (every lane of the segment gets all S_j).
template <int RMAX, int W, int P>
__device__ __forceinline__ void seg_syndromes(const RsSmem& T, const uint32_t (&sym)[P], int lane,
                                              uint32_t (&S)[RMAX]) {
    const int n = T.n, r = T.r, q1 = T.q1;
    const int sl = lane & (W - 1);
#pragma unroll
    for (int j = 0; j < RMAX; ++j) S[j] = 0;
#pragma unroll(P > 4 ? 1 : P)  // long codes: a rolled position loop keeps the code in the I-cache
    for (int p = 0; p < P; ++p) {
        const int i = sl + W * p;
        const uint32_t v = sym[p];
        if (i < n && v) {
            int lg = static_cast<int>(T.log[v]) + static_cast<int>(T.logv[i]);
            if (lg >= q1) lg -= q1;
            const int step = i % q1;
#pragma unroll
            for (int j = 0; j < RMAX; ++j) {
                if (j < r) S[j] ^= T.exp2[lg];
                lg += step;
                if (lg >= q1) lg -= q1;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) S[j] ^= __shfl_xor_sync(0xffffffffu, S[j], o);
    }
}

// Error locator and values from the syndromes (segment-uniform S[0..r-1]):
// Berlekamp-Massey on S_0..S_{2t-1}, lane-parallel Chien search over the n
// valid locators, Forney. err[p] = error value at position sl + W p. Returns
// the number of nonzero error values (segment-uniform), or -1 when the
// locator is not a product of distinct valid linear factors of degree <= t.
// BM keeps x^shift B pre-shifted (O(t) register moves per step instead of an
// O(t^2) select); the Chien search evaluates Lambda from precomputed logs of
// its coefficients, and Omega and Lambda' are formed only in lanes that hold a
// root.
template <int TMAX, int W, int P>
__device__ __forceinline__ int seg_locate(const RsSmem& T, const uint32_t (&S)[2 * TMAX + 1], int lane,
                                          uint32_t (&err)[P]) {
    constexpr int RMAX = 2 * TMAX + 1;
    constexpr int DMAX = TMAX + 1;  // Lambda has degree <= t on success; one more slot detects deg > t
    const int n = T.n, t = T.t, q1 = T.q1;
    const int sl = lane & (W - 1);
    uint32_t Lam[DMAX + 1], xB[DMAX + 1];
#pragma unroll
    for (int i = 0; i <= DMAX; ++i) Lam[i] = xB[i] = 0;
    Lam[0] = 1;
    xB[1] = 1;  // x * B, B = 1
    int L = 0, xdeg = 1;  // xdeg = deg(x^shift B), exact
    uint32_t bdisc = 1;
    // An update with deg(x^shift B) > DMAX would need coefficients the arrays
    // drop; it implies L > t at the end (deg(x^shift B) <= max L), a failure.
    bool overflow = false;
#pragma unroll
    for (int step = 0; step < 2 * TMAX; ++step) {
        if (step < 2 * t) {
            uint32_t d = S[step];
#pragma unroll
            for (int i = 1; i <= DMAX && i <= step; ++i)
                if (i <= L) d ^= gf_mul(T, Lam[i], S[step - i]);
            uint32_t nxB[DMAX + 1];
            if (d == 0) {
                ++xdeg;
                nxB[0] = 0;
#pragma unroll
                for (int i = 1; i <= DMAX; ++i) nxB[i] = xB[i - 1];
            } else {
                const uint32_t coef = gf_div(T, d, bdisc);
                const bool grow = 2 * L <= step;
                overflow |= xdeg > DMAX;
                uint32_t src[DMAX + 1];
                int dl = 0;
#pragma unroll
                for (int i = 0; i <= DMAX; ++i) {
                    src[i] = grow ? Lam[i] : xB[i];
                    if (Lam[i]) dl = i;
                }
                xdeg = grow ? dl + 1 : xdeg + 1;
#pragma unroll
                for (int i = 0; i <= DMAX; ++i) Lam[i] ^= gf_mul(T, coef, xB[i]);
                nxB[0] = 0;
#pragma unroll
                for (int i = 1; i <= DMAX; ++i) nxB[i] = src[i - 1];
                if (grow) {
                    L = step + 1 - L;
                    bdisc = d;
                }
            }
#pragma unroll
            for (int i = 0; i <= DMAX; ++i) xB[i] = nxB[i];
        }
    }
    int deg = 0;
#pragma unroll
    for (int i = 0; i <= DMAX; ++i)
        if (Lam[i]) deg = i;
    bool fail = L > t || deg != L || overflow;

    int lgl[DMAX + 1];  // log Lambda_d, -1 for a zero coefficient
#pragma unroll
    for (int d = 0; d <= DMAX; ++d) lgl[d] = Lam[d] ? static_cast<int>(T.log[Lam[d]]) : -1;

    int roots = 0, changed = 0;
    bool badlane = false;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int i = sl + W * p;
        err[p] = 0;
        bool root = false;
        if (i < n && !fail) {
            const int li = i % q1;            // log X_i
            const int linv = (q1 - li) % q1;  // log X_i^{-1}
            uint32_t val = 0;
            int lx = 0;  // log x^d, d = 0..
#pragma unroll
            for (int dgr = 0; dgr <= TMAX; ++dgr) {
                if (lgl[dgr] >= 0) val ^= T.exp2[lgl[dgr] + lx];
                lx += linv;
                if (lx >= q1) lx -= q1;
            }
            root = (val == 0);
            if (root) {
                // Lambda'(x) = sum_{d odd} Lam_d x^{d-1}; Omega = S Lambda mod x^{2t}
                uint32_t dval = 0, oval = 0;
                lx = 0;
#pragma unroll
                for (int dgr = 0; dgr < 2 * TMAX; ++dgr) {
                    if (dgr < 2 * t) {
                        uint32_t om = 0;
#pragma unroll
                        for (int k2 = 0; k2 <= dgr && k2 <= TMAX; ++k2) om ^= gf_mul(T, Lam[k2], S[dgr - k2]);
                        if (om) oval ^= T.exp2[T.log[om] + lx];
                    }
                    if (dgr + 1 <= TMAX && ((dgr + 1) & 1) && lgl[dgr + 1] >= 0) dval ^= T.exp2[lgl[dgr + 1] + lx];
                    lx += linv;
                    if (lx >= q1) lx -= q1;
                }
                if (dval == 0) {
                    badlane = true;  // repeated root: not a valid error locator
                } else {
                    // Y = X * Omega(X^-1) / Lambda'(X^-1); e = Y / v_i
                    uint32_t Y = gf_div(T, oval, dval);
                    if (Y) Y = T.exp2[T.log[Y] + li];
                    uint32_t e = 0;
                    if (Y) {
                        int le = static_cast<int>(T.log[Y]) - static_cast<int>(T.logv[i]);
                        if (le < 0) le += q1;
                        e = T.exp2[le];
                    }
                    err[p] = e;
                }
            }
        }
        roots += __popc(seg_ballot<W>(root, lane));
        changed += __popc(seg_ballot<W>(err[p] != 0, lane));
    }
    if (seg_ballot<W>(badlane, lane) != 0 || roots != L) fail = true;
    return fail ? -1 : changed;
}

// Long codes (one codeword per warp, t up to 31): Berlekamp-Massey with the
// locator spread over the lanes — lane i holds Lambda_i and B_i, lane j holds
// S_j and S_{j+32} — so a step is one discrepancy reduction (a butterfly)
// and one shifted update (a shuffle) instead of O(t^2) work in every lane.
// Omega_j is formed the same way; the Chien search and Forney then run per
// position with the coefficients gathered into every lane (log domain).
// Same contract as seg_locate.
template <int TMAX, int P>
__device__ __forceinline__ int warp_locate_lp(const RsSmem& T, const uint32_t (&S)[2 * TMAX + 1], int lane,
                                              uint32_t (&err)[P]) {
    static_assert(TMAX <= 31, "lane-parallel locator holds Lambda_0..Lambda_31");
    constexpr int RMAX = 2 * TMAX + 1;
    const int n = T.n, t = T.t, q1 = T.q1;
    // distribute the syndromes: lane j <- S_j, S_{j+32}
    uint32_t slo = 0, shi = 0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
        if (j < 32 && j == lane) slo = S[j];
        if (j >= 32 && j - 32 == lane) shi = S[j];
    }
    uint32_t lam = lane == 0 ? 1u : 0u, bb = lam, bdisc = 1;
    int L = 0, shift = 1;
    for (int step = 0; step < 2 * t; ++step) {  // warp-uniform
        const int idx = step - lane;             // S_{step - i} for i = lane
        const uint32_t s_lo = __shfl_sync(0xffffffffu, slo, idx & 31);
        const uint32_t s_hi = __shfl_sync(0xffffffffu, shi, (idx - 32) & 31);
        const uint32_t sv = idx < 0 ? 0u : (idx < 32 ? s_lo : s_hi);
        uint32_t d = (lane <= L) ? gf_mul(T, lam, sv) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d ^= __shfl_xor_sync(0xffffffffu, d, o);
        if (d == 0) {
            ++shift;
        } else {
            const uint32_t coef = gf_div(T, d, bdisc);
            uint32_t bs = __shfl_up_sync(0xffffffffu, bb, shift < 32 ? shift : 0);
            if (lane < shift) bs = 0;
            const uint32_t nl = lam ^ gf_mul(T, coef, bs);
            if (2 * L <= step) {
                bb = lam;
                L = step + 1 - L;
                bdisc = d;
                shift = 1;
            } else {
                ++shift;
            }
            lam = nl;
        }
    }
    const uint32_t nz = __ballot_sync(0xffffffffu, lam != 0);
    const int deg = 31 - __clz(nz);
    bool fail = L > t || deg != L;
    // Omega_j = sum_{i <= j} Lambda_i S_{j-i}, j < 2t: lane j forms Omega_j and Omega_{j+32}
    uint32_t olo = 0, ohi = 0;
    for (int i = 0; i <= L && i < 32; ++i) {  // warp-uniform
        const uint32_t li = __shfl_sync(0xffffffffu, lam, i);
        const int a = lane - i;  // S_{lane - i}
        const uint32_t sa = __shfl_sync(0xffffffffu, slo, a & 31);
        const uint32_t sb_lo = __shfl_sync(0xffffffffu, slo, (a + 32) & 31);  // S_{lane + 32 - i}, < 32
        const uint32_t sb_hi = __shfl_sync(0xffffffffu, shi, a & 31);         // S_{lane + 32 - i}, >= 32
        if (a >= 0) olo ^= gf_mul(T, li, sa);
        ohi ^= gf_mul(T, li, a >= 0 ? sb_hi : sb_lo);
    }
    if (lane >= 2 * t) olo = 0;
    if (lane + 32 >= 2 * t) ohi = 0;
    // gather the coefficients (logs; 0xFFFF marks a zero coefficient)
    uint16_t lgl[32], lgo[2 * TMAX];
#pragma unroll
    for (int d = 0; d < 32; ++d) {
        const uint32_t c = __shfl_sync(0xffffffffu, lam, d);
        lgl[d] = (d <= TMAX && c) ? static_cast<uint16_t>(T.log[c]) : 0xFFFFu;
    }
#pragma unroll
    for (int j = 0; j < 2 * TMAX; ++j) {
        const uint32_t c = j < 32 ? __shfl_sync(0xffffffffu, olo, j) : __shfl_sync(0xffffffffu, ohi, (j - 32) & 31);
        lgo[j] = c ? static_cast<uint16_t>(T.log[c]) : 0xFFFFu;
    }
    int roots = 0, changed = 0;
    bool badlane = false;
#pragma unroll 1  // rolled: the unrolled 8-position Chien/Forney body overflowed the I-cache (ncu: 92 % no_instructions)
    for (int p = 0; p < P; ++p) {
        const int i = lane + 32 * p;
        err[p] = 0;
        bool root = false;
        if (i < n && !fail) {
            const int li = i % q1;
            const int linv = (q1 - li) % q1;
            uint32_t val = 0, dval = 0, oval = 0;
            int lx = 0;
#pragma unroll
            for (int dgr = 0; dgr <= TMAX; ++dgr) {
                if (lgl[dgr] != 0xFFFFu) {
                    val ^= T.exp2[lgl[dgr] + lx];
                    if (dgr & 1) {
                        int lprev = lx - linv;
                        if (lprev < 0) lprev += q1;
                        dval ^= T.exp2[lgl[dgr] + lprev];
                    }
                }
                lx += linv;
                if (lx >= q1) lx -= q1;
            }
            root = (val == 0);
            if (root) {
                lx = 0;
#pragma unroll
                for (int j = 0; j < 2 * TMAX; ++j) {
                    if (lgo[j] != 0xFFFFu) oval ^= T.exp2[lgo[j] + lx];
                    lx += linv;
                    if (lx >= q1) lx -= q1;
                }
                if (dval == 0) {
                    badlane = true;
                } else {
                    uint32_t Y = gf_div(T, oval, dval);
                    if (Y) Y = T.exp2[T.log[Y] + li];
                    uint32_t e = 0;
                    if (Y) {
                        int le = static_cast<int>(T.log[Y]) - static_cast<int>(T.logv[i]);
                        if (le < 0) le += q1;
                        e = T.exp2[le];
                    }
                    err[p] = e;
                }
            }
        }
        roots += __popc(__ballot_sync(0xffffffffu, root));
        changed += __popc(__ballot_sync(0xffffffffu, err[p] != 0));
    }
    if (__any_sync(0xffffffffu, badlane) || roots != L) fail = true;
    return fail ? -1 : changed;
}

// Bounded-distance decode of symbol words, W lanes per codeword. sym[p] holds
// symbol sl + W p. On return (all lanes of the segment): errors_corrected or
// -1; sym[] corrected on success. A success requires every one of the n-k
// checks to vanish on the corrected word (syndromes are linear: the error
// pattern's syndromes must equal the received word's) and at most t changed
// symbols.
template <int TMAX, int W, int P>
__device__ __forceinline__ int rs_seg_bm(const RsSmem& T, uint32_t (&sym)[P], int lane) {
    constexpr int RMAX = 2 * TMAX + 1;
    uint32_t S[RMAX];
    seg_syndromes<RMAX, W, P>(T, sym, lane, S);
    uint32_t anyS = 0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) anyS |= S[j];
    if (!__any_sync(0xffffffffu, anyS != 0)) return 0;  // warp-uniform fast path
    uint32_t err[P];
    int changed;
    if constexpr (W == 32 && TMAX >= 16) changed = warp_locate_lp<TMAX, P>(T, S, lane, err);
    else changed = seg_locate<TMAX, W, P>(T, S, lane, err);
    uint32_t S2[RMAX];
    seg_syndromes<RMAX, W, P>(T, err, lane, S2);  // recheck all n-k checks
    uint32_t bad = 0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) bad |= S2[j] ^ S[j];
    if (anyS == 0) return 0;
    if (changed < 0 || bad || changed > T.t) return -1;
#pragma unroll
    for (int p = 0; p < P; ++p) sym[p] ^= err[p];
    return changed;
}

// One codeword per warp (the detect completion kernel's general-t path).
template <int TMAX, int P>
__device__ __forceinline__ int rs_warp_bm(const RsSmem& T, uint32_t (&sym)[P], int lane) {
    return rs_seg_bm<TMAX, 32, P>(T, sym, lane);
}

}  // namespace qrm
