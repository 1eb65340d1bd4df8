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
//   * rs_warp_bm    — any t, one codeword per warp: lane-parallel syndromes
//     (xor butterfly), Berlekamp-Massey, lane-parallel Chien search over the n
//     valid locators only, Forney, then a full n-k syndrome recheck.
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

// Partial syndromes of this lane's positions, reduced across the warp:
// S_j = xor_i r_i v_i X_i^j for j < n-k (all lanes receive all S_j).
template <int RMAX, int P>
__device__ __forceinline__ void rs_warp_syndromes(const RsSmem& T, const uint32_t (&sym)[P], int lane,
                                                  uint32_t (&S)[RMAX]) {
    const int n = T.n, r = T.r, q1 = T.q1;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) S[j] = 0;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int i = lane + 32 * p;
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
        if (j < r) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) S[j] ^= __shfl_xor_sync(0xffffffffu, S[j], o);
        }
    }
}

// ------------------------------------------------------------ warp BM ----
// One codeword per warp. sym[p] holds symbol i = lane + 32 p (p < P).
// On return (all lanes): nerr = errors_corrected or -1; sym[] corrected.
template <int TMAX, int P>
__device__ __forceinline__ int rs_warp_bm(const RsSmem& T, uint32_t (&sym)[P], int lane) {
    constexpr int RMAX = 2 * TMAX + 1;
    const int n = T.n, t = T.t, q1 = T.q1;
    // Lane-parallel syndromes: each lane folds its positions (log-domain,
    // X_i^j stepped incrementally), then one xor butterfly per check.
    uint32_t S[RMAX];
    rs_warp_syndromes<RMAX, P>(T, sym, lane, S);
    uint32_t anyS = 0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) anyS |= S[j];
    if (anyS == 0) return 0;

    // Berlekamp-Massey on S_0..S_{2t-1} (warp-uniform; every lane runs it).
    uint32_t Lam[RMAX + 1], B[RMAX + 1];
#pragma unroll
    for (int i = 0; i <= RMAX; ++i) Lam[i] = B[i] = 0;
    Lam[0] = B[0] = 1;
    int L = 0, shift = 1;
    uint32_t bdisc = 1;
#pragma unroll
    for (int step = 0; step < 2 * TMAX; ++step) {
        if (step < 2 * t) {
            uint32_t d = S[step];
#pragma unroll
            for (int i = 1; i <= 2 * TMAX; ++i)
                if (i <= L && i <= step) d ^= gf_mul(T, Lam[i], S[step - i]);
            if (d == 0) {
                ++shift;
            } else {
                const uint32_t coef = gf_div(T, d, bdisc);
                uint32_t Tmp[RMAX + 1];
#pragma unroll
                for (int i = 0; i <= RMAX; ++i) Tmp[i] = Lam[i];
                // Lam -= coef * x^shift * B
#pragma unroll
                for (int i = 0; i <= RMAX; ++i) {
                    uint32_t bi = 0;
#pragma unroll
                    for (int s2 = 1; s2 <= RMAX; ++s2)
                        if (s2 == shift && i - s2 >= 0) bi = B[i - s2];
                    Lam[i] ^= gf_mul(T, coef, bi);
                }
                if (2 * L <= step) {
                    L = step + 1 - L;
#pragma unroll
                    for (int i = 0; i <= RMAX; ++i) B[i] = Tmp[i];
                    bdisc = d;
                    shift = 1;
                } else {
                    ++shift;
                }
            }
        }
    }
    if (L > t) return -1;
    // deg Lambda must equal L
    int deg = 0;
#pragma unroll
    for (int i = 0; i <= RMAX; ++i)
        if (Lam[i]) deg = i;
    if (deg != L) return -1;

    // Omega = S * Lambda mod x^{2t}
    uint32_t Om[2 * TMAX];
#pragma unroll
    for (int j = 0; j < 2 * TMAX; ++j) {
        uint32_t o = 0;
#pragma unroll
        for (int i = 0; i <= j; ++i)
            if (j < 2 * t) o ^= gf_mul(T, Lam[i], S[j - i]);
        Om[j] = o;
    }

    // Chien search over the n valid locators + Forney, lane-parallel.
    int roots = 0, changed = 0;
    bool badlane = false;
    uint32_t err[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int i = lane + 32 * p;
        err[p] = 0;
        bool root = false;
        if (i < n) {
            const int li = i % q1;                 // log X_i
            const int linv = (q1 - li) % q1;       // log X_i^{-1}
            uint32_t val = 0, dval = 0, oval = 0;
            int lx = 0;                            // log x^d, d = 0..
#pragma unroll
            for (int dgr = 0; dgr <= RMAX; ++dgr) {
                if (dgr <= L && Lam[dgr]) {
                    const uint32_t term = T.exp2[T.log[Lam[dgr]] + lx];
                    val ^= term;
                }
                if (dgr >= 1 && (dgr & 1) && dgr <= L && Lam[dgr]) {  // Lambda' = sum_{d odd} Lam_d x^{d-1}
                    int lprev = lx - linv;
                    if (lprev < 0) lprev += q1;
                    dval ^= T.exp2[T.log[Lam[dgr]] + lprev];
                }
                if (dgr < 2 * TMAX && dgr < 2 * t && Om[dgr]) oval ^= T.exp2[T.log[Om[dgr]] + lx];
                lx += linv;
                if (lx >= q1) lx -= q1;
            }
            root = (val == 0);
            if (root) {
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
        const unsigned bal = __ballot_sync(0xffffffffu, root);
        roots += __popc(bal);
        changed += __popc(__ballot_sync(0xffffffffu, err[p] != 0));
    }
    if (__any_sync(0xffffffffu, badlane)) return -1;
    if (roots != L) return -1;

    // Apply and recheck every parity check (n-k of them) on the corrected word.
#pragma unroll
    for (int p = 0; p < P; ++p) sym[p] ^= err[p];
    uint32_t S2[RMAX];
    rs_warp_syndromes<RMAX, P>(T, sym, lane, S2);
    uint32_t bad = 0;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) bad |= S2[j];
    if (bad || changed > t) return -1;
    return changed;
}

}  // namespace qrm
