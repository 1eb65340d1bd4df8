// Batched Reed-Solomon decoding kernels (replace bw_decode, rs.cpp:188-196)
// and the RS stress-word generator used by the RS-only benchmark.
#include <cuda_runtime.h>


#include "qrm_device.cuh"
#include "qrm_rs.cuh"
#include "qrm_types.h"

namespace qrm {

// One codeword per thread (t = 1 codes, n*m <= 64): HBM-bound, 8 B in + 9 B out.
__global__ void __launch_bounds__(256) rs_t1_packed_kernel(const RsTables* __restrict__ g,
                                                          const uint64_t* __restrict__ words, int64_t count,
                                                          uint64_t* __restrict__ cw_out, int8_t* __restrict__ nerr_out) {
    __shared__ RsSmem T;
    rs_stage_tables(T, g, threadIdx.x, blockDim.x);
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t w = __ldcs(words + i);
        uint64_t cw = 0;
        const int e = rs_t1_packed(T, w, cw);
        __stcs(cw_out + i, e >= 0 ? cw : 0ull);
        __stcs(reinterpret_cast<signed char*>(nerr_out) + i, static_cast<signed char>(e));
    }
}

// Vectorised form: each thread decodes 4 consecutive words (two 16-byte
// loads issued before any compute, so each thread keeps 32 B in flight);
// requires 16-byte aligned word arrays and 4-byte aligned nerr. The code shape
// (MB syndrome bits per symbol, R = n-k) is compile-time and the syndrome
// masks live in registers.
template <int MB, int R>
__global__ void __launch_bounds__(256) rs_t1_packed_x4_kernel(const RsTables* __restrict__ g,
                                                             const ulonglong2* __restrict__ words, int64_t groups,
                                                             ulonglong2* __restrict__ cw_out,
                                                             uint32_t* __restrict__ nerr_out) {
    __shared__ RsSmem T;
    rs_stage_tables(T, g, threadIdx.x, blockDim.x);
    uint64_t mk[R * MB];
#pragma unroll
    for (int j = 0; j < R * MB; ++j) mk[j] = __ldg(&g->synd_mask[j]);
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < groups; i += stride) {
        const ulonglong2 a = __ldcs(words + 2 * i);
        const ulonglong2 b = __ldcs(words + 2 * i + 1);
        uint64_t w[4] = {a.x, a.y, b.x, b.y}, c[4];
        uint32_t ne = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint64_t cw;
            const int e = rs_t1_fixed<MB, R>(T, mk, w[j], cw);
            c[j] = e >= 0 ? cw : 0ull;
            ne |= (static_cast<uint32_t>(e) & 0xFFu) << (8 * j);
        }
        __stcs(cw_out + 2 * i, make_ulonglong2(c[0], c[1]));
        __stcs(cw_out + 2 * i + 1, make_ulonglong2(c[2], c[3]));
        __stcs(nerr_out + i, ne);
    }
}

// General t, packed words (n*m <= 64). A warp owns chunks of 32 consecutive
// words (one coalesced 8-byte load per lane, the next chunk prefetched while
// this one is decoded). Syndromes are GF(2)-linear parities of the packed
// word, so each lane first forms its own word's r*m syndrome bits (popc over
// the masks); words with a nonzero syndrome are then decoded W lanes per word,
// 32/W at a time: the segment takes the word's syndromes by shuffle, runs
// Berlekamp-Massey, the lane-parallel Chien search over positions sl + W p and
// Forney (seg_locate), and ORs the corrections into the word; the owning lane
// receives the result and rechecks all n-k checks on it. Results are written
// back with one coalesced store per lane.
//
// With a CodebookTable (row f1: the reference's CorrectionCache, detect.cpp:
// 86-128, as a device memo) each lane first probes the table for its word; hits
// skip the decode, and decoded words are inserted (slot claimed by CAS, value
// written, then the key published behind a fence, so a reader that sees the
// key sees the value). The memo is transparent: a decode is a pure function
// of the word.
template <int W, int P, int TMAX, bool CACHED>
__global__ void __launch_bounds__(256) rs_seg_packed_kernel(const RsTables* __restrict__ g,
                                                           const uint64_t* __restrict__ words, int64_t count,
                                                           uint64_t* __restrict__ cw_out,
                                                           int8_t* __restrict__ nerr_out, CodebookTable cache) {
    __shared__ RsSmem T;
    rs_stage_tables(T, g, threadIdx.x, blockDim.x);
    __syncthreads();
    constexpr int RMAX = 2 * TMAX + 1;
    constexpr int kPerRound = 32 / W;
    const int lane = threadIdx.x & 31;
    const int sl = lane & (W - 1);
    const int seg = lane / W;
    const int m = T.m, n = T.n, r = T.r, t = T.t, nm = T.nmask;
    const uint32_t smask = (1u << m) - 1;
    auto syndrome_bits = [&](uint64_t w) {
        uint64_t sb = 0;
        for (int b = 0; b < nm; ++b) {
            const uint64_t x = w & T.synd_mask[b];
            sb |= static_cast<uint64_t>(__popc(static_cast<uint32_t>(x) ^ static_cast<uint32_t>(x >> 32)) & 1) << b;
        }
        return sb;
    };
    const int64_t warp_id = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 32;
    int64_t base = warp_id * 32;
    uint64_t wnext = base + lane < count ? __ldcs(words + base + lane) : 0ull;
    for (; base < count; base += stride) {  // warp-uniform loop
        const int64_t i = base + lane;
        const bool live = i < count;
        const uint64_t w = wnext;
        if (base + stride + lane < count) wnext = __ldcs(words + base + stride + lane);
        uint64_t cw = w;
        int nerr = 0;
        bool hit = false;
        uint64_t slot0 = 0;
        if constexpr (CACHED) {
            if (live) {
                slot0 = mix64(w) & cache.mask;
#pragma unroll 1
                for (int pr = 0; pr < kCodebookProbes; ++pr) {
                    const uint64_t sidx = (slot0 + pr) & cache.mask;
                    const uint64_t key = *reinterpret_cast<volatile const uint64_t*>(cache.keys + sidx);
                    if (key == w) {
                        __threadfence();  // acquire: the value was published before the key
                        cw = cache.vals[sidx];
                        nerr = cache.nerr[sidx];
                        hit = true;
                        break;
                    }
                    if (key == kCodebookEmpty) break;
                }
            }
        }
        const uint64_t sb = (live && !hit) ? syndrome_bits(w) : 0ull;
        uint32_t pending = __ballot_sync(0xffffffffu, sb != 0);
        const int my_rank = __popc(pending & ((1u << lane) - 1));  // among the words needing correction
        int round_base = 0;
        while (pending) {  // warp-uniform: kPerRound words per round
            uint32_t rest = pending;  // this segment's word: the seg-th set bit of pending (32: none)
#pragma unroll
            for (int q = 0; q < kPerRound - 1; ++q)
                if (q < seg) rest &= rest - 1;
            const int j = rest ? __ffs(rest) - 1 : 32;
            const int src = j < 32 ? j : 0;
            const uint64_t wj = __shfl_sync(0xffffffffu, w, src);
            const uint64_t sb_src = __shfl_sync(0xffffffffu, sb, src);  // every lane shuffles (no divergent sync)
            const uint64_t sj = j < 32 ? sb_src : 0ull;
            uint32_t S[RMAX];
#pragma unroll
            for (int q = 0; q < RMAX; ++q) S[q] = q < r ? static_cast<uint32_t>(sj >> (q * m)) & smask : 0u;
            uint32_t err[P];
            const int changed = seg_locate<TMAX, W, P>(T, S, lane, err);
            uint64_t part = 0;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int pos = sl + W * q;
                if (pos < n && changed > 0) part |= static_cast<uint64_t>(err[q]) << (m * (n - 1 - pos));
            }
#pragma unroll
            for (int o = W / 2; o > 0; o >>= 1) part |= __shfl_xor_sync(0xffffffffu, part, o);
            // the owning lane takes its word's result from segment (rank - round_base)
            const int from = (my_rank - round_base) * W;
            const bool mine = sb != 0 && my_rank >= round_base && my_rank < round_base + kPerRound;
            const uint64_t got_part = __shfl_sync(0xffffffffu, part, mine ? from : 0);
            const int got_changed = __shfl_sync(0xffffffffu, changed, mine ? from : 0);
            if (mine) {
                const uint64_t c2 = w ^ got_part;
                if (got_changed < 0 || got_changed > t || syndrome_bits(c2) != 0) {
                    nerr = -1;
                } else {
                    nerr = got_changed;
                    cw = c2;
                }
            }
#pragma unroll
            for (int q = 0; q < kPerRound; ++q) pending &= pending - 1;  // drop this round's words
            round_base += kPerRound;
        }
        if constexpr (CACHED) {
            if (live && !hit && sb != 0) {  // memoise decoded (and failed) words
#pragma unroll 1
                for (int pr = 0; pr < kCodebookProbes; ++pr) {
                    const uint64_t sidx = (slot0 + pr) & cache.mask;
                    const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(cache.keys + sidx),
                                                             kCodebookEmpty, kCodebookBusy);
                    if (old == kCodebookEmpty) {
                        cache.vals[sidx] = cw;
                        cache.nerr[sidx] = static_cast<int8_t>(nerr);
                        __threadfence();  // release: value before key
                        *reinterpret_cast<volatile uint64_t*>(cache.keys + sidx) = w;
                        break;
                    }
                    if (old == w) break;  // another lane inserted it
                }
            }
        }
        if (live) {
            __stcs(cw_out + i, nerr >= 0 ? cw : 0ull);
            __stcs(reinterpret_cast<signed char*>(nerr_out) + i, static_cast<signed char>(nerr));
        }
    }
}

// General t, symbol bytes: one codeword per segment of W lanes (n <= 32), or
// per warp with P symbols per lane (n <= 32 P).
template <int TMAX, int W, int P>
__global__ void __launch_bounds__(256, (W == 32 && TMAX >= 16) ? 2 : 1) rs_seg_symbols_kernel(const RsTables* __restrict__ g,
                                                            const uint8_t* __restrict__ recv, int64_t count,
                                                            uint8_t* __restrict__ cw_out,
                                                            int8_t* __restrict__ nerr_out) {
    __shared__ RsSmem T;
    rs_stage_tables(T, g, threadIdx.x, blockDim.x);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int sl = lane & (W - 1);
    constexpr int kPerWarp = 32 / W;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int n = T.n;
    for (int64_t base = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kPerWarp;
         base < count; base += warps * kPerWarp) {  // warp-uniform loop
        const int64_t i = base + lane / W;
        const bool live = i < count;
        uint32_t sym[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int pos = sl + W * p;
            sym[p] = (live && pos < n) ? recv[i * n + pos] : 0u;
        }
        const int e = rs_seg_bm<TMAX, W, P>(T, sym, lane);
        if (live) {
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const int pos = sl + W * p;
                if (pos < n) cw_out[i * n + pos] = e >= 0 ? static_cast<uint8_t>(sym[p]) : 0;
            }
            if (sl == 0) nerr_out[i] = static_cast<int8_t>(e);
        }
    }
}

// RS stress words (SURVEY 8d recipe, counter-RNG per word so any slice is
// reproducible): random k*m-bit message -> systematic encode (parity bits are
// GF(2)-linear in the message: parity bit b = parity(msg & enc_mask[b])) ->
// e errors at distinct positions, each XOR (1 + below(q-1)); e ~ U{0..t} for
// 90% of words and U{t+1..3} for the other 10%.
__global__ void rs_stress_kernel(const RsTables* __restrict__ g, const uint64_t* __restrict__ enc_mask,
                                 uint64_t seed, int64_t count, uint64_t* __restrict__ msg_out,
                                 uint64_t* __restrict__ word_out, int8_t* __restrict__ nerr_true) {
    const int m = g->m, n = g->n, k = g->k, t = g->t, q1 = g->q1;
    const int rb = (n - k) * m, kb = k * m;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t u = static_cast<uint64_t>(i);
        const uint64_t msg = rng_word(seed, 0, u) & (kb == 64 ? ~0ull : ((1ull << kb) - 1));
        uint64_t par = 0;
        for (int b = 0; b < rb; ++b) par |= static_cast<uint64_t>(__popcll(msg & enc_mask[b]) & 1) << b;
        uint64_t w = (msg << rb) | par;
        int e;
        const bool beyond = rng_below(seed, 1, u, 10) == 0 && t + 1 <= 3;
        if (beyond) e = t + 1 + static_cast<int>(rng_below(seed, 2, u, static_cast<uint64_t>(3 - t)));
        else e = static_cast<int>(rng_below(seed, 2, u, static_cast<uint64_t>(t + 1)));
        if (e > n) e = n;
        uint32_t used = 0;  // n <= 32 for packed words
        uint64_t ctr = 0;
        for (int j = 0; j < e; ++j) {
            int pos;
            do {
                pos = static_cast<int>(rng_below(seed, 3 + u * 2, ctr++, static_cast<uint64_t>(n)));
            } while ((used >> pos) & 1);
            used |= 1u << pos;
            const uint64_t val = 1 + rng_below(seed, 4 + u * 2, static_cast<uint64_t>(j), static_cast<uint64_t>(q1));
            w ^= val << (m * (n - 1 - pos));
        }
        msg_out[i] = msg;
        word_out[i] = w;
        nerr_true[i] = static_cast<int8_t>(e);
    }
}

// RS stress words for symbol codes (any n): one warp per word. Message
// symbols are counter-RNG draws; the parity symbols are GF(2^m)-linear in the
// message (encoding is linear), parity_c = xor_j a_j * G[j][c] with G[j] the
// parity of the j-th unit message (host rs_encode), staged in shared memory.
// Errors as in rs_stress_kernel: e ~ U{0..t} for 90% of words and
// U{t+1..t+2} for the other 10%, at distinct positions, each XOR (1 + below(q-1)).
__global__ void __launch_bounds__(256) rs_stress_symbols_kernel(const RsTables* __restrict__ g,
                                                               const uint8_t* __restrict__ gpar, uint64_t seed,
                                                               int64_t count, uint8_t* __restrict__ true_cw,
                                                               uint8_t* __restrict__ recv,
                                                               int8_t* __restrict__ nerr_true) {
    extern __shared__ uint8_t sg[];  // [k][r] parity generator
    __shared__ RsSmem T;
    rs_stage_tables(T, g, threadIdx.x, blockDim.x);
    const int n = g->n, k = g->k, r = g->r, t = g->t, q1 = g->q1, m = g->m;
    for (int i = threadIdx.x; i < k * r; i += blockDim.x) sg[i] = gpar[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); w < count;
         w += warps) {
        const uint64_t u = static_cast<uint64_t>(w);
        uint8_t* tc = true_cw + w * n;
        uint8_t* rc = recv + w * n;
        for (int c0 = 0; c0 < ((r + 31) & ~31); c0 += 32) {
            const int c = c0 + lane;
            uint32_t par = 0;
            for (int j = 0; j < k; ++j) {
                const uint32_t a = static_cast<uint32_t>(rng_word(seed, 0, u * 256 + j)) & (q1 > 0 ? ((1u << m) - 1) : 0u);
                if (c < r) par ^= gf_mul(T, a, sg[j * r + c]);
                if (c0 == 0 && (j & 31) == lane) {
                    tc[j] = static_cast<uint8_t>(a);
                    rc[j] = static_cast<uint8_t>(a);
                }
            }
            if (c < r) {
                tc[k + c] = static_cast<uint8_t>(par);
                rc[k + c] = static_cast<uint8_t>(par);
            }
        }
        __syncwarp();
        if (lane == 0) {
            int e;
            if (rng_below(seed, 1, u, 10) == 0) e = t + 1 + static_cast<int>(rng_below(seed, 2, u, 2));
            else e = static_cast<int>(rng_below(seed, 2, u, static_cast<uint64_t>(t + 1)));
            if (e > n) e = n;
            uint32_t used[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            uint64_t ctr = 0;
            for (int j = 0; j < e; ++j) {
                int pos;
                do {
                    pos = static_cast<int>(rng_below(seed, 3 + u * 2, ctr++, static_cast<uint64_t>(n)));
                } while ((used[pos >> 5] >> (pos & 31)) & 1);
                used[pos >> 5] |= 1u << (pos & 31);
                rc[pos] ^= static_cast<uint8_t>(1 + rng_below(seed, 4 + u * 2, static_cast<uint64_t>(j), static_cast<uint64_t>(q1)));
            }
            nerr_true[w] = static_cast<int8_t>(e);
        }
        __syncwarp();
    }
}

cudaError_t launch_rs_stress_symbols(const RsTables* tab, const uint8_t* gpar, int k, int r, uint64_t seed,
                                     int64_t count, uint8_t* true_cw, uint8_t* recv, int8_t* nerr_true,
                                     cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    const size_t smem = static_cast<size_t>(k) * r;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(rs_stress_symbols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    rs_stress_symbols_kernel<<<static_cast<unsigned>(blocks), 256, smem, st>>>(tab, gpar, seed, count, true_cw, recv,
                                                                               nerr_true);
    return cudaGetLastError();
}

cudaError_t launch_rs_packed(const RsTables* tab, int m, int n, int r, int t, int algo, const uint64_t* words,
                             int64_t count, uint64_t* cw, int8_t* nerr, int sm_count, cudaStream_t st,
                             CodebookTable cache) {
    if (count <= 0) return cudaSuccess;
    const int sms = sm_count > 0 ? sm_count : 148;
    if (algo == 1) {
        const bool vec = (reinterpret_cast<uintptr_t>(words) % 16 == 0) && (reinterpret_cast<uintptr_t>(cw) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(nerr) % 4 == 0);
        const int64_t groups = vec ? count / 4 : 0;
        if (groups > 0) {
            int64_t blocks = (groups + 255) / 256;
            const int64_t cap = static_cast<int64_t>(sms) * 16;
            if (blocks > cap) blocks = cap;
            const auto* wv = reinterpret_cast<const ulonglong2*>(words);
            auto* cv = reinterpret_cast<ulonglong2*>(cw);
            auto* nv = reinterpret_cast<uint32_t*>(nerr);
            const unsigned gb = static_cast<unsigned>(blocks);
            if (m == 4 && r == 3) rs_t1_packed_x4_kernel<4, 3><<<gb, 256, 0, st>>>(tab, wv, groups, cv, nv);
            else if (m == 4) rs_t1_packed_x4_kernel<4, 2><<<gb, 256, 0, st>>>(tab, wv, groups, cv, nv);
            else if (r == 3) rs_t1_packed_x4_kernel<8, 3><<<gb, 256, 0, st>>>(tab, wv, groups, cv, nv);
            else rs_t1_packed_x4_kernel<8, 2><<<gb, 256, 0, st>>>(tab, wv, groups, cv, nv);
        }
        const int64_t done = groups * 4, rest = count - done;
        if (rest > 0) {
            int64_t blocks = (rest + 255) / 256;
            const int64_t cap = static_cast<int64_t>(sms) * 8;
            if (blocks > cap) blocks = cap;
            rs_t1_packed_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(tab, words + done, rest, cw + done,
                                                                               nerr + done);
        }
    } else {
        // 4 lanes per word (8 words per round): measured 11.3 G words/s on gf16-15-12 stress words
        // against 9.5 (8 lanes) and 6.7 (16 lanes) — the segment-uniform work (BM) amortises over
        // more words. Packed words have n <= 15 (m = 4) or n <= 8 (m = 8): 4 or 2 positions per lane.
        int64_t blocks = (count + 255) / 256;
        const int64_t cap = static_cast<int64_t>(sms) * 16;
        if (blocks > cap) blocks = cap;
        const unsigned b = static_cast<unsigned>(blocks);
#define QRM_SEGP(P, TM)                                                                                       \
    (cache.keys ? (rs_seg_packed_kernel<4, P, TM, true><<<b, 256, 0, st>>>(tab, words, count, cw, nerr, cache), 0) \
                : (rs_seg_packed_kernel<4, P, TM, false><<<b, 256, 0, st>>>(tab, words, count, cw, nerr, cache), 0))
        if (n <= 8 && t <= 1) QRM_SEGP(2, 1);
        else if (n <= 8 && t <= 2) QRM_SEGP(2, 2);
        else if (n <= 8) QRM_SEGP(2, 4);
        else if (t <= 1) QRM_SEGP(4, 1);
        else if (t <= 2) QRM_SEGP(4, 2);
        else if (t <= 4) QRM_SEGP(4, 4);
        else QRM_SEGP(4, 8);
#undef QRM_SEGP
    }
    return cudaGetLastError();
}

cudaError_t launch_rs_symbols(const RsTables* tab, int n, int t, const uint8_t* recv, int64_t count, uint8_t* cw,
                              int8_t* nerr, int sm_count, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    const int sms = sm_count > 0 ? sm_count : 148;
    // narrow segments for short codes (W = 4 or 8 lanes, 4 positions each), a warp per long codeword
    const int W = n <= 16 ? 4 : n <= 32 ? 8 : 32;
    int64_t blocks = (count * W + 255) / 256;
    const int64_t cap = static_cast<int64_t>(sms) * 16;
    if (blocks > cap) blocks = cap;
    const unsigned b = static_cast<unsigned>(blocks);
    // t <= (n - 1) / 2: n <= 16 -> t <= 7, n <= 32 -> t <= 15
    if (n <= 16) {
        if (t <= 1) rs_seg_symbols_kernel<1, 4, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 2) rs_seg_symbols_kernel<2, 4, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 4) rs_seg_symbols_kernel<4, 4, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else rs_seg_symbols_kernel<8, 4, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
    } else if (n <= 32) {
        if (t <= 2) rs_seg_symbols_kernel<2, 8, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 4) rs_seg_symbols_kernel<4, 8, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 8) rs_seg_symbols_kernel<8, 8, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else rs_seg_symbols_kernel<16, 8, 4><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
    }
    if (n > 32) {
        if (t <= 2) rs_seg_symbols_kernel<2, 32, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 4) rs_seg_symbols_kernel<4, 32, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 8) rs_seg_symbols_kernel<8, 32, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 16) rs_seg_symbols_kernel<16, 32, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else rs_seg_symbols_kernel<31, 32, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
    }
    return cudaGetLastError();
}

cudaError_t launch_rs_stress(const RsTables* tab, const uint64_t* enc_mask, uint64_t seed, int64_t count,
                             uint64_t* msg, uint64_t* words, int8_t* nerr_true, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    rs_stress_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(tab, enc_mask, seed, count, msg, words, nerr_true);
    return cudaGetLastError();
}

}  // namespace qrm
