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

// One codeword per warp, packed words (n <= 32 symbols).
template <int TMAX>
__global__ void __launch_bounds__(256) rs_warp_packed_kernel(const RsTables* __restrict__ g,
                                                            const uint64_t* __restrict__ words, int64_t count,
                                                            uint64_t* __restrict__ cw_out,
                                                            int8_t* __restrict__ nerr_out) {
    __shared__ RsSmem T;
    rs_stage_tables(T, g, threadIdx.x, blockDim.x);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int m = T.m, n = T.n;
    const uint32_t smask = (1u << m) - 1;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < count;
         i += warps) {
        const uint64_t w = words[i];
        uint32_t sym[1];
        sym[0] = lane < n ? static_cast<uint32_t>((w >> (m * (n - 1 - lane))) & smask) : 0u;
        const int e = rs_warp_bm<TMAX, 1>(T, sym, lane);
        uint64_t part = (e >= 0 && lane < n) ? static_cast<uint64_t>(sym[0]) << (m * (n - 1 - lane)) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part |= __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) {
            cw_out[i] = part;
            nerr_out[i] = static_cast<int8_t>(e);
        }
    }
}

// One codeword per warp, symbol bytes (any n <= 255).
template <int TMAX, int P>
__global__ void __launch_bounds__(256) rs_warp_symbols_kernel(const RsTables* __restrict__ g,
                                                             const uint8_t* __restrict__ recv, int64_t count,
                                                             uint8_t* __restrict__ cw_out,
                                                             int8_t* __restrict__ nerr_out) {
    __shared__ RsSmem T;
    rs_stage_tables(T, g, threadIdx.x, blockDim.x);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int n = T.n;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < count;
         i += warps) {
        uint32_t sym[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int pos = lane + 32 * p;
            sym[p] = pos < n ? recv[i * n + pos] : 0u;
        }
        const int e = rs_warp_bm<TMAX, P>(T, sym, lane);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int pos = lane + 32 * p;
            if (pos < n) cw_out[i * n + pos] = e >= 0 ? static_cast<uint8_t>(sym[p]) : 0;
        }
        if (lane == 0) nerr_out[i] = static_cast<int8_t>(e);
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

cudaError_t launch_rs_packed(const RsTables* tab, int m, int r, int t, int algo, const uint64_t* words,
                             int64_t count, uint64_t* cw, int8_t* nerr, int sm_count, cudaStream_t st) {
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
        int64_t blocks = (count + 7) / 8;
        const int64_t cap = static_cast<int64_t>(sms) * 16;
        if (blocks > cap) blocks = cap;
        const unsigned b = static_cast<unsigned>(blocks);
        if (t <= 1) rs_warp_packed_kernel<1><<<b, 256, 0, st>>>(tab, words, count, cw, nerr);
        else if (t <= 2) rs_warp_packed_kernel<2><<<b, 256, 0, st>>>(tab, words, count, cw, nerr);
        else if (t <= 4) rs_warp_packed_kernel<4><<<b, 256, 0, st>>>(tab, words, count, cw, nerr);
        else rs_warp_packed_kernel<8><<<b, 256, 0, st>>>(tab, words, count, cw, nerr);
    }
    return cudaGetLastError();
}

cudaError_t launch_rs_symbols(const RsTables* tab, int n, int t, const uint8_t* recv, int64_t count, uint8_t* cw,
                              int8_t* nerr, int sm_count, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    const int sms = sm_count > 0 ? sm_count : 148;
    int64_t blocks = (count + 7) / 8;
    const int64_t cap = static_cast<int64_t>(sms) * 16;
    if (blocks > cap) blocks = cap;
    const unsigned b = static_cast<unsigned>(blocks);
    if (n <= 32) {
        if (t <= 1) rs_warp_symbols_kernel<1, 1><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 2) rs_warp_symbols_kernel<2, 1><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 4) rs_warp_symbols_kernel<4, 1><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 8) rs_warp_symbols_kernel<8, 1><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else rs_warp_symbols_kernel<16, 1><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
    } else {
        if (t <= 2) rs_warp_symbols_kernel<2, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 4) rs_warp_symbols_kernel<4, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else if (t <= 8) rs_warp_symbols_kernel<8, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
        else rs_warp_symbols_kernel<16, 8><<<b, 256, 0, st>>>(tab, recv, count, cw, nerr);
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
