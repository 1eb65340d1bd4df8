// Device-side building blocks shared by the sm_100a kernels.
//
//  * counter RNG (reference include/qrmark/rng.hpp:13-39), usable on host and device
//  * tile selection (reference src/tiling.cpp:23-47)
//  * thin PTX wrappers: mbarrier, cp.async, proxy fences, tcgen05 (TMEM alloc,
//    MMA, commit, ld) — written for sm_100a only.
#pragma once

#include <cstdint>

#include "qrm_types.h"

#define QRM_HD __host__ __device__ __forceinline__
#define QRM_D __device__ __forceinline__

namespace qrm {

// ---------------------------------------------------------------- rng ----
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

QRM_HD uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

QRM_HD uint64_t rng_word(uint64_t seed, uint64_t stream, uint64_t ctr) {
    const uint64_t key = mix64(seed + kGolden * (stream + 1));
    return mix64(key ^ (ctr * 0xd6e8feb86659fd93ULL) ^ (ctr >> 32));
}

QRM_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

QRM_HD uint64_t rng_below(uint64_t seed, uint64_t stream, uint64_t ctr, uint64_t bound) {
    return mulhi64(rng_word(seed, stream, ctr), bound);
}

QRM_HD double rng_unit(uint64_t seed, uint64_t stream, uint64_t ctr) {
    return static_cast<double>(rng_word(seed, stream, ctr) >> 11) * 0x1.0p-53;
}

// Tile origin inside the w x h working image (tiling.cpp:23-47).
// strategy: 0 random, 1 random_grid, 2 fixed.
QRM_HD void select_tile(int w, int h, int l, int strategy, uint64_t seed, uint64_t draw, int& x, int& y) {
    if (strategy == QRM_TILE_FIXED) {
        x = 0;
        y = 0;
    } else if (strategy == QRM_TILE_RANDOM) {
        x = static_cast<int>(rng_below(seed, 2 * draw, 0, static_cast<uint64_t>(w - l) + 1));
        y = static_cast<int>(rng_below(seed, 2 * draw + 1, 0, static_cast<uint64_t>(h - l) + 1));
    } else {
        // cols*rows < 2^31 here (w, h are int), so the cell index fits 32 bits:
        // 32-bit div/mod instead of a 64-bit division subroutine.
        const uint32_t cols = static_cast<uint32_t>(w / l), rows = static_cast<uint32_t>(h / l);
        const uint32_t cell = static_cast<uint32_t>(rng_below(seed, draw, 0, static_cast<uint64_t>(cols) * rows));
        x = static_cast<int>(cell % cols) * l;
        y = static_cast<int>(cell / cols) * l;
    }
}

#ifdef __CUDACC__
// --------------------------------------------------------------- smem ----
QRM_D uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// ----------------------------------------------------------- mbarrier ----
QRM_D void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

QRM_D void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

QRM_D void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}

QRM_D bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

QRM_D void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// ----------------------------------------------------------- cp.async ----
// 16-byte global->shared copy through L2 only (.cg); src_bytes < 16 zero-fills.
QRM_D void cp_async16(uint32_t dst_smem, const void* src, uint32_t src_bytes = 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst_smem), "l"(src), "r"(src_bytes)
                 : "memory");
}
// As cp_async16 with an explicit L2 fill-size hint (64 / 128 / 256 B).
QRM_D void cp_async16_l2_64(uint32_t dst_smem, const void* src) {
    asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
QRM_D void cp_async16_l2_256(uint32_t dst_smem, const void* src) {
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
QRM_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
QRM_D void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Arrive on `bar` once all cp.async previously issued by this thread have
// landed in shared memory (the barrier's count must include this thread).
QRM_D void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Fire-and-forget L2 prefetch of `bytes` (multiple of 16, 16-B aligned).
QRM_D void prefetch_l2_bulk(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// Prefetch the line holding `p` into L2 (plain LSU prefetch).
QRM_D void prefetch_l2_line(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// Make generic-proxy shared-memory writes visible to the async proxy (tcgen05.mma).
QRM_D void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ tcgen05 ----
template <uint32_t kCols>
QRM_D void tmem_alloc(uint32_t* dst_smem_slot) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
QRM_D void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

QRM_D void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
QRM_D void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem], kind::i8 (u8 x s8 -> s32).
QRM_D void umma_i8(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 x bf16 -> f32).
QRM_D void umma_bf16(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
        : "memory");
}

QRM_D void umma_tf32(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
        : "memory");
}

// As umma_bf16, with output lanes disabled (mask bit set = lane not written):
// mask[q] covers lanes 32q..32q+31.
QRM_D void umma_bf16_masked(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate,
                            uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate), "r"(m0), "r"(m1), "r"(m2), "r"(m3)
        : "memory");
}

// mbarrier arrive that also sets the expected transaction bytes (TMA / bulk copies).
QRM_D void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// 4-D TMA tile load global -> shared, completion on an mbarrier (tx bytes).
QRM_D void tma_load_4d(uint32_t dst_smem, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(dst_smem),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

// 3-D TMA tile load global -> shared, completion on an mbarrier (tx bytes).
QRM_D void tma_load_3d(uint32_t dst_smem, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst_smem),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// TMA tensor store shared -> global (bulk-group completion).
QRM_D void tma_store_2d(const void* tmap, uint32_t src_smem, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
                 "r"(src_smem), "r"(c0), "r"(c1)
                 : "memory");
}
QRM_D void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until at most N committed bulk groups still READ their shared source.
template <int N>
QRM_D void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
QRM_D void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
QRM_D void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Contiguous bulk copy global -> shared (bytes % 16 == 0), completion on an mbarrier.
QRM_D void bulk_load(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One elected lane of a converged warp (elect.sync).
QRM_D bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t.reg .b32 r;\n\t"
        "elect.sync r|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// Arrive (once) on an mbarrier when all previously issued tcgen05.mma of this
// thread have completed. Implies tcgen05.fence::before_thread_sync.
QRM_D void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread.
QRM_D void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
QRM_D void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major operand in the 128-byte swizzle
// canonical layout (rows of 128 B, 8-row groups 1024 B apart).
QRM_D uint64_t sw128_kmajor_desc(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);  // start address
    d |= static_cast<uint64_t>(1) << 16;                    // LBO (ignored for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;            // SBO: 8-row group stride
    d |= static_cast<uint64_t>(1) << 46;                    // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;                    // SWIZZLE_128B
    return d;
}

// Instruction descriptor (kind::i8): D s32, A u8, B s8, both K-major.
QRM_HD uint32_t idesc_i8_u8s8(int M, int N) {
    return (2u << 4) | (0u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

// Instruction descriptor (kind::f16): D f32, A bf16, B bf16, both K-major.
QRM_HD uint32_t idesc_bf16_f32(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

// Instruction descriptor (kind::tf32): D f32, A tf32, B tf32, both K-major.
QRM_HD uint32_t idesc_tf32_f32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

// ------------------------------------------- programmatic dependent launch ----
// The next kernel in the stream may begin launching (its prologue overlaps
// this kernel's tail); it must griddep_wait() before touching our outputs.
QRM_D void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Wait until the previous kernel in the stream has completed and its writes
// are visible (a no-op when this kernel was not launched with PDL).
QRM_D void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ----------------------------------------------------------- clusters ----
QRM_D uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
QRM_D uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// Full cluster barrier: writes before it (incl. DSMEM stores) are visible after it.
QRM_D void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Split cluster barrier (a thread may do work between its arrive and its wait).
QRM_D void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
QRM_D void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// Address of the same shared-memory offset in CTA `rank` of the cluster.
QRM_D uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}
QRM_D void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}


// -------------------------------------------------- CTA pair (cta_group::2) ----
// Both CTAs of the pair execute alloc/dealloc from the same warp; the column
// range is mirrored in the two TMEMs.
template <uint32_t kCols>
QRM_D void tmem_alloc_pair(uint32_t* dst_smem_slot) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem_slot)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
QRM_D void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
// D[256 x N] (+)= A[256 x K] * B[K x N] over the pair (issued by the even CTA):
// A rows 0-127 / 128-255 and B columns 0..N/2-1 / N/2..N-1 come from the same
// smem offsets of CTA 0 / CTA 1; D rows land in each CTA's own TMEM. Eight
// 32-lane disable masks cover the 256 output rows.
QRM_D void umma_bf16_pair_masked(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc,
                                 uint32_t accumulate, uint32_t m0, uint32_t m1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %6, %5, %6, %5, %6, %5, %6}, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate), "r"(m0), "r"(m1)
        : "memory");
}
// Commit of the pair's MMAs, arriving once on the barrier at this smem offset
// in every CTA of `mask`.
QRM_D void umma_commit_pair_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// Arrive on an mbarrier of another CTA of the cluster (address from map_to_rank).
// Default semantics (.release at CTA scope), as CUTLASS's ClusterBarrier does:
// a .release.cluster arrive waits for all of the thread's outstanding writes
// (the epilogue's output stores) to reach cluster scope, and measured as half
// of the pair kernel's warp stalls. The barriers only order TMEM/smem reuse,
// which tcgen05.wait::ld / the fences before the arrive already cover.
QRM_D void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
QRM_D void mbar_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr), "r"(bytes)
                 : "memory");
}
// 4-D TMA load into this CTA's smem whose completion is signalled on a barrier
// of either CTA of the pair (cluster address).
QRM_D void tma_load_4d_pair(uint32_t dst_smem, const void* tmap, int c0, int c1, int c2, int c3, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4, %5}], [%6];" ::"r"(dst_smem),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_cluster)
        : "memory");
}

// Byte offset of 16-byte chunk `c` of row `r` inside a 128B-swizzled K-major tile.
QRM_HD uint32_t sw128_offset(uint32_t r, uint32_t c) { return r * 128u + ((c ^ (r & 7u)) << 4); }
#endif  // __CUDACC__

}  // namespace qrm
