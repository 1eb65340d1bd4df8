// PCIe probe: how fast can the tile windows of a pinned host batch reach the
// device? (copy engine vs zero-copy kernel reads at several granularities)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_probe scripts/pcie_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <thread>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

constexpr int W = 256, H = 256, L = 64, ROWB = 3 * L, PITCH = 3 * W, IMG = W * H * 3, K = 3 * L * L;

// one 16-B chunk per thread: rows of 12 chunks; NB rows per thread in flight
template <int NB>
__global__ void gather16(const uint8_t* __restrict__ host, const int* __restrict__ org, int count, uint8_t* __restrict__ dst) {
    const int64_t total = static_cast<int64_t>(count) * L * 12;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; base < total; base += stride * NB) {
        uint4 v[NB];
        int64_t idx[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            idx[j] = base + j * stride;
            if (idx[j] < total) {
                const int64_t img = idx[j] / (L * 12);
                const int r = static_cast<int>((idx[j] / 12) % L), c = static_cast<int>(idx[j] % 12);
                const uint8_t* s = host + img * IMG + static_cast<int64_t>(org[2 * img + 1] + r) * PITCH + org[2 * img] * 3 + c * 16;
                v[j] = *reinterpret_cast<const uint4*>(s);
            }
        }
#pragma unroll
        for (int j = 0; j < NB; ++j)
            if (idx[j] < total) {
                const int64_t img = idx[j] / (L * 12);
                const int r = static_cast<int>((idx[j] / 12) % L), c = static_cast<int>(idx[j] % 12);
                *reinterpret_cast<uint4*>(dst + img * K + r * ROWB + c * 16) = v[j];
            }
    }
}

// warp per window row-group: lanes read whole aligned 128-B lines covering the row (over-read)
__global__ void gather_lines(const uint8_t* __restrict__ host, const int* __restrict__ org, int count, uint8_t* __restrict__ dst) {
    // each warp: 2 rows; each row 192 B at 64-B alignment -> covered by 256 B (2 lines) -> 16 lanes x 16 B
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); w < static_cast<int64_t>(count) * L / 2; w += warps) {
        const int64_t img = w / (L / 2);
        const int r = static_cast<int>(w % (L / 2)) * 2 + (lane >> 4);
        const int64_t rowoff = static_cast<int64_t>(org[2 * img + 1] + r) * PITCH + org[2 * img] * 3;
        const int64_t aligned = rowoff & ~int64_t(127);
        const int shift = static_cast<int>(rowoff - aligned);  // 0 or 64
        const int c = lane & 15;
        const uint4 v = *reinterpret_cast<const uint4*>(host + img * IMG + aligned + c * 16);
        const int pos = c * 16 - shift;
        if (pos >= 0 && pos < ROWB) *reinterpret_cast<uint4*>(dst + img * K + r * ROWB + pos) = v;
    }
}

__global__ void seq_read(const uint4* __restrict__ host, int64_t n16, uint4* __restrict__ dst) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = host[i];
}


// TMA bulk copies (cp.async.bulk global->shared) of whole 192-B window rows
// straight from mapped host memory, then to HBM: one warp per image.
__global__ void gather_bulk(const uint8_t* __restrict__ host, const int* __restrict__ org, int count, uint8_t* __restrict__ dst) {
    __shared__ __align__(128) uint8_t buf[3][K];
    __shared__ __align__(8) uint64_t bar[3];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t phase = 0;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[w])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    for (int64_t img = blockIdx.x * 3 + w; img < count; img += gridDim.x * 3) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[w]);
        if (lane == 0)
            asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(b), "r"(K) : "memory");
        __syncwarp();
        for (int r = lane; r < L; r += 32) {
            const uint8_t* s = host + img * IMG + static_cast<int64_t>(org[2 * img + 1] + r) * PITCH + org[2 * img] * 3;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&buf[w][r * ROWB])), "l"(s), "r"(ROWB), "r"(b) : "memory");
        }
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(b), "r"(phase) : "memory");
        phase ^= 1;
        const uint4* src = reinterpret_cast<const uint4*>(buf[w]);
        uint4* d = reinterpret_cast<uint4*>(dst + img * K);
        for (int i = lane; i < K / 16; i += 32) d[i] = src[i];
        __syncwarp();
    }
}

// zero-copy reads of the 64 FULL rows holding the window (contiguous 48 KB per image)
__global__ void rowblock_read(const uint4* __restrict__ host, const int* __restrict__ org, int count, uint4* __restrict__ dst) {
    const int64_t per = static_cast<int64_t>(L) * PITCH / 16;
    const int64_t total = per * count;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t img = i / per, j = i % per;
        dst[(i / 3) % (static_cast<int64_t>(count) * K / 16)] = host[(img * IMG + static_cast<int64_t>(org[2 * img + 1]) * PITCH) / 16 + j];
    }
}

int main() {
    const int count = 4096;
    uint8_t* h = nullptr;
    CK(cudaHostAlloc(&h, static_cast<size_t>(count) * IMG, cudaHostAllocMapped));
    for (size_t i = 0; i < static_cast<size_t>(count) * IMG; i += 4096) h[i] = static_cast<uint8_t>(i);
    std::vector<int> org(2 * count);
    for (int i = 0; i < count; ++i) {
        org[2 * i] = ((i * 7) % 4) * 64;
        org[2 * i + 1] = ((i * 13) % 4) * 64;
    }
    int* dorg;
    uint8_t *dst, *dimgs, *dh;
    CK(cudaMalloc(&dorg, sizeof(int) * 2 * count));
    CK(cudaMemcpy(dorg, org.data(), sizeof(int) * 2 * count, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dst, static_cast<size_t>(count) * K));
    CK(cudaMalloc(&dimgs, static_cast<size_t>(count) * IMG));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dh), h, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, double bytes, auto fn) {
        for (int i = 0; i < 2; ++i) fn();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        const int reps = 5;
        for (int i = 0; i < reps; ++i) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        printf("{\"probe\": \"%s\", \"ms\": %.4f, \"GBps\": %.2f, \"images_per_s\": %.0f}\n", name, ms, bytes / ms / 1e6,
               count / ms * 1e3);
        fflush(stdout);
    };
    const double wbytes = static_cast<double>(count) * K;
    timeit("memcpy_h2d_windows_size(50MB contiguous)", wbytes, [&] { cudaMemcpyAsync(dst, h, count * static_cast<size_t>(K), cudaMemcpyHostToDevice); });
    timeit("memcpy_h2d_full_images(805MB)", static_cast<double>(count) * IMG,
           [&] { cudaMemcpyAsync(dimgs, h, static_cast<size_t>(count) * IMG, cudaMemcpyHostToDevice); });
    timeit("zero_copy_seq_read(50MB)", wbytes, [&] { seq_read<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(dh), count * static_cast<int64_t>(K) / 16, reinterpret_cast<uint4*>(dst)); });
    timeit("gather16_nb1", wbytes, [&] { gather16<1><<<148 * 8, 256>>>(dh, dorg, count, dst); });
    timeit("gather16_nb4", wbytes, [&] { gather16<4><<<148 * 8, 256>>>(dh, dorg, count, dst); });
    timeit("gather16_nb8_g4", wbytes, [&] { gather16<8><<<148 * 4, 256>>>(dh, dorg, count, dst); });
    timeit("gather_lines(256B per 192B row)", wbytes, [&] { gather_lines<<<148 * 8, 256>>>(dh, dorg, count, dst); });
    timeit("gather_bulk(TMA 192B rows from host)", wbytes, [&] { gather_bulk<<<148 * 2, 96>>>(dh, dorg, count, dst); });
    timeit("gather_bulk_g8", wbytes, [&] { gather_bulk<<<148 * 6, 96>>>(dh, dorg, count, dst); });
    timeit("rowblock_zero_copy(48KB/img read)", wbytes, [&] { rowblock_read<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(dh), dorg, count, reinterpret_cast<uint4*>(dst)); });
    {   // copy engine: one contiguous 48-KB row block per image (4x the window bytes)
        uint8_t* drows;
        CK(cudaMalloc(&drows, static_cast<size_t>(count) * L * PITCH));
        timeit("memcpy_rowblocks_4096_calls", wbytes, [&] {
            for (int i = 0; i < count; ++i)
                cudaMemcpyAsync(drows + static_cast<size_t>(i) * L * PITCH, h + static_cast<size_t>(i) * IMG + static_cast<size_t>(org[2 * i + 1]) * PITCH,
                                static_cast<size_t>(L) * PITCH, cudaMemcpyHostToDevice);
        });
        timeit("memcpy2d_windows_4096_calls", wbytes, [&] {
            for (int i = 0; i < count; ++i)
                cudaMemcpy2DAsync(dst + static_cast<size_t>(i) * K, ROWB, h + static_cast<size_t>(i) * IMG + static_cast<size_t>(org[2 * i + 1]) * PITCH + org[2 * i] * 3,
                                  PITCH, ROWB, L, cudaMemcpyHostToDevice);
        });
#if CUDART_VERSION >= 12080
        std::vector<void*> dsts(count), srcs(count);
        std::vector<size_t> sizes(count, static_cast<size_t>(L) * PITCH);
        for (int i = 0; i < count; ++i) {
            dsts[i] = drows + static_cast<size_t>(i) * L * PITCH;
            srcs[i] = h + static_cast<size_t>(i) * IMG + static_cast<size_t>(org[2 * i + 1]) * PITCH;
        }
        cudaMemcpyAttributes attr{};
        attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        attr.srcLocHint.type = cudaMemLocationTypeHost;
        attr.dstLocHint.type = cudaMemLocationTypeDevice;
        size_t ai = 0, fail = 0;
        timeit("memcpy_batch_rowblocks", wbytes, [&] {
            cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), count, &attr, &ai, 1, &fail, 0);
        });
        printf("batch fail idx %zu err %s\n", fail, cudaGetErrorString(cudaGetLastError()));
#endif
    }
    {   // host gather into pinned staging with T threads, then one H2D
        uint8_t* stage;
        CK(cudaHostAlloc(&stage, static_cast<size_t>(count) * K, cudaHostAllocDefault));
        unsigned hc = std::thread::hardware_concurrency();
        printf("{\"host_threads\": %u}\n", hc);
        for (unsigned T : {1u, 2u, 4u, 8u, 16u, 32u}) {
            if (T > 2 * hc) break;
            auto gather = [&](int t) {
                for (int i = t; i < count; i += T) {
                    const uint8_t* s = h + static_cast<size_t>(i) * IMG + static_cast<size_t>(org[2 * i + 1]) * PITCH + org[2 * i] * 3;
                    uint8_t* d = stage + static_cast<size_t>(i) * K;
                    for (int r = 0; r < L; ++r) memcpy(d + r * ROWB, s + static_cast<size_t>(r) * PITCH, ROWB);
                }
            };
            double best = 1e30;
            for (int rep = 0; rep < 5; ++rep) {
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> th;
                for (unsigned t = 0; t < T; ++t) th.emplace_back(gather, t);
                for (auto& x : th) x.join();
                double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                if (ms < best) best = ms;
            }
            printf("{\"probe\": \"host_gather_T%u\", \"ms\": %.4f, \"GBps\": %.2f, \"images_per_s\": %.0f}\n", T, best, wbytes / best / 1e6, count / best * 1e3);
        }
        timeit("memcpy_h2d_staged_windows", wbytes, [&] { cudaMemcpyAsync(dst, stage, count * static_cast<size_t>(K), cudaMemcpyHostToDevice); });
    }
    {   // hybrid: half the windows by zero-copy gather, half by DMA of a pre-gathered pinned buffer, concurrently
        uint8_t* stage2;
        CK(cudaHostAlloc(&stage2, static_cast<size_t>(count) * K, cudaHostAllocDefault));
        cudaStream_t s1, s2;
        CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        for (double frac : {0.5, 0.6, 0.7, 0.8}) {
            const int na = static_cast<int>(count * frac);
            char name[64];
            snprintf(name, sizeof name, "hybrid_zero_copy_%.1f_plus_dma", frac);
            timeit(name, wbytes, [&] {
                gather16<4><<<148 * 2, 256, 0, s1>>>(dh, dorg, na, dst);
                cudaMemcpyAsync(dst + static_cast<size_t>(na) * K, stage2 + static_cast<size_t>(na) * K,
                                static_cast<size_t>(count - na) * K, cudaMemcpyHostToDevice, s2);
                cudaStreamSynchronize(s1);
                cudaStreamSynchronize(s2);
            });
        }
    }
    {   // device-resident images: how fast can the window gather pattern stream from HBM?
        const int dcount = 16384;
        uint8_t *dpool, *dwin;
        int* dorg2;
        CK(cudaMalloc(&dpool, static_cast<size_t>(dcount) * IMG));
        CK(cudaMemset(dpool, 1, static_cast<size_t>(dcount) * IMG));
        CK(cudaMalloc(&dwin, static_cast<size_t>(dcount) * K));
        std::vector<int> org2(2 * dcount);
        for (int i = 0; i < dcount; ++i) {
            org2[2 * i] = ((i * 7) % 4) * 64;
            org2[2 * i + 1] = ((i * 13) % 4) * 64;
        }
        CK(cudaMalloc(&dorg2, sizeof(int) * 2 * dcount));
        CK(cudaMemcpy(dorg2, org2.data(), sizeof(int) * 2 * dcount, cudaMemcpyHostToDevice));
        for (int n : {4096, 16384}) {
            const double wb = static_cast<double>(n) * K;
            char name[64];
            snprintf(name, sizeof name, "hbm_gather16_nb4_%d", n);
            timeit(name, wb, [&] { gather16<4><<<148 * 8, 256>>>(dpool, dorg2, n, dwin); });
            snprintf(name, sizeof name, "hbm_gather_lines_%d", n);
            timeit(name, wb, [&] { gather_lines<<<148 * 8, 256>>>(dpool, dorg2, n, dwin); });
            snprintf(name, sizeof name, "hbm_seq_copy_%d", n);
            timeit(name, wb, [&] { seq_read<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(dpool) + (n * static_cast<int64_t>(K) / 16), n * static_cast<int64_t>(K) / 16, reinterpret_cast<uint4*>(dwin)); });
        }
    }
    return 0;
}
