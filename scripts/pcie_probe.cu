// PCIe probe: how fast can the tile windows of a pinned host batch reach the
// device? (copy engine vs zero-copy kernel reads at several granularities)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_probe scripts/pcie_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
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
    return 0;
}
