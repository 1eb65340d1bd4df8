// Host pipeline mode 2/3 probe: CPU gather of 4,096 windows into pinned
// staging, then one H2D of the staging buffer. Times the H2D right after a
// gather (dirty CPU cache lines) with regular vs non-temporal (streaming)
// stores, and the H2D of an idle buffer.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/scp scripts/stage_copy_probe.cu
#include <cuda_runtime.h>
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static void gather(const uint8_t* pool, uint8_t* stage, int B, int T, bool nt, long rot) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([=] {
            for (int i = t; i < B; i += T) {
                const int img = static_cast<int>((rot * B + i) % 16384);
                const uint8_t* s = pool + static_cast<size_t>(img) * 196608 + ((i * 7) % 4) * 64 * 768 + ((i * 13) % 4) * 192;
                uint8_t* d = stage + static_cast<size_t>(i) * 12288;
                for (int r = 0; r < 64; ++r) {
                    if (nt) {
                        const __m128i* src = reinterpret_cast<const __m128i*>(s + r * 768);
                        __m128i* dst = reinterpret_cast<__m128i*>(d + r * 192);
                        for (int k = 0; k < 12; ++k) _mm_stream_si128(dst + k, _mm_loadu_si128(src + k));
                    } else {
                        std::memcpy(d + r * 192, s + r * 768, 192);
                    }
                }
            }
            if (nt) _mm_sfence();
        });
    for (auto& x : th) x.join();
}
int main() {
    const int B = 4096;
    uint8_t *pool, *stage, *dst;
    cudaHostAlloc(&pool, 16384ull * 196608, cudaHostAllocMapped);
    memset(pool, 1, 16384ull * 196608);
    cudaHostAlloc(&stage, static_cast<size_t>(B) * 12288, cudaHostAllocDefault);
    memset(stage, 0, static_cast<size_t>(B) * 12288);
    cudaMalloc(&dst, static_cast<size_t>(B) * 12288);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int variant = 0; variant < 3; ++variant) {
        double gsum = 0, csum = 0;
        const int reps = 20;
        for (int r = 0; r < reps; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            if (variant < 2) gather(pool, stage, B, 16, variant == 1, r);
            gsum += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            cudaEventRecord(e0, st);
            cudaMemcpyAsync(dst, stage, static_cast<size_t>(B) * 12288, cudaMemcpyHostToDevice, st);
            cudaEventRecord(e1, st);
            cudaStreamSynchronize(st);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            csum += ms;
        }
        const char* name[] = {"gather_memcpy_then_h2d", "gather_stream_stores_then_h2d", "h2d_only"};
        printf("{\"probe\": \"%s\", \"gather_ms\": %.3f, \"h2d_ms\": %.3f, \"h2d_GBps\": %.2f}\n", name[variant],
               gsum / reps, csum / reps, B * 12288.0 / (csum / reps) / 1e6);
    }
}
