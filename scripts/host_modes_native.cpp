// qrm_detect_host throughput per transfer mode from a plain C++ process (no
// Python / torch): pinned 16,384-image pool, batch 4096, plan [1,1,1] x 4096.
//   g++ -O2 -std=c++17 scripts/host_modes_native.cpp -Iinclude -Lpaper_2509_02447_b200/_lib -lqrmark_b200 \
//       -Wl,-rpath,$PWD/paper_2509_02447_b200/_lib -L/usr/local/cuda/lib64 -lcudart -o /tmp/hmn
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include "qrmark_gpu.h"
int main(int argc, char** argv) {
    const int n = 16384, B = 4096, W = 256, H = 256;
    const size_t img = static_cast<size_t>(W) * H * 3;
    uint8_t* pool = nullptr;
    cudaHostAlloc(&pool, n * img, cudaHostAllocMapped);
    for (size_t i = 0; i < n * img; ++i) pool[i] = static_cast<uint8_t>(i * 2654435761u >> 13);
    std::vector<uint8_t> msg(48, 1);
    qrm_config cfg{4, 15, 12, 64, QRM_TILE_RANDOM_GRID, 0, 1, 0.04, msg.data(), 1e-6};
    qrm_ctx* ctx = nullptr;
    if (qrm_ctx_create(0, &cfg, &ctx) != QRM_OK) { printf("ctx fail %s\n", qrm_last_error()); return 1; }
    qrm_record* out = nullptr;
    cudaHostAlloc(&out, sizeof(qrm_record) * B, cudaHostAllocDefault);
    qrm_plan plan{{1, 1, 1}, {B, B, B}};
    {   // raw H2D of a freshly written pinned buffer, before and after the library's calls
        uint8_t *hs, *d;
        cudaHostAlloc(&hs, B * 12288ull, cudaHostAllocDefault);
        cudaMalloc(&d, B * 12288ull);
        cudaStream_t st;
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto raw = [&](const char* tag) {
            memset(hs, 3, B * 12288ull);
            cudaEventRecord(e0, st);
            cudaMemcpyAsync(d, hs, B * 12288ull, cudaMemcpyHostToDevice, st);
            cudaEventRecord(e1, st);
            cudaStreamSynchronize(st);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"raw_h2d\": \"%s\", \"ms\": %.3f}\n", tag, ms);
        };
        raw("after ctx create");
        raw("after ctx create");
        for (int i = 0; i < 2; ++i) qrm_detect_host(ctx, pool, B, W, H, img, 0, out, &plan, 2, nullptr);
        raw("after mode 2 calls");
        raw("after mode 2 calls");
    }
    const double fracs[] = {0.0, 0.0, 0.4, 0.5, 0.6, 0.7};
    const int modes[] = {0, 2, 3, 3, 3, 3};
    for (int mi = 0; mi < 6; ++mi) {
        const int mode = modes[mi];
        if (mode == 3) qrm_ctx_set_transfer_split(ctx, fracs[mi]);
        for (int i = 0; i < 3; ++i) qrm_detect_host(ctx, pool + (i % 4) * B * img, B, W, H, img, i * B, out, &plan, mode, nullptr);
        const int reps = 12;
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < reps; ++i)
            if (qrm_detect_host(ctx, pool + (i % 4) * B * img, B, W, H, img, i * B, out, &plan, mode, nullptr) != QRM_OK) {
                printf("fail %s\n", qrm_last_error());
                return 1;
            }
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("{\"mode\": %d, \"frac\": %.1f, \"img_per_s\": %.0f}\n", mode, fracs[mi], reps * static_cast<double>(B) / s);
    }
    qrm_ctx_destroy(ctx);
}
