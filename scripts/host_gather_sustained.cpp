// Sustained host window-gather rate (the CPU half of host-pipeline modes 2/3):
// T threads copy 64 x 192-B rows per image out of a 16,384-image pool into a
// staging buffer, repeatedly for ~2 s; prints GB/s of windows per T.
//   g++ -O3 -std=c++17 -pthread scripts/host_gather_sustained.cpp -o /tmp/hgs && /tmp/hgs
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
    const int n = 16384, IMG = 256 * 256 * 3, K = 12288, B = 4096;
    std::vector<uint8_t> pool(static_cast<size_t>(n) * IMG, 1), stage(static_cast<size_t>(B) * K);
    for (int T : {1, 4, 8, 12, 16}) {
        auto t0 = std::chrono::steady_clock::now();
        double secs = 0;
        long batches = 0;
        while (secs < 2.0) {
            std::vector<std::thread> th;
            const long b0 = batches;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    for (int i = t; i < B; i += T) {
                        const int img = static_cast<int>((b0 * B + i) % n);
                        const uint8_t* s = pool.data() + static_cast<size_t>(img) * IMG + ((i * 7) % 4) * 64 * 768 + ((i * 13) % 4) * 192;
                        for (int r = 0; r < 64; ++r) std::memcpy(stage.data() + static_cast<size_t>(i) * K + r * 192, s + r * 768, 192);
                    }
                });
            for (auto& x : th) x.join();
            ++batches;
            secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        printf("{\"threads\": %d, \"batches\": %ld, \"GBps\": %.2f, \"windows_per_s\": %.0f}\n", T, batches,
               batches * static_cast<double>(B) * K / secs / 1e9, batches * static_cast<double>(B) / secs);
    }
}
