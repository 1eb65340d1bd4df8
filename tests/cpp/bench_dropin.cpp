// End-to-end throughput of the C++ drop-in: qrmark::detect_batch over a
// std::vector<ImageBuffer> (detect.hpp:145-149), the call a user of the
// reference makes, at BASELINE configs[1] (256x256, batch 4096, defaults of
// cli.cpp:55-65). Every image is its own pageable ImageBuffer; each call builds
// its DetectionContext (as the reference does), gathers only the tile windows
// into the context's pinned staging ring, decodes on the GPU and returns
// DetectionRecords with the CorrectionCache hit flags.
//
//   bench_dropin <raw u8 file: N x H x W x 3> N W H steps warmup
//
// Prints one JSON object: images/s over the timed calls (host wall clock around
// each detect_batch; results are on the host when it returns), per-call ms,
// the DeskReport of the last call and the verified count of the last call.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "qrmark/detect.hpp"
#include "qrmark/rng.hpp"
#include "qrmark/rs.hpp"

using namespace qrmark;

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: %s raw N W H steps warmup\n", argv[0]);
        return 2;
    }
    const char* path = argv[1];
    const long n = std::atol(argv[2]);
    const int w = std::atoi(argv[3]), h = std::atoi(argv[4]);
    const int steps = std::atoi(argv[5]), warmup = std::atoi(argv[6]);
    std::vector<ImageBuffer> images;
    images.reserve(n);
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        std::perror(path);
        return 2;
    }
    for (long i = 0; i < n; ++i) {
        images.push_back(ImageBuffer::make_byte(w, h));
        if (std::fread(images.back().bytes.data(), 1, images.back().bytes.size(), f) != images.back().bytes.size()) {
            std::fprintf(stderr, "short read\n");
            return 2;
        }
    }
    std::fclose(f);
    // DetectionConfig of cmd_detect / cmd_bench with the defaults (cli.cpp:47-65)
    CodeParams code = resolve_profile("gf16-15-12");
    BitVec msg(code.message_bits());
    for (int i = 0; i < code.message_bits(); ++i) msg[i] = rng_word(1, 0x6d73, i) & 1;
    DetectionConfig cfg = DetectionConfig::make(code, TileSpec{64, TileStrategy::random_grid, 0}, 1, 0.04, msg);

    DeskReport rep;
    std::vector<DetectionRecord> recs;
    for (int i = 0; i < warmup; ++i) recs = detect_batch(images, cfg, nullptr, nullptr, &rep);
    std::vector<double> ms;
    for (int i = 0; i < steps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        recs = detect_batch(images, cfg, nullptr, nullptr, &rep);
        ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    double total = 0.0;
    for (double v : ms) total += v;
    long verified = 0;
    for (const auto& r : recs) verified += r.verified;
    std::vector<double> sorted = ms;
    std::sort(sorted.begin(), sorted.end());
    std::printf("{\"images_per_s\": %.1f, \"ms_per_call_mean\": %.4f, \"ms_per_call_median\": %.4f, "
                "\"calls\": %d, \"images_per_call\": %ld, \"verified_last\": %ld, "
                "\"desk_report_last\": {\"wall_ns\": %lld, \"stage_busy_ns\": [%lld, %lld, %lld], "
                "\"stage_workers\": [%d, %d, %d]}}\n",
                static_cast<double>(n) * steps / (total / 1e3), total / steps, sorted[sorted.size() / 2], steps, n,
                verified, static_cast<long long>(rep.wall_ns), static_cast<long long>(rep.stage_busy_ns[0]),
                static_cast<long long>(rep.stage_busy_ns[1]), static_cast<long long>(rep.stage_busy_ns[2]),
                rep.stage_workers[0], rep.stage_workers[1], rep.stage_workers[2]);
    return 0;
}
