// C++ tests of the drop-in API (include/qrmark/*.hpp over libqrmark_b200.so).
// The cases mirror the reference's own suites (proj/tests/test_gf.cpp,
// test_rs.cpp, test_image.cpp) and the SPEC examples for tiling, stego,
// detect and sched, so a caller of the reference API sees the same behaviour.
//
//   test_dropin host   — host-side API (no GPU needed)
//   test_dropin gpu    — GPU-backed API (bw_decode, preprocess, extract, detect)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>

#include "qrmark/detect.hpp"
#include "qrmark/gf.hpp"
#include "qrmark/image.hpp"
#include "qrmark/rng.hpp"
#include "qrmark/rs.hpp"
#include "qrmark/sched.hpp"
#include "qrmark/sim.hpp"
#include "qrmark/stego.hpp"
#include "qrmark/tiling.hpp"
#include "qrmark/transforms.hpp"
#include "qrmark_gpu.h"

using namespace qrmark;

static int g_checks = 0, g_fail = 0;
#define CHECK(x)                                                          \
    do {                                                                  \
        ++g_checks;                                                       \
        if (!(x)) {                                                       \
            ++g_fail;                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);      \
        }                                                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                          \
    do {                                                                  \
        ++g_checks;                                                       \
        bool ok_ = false;                                                 \
        try {                                                             \
            (void)(expr);                                                 \
        } catch (const T&) {                                              \
            ok_ = true;                                                   \
        } catch (...) {                                                   \
        }                                                                 \
        if (!ok_) {                                                       \
            ++g_fail;                                                     \
            std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
        }                                                                 \
    } while (0)

static uint16_t clmul_mod(uint16_t a, uint16_t b, uint32_t poly, int m) {
    uint32_t acc = 0;
    for (int i = 0; i < m; ++i)
        if ((b >> i) & 1) acc ^= static_cast<uint32_t>(a) << i;
    for (int d = 2 * m - 2; d >= m; --d)
        if ((acc >> d) & 1) acc ^= poly << (d - m);
    return static_cast<uint16_t>(acc);
}

static BitVec random_bits(CounterRng& rng, size_t n) {
    BitVec b(n);
    for (auto& v : b) v = rng.next() & 1;
    return b;
}

// ------------------------------------------------------------------ host
static void host_gf() {
    const FieldSpec& f = FieldSpec::gf16();
    for (uint16_t a = 0; a < 16; ++a)
        for (uint16_t b = 0; b < 16; ++b) CHECK(f.mul(a, b) == clmul_mod(a, b, f.primitive_poly(), 4));
    for (uint16_t a = 1; a < 16; ++a) CHECK(f.mul(a, f.inv(a)) == 1);
    CHECK_THROWS_AS(f.inv(0), DivisionByZero);
    CHECK_THROWS_AS(f.div(3, 0), DivisionByZero);
    CHECK_THROWS_AS(f.mul(16, 1), InvalidInput);
    const FieldSpec& g = FieldSpec::gf256();
    CounterRng rng(5, 0);
    for (int i = 0; i < 10000; ++i) {
        uint16_t a = rng.below(256), b = rng.below(256), c = rng.below(256);
        CHECK(g.mul(a, b) == clmul_mod(a, b, 0x11d, 8));
        CHECK(g.mul(a, g.add(b, c)) == g.add(g.mul(a, b), g.mul(a, c)));
    }
    std::set<uint16_t> seen;
    for (int i = 0; i < 255; ++i) seen.insert(g.alpha_pow(i));
    CHECK(seen.size() == 255);
    CHECK(g.pow(2, 255) == 1);
    // Poly: divmod identity and Lagrange evaluate-back
    Poly num(g, {3, 7, 0, 9, 200}), den(g, {5, 1});
    auto [q, r] = Poly::divmod(num, den);
    CHECK(q * den + r == num);
    CHECK(r.degree() < den.degree());
    CHECK_THROWS_AS(Poly::divmod(num, Poly::zero(g)), DivisionByZero);
    std::vector<std::pair<uint16_t, uint16_t>> pts = {{1, 9}, {2, 4}, {4, 77}, {8, 0}};
    Poly p = lagrange_interpolate(g, pts);
    for (auto [x, y] : pts) CHECK(p.eval(x) == y);
    std::vector<std::pair<uint16_t, uint16_t>> dup = {{1, 9}, {1, 4}};
    CHECK_THROWS_AS(lagrange_interpolate(g, dup), InvalidInput);
    FieldElement e1(3, f), e2(5, g);
    CHECK_THROWS_AS(e1 + e2, InvalidInput);
}

static void host_rs_encode() {
    BitVec bits = {0, 1, 0, 1, 1, 1, 1, 0};
    auto sym = bits_to_symbols(bits, 4);
    CHECK(sym.size() == 2 && sym[0] == 0x5 && sym[1] == 0xe);
    CHECK(symbols_to_bits(sym, 4) == bits);
    CHECK(bits_to_hex(bits) == "5e");
    CHECK(hex_to_bits("5e", 8) == bits);
    CHECK_THROWS_AS(hex_to_bits("5e", 12), InvalidInput);
    CodeParams g16 = resolve_profile("gf16-15-12");
    CHECK(g16.n == 15 && g16.k == 12 && g16.t == 1 && g16.message_bits() == 48 && g16.codeword_bits() == 60);
    CodeParams g256 = resolve_profile("gf256-dynamic", 48);
    CHECK(g256.field->bits() == 8 && g256.k == 6 && g256.n == 8 && g256.t == 1);
    CHECK_THROWS_AS(resolve_profile("nope"), InvalidInput);
    CHECK_THROWS_AS(resolve_profile("gf256-dynamic", 42), InvalidInput);
    CHECK_THROWS_AS(CodeParams::make(FieldSpec::gf16(), 16, 12), InvalidInput);
    CHECK(rs_encode(BitVec(48, 0), g16) == BitVec(60, 0));
    CounterRng rng(21, 0);
    for (int i = 0; i < 50; ++i) {
        BitVec m = random_bits(rng, 48);
        BitVec w = rs_encode(m, g16);
        CHECK(w.size() == 60);
        CHECK(BitVec(w.begin(), w.begin() + 48) == m);
    }
    CHECK_THROWS_AS(rs_encode(BitVec(47, 0), g16), InvalidInput);
    // the key message and codeword of the reference defaults
    BitVec msg(48);
    for (int i = 0; i < 48; ++i) msg[i] = rng_word(1, 0x6d73, i) & 1;
    CHECK(bits_to_hex(msg) == "b1b8528ad785");
    CHECK(bits_to_hex(rs_encode(msg, g16)) == "b1b8528ad7859a0");
    // rs_aware_loss / accuracies (test_rs.cpp:165-218)
    BitVec a(48, 0), b = a, c = a;
    CHECK(rs_aware_loss(a, a, g16) == 0.0);
    b[0] = 1;
    CHECK(rs_aware_loss(b, a, g16) == 0.0);
    c[0] = c[4] = c[9] = 1;
    CHECK(rs_aware_loss(c, a, g16) == 4.0);
    CHECK(bit_accuracy(a, a) == 1.0);
    CHECK(std::fabs(bit_accuracy(a, b) - 47.0 / 48.0) < 1e-12);
    CHECK(word_accuracy({a, b}, {a, a}) == 0.5);
    CHECK(verify_threshold(48, 1e-6) == 41 && verify_threshold(60, 1e-6) == 49 && verify_threshold(64, 1e-6) == 51);
    CHECK(verify_threshold(48, std::ldexp(1.0, -48)) == 48);
    CHECK(verify(a, a, 1e-6) && !verify(a, BitVec(48, 1), 1e-6));
}

static void host_tiling_sched() {
    CHECK(grid_cells(256, 256, 64).size() == 16);
    CHECK(grid_cells(256, 256, 80).size() == 9);
    CHECK(grid_cells(300, 200, 100).size() == 6);
    CHECK((select_tile(256, 256, TileSpec{64, TileStrategy::fixed, 0}, 9) == TileRef{0, 0, 64}));
    CHECK_THROWS_AS(select_tile(32, 32, TileSpec{64, TileStrategy::random_grid, 0}, 0), InvalidInput);
    int counts[16] = {0};
    for (uint64_t d = 0; d < 100000; ++d) {
        TileRef t = select_tile(256, 256, TileSpec{64, TileStrategy::random_grid, 3}, d);
        CHECK(t.x % 64 == 0 && t.y % 64 == 0);
        counts[(t.y / 64) * 4 + t.x / 64]++;
    }
    for (int c : counts) CHECK(std::abs(c - 6250) < 3 * std::sqrt(6250.0));
    CHECK(parse_tile_strategy("random") == TileStrategy::random);
    CHECK(tile_strategy_name(TileStrategy::random_grid) == "random_grid");
    // Alg.1: budget / memory respected, every stage has a stream
    StageProfile prof;
    prof.b0 = 16;
    prof.time = {5.0, 7.0, 28.0};
    prof.memory = {1000.0, 500.0, 10.0};
    StreamPlan plan = allocate_streams(prof, 256, 16, 1e9, 0.0, 2);
    CHECK(plan.streams.size() == 3 && plan.total_streams() <= 16);
    for (int s : plan.streams) CHECK(s >= 1);
    CHECK(mem_ok(plan.streams, plan.minibatch, prof.memory, 1e9));
    CHECK(plan.bottleneck <= stage_time(prof, 2, 1, plan.minibatch[2]));
    CHECK_THROWS_AS(allocate_streams(prof, 256, 2, 1e9, 0.0, 2), InvalidInput);
    CHECK_THROWS_AS(allocate_streams(prof, 256, 16, 1.0, 0.0, 2), InfeasibleConfig);
    // Alg.2: latency and units conserved, m_unit >= b_min
    std::vector<Task> tasks;
    double total = 0.0;
    for (int i = 0; i < 9; ++i) {
        Task t;
        t.id = i;
        t.latency = 1.0 + i % 4;
        t.memory = 2.0;
        t.units = 3;
        tasks.push_back(t);
        total += t.latency;
    }
    StreamSchedule s = lpt_schedule(tasks, 3, 0.25, 1e9, 1, 64);
    CHECK(std::fabs(s.total_latency() - total) < 1e-9);
    int units = 0;
    for (auto& st : s.streams)
        for (auto& t : st) units += t.units;
    CHECK(units == 27);
    CHECK(s.m_unit >= 1 && s.makespan() <= total);
    // measure_stages with a scripted clock (sim.cpp:214-238)
    int64_t clock = 0;
    std::vector<StageBench> benches = {{"a", [&] { clock += 3000000; }, 10.0, 0.5},
                                       {"b", [&] { clock += 1000000; }, 20.0, 0.0}};
    StageProfile mp = measure_stages(benches, 3, 16.0, [&] { return clock; });
    CHECK(mp.time.size() == 2 && std::fabs(mp.time[0] - 3.0) < 1e-9 && std::fabs(mp.time[1] - 1.0) < 1e-9);
    CHECK(std::fabs(mp.prep[0] - 1.5) < 1e-9 && mp.memory[1] == 20.0 && mp.b0 == 16.0);
}

// ------------------------------------------------------------------- gpu
// CorrectionCache's LRU eviction (detect.cpp:86-128) against the C-ABI's
// replay (qrm_cache_hits, pinned to the reference's own JSON output in
// tests/test_formats.py), with eviction by capacity and by staleness.
static void host_cache() {
    CounterRng rng(31, 0);
    for (auto [cap, stale] : {std::pair<size_t, uint64_t>{4, 1u << 20}, {16, 7}, {3, 2}, {4096, 1u << 20}}) {
        CorrectionCache cache(CacheConfig{true, cap, stale}), packed(CacheConfig{true, cap, stale});
        std::vector<qrm_record> recs(3000);
        std::vector<uint8_t> want(recs.size());
        for (size_t i = 0; i < recs.size(); ++i) {
            // a skewed stream: a few hot words and a long tail
            const uint64_t r = rng.next();
            const uint64_t word = (r & 3) ? (r >> 8) % 9 : (r >> 8) % 400;
            recs[i] = qrm_record{};
            recs[i].raw = word;
        }
        CHECK(qrm_cache_hits(recs.data(), static_cast<int64_t>(recs.size()), static_cast<int64_t>(cap), stale,
                             want.data()) == QRM_OK);
        size_t hits = 0;
        for (size_t i = 0; i < recs.size(); ++i) {
            BitVec raw(60);
            for (int b = 0; b < 60; ++b) raw[b] = (recs[i].raw >> (59 - b)) & 1;
            const bool h = cache.record(raw, std::optional<DecodeResult>{});
            CHECK(h == (want[i] != 0));
            CHECK(packed.record_packed(recs[i].raw, 60, [] { return std::optional<DecodeResult>{}; }) == h);
            hits += h;
        }
        CHECK(cache.hits() == hits && cache.size() <= cap);
        CorrectionCache batch(CacheConfig{true, cap, stale});
        std::vector<uint8_t> bh(recs.size(), 2);
        batch.record_packed_batch(&recs[0].raw, recs.size(), sizeof(qrm_record) / sizeof(uint64_t), 60,
                                  [](size_t) { return std::optional<DecodeResult>{}; }, bh.data());
        CHECK(bh == want && batch.hits() == hits);
    }
}

static void gpu_rs() {
    CounterRng rng(22, 0);
    for (const char* name : {"gf16-15-12", "gf256-dynamic"}) {
        CodeParams p = resolve_profile(name, 48);
        std::vector<BitVec> words, msgs;
        for (int i = 0; i < 200; ++i) {
            msgs.push_back(random_bits(rng, p.message_bits()));
            words.push_back(rs_encode(msgs.back(), p));
        }
        auto res = bw_decode_batch(words, p);
        for (int i = 0; i < 200; ++i) {
            CHECK(res[i].has_value());
            if (res[i]) CHECK(res[i]->message == msgs[i] && res[i]->codeword == words[i] && res[i]->errors_corrected == 0);
        }
    }
    // exhaustive single-symbol corruption (test_rs.cpp:93-114)
    CodeParams p = resolve_profile("gf16-15-12");
    CounterRng r23(23, 0);
    for (int trial = 0; trial < 10; ++trial) {
        BitVec msg = random_bits(r23, 48);
        auto sym = bits_to_symbols(rs_encode(msg, p), 4);
        std::vector<BitVec> bad;
        for (int pos = 0; pos < 15; ++pos)
            for (uint16_t wrong = 0; wrong < 16; ++wrong)
                if (wrong != sym[pos]) {
                    auto c = sym;
                    c[pos] = wrong;
                    bad.push_back(symbols_to_bits(c, 4));
                }
        auto res = bw_decode_batch(bad, p);
        for (auto& r : res) CHECK(r && r->message == msg && r->errors_corrected == 1);
    }
    // t = 2 (test_rs.cpp:116-134)
    CodeParams p2 = CodeParams::make(FieldSpec::gf256(), 12, 8);
    CounterRng r24(24, 0);
    for (int trial = 0; trial < 150; ++trial) {
        BitVec msg = random_bits(r24, 64);
        auto s = bits_to_symbols(rs_encode(msg, p2), 8);
        int a = r24.below(12), b = r24.below(12);
        while (b == a) b = r24.below(12);
        s[a] ^= 1 + r24.below(255);
        s[b] ^= 1 + r24.below(255);
        auto r = bw_decode(symbols_to_bits(s, 8), p2);
        CHECK(r && r->message == msg && r->errors_corrected == 2);
    }
    // beyond capacity never silently passes (test_rs.cpp:136-163)
    CounterRng r25(25, 0);
    int failures = 0;
    for (int trial = 0; trial < 300; ++trial) {
        BitVec msg = random_bits(r25, 48);
        auto s = bits_to_symbols(rs_encode(msg, p), 4);
        int q[3];
        q[0] = r25.below(15);
        do q[1] = r25.below(15);
        while (q[1] == q[0]);
        do q[2] = r25.below(15);
        while (q[2] == q[0] || q[2] == q[1]);
        for (int k : q) s[k] ^= 1 + r25.below(15);
        auto r = bw_decode(symbols_to_bits(s, 4), p);
        if (!r) ++failures;
        else CHECK(r->message != msg && r->errors_corrected <= p.t);
    }
    CHECK(failures > 0);
    CHECK_THROWS_AS(bw_decode(BitVec(59, 0), p), InvalidInput);
}

static ImageBuffer noise_image(uint64_t seed, int w, int h) {
    ImageBuffer img = ImageBuffer::make_byte(w, h);
    CounterRng rng(seed, 1);
    for (auto& b : img.bytes) b = static_cast<uint8_t>(rng.below(256));
    return img;
}

static void gpu_image() {
    ImageBuffer big = noise_image(3, 512, 512);
    ImageBuffer out = preprocess(big);
    CHECK(out.width == 256 && out.height == 256 && out.form == PixelForm::normalized);
    for (int probe = 0; probe < 64; ++probe) {
        int x = probe * 4 + 1, y = probe * 3 + 2;
        CHECK(out.atf(x, y, 1) == static_cast<float>(big.at8(x + 128, y + 128, 1) / 127.5 - 1.0));
    }
    ImageBuffer img = noise_image(4, 256, 256);
    ImageBuffer o2 = preprocess(img);
    for (int probe = 0; probe < 256; ++probe) {
        int x = probe, y = (probe * 7) % 256;
        CHECK(o2.atf(x, y, 0) == static_cast<float>(img.at8(x, y, 0) / 127.5 - 1.0));
    }
    for (auto [w, h] : {std::pair{1, 1}, {3, 200}, {100, 300}, {255, 255}}) {
        ImageBuffer o = preprocess(noise_image(5, w, h));
        CHECK(o.width == 256 && o.height == 256);
        for (float v : o.values) CHECK(v >= -1.0f && v <= 1.0f);
    }
    CounterRng rng(31, 0);
    for (int trial = 0; trial < 20; ++trial) {
        int w = 1 + rng.below(480), h = 1 + rng.below(480);
        ImageBuffer im = noise_image(100 + trial, w, h);
        CHECK(preprocess_fused(im).values == preprocess(im).values);
    }
    // staged primitives compose to preprocess
    ImageBuffer small = noise_image(9, 200, 150);
    ImageBuffer staged = normalize(center_crop(resize_bilinear(small, 341, 256), 256, 256));
    CHECK(staged.values == preprocess(small).values);
    ImageBuffer n = normalize(img);
    CHECK(center_crop(n, 64, 64).atf(0, 0, 0) == n.atf(96, 96, 0));
    ImageBuffer t = extract_tile(img, TileRef{64, 128, 64});
    CHECK(t.at8(5, 7, 2) == img.at8(69, 135, 2));
    CHECK_THROWS_AS(extract_tile(img, TileRef{224, 0, 64}), InvalidInput);
    CHECK_THROWS_AS(normalize(n), InvalidInput);
    ImageBuffer syn = synthetic_image(1000, 64, 48);
    CHECK(syn.width == 64 && syn.height == 48 && syn.bytes.size() == 64 * 48 * 3);
}

static void host_ppm() {
    ImageBuffer img = noise_image(12, 37, 21);
    const std::string path = "/tmp/qrm_dropin_test.ppm";
    write_ppm(img, path);
    ImageBuffer back = read_ppm(path);
    CHECK(back.width == 37 && back.height == 21 && back.bytes == img.bytes);
    CHECK_THROWS_AS(read_ppm("/tmp/qrm_no_such_file.ppm"), InvalidInput);
    CHECK_THROWS_AS(write_ppm(ImageBuffer::make_normalized(2, 2), path), InvalidInput);
    std::remove(path.c_str());
}

static void gpu_stego_detect() {
    WatermarkKey key{1, 60, 0.04};
    SpreadSpectrumCodec codec(key, 64);
    CounterRng rng(8, 0);
    ImageBuffer tile = normalize(noise_image(77, 64, 64));
    for (int trial = 0; trial < 5; ++trial) {
        BitVec bits = random_bits(rng, 60);
        SoftBits s = codec.extract(codec.embed(tile, bits));
        CHECK(harden(s) == bits);
    }
    SoftBits z = codec.extract(ImageBuffer::make_normalized(64, 64));
    for (double v : z.values) CHECK(v == 0.0);
    CHECK(std::fabs(codec.pattern_correlation(0, 1)) < 0.1 && codec.pattern_correlation(2, 2) == 1.0);
    CHECK_THROWS_AS(codec.extract(ImageBuffer::make_normalized(32, 32)), InvalidInput);
    // detection on the cmd_bench corpus recipe (cli.cpp:404-411)
    CodeParams code = resolve_profile("gf16-15-12");
    BitVec msg(48);
    for (int i = 0; i < 48; ++i) msg[i] = rng_word(1, 0x6d73, i) & 1;
    DetectionConfig cfg = DetectionConfig::make(code, TileSpec{64, TileStrategy::random_grid, 0}, 1, 0.04, msg);
    BitVec cw = rs_encode(msg, code);
    std::vector<ImageBuffer> pos, neg;
    for (int i = 0; i < 24; ++i) {
        ImageBuffer n = normalize(synthetic_image(1000 + i, 256, 256));
        embed_image_grid(n, codec, cw);
        pos.push_back(denormalize(n));
        neg.push_back(synthetic_image(5000 + i, 256, 256));
    }
    auto rp = detect_batch(pos, cfg);
    auto rn = detect_batch(neg, cfg);
    for (size_t i = 0; i < rp.size(); ++i) {
        CHECK(rp[i].image_index == i);
        CHECK(rp[i].cache_hit == (i > 0));  // one raw word: the codebook hits after the first (detect.cpp:326-333)
        CHECK(rp[i].verified && rp[i].corrected && *rp[i].corrected == msg && rp[i].errors_corrected == 0);
        CHECK(rp[i].bit_acc == 1.0);
        CHECK(!rn[i].verified);
    }
    // worker/plan invariance and detect_one equivalence
    StreamPlan plan{{2, 3, 2}, {5, 5, 5}, 0.0};
    DeskReport rep;
    auto rq = detect_batch(pos, cfg, &plan, nullptr, &rep);
    CHECK(rep.items == pos.size() && rep.stage_workers[1] == 3);
    DetectionContext ctx(cfg);
    for (size_t i = 0; i < rp.size(); ++i) {
        CHECK(semantic_equal(rp[i], rq[i]));
        CHECK(semantic_equal(rp[i], ctx.detect_one(pos[i], i)));
    }
    // DeskReport and StageLatencies are filled from the stage streams' events
    CHECK(rep.wall_ns > 0 && rep.stage_busy_ns[0] > 0 && rep.stage_busy_ns[1] > 0 && rep.stage_busy_ns[2] > 0);
    for (const auto& r : rq) CHECK(r.stage_ns.preprocess_ns > 0 && r.stage_ns.extract_ns > 0 && r.stage_ns.correct_ns > 0);
    // SyntheticStageLoad holds each stage's stream load_ns per image (detect.cpp:304, 318, 336)
    {
        SyntheticStageLoad load{0, 200000, 50000};  // 0.2 ms per image on decode, 0.05 ms on correct
        StreamPlan one{{1, 1, 1}, {8}, 0.0};         // minibatch of any length: its largest entry (detect.cpp:266)
        DeskReport lr;
        auto rl = detect_batch(pos, cfg, &one, &load, &lr);
        CHECK(lr.stage_busy_ns[1] >= static_cast<int64_t>(pos.size()) * 200000);
        CHECK(lr.stage_busy_ns[2] >= static_cast<int64_t>(pos.size()) * 50000);
        CHECK(lr.wall_ns >= static_cast<int64_t>(pos.size()) * 200000);
        for (size_t i = 0; i < rl.size(); ++i) {
            CHECK(semantic_equal(rl[i], rp[i]));
            CHECK(rl[i].stage_ns.extract_ns >= 8 * 200000);  // its mini-batch of 8 held the decode stream
        }
        CHECK_THROWS_AS(detect_batch(std::vector<ImageBuffer>{pos[0], noise_image(4, 300, 200)}, cfg, nullptr, &load),
                        InvalidInput);
    }
    {
        StreamPlan bad{{1, 1}, {4, 4}, 0.0};
        CHECK_THROWS_AS(detect_batch(pos, cfg, &bad), InvalidInput);
        DeskReport er;
        CHECK(detect_batch(std::vector<ImageBuffer>{}, cfg, &bad, nullptr, &er).empty() && er.items == 0);
    }
    // ragged inputs through the same entry
    std::vector<ImageBuffer> mixed = {pos[0], noise_image(4, 300, 200), noise_image(5, 100, 90)};
    auto rm = detect_batch(mixed, cfg);
    CHECK(rm.size() == 3 && semantic_equal(rm[0], rp[0]));
    CHECK_THROWS_AS(detect_batch(std::vector<ImageBuffer>{ImageBuffer::make_normalized(8, 8)}, cfg), InvalidInput);
    // the codebook cache is transparent
    CorrectionCache cache(CacheConfig{true, 2, 1u << 20});
    auto [r1, h1] = cache.correct(rp[0].raw_bits, code);
    auto [r2, h2] = cache.correct(rp[0].raw_bits, code);
    CHECK(!h1 && h2 && r1 && r2 && r1->message == r2->message && cache.hits() == 1);
    // warm-up profile of the device stages feeds Algorithm 1
    StageProfile prof = warmup_profile(pos, 2, cfg);
    CHECK(prof.stages() == 3 && prof.b0 == 16.0);
    for (double t : prof.time) CHECK(t > 0.0);
    StreamPlan p2 = allocate_streams(prof, 24, 8, 1e12, 0.0, 2);
    auto [rr, rrep] = run_desk(p2, pos, cfg);
    for (size_t i = 0; i < rr.size(); ++i) CHECK(semantic_equal(rr[i], rp[i]));
}

// The learned extractor through the same entry points (DetectionConfig::extractor).
static void gpu_conv_detect() {
    CodeParams code = resolve_profile("gf16-15-12");
    BitVec msg(48);
    for (int i = 0; i < 48; ++i) msg[i] = rng_word(1, 0x6d73, i) & 1;
    DetectionConfig cfg = DetectionConfig::make(code, TileSpec{64, TileStrategy::random_grid, 0}, 1, 0.04, msg);
    cfg.extractor = ExtractorKind::conv;
    cfg.conv_weight_seed = 7;
    std::vector<ImageBuffer> imgs;
    for (int i = 0; i < 12; ++i) imgs.push_back(synthetic_image(1000 + i, 256, 256));
    auto r1 = detect_batch(imgs, cfg);
    StreamPlan plan{{1, 2, 1}, {5, 5, 5}, 0.0};
    auto r2 = detect_batch(imgs, cfg, &plan);
    DetectionContext ctx(cfg);
    CHECK(r1.size() == imgs.size());
    BitVec kcw = rs_encode(msg, code);
    for (size_t i = 0; i < r1.size(); ++i) {
        CHECK(semantic_equal(r1[i], r2[i]));
        CHECK(semantic_equal(r1[i], ctx.detect_one(imgs[i], i)));
        // RS + verify on the extractor's own hard bits equal the reference chain
        auto d = bw_decode(r1[i].raw_bits, code);
        CHECK(d.has_value() == r1[i].corrected.has_value());
        if (d) CHECK(*r1[i].corrected == d->message && r1[i].errors_corrected == d->errors_corrected);
        CHECK(r1[i].bit_acc == bit_accuracy(r1[i].raw_bits, kcw));
    }
    // sharded over several device contexts (here all on device 0): same records
    DetectionConfig multi = cfg;
    multi.devices = {0, 0, 0};
    auto r4 = detect_batch(imgs, multi);
    for (size_t i = 0; i < r4.size(); ++i) CHECK(semantic_equal(r1[i], r4[i]));
    // the spread-spectrum default is unaffected by a conv context alive beside it
    cfg.extractor = ExtractorKind::spread_spectrum;
    auto r3 = detect_batch(imgs, cfg);
    bool differs = false;
    for (size_t i = 0; i < r3.size(); ++i) differs |= r3[i].raw_bits != r1[i].raw_bits;
    CHECK(differs);
}

int main(int argc, char** argv) {
    const std::string which = argc > 1 ? argv[1] : "all";
    struct Case {
        const char* name;
        bool gpu;
        void (*fn)();
    } cases[] = {{"gf", false, host_gf},          {"rs_encode", false, host_rs_encode},
                 {"tiling_sched", false, host_tiling_sched}, {"ppm", false, host_ppm}, {"cache", false, host_cache}, {"rs_gpu", true, gpu_rs},
                 {"image_gpu", true, gpu_image},  {"stego_detect_gpu", true, gpu_stego_detect},
                 {"conv_detect_gpu", true, gpu_conv_detect}};
    for (auto& c : cases) {
        if ((which == "host" && c.gpu) || (which == "gpu" && !c.gpu)) continue;
        const int before = g_fail;
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("FAIL %s: uncaught %s\n", c.name, e.what());
        }
        std::printf("%-20s %s\n", c.name, g_fail == before ? "ok" : "FAILED");
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
