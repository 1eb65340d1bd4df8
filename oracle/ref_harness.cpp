// C-ABI shim over the UNMODIFIED reference library (TEST INFRASTRUCTURE ONLY).
//
// Compiled together with /root/reference/proj/src/{gf,rs,image,transforms,tiling,
// stego,sched,detect,sim,json_io}.cpp by oracle/Makefile into oracle/_ref/libqrmark_ref.so.
// Every entry point calls the reference's own public API; nothing here
// re-implements reference arithmetic except `default_message`, which lives in
// cli.cpp (not compiled: it needs CLI11) and is restated from cli.cpp:47-51.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline / reference
// arm may load this library.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "qrmark/detect.hpp"
#include "qrmark/gf.hpp"
#include "qrmark/image.hpp"
#include "qrmark/json_io.hpp"
#include "qrmark/rng.hpp"
#include "qrmark/rs.hpp"
#include "qrmark/sched.hpp"
#include "qrmark/sim.hpp"
#include "qrmark/stego.hpp"
#include "qrmark/tiling.hpp"
#include "qrmark/transforms.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace qrmark;

namespace {

thread_local std::string g_err;

// 0 ok; 1 InvalidInput; 2 DivisionByZero; 3 InfeasibleConfig; 4 other
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const InvalidInput& e) {
        g_err = e.what();
        return 1;
    } catch (const DivisionByZero& e) {
        g_err = e.what();
        return 2;
    } catch (const InfeasibleConfig& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

CodeParams code_of(int m, int n, int k) {
    if (m == 4) return CodeParams::make(FieldSpec::gf16(), n, k);
    if (m == 8) return CodeParams::make(FieldSpec::gf256(), n, k);
    throw InvalidInput("harness: symbol size must be 4 or 8");
}

int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

BitVec unpack_word(uint64_t w, int nbits) {
    BitVec b(nbits);
    for (int i = 0; i < nbits; ++i) b[i] = (w >> (nbits - 1 - i)) & 1;
    return b;
}

uint64_t pack_word(const BitVec& b) {
    uint64_t w = 0;
    for (uint8_t v : b) w = (w << 1) | (v & 1);
    return w;
}

TileStrategy strategy_of(int s) {
    switch (s) {
        case 0: return TileStrategy::random;
        case 1: return TileStrategy::random_grid;
        case 2: return TileStrategy::fixed;
    }
    throw InvalidInput("harness: bad strategy");
}

}  // namespace

extern "C" {

struct ref_detect_cfg {
    int m, n, k;
    int tile_size;
    int strategy;  // 0 random, 1 random_grid, 2 fixed
    uint64_t tile_seed;
    uint64_t key_seed;
    double alpha;
    const uint8_t* key_message;  // k*m bits, one per byte
    int rs_workers;
    double fpr;
    int cache_enabled;
    uint64_t cache_capacity;
    uint64_t stale_after;
};

struct ref_records {
    uint8_t* raw_bits;       // count * n*m
    uint8_t* has_corrected;  // count
    uint8_t* corrected;      // count * k*m
    int32_t* errors;         // count
    double* bit_acc;         // count
    uint8_t* verified;       // count
    uint8_t* cache_hit;      // count (may be null)
};

}  // extern "C"

namespace {

DetectionConfig config_of(const ref_detect_cfg* c) {
    CodeParams code = code_of(c->m, c->n, c->k);
    BitVec msg(c->key_message, c->key_message + code.message_bits());
    TileSpec tile{c->tile_size, strategy_of(c->strategy), c->tile_seed};
    DetectionConfig cfg = DetectionConfig::make(code, tile, c->key_seed, c->alpha, msg);
    cfg.rs_workers = c->rs_workers;
    cfg.fpr_target = c->fpr;
    cfg.cache.enabled = c->cache_enabled != 0;
    cfg.cache.capacity = c->cache_capacity;
    cfg.cache.stale_after = c->stale_after;
    return cfg;
}

void store_record(const DetectionRecord& r, size_t slot, const CodeParams& code, ref_records* out) {
    const int nb = code.codeword_bits(), kb = code.message_bits();
    std::memcpy(out->raw_bits + slot * nb, r.raw_bits.data(), nb);
    out->has_corrected[slot] = r.corrected.has_value();
    if (r.corrected) std::memcpy(out->corrected + slot * kb, r.corrected->data(), kb);
    else std::memset(out->corrected + slot * kb, 0, kb);
    out->errors[slot] = r.errors_corrected;
    out->bit_acc[slot] = r.bit_acc;
    out->verified[slot] = r.verified;
    if (out->cache_hit) out->cache_hit[slot] = r.cache_hit;
}

std::vector<ImageBuffer> images_of(const uint8_t* const* imgs, const int* ws, const int* hs, int64_t count) {
    std::vector<ImageBuffer> v;
    v.reserve(count);
    for (int64_t i = 0; i < count; ++i) {
        ImageBuffer b = ImageBuffer::make_byte(ws[i], hs[i]);
        std::memcpy(b.bytes.data(), imgs[i], b.bytes.size());
        v.push_back(std::move(b));
    }
    return v;
}

}  // namespace

REF_API int ref_abi_version() { return 3; }
REF_API const char* ref_last_error() { return g_err.c_str(); }

REF_API int ref_resolve_profile(const char* name, int payload_bits, int* m, int* n, int* k, int* t) {
    return guarded([&] {
        CodeParams p = resolve_profile(name, payload_bits);
        *m = p.field->bits();
        *n = p.n;
        *k = p.k;
        *t = p.t;
    });
}

// cli.cpp:47-51 (default_message) — restated because cli.cpp is not compiled.
REF_API void ref_default_message(uint64_t key_seed, int n_bits, uint8_t* out) {
    for (int i = 0; i < n_bits; ++i) out[i] = rng_word(key_seed, 0x6d73, i) & 1;
}

REF_API uint64_t ref_rng_word(uint64_t s, uint64_t st, uint64_t c) { return rng_word(s, st, c); }
REF_API uint64_t ref_rng_below(uint64_t s, uint64_t st, uint64_t c, uint64_t b) { return rng_below(s, st, c, b); }
REF_API double ref_rng_unit(uint64_t s, uint64_t st, uint64_t c) { return rng_unit(s, st, c); }

REF_API int ref_gf_mul(int m, int a, int b, int* out) {
    return guarded([&] {
        const FieldSpec& f = m == 4 ? FieldSpec::gf16() : FieldSpec::gf256();
        *out = f.mul(static_cast<uint16_t>(a), static_cast<uint16_t>(b));
    });
}

REF_API int ref_rs_encode(int m, int n, int k, const uint8_t* msg_bits, uint8_t* cw_bits) {
    return guarded([&] {
        CodeParams p = code_of(m, n, k);
        BitVec msg(msg_bits, msg_bits + p.message_bits());
        BitVec cw = rs_encode(msg, p);
        std::memcpy(cw_bits, cw.data(), cw.size());
    });
}

// Returns 1 decoded, 0 decode failure, <0 -(exception code).
REF_API int ref_bw_decode(int m, int n, int k, const uint8_t* bits, uint8_t* msg_out, uint8_t* cw_out,
                          int* errors) {
    int decoded = 0;
    int rc = guarded([&] {
        CodeParams p = code_of(m, n, k);
        BitVec r(bits, bits + p.codeword_bits());
        auto res = bw_decode(r, p);
        if (res) {
            decoded = 1;
            if (msg_out) std::memcpy(msg_out, res->message.data(), res->message.size());
            if (cw_out) std::memcpy(cw_out, res->codeword.data(), res->codeword.size());
            *errors = res->errors_corrected;
        } else {
            *errors = 0;
        }
    });
    return rc ? -rc : decoded;
}

// Batch bw_decode over packed words (n*m <= 64, MSB-first) on `threads`
// std::threads. nerr_out = errors_corrected, or -1 for a decode failure.
// Returns wall-clock ns of the decode loop (the CPU RS baseline).
REF_API int64_t ref_bw_decode_packed(int m, int n, int k, const uint64_t* words, int64_t count, int threads,
                                     uint64_t* cw_out, int8_t* nerr_out) {
    int64_t wall = -1;
    guarded([&] {
        CodeParams p = code_of(m, n, k);
        const int nb = p.codeword_bits();
        if (nb > 64) throw InvalidInput("harness: packed words need n*m <= 64");
        threads = std::max(1, threads);
        std::atomic<int64_t> next{0};
        const int64_t chunk = 4096;
        auto worker = [&] {
            while (true) {
                int64_t b = next.fetch_add(chunk);
                if (b >= count) break;
                int64_t e = std::min(count, b + chunk);
                for (int64_t i = b; i < e; ++i) {
                    auto res = bw_decode(unpack_word(words[i], nb), p);
                    if (res) {
                        cw_out[i] = pack_word(res->codeword);
                        nerr_out[i] = static_cast<int8_t>(res->errors_corrected);
                    } else {
                        cw_out[i] = 0;
                        nerr_out[i] = -1;
                    }
                }
            }
        };
        int64_t t0 = now_ns();
        std::vector<std::thread> pool;
        for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
        worker();
        for (auto& th : pool) th.join();
        wall = now_ns() - t0;
    });
    return wall;
}

// Symbol-array batch decode for codes wider than 64 bits (e.g. (12,8) GF(256)).
// recv: count*n symbols (one byte each); cw_out: count*n; nerr_out: errors or -1.
REF_API int ref_bw_decode_symbols(int m, int n, int k, const uint8_t* recv, int64_t count, uint8_t* cw_out,
                                  int8_t* nerr_out) {
    return guarded([&] {
        CodeParams p = code_of(m, n, k);
        std::vector<uint16_t> sym(n);
        for (int64_t i = 0; i < count; ++i) {
            for (int j = 0; j < n; ++j) sym[j] = recv[i * n + j];
            auto res = bw_decode(symbols_to_bits(sym, m), p);
            if (res) {
                auto cs = bits_to_symbols(res->codeword, m);
                for (int j = 0; j < n; ++j) cw_out[i * n + j] = static_cast<uint8_t>(cs[j]);
                nerr_out[i] = static_cast<int8_t>(res->errors_corrected);
            } else {
                std::memset(cw_out + i * n, 0, n);
                nerr_out[i] = -1;
            }
        }
    });
}

// The same over `threads` host threads, returning the wall time in ns (the RS
// CPU baseline for symbol codes, e.g. GF(2^8) (12,8) and (255,223)).
REF_API int64_t ref_bw_decode_symbols_mt(int m, int n, int k, const uint8_t* recv, int64_t count, int threads,
                                         uint8_t* cw_out, int8_t* nerr_out) {
    int64_t wall = -1;
    guarded([&] {
        CodeParams p = code_of(m, n, k);
        threads = std::max(1, threads);
        std::atomic<int64_t> next{0};
        const int64_t chunk = 1024;
        auto worker = [&] {
            std::vector<uint16_t> sym(n);
            while (true) {
                int64_t b = next.fetch_add(chunk);
                if (b >= count) break;
                int64_t e = std::min(count, b + chunk);
                for (int64_t i = b; i < e; ++i) {
                    for (int j = 0; j < n; ++j) sym[j] = recv[i * n + j];
                    auto res = bw_decode(symbols_to_bits(sym, m), p);
                    if (res) {
                        auto cs = bits_to_symbols(res->codeword, m);
                        for (int j = 0; j < n; ++j) cw_out[i * n + j] = static_cast<uint8_t>(cs[j]);
                        nerr_out[i] = static_cast<int8_t>(res->errors_corrected);
                    } else {
                        std::memset(cw_out + i * n, 0, n);
                        nerr_out[i] = -1;
                    }
                }
            }
        };
        int64_t t0 = now_ns();
        std::vector<std::thread> pool;
        for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
        worker();
        for (auto& th : pool) th.join();
        wall = now_ns() - t0;
    });
    return wall;
}

REF_API int ref_verify_threshold(int n_bits, double fpr, int* tau) {
    return guarded([&] { *tau = verify_threshold(n_bits, fpr); });
}

REF_API int ref_synthetic_image(uint64_t seed, int w, int h, uint8_t* out) {
    return guarded([&] {
        ImageBuffer img = synthetic_image(seed, w, h);
        std::memcpy(out, img.bytes.data(), img.bytes.size());
    });
}

// cmd_bench corpus recipe (cli.cpp:404-411): synthetic_image(first_seed + i)
// -> normalize -> embed_image_grid(key codeword) -> denormalize. embed=0 gives
// the un-watermarked negatives.
REF_API int ref_make_corpus(uint64_t first_seed, int64_t count, int w, int h, uint64_t key_seed, double alpha,
                            int m, int n, int k, int tile, int embed, int threads, uint8_t* out) {
    return guarded([&] {
        CodeParams code = code_of(m, n, k);
        BitVec msg(code.message_bits());
        ref_default_message(key_seed, code.message_bits(), msg.data());
        BitVec word = rs_encode(msg, code);
        WatermarkKey key{key_seed, code.codeword_bits(), alpha};
        SpreadSpectrumCodec codec(key, tile);
        const size_t bytes = static_cast<size_t>(w) * h * 3;
        std::atomic<int64_t> next{0};
        auto worker = [&] {
            while (true) {
                int64_t i = next.fetch_add(1);
                if (i >= count) break;
                ImageBuffer img = synthetic_image(first_seed + static_cast<uint64_t>(i), w, h);
                if (embed) {
                    ImageBuffer norm = normalize(img);
                    embed_image_grid(norm, codec, word);
                    img = denormalize(norm);
                }
                std::memcpy(out + static_cast<size_t>(i) * bytes, img.bytes.data(), bytes);
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < std::max(1, threads); ++t) pool.emplace_back(worker);
        worker();
        for (auto& th : pool) th.join();
    });
}

REF_API int ref_preprocess(const uint8_t* img, int w, int h, int fused, float* out) {
    return guarded([&] {
        ImageBuffer b = ImageBuffer::make_byte(w, h);
        std::memcpy(b.bytes.data(), img, b.bytes.size());
        ImageBuffer r = fused ? preprocess_fused(b) : preprocess(b);
        std::memcpy(out, r.values.data(), r.values.size() * sizeof(float));
    });
}

REF_API int ref_resize_bilinear(const uint8_t* img, int w, int h, int ow, int oh, uint8_t* out) {
    return guarded([&] {
        ImageBuffer b = ImageBuffer::make_byte(w, h);
        std::memcpy(b.bytes.data(), img, b.bytes.size());
        ImageBuffer r = resize_bilinear(b, ow, oh);
        std::memcpy(out, r.bytes.data(), r.bytes.size());
    });
}

REF_API int ref_select_tile(int w, int h, int l, int strategy, uint64_t seed, uint64_t draw, int* x, int* y) {
    return guarded([&] {
        TileRef t = select_tile(w, h, TileSpec{l, strategy_of(strategy), seed}, draw);
        *x = t.x;
        *y = t.y;
    });
}

REF_API int ref_grid_cells(int w, int h, int l, int* xy_out, int cap, int* count) {
    return guarded([&] {
        auto cells = grid_cells(w, h, l);
        *count = static_cast<int>(cells.size());
        for (int i = 0; i < std::min(cap, *count); ++i) {
            xy_out[2 * i] = cells[i].x;
            xy_out[2 * i + 1] = cells[i].y;
        }
    });
}

// SpreadSpectrumCodec::extract on a normalized l*l*3 tile.
REF_API int ref_extract(uint64_t key_seed, int n_bits, double alpha, int l, const float* tile, double* soft) {
    return guarded([&] {
        SpreadSpectrumCodec codec(WatermarkKey{key_seed, n_bits, alpha}, l);
        ImageBuffer t = ImageBuffer::make_normalized(l, l);
        std::memcpy(t.values.data(), tile, t.values.size() * sizeof(float));
        SoftBits s = codec.extract(t);
        std::memcpy(soft, s.values.data(), s.values.size() * sizeof(double));
    });
}

// The codec's +-1 planes, recovered through the public residual(): with a
// single set bit the residual is P_i - sum_{j!=i} P_j; with none it is
// -sum_j P_j; their half-difference is P_i.
REF_API int ref_pattern(uint64_t key_seed, int n_bits, int l, int bit, int8_t* out) {
    return guarded([&] {
        SpreadSpectrumCodec codec(WatermarkKey{key_seed, n_bits, 0.04}, l);
        BitVec zero(n_bits, 0), one(n_bits, 0);
        one[bit] = 1;
        auto a = codec.residual(one), b = codec.residual(zero);
        for (size_t i = 0; i < a.size(); ++i) out[i] = static_cast<int8_t>((a[i] - b[i]) / 2.0f);
    });
}

// DetectionContext::detect_one over a batch with draw_index = first_draw + i,
// sequential, one context (cache follows the reference's own policy).
REF_API int ref_detect_sequential(const uint8_t* const* imgs, const int* ws, const int* hs, int64_t count,
                                  uint64_t first_draw, const ref_detect_cfg* c, ref_records* out) {
    return guarded([&] {
        DetectionConfig cfg = config_of(c);
        DetectionContext ctx(cfg);
        for (int64_t i = 0; i < count; ++i) {
            ImageBuffer b = ImageBuffer::make_byte(ws[i], hs[i]);
            std::memcpy(b.bytes.data(), imgs[i], b.bytes.size());
            DetectionRecord r = ctx.detect_one(b, first_draw + static_cast<uint64_t>(i));
            store_record(r, static_cast<size_t>(i), cfg.code, out);
        }
    });
}

// The reference pipeline: detect_batch (detect.cpp:250) with an optional
// 3-stage StreamPlan (worker counts + mini-batches). Returns DeskReport.wall_ns
// (the images are copied into ImageBuffers before the clock starts).
REF_API int64_t ref_detect_batch(const uint8_t* const* imgs, const int* ws, const int* hs, int64_t count,
                                 const ref_detect_cfg* c, const int* streams3, const int* minibatch3,
                                 ref_records* out) {
    int64_t wall = -1;
    guarded([&] {
        DetectionConfig cfg = config_of(c);
        std::vector<ImageBuffer> images = images_of(imgs, ws, hs, count);
        StreamPlan plan;
        const StreamPlan* pp = nullptr;
        if (streams3) {
            plan.streams = {streams3[0], streams3[1], streams3[2]};
            plan.minibatch = {minibatch3[0], minibatch3[1], minibatch3[2]};
            pp = &plan;
        }
        DeskReport rep;
        auto recs = detect_batch(images, cfg, pp, nullptr, &rep);
        if (out)
            for (size_t i = 0; i < recs.size(); ++i) store_record(recs[i], i, cfg.code, out);
        wall = rep.wall_ns;
    });
    return wall;
}


// read_ppm (image.cpp:129-146). dst == nullptr: header only.
REF_API int ref_read_ppm(const char* path, uint8_t* dst, int64_t cap, int* w, int* h) {
    return guarded([&] {
        ImageBuffer img = read_ppm(path);
        *w = img.width;
        *h = img.height;
        if (dst) {
            if (cap < static_cast<int64_t>(img.bytes.size())) throw InvalidInput("harness: buffer too small");
            std::memcpy(dst, img.bytes.data(), img.bytes.size());
        }
    });
}

// write_ppm (image.cpp:148-156).
REF_API int ref_write_ppm(const char* path, const uint8_t* img, int w, int h) {
    return guarded([&] {
        ImageBuffer b = ImageBuffer::make_byte(w, h);
        std::memcpy(b.bytes.data(), img, b.bytes.size());
        write_ppm(b, path);
    });
}

// cmd_detect's "records" (cli.cpp:234, 279-281): detect_batch over the images,
// then json::array of record_to_json(rec, deterministic = true), dump(2).
// Returns the length; copies at most cap-1 bytes + NUL into out.
REF_API int64_t ref_detect_json(const uint8_t* const* imgs, const int* ws, const int* hs, int64_t count,
                                const ref_detect_cfg* c, char* out, int64_t cap) {
    int64_t len = -1;
    guarded([&] {
        DetectionConfig cfg = config_of(c);
        std::vector<ImageBuffer> images = images_of(imgs, ws, hs, count);
        auto recs = detect_batch(images, cfg);
        nlohmann::json arr = nlohmann::json::array();
        for (const auto& r : recs) arr.push_back(record_to_json(r, true));
        const std::string s = arr.dump(2);
        len = static_cast<int64_t>(s.size());
        if (out && cap > 0) {
            const int64_t n = std::min<int64_t>(cap - 1, len);
            std::memcpy(out, s.data(), static_cast<size_t>(n));
            out[n] = '\0';
        }
    });
    return len;
}


// apply_attack (transforms.cpp:289-362) via TransformSpec::parse (the CLI's
// names). out: bytes, or floats for "normalize" (*is_float = 1).
REF_API int ref_apply_attack(const uint8_t* img, int w, int h, const char* op, double param, void* out, int64_t cap,
                             int* ow, int* oh, int* is_float) {
    return guarded([&] {
        ImageBuffer b = ImageBuffer::make_byte(w, h);
        std::memcpy(b.bytes.data(), img, b.bytes.size());
        ImageBuffer r = apply_attack(b, TransformSpec::parse(op, param));
        *ow = r.width;
        *oh = r.height;
        *is_float = r.form == PixelForm::normalized;
        const int64_t bytes = *is_float ? static_cast<int64_t>(r.values.size() * sizeof(float))
                                        : static_cast<int64_t>(r.bytes.size());
        if (out) {
            if (cap < bytes) throw InvalidInput("harness: buffer too small");
            std::memcpy(out, *is_float ? static_cast<const void*>(r.values.data()) : r.bytes.data(), bytes);
        }
    });
}

// allocate_streams (sched.cpp:50). Returns the error code (0 ok).
REF_API int ref_allocate_streams(int stages, const double* time, const double* memory, double b0,
                                 int global_batch, int budget, double m_cap, double eps, int stall_cap,
                                 int* streams_out, int* mb_out, double* bottleneck) {
    return guarded([&] {
        StageProfile prof;
        prof.b0 = b0;
        prof.time.assign(time, time + stages);
        prof.memory.assign(memory, memory + stages);
        StreamPlan p = allocate_streams(prof, global_batch, budget, m_cap, eps, stall_cap);
        for (int k = 0; k < stages; ++k) {
            streams_out[k] = p.streams[k];
            mb_out[k] = p.minibatch[k];
        }
        *bottleneck = p.bottleneck;
    });
}

// lpt_schedule (sched.cpp:177). Pieces are written stream by stream in
// placement order: (stream, id, units, latency, memory, mb).
REF_API int ref_lpt_schedule(int ntasks, const int* ids, const double* lat, const double* mem, const int* units,
                             int streams, double lambda, double m_cap, int b_min, int global_batch, int cap,
                             int* p_stream, int* p_id, int* p_units, double* p_lat, double* p_mem, int* p_mb,
                             int* n_pieces, double* loads_out, int* m_unit) {
    return guarded([&] {
        std::vector<Task> tasks(ntasks);
        for (int i = 0; i < ntasks; ++i) {
            tasks[i].id = ids[i];
            tasks[i].latency = lat[i];
            tasks[i].memory = mem[i];
            tasks[i].units = units[i];
        }
        StreamSchedule s = lpt_schedule(tasks, streams, lambda, m_cap, b_min, global_batch);
        int c = 0;
        for (int st = 0; st < streams; ++st) {
            loads_out[st] = s.loads[st];
            for (const Task& t : s.streams[st]) {
                if (c < cap) {
                    p_stream[c] = st;
                    p_id[c] = t.id;
                    p_units[c] = t.units;
                    p_lat[c] = t.latency;
                    p_mem[c] = t.memory;
                    p_mb[c] = t.mb;
                }
                ++c;
            }
        }
        *n_pieces = c;
        *m_unit = s.m_unit;
    });
}

// measure_stages (sim.cpp:214) with a scripted clock: clock_values is read in
// order, one value per now_ns() call; run_batch is a no-op.
REF_API int ref_measure_stages_scripted(int stages, int iters, double b0, const int64_t* clock_values,
                                        const double* mem, const double* prep_share, double* time_out,
                                        double* prep_out) {
    return guarded([&] {
        std::vector<StageBench> benches;
        for (int k = 0; k < stages; ++k)
            benches.push_back({"s" + std::to_string(k), [] {}, mem[k], prep_share[k]});
        size_t pos = 0;
        auto clock = [&] { return clock_values[pos++]; };
        StageProfile p = measure_stages(benches, iters, b0, clock);
        for (int k = 0; k < stages; ++k) {
            time_out[k] = p.time[k];
            prep_out[k] = p.prep[k];
        }
    });
}
