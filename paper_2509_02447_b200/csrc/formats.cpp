// The wire and on-disk formats either side of the detection path (SURVEY
// §8f row 4), host C++:
//
//  * PPM P6 read/write with the reference's grammar (image.cpp:106-156):
//    whitespace and '#' comments between header tokens, maxval 255 only, one
//    whitespace byte before the raster, the same InvalidInput messages. The
//    batch reader decodes many same-size files in parallel straight into a
//    caller buffer (normally pinned memory that qrm_detect_host then reads
//    over PCIe), which is the ingest half of cmd_detect (cli.cpp:22-45).
//  * The detection records as JSON: record_to_json (json_io.cpp:98-120) for
//    every record, as the "records" array of cmd_detect's report
//    (cli.cpp:279-281), in nlohmann::json's dump(2) layout (keys in sorted
//    order, two-space indent, shortest round-trip doubles with ".0" on
//    integral values), so reports diff byte-for-byte against the reference.
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <thread>
#include <vector>

#include "host_code.hpp"
#include "qrm_types.h"

namespace qrm {
namespace {

struct File {
    FILE* f = nullptr;
    explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// read_ppm_token (image.cpp:108-124): skip whitespace and '#' comment lines,
// then a decimal integer (operator>> semantics: optional sign, digits).
bool ppm_token(FILE* f, int& value) {
    int c;
    while (true) {
        c = std::fgetc(f);
        if (c == '#') {
            while (c != '\n' && c != EOF) c = std::fgetc(f);
            if (c == EOF) return false;
        } else if (c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r') {
            continue;
        } else {
            break;
        }
    }
    bool neg = false;
    if (c == '+' || c == '-') {
        neg = c == '-';
        c = std::fgetc(f);
    }
    if (c < '0' || c > '9') return false;
    long long v = 0;
    while (c >= '0' && c <= '9') {
        v = v * 10 + (c - '0');
        if (v > 0x7fffffffLL) return false;
        c = std::fgetc(f);
    }
    if (c != EOF) std::ungetc(c, f);
    value = static_cast<int>(neg ? -v : v);
    return true;
}

// Header of a P6 file; on success the stream sits at the first raster byte.
qrm_status ppm_header(FILE* f, const std::string& name, int& w, int& h) {
    char magic[2];
    if (std::fread(magic, 1, 2, f) != 2 || magic[0] != 'P' || magic[1] != '6')
        return report_error(QRM_INVALID_INPUT, name + ": not a P6 PPM");
    int maxval = 0;
    if (!ppm_token(f, w) || !ppm_token(f, h) || !ppm_token(f, maxval))
        return report_error(QRM_INVALID_INPUT, "malformed PPM header");
    if (maxval != 255) return report_error(QRM_INVALID_INPUT, name + ": only maxval 255 supported");
    if (w <= 0 || h <= 0) return report_error(QRM_INVALID_INPUT, "image dimensions must be positive");
    std::fgetc(f);  // single whitespace before the raster (image.cpp:138)
    return QRM_OK;
}

qrm_status ppm_read(const char* path, uint8_t* dst, int64_t cap, int* w_out, int* h_out) {
    if (!path) return report_error(QRM_INVALID_INPUT, "null path");
    const std::string name(path);
    File in(path, "rb");
    if (!in.f) return report_error(QRM_INVALID_INPUT, "cannot open " + name);
    int w = 0, h = 0;
    qrm_status s = ppm_header(in.f, name, w, h);
    if (s != QRM_OK) return s;
    if (w_out) *w_out = w;
    if (h_out) *h_out = h;
    if (!dst) return QRM_OK;  // header query
    const int64_t bytes = static_cast<int64_t>(w) * h * 3;
    if (cap < bytes) return report_error(QRM_INVALID_INPUT, name + ": destination smaller than the raster");
    if (static_cast<int64_t>(std::fread(dst, 1, static_cast<size_t>(bytes), in.f)) != bytes)
        return report_error(QRM_INVALID_INPUT, name + ": truncated raster data");
    return QRM_OK;
}

// A double as nlohmann::json's dump writes it: the digit string laid out by
// its format_buffer with min_exp = -4, max_exp = 15 (plain notation with ".0"
// on integral values while the decimal point falls in (-4, 15], else
// d.ddde+XX). Digits are the shortest round-trip ones (std::to_chars);
// nlohmann's grisu2 emits the same digits for every bit_acc value m/n with
// n <= 64 (checked exhaustively against json.hpp) — the only doubles a record
// holds — and can differ in the last place for rare other doubles.
void append_double(std::string& out, double v) {
    if (!std::isfinite(v)) {  // nlohmann dumps NaN/inf as null
        out += "null";
        return;
    }
    if (v == 0.0) {
        out += std::signbit(v) ? "-0.0" : "0.0";
        return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
    std::string sci(buf, r.ptr);  // [-]d[.ddd]e[+-]XX
    std::string sign;
    if (sci[0] == '-') {
        sign = "-";
        sci.erase(0, 1);
    }
    const size_t epos = sci.find('e');
    const int exp10 = std::atoi(sci.c_str() + epos + 1);
    std::string digits;
    for (size_t i = 0; i < epos; ++i)
        if (sci[i] != '.') digits += sci[i];
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // value = 0.d1d2...dk x 10^n
    std::string o;
    if (k <= n && n <= 15) {
        o = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        o = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
    } else if (-4 < n && n <= 0) {
        o = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
    } else {
        o = digits.substr(0, 1);
        if (k > 1) o += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        o += eb;
    }
    out += sign + o;
}

std::string hex_of(uint64_t word, int bits) {
    // bits_to_hex (rs.cpp:27-36): MSB-first nibbles, lowercase
    static const char* kHex = "0123456789abcdef";
    std::string s;
    for (int i = 0; i < bits / 4; ++i) s += kHex[(word >> (bits - 4 * (i + 1))) & 0xF];
    return s;
}

// DetectionRecord::cache_hit: the codebook's policy (CorrectionCache::correct +
// evict_locked, detect.cpp:86-128) replayed over the records in index order —
// the reference with one correct worker. Keys are the raw words (pack_bits is a
// bijection of them); every call has its own tick, so "oldest" is unique and an
// ordered map by last access replaces the reference's linear scan.
void cache_replay(const qrm_record* recs, int64_t count, int64_t capacity, uint64_t stale_after, uint8_t* hit) {
    std::unordered_map<uint64_t, uint64_t> last;  // word -> last access tick
    std::map<uint64_t, uint64_t> by_tick;         // last access tick -> word
    uint64_t tick = 0;
    auto evict = [&] {
        while (!by_tick.empty() && tick - by_tick.begin()->first > stale_after) {
            last.erase(by_tick.begin()->second);
            by_tick.erase(by_tick.begin());
        }
        while (static_cast<int64_t>(last.size()) > capacity) {
            last.erase(by_tick.begin()->second);
            by_tick.erase(by_tick.begin());
        }
    };
    for (int64_t i = 0; i < count; ++i) {
        ++tick;
        evict();
        const uint64_t key = recs[i].raw;
        auto it = last.find(key);
        hit[i] = it != last.end();
        if (it != last.end()) {
            by_tick.erase(it->second);
            it->second = tick;
            by_tick[tick] = key;
            continue;
        }
        last[key] = tick;
        by_tick[tick] = key;
        evict();
    }
}

}  // namespace
}  // namespace qrm

using namespace qrm;

extern "C" {

QRM_EXPORT qrm_status qrm_ppm_read(const char* path, uint8_t* dst, int64_t cap, int* w, int* h) {
    return ppm_read(path, dst, cap, w, h);
}

QRM_EXPORT qrm_status qrm_ppm_write(const char* path, const uint8_t* img, int w, int h) {
    if (!path || !img) return report_error(QRM_INVALID_INPUT, "null argument");
    if (w <= 0 || h <= 0) return report_error(QRM_INVALID_INPUT, "image dimensions must be positive");
    File out(path, "wb");
    if (!out.f) return report_error(QRM_INVALID_INPUT, std::string("cannot write ") + path);
    std::fprintf(out.f, "P6\n%d %d\n255\n", w, h);  // write_ppm (image.cpp:148-155)
    const size_t bytes = static_cast<size_t>(w) * h * 3;
    if (std::fwrite(img, 1, bytes, out.f) != bytes)
        return report_error(QRM_INVALID_INPUT, std::string("cannot write ") + path);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_ppm_read_batch(const char* const* paths, int64_t count, int w, int h, uint8_t* dst,
                                         int64_t image_stride, int threads, int32_t* status) {
    if (count < 0 || (count > 0 && (!paths || !dst))) return report_error(QRM_INVALID_INPUT, "null argument");
    if (w <= 0 || h <= 0) return report_error(QRM_INVALID_INPUT, "image dimensions must be positive");
    const int64_t bytes = static_cast<int64_t>(w) * h * 3;
    if (image_stride < bytes) return report_error(QRM_INVALID_INPUT, "image stride smaller than an image");
    const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : 8, count)));
    std::vector<std::string> errs(static_cast<size_t>(count));
    auto work = [&](int t) {
        for (int64_t i = t; i < count; i += nt) {
            int fw = 0, fh = 0;
            qrm_status s = ppm_read(paths[i], dst + i * image_stride, bytes, &fw, &fh);
            if (s == QRM_OK && (fw != w || fh != h)) {
                s = QRM_INVALID_INPUT;
                report_error(s, std::string(paths[i]) + ": size differs from the batch");
            }
            if (s != QRM_OK) {
                // qrm_last_error is per thread: carry the message to the caller's thread
                errs[static_cast<size_t>(i)] = qrm_last_error();
            }
            if (status) status[i] = s;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int64_t i = 0; i < count; ++i)
        if (!errs[static_cast<size_t>(i)].empty()) return report_error(QRM_INVALID_INPUT, errs[static_cast<size_t>(i)]);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_cache_hits(const qrm_record* recs, int64_t count, int64_t capacity, uint64_t stale_after,
                                     uint8_t* hit) {
    if (count < 0 || (count > 0 && (!recs || !hit))) return report_error(QRM_INVALID_INPUT, "null argument");
    if (capacity < 0) return report_error(QRM_INVALID_INPUT, "bad cache capacity");
    cache_replay(recs, count, capacity, stale_after, hit);
    return QRM_OK;
}

QRM_EXPORT qrm_status qrm_records_json(const qrm_record* recs, int64_t count, int n_bits, int k_bits,
                                       int64_t first_index, int cache_enabled, int64_t cache_capacity,
                                       uint64_t stale_after, char* out, int64_t cap, int64_t* len) {
    if (count < 0 || (count > 0 && !recs) || !len) return report_error(QRM_INVALID_INPUT, "null argument");
    if (n_bits <= 0 || n_bits > 64 || k_bits <= 0 || k_bits > n_bits)
        return report_error(QRM_INVALID_INPUT, "bad code widths");
    if (cache_enabled && cache_capacity < 0) return report_error(QRM_INVALID_INPUT, "bad cache capacity");
    std::vector<uint8_t> hit(static_cast<size_t>(count), 0);
    if (cache_enabled) cache_replay(recs, count, cache_capacity, stale_after, hit.data());
    // json::array of record_to_json(rec, deterministic = true) (json_io.cpp:98-120),
    // dump(2): keys sorted as nlohmann's std::map orders them.
    std::string s;
    if (count == 0) {
        s = "[]";
    } else {
        s = "[\n";
        for (int64_t i = 0; i < count; ++i) {
            const qrm_record& r = recs[i];
            const bool decoded = r.status == QRM_REC_DECODED;
            s += "  {\n    \"bit_acc\": ";
            append_double(s, static_cast<double>(r.matches) / n_bits);  // bit_accuracy (rs.cpp:215-221)
            s += hit[static_cast<size_t>(i)] ? ",\n    \"cache_hit\": true" : ",\n    \"cache_hit\": false";
            s += ",\n    \"corrected_hex\": ";
            if (decoded)
                s += k_bits % 4 == 0 ? "\"" + hex_of(r.msg, k_bits) + "\"" : "\"\"";
            else
                s += "null";
            s += ",\n    \"errors_corrected\": " + std::to_string(decoded ? r.errors : 0);
            s += ",\n    \"index\": " + std::to_string(first_index + i);
            s += ",\n    \"raw_hex\": \"" + (n_bits % 4 == 0 ? hex_of(r.raw, n_bits) : std::string()) + "\"";
            s += ",\n    \"stage_ns\": {\n      \"correct\": 0,\n      \"extract\": 0,\n      \"preprocess\": 0\n    }";
            s += ",\n    \"verified\": ";
            s += r.verified ? "true" : "false";
            s += "\n  }";
            s += i + 1 < count ? ",\n" : "\n";
        }
        s += "]";
    }
    *len = static_cast<int64_t>(s.size());
    if (out && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
        std::memcpy(out, s.data(), static_cast<size_t>(n));
        out[n] = '\0';
    }
    return QRM_OK;
}

}  // extern "C"
