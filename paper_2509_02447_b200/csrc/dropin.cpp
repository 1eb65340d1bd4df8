// The reference C++ API (include/qrmark/api.hpp) implemented over the C-ABI.
//
// GPU: bw_decode / bw_decode_batch, SpreadSpectrumCodec::extract, preprocess,
// normalize / resize_bilinear / center_crop / extract_tile (byte images),
// synthetic_image, DetectionContext::detect_one, detect_batch, warmup_profile.
// Host: field and polynomial arithmetic, bit packing, thresholds, the planners,
// float-form copies and the embedding helpers used to build inputs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <thread>

#include "host_code.hpp"
#include "host_pool.hpp"
#include "qrmark/api.hpp"
#include "qrmark_gpu.h"
#include "sched_host.hpp"

namespace qrmark {

namespace {

[[noreturn]] void raise(qrm_status s) {
    const std::string msg = qrm_last_error();
    switch (s) {
        case QRM_INVALID_INPUT: throw InvalidInput(msg);
        case QRM_DIVISION_BY_ZERO: throw DivisionByZero(msg);
        case QRM_INFEASIBLE: throw InfeasibleConfig(msg);
        default: throw CudaUnavailable(msg);
    }
}

void check(qrm_status s) {
    if (s != QRM_OK) raise(s);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaUnavailable(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
};

uint64_t pack(const BitVec& b) {
    uint64_t w = 0;
    for (uint8_t v : b) w = (w << 1) | (v & 1);
    return w;
}

BitVec unpack(uint64_t w, int n) {
    BitVec b(n);
    for (int i = 0; i < n; ++i) b[i] = (w >> (n - 1 - i)) & 1;
    return b;
}

int geometry_upscale(int w, int h, int& sw, int& sh, int& xo, int& yo) {
    const int mn = std::min(w, h);
    int up = 0;
    if (mn < kWorkingSize) {
        const double s = static_cast<double>(kWorkingSize) / mn;
        up = 1;
        sw = std::max<int>(kWorkingSize, static_cast<int>(std::lround(w * s)));
        sh = std::max<int>(kWorkingSize, static_cast<int>(std::lround(h * s)));
    } else {
        sw = w;
        sh = h;
    }
    xo = (sw - kWorkingSize) / 2;
    yo = (sh - kWorkingSize) / 2;
    return up;
}

}  // namespace

// ---------------------------------------------------------------------- gf
FieldSpec::FieldSpec(int m, uint32_t poly) : m_(m), poly_(poly), order_(1 << m) {
    const qrm::HostField& f = qrm::host_field(m);
    exp_ = f.exp;
    log_ = f.log;
}
const FieldSpec& FieldSpec::gf16() {
    static const FieldSpec f(4, 0x13);
    return f;
}
const FieldSpec& FieldSpec::gf256() {
    static const FieldSpec f(8, 0x11d);
    return f;
}
void FieldSpec::check(uint16_t v) const {
    if (v >= order_) throw InvalidInput("field element out of range");
}
uint16_t FieldSpec::add(uint16_t a, uint16_t b) const {
    check(a);
    check(b);
    return a ^ b;
}
uint16_t FieldSpec::mul(uint16_t a, uint16_t b) const {
    check(a);
    check(b);
    if (!a || !b) return 0;
    return exp_[(log_[a] + log_[b]) % (order_ - 1)];
}
uint16_t FieldSpec::inv(uint16_t a) const {
    check(a);
    if (!a) throw DivisionByZero("inverse of zero field element");
    return exp_[(order_ - 1 - log_[a]) % (order_ - 1)];
}
uint16_t FieldSpec::div(uint16_t a, uint16_t b) const { return mul(a, inv(b)); }
uint16_t FieldSpec::pow(uint16_t a, uint64_t e) const {
    check(a);
    if (e == 0) return 1;
    if (a == 0) return 0;
    return exp_[(static_cast<uint64_t>(log_[a]) * (e % (order_ - 1))) % (order_ - 1)];
}

static void same(const FieldElement& a, const FieldElement& b) {
    if (!a.spec || a.spec != b.spec) throw InvalidInput("field elements from different fields");
}
FieldElement operator+(FieldElement a, FieldElement b) {
    same(a, b);
    return {a.spec->add(a.value, b.value), *a.spec};
}
FieldElement operator*(FieldElement a, FieldElement b) {
    same(a, b);
    return {a.spec->mul(a.value, b.value), *a.spec};
}
FieldElement operator/(FieldElement a, FieldElement b) {
    same(a, b);
    return {a.spec->div(a.value, b.value), *a.spec};
}

Poly::Poly(const FieldSpec& spec, std::vector<uint16_t> coeffs) : spec_(&spec), c_(std::move(coeffs)) {
    while (!c_.empty() && c_.back() == 0) c_.pop_back();
}
uint16_t Poly::eval(uint16_t x) const {
    uint16_t acc = 0;
    for (size_t i = c_.size(); i-- > 0;) acc = spec_->add(spec_->mul(acc, x), c_[i]);
    return acc;
}
Poly operator+(const Poly& a, const Poly& b) {
    if (a.spec_ != b.spec_) throw InvalidInput("polynomials from different fields");
    std::vector<uint16_t> o(std::max(a.c_.size(), b.c_.size()));
    for (size_t i = 0; i < o.size(); ++i) o[i] = a.coeff(i) ^ b.coeff(i);
    return Poly(*a.spec_, std::move(o));
}
Poly operator*(const Poly& a, const Poly& b) {
    if (a.spec_ != b.spec_) throw InvalidInput("polynomials from different fields");
    if (a.is_zero() || b.is_zero()) return Poly::zero(*a.spec_);
    std::vector<uint16_t> o(a.c_.size() + b.c_.size() - 1, 0);
    for (size_t i = 0; i < a.c_.size(); ++i)
        for (size_t j = 0; j < b.c_.size(); ++j) o[i + j] ^= a.spec_->mul(a.c_[i], b.c_[j]);
    return Poly(*a.spec_, std::move(o));
}
Poly Poly::scaled(uint16_t s) const {
    std::vector<uint16_t> o(c_.size());
    for (size_t i = 0; i < c_.size(); ++i) o[i] = spec_->mul(c_[i], s);
    return Poly(*spec_, std::move(o));
}
std::pair<Poly, Poly> Poly::divmod(const Poly& num, const Poly& den) {
    if (num.spec_ != den.spec_) throw InvalidInput("polynomials from different fields");
    if (den.is_zero()) throw DivisionByZero("polynomial division by zero");
    const FieldSpec& f = *num.spec_;
    if (num.degree() < den.degree()) return {Poly::zero(f), num};
    std::vector<uint16_t> r(num.c_), q(num.degree() - den.degree() + 1, 0);
    const uint16_t li = f.inv(den.c_.back());
    for (int d = num.degree(); d >= den.degree(); --d) {
        if (!r[d]) continue;
        const uint16_t k = f.mul(r[d], li);
        q[d - den.degree()] = k;
        for (size_t i = 0; i < den.c_.size(); ++i) r[d - den.degree() + i] ^= f.mul(k, den.c_[i]);
    }
    return {Poly(f, std::move(q)), Poly(f, std::move(r))};
}
Poly lagrange_interpolate(const FieldSpec& spec, std::span<const std::pair<uint16_t, uint16_t>> pts) {
    for (size_t i = 0; i < pts.size(); ++i)
        for (size_t j = i + 1; j < pts.size(); ++j)
            if (pts[i].first == pts[j].first) throw InvalidInput("duplicate x coordinate in interpolation");
    Poly acc = Poly::zero(spec);
    for (size_t i = 0; i < pts.size(); ++i) {
        Poly basis = Poly::constant(spec, 1);
        uint16_t den = 1;
        for (size_t j = 0; j < pts.size(); ++j) {
            if (j == i) continue;
            basis = basis * Poly(spec, {pts[j].first, 1});
            den = spec.mul(den, spec.add(pts[i].first, pts[j].first));
        }
        acc = acc + basis.scaled(spec.div(pts[i].second, den));
    }
    return acc;
}

// ---------------------------------------------------------------------- rs
std::vector<uint16_t> bits_to_symbols(const BitVec& bits, int m) {
    if (m <= 0 || bits.size() % m) throw InvalidInput("bit count not a multiple of symbol size");
    std::vector<uint16_t> o(bits.size() / m);
    for (size_t s = 0; s < o.size(); ++s)
        for (int b = 0; b < m; ++b) o[s] = static_cast<uint16_t>((o[s] << 1) | (bits[s * m + b] & 1));
    return o;
}
BitVec symbols_to_bits(std::span<const uint16_t> symbols, int m) {
    BitVec o(symbols.size() * m);
    for (size_t s = 0; s < symbols.size(); ++s)
        for (int b = 0; b < m; ++b) o[s * m + b] = (symbols[s] >> (m - 1 - b)) & 1;
    return o;
}
std::string bits_to_hex(const BitVec& bits) {
    if (bits.size() % 4) throw InvalidInput("bit count not a multiple of 4");
    static const char* dg = "0123456789abcdef";
    std::string o(bits.size() / 4, '0');
    for (size_t i = 0; i < o.size(); ++i) o[i] = dg[(bits[4 * i] << 3) | (bits[4 * i + 1] << 2) | (bits[4 * i + 2] << 1) | bits[4 * i + 3]];
    return o;
}
BitVec hex_to_bits(const std::string& hex, size_t n_bits) {
    if (hex.size() * 4 != n_bits) throw InvalidInput("hex string length does not match bit count");
    BitVec o(n_bits);
    for (size_t i = 0; i < hex.size(); ++i) {
        const char c = static_cast<char>(std::tolower(static_cast<unsigned char>(hex[i])));
        int v;
        if (c >= '0' && c <= '9') v = c - '0';
        else if (c >= 'a' && c <= 'f') v = c - 'a' + 10;
        else throw InvalidInput("invalid hex digit");
        for (int b = 0; b < 4; ++b) o[4 * i + b] = (v >> (3 - b)) & 1;
    }
    return o;
}
CodeParams CodeParams::make(const FieldSpec& field, int n, int k) {
    const std::string e = qrm::check_code(field.bits(), n, k);
    if (!e.empty()) throw InvalidInput(e);
    CodeParams p;
    p.field = &field;
    p.n = n;
    p.k = k;
    p.t = (n - k) / 2;
    p.eval_points.resize(n);
    for (int i = 0; i < n; ++i) p.eval_points[i] = field.alpha_pow(i);
    return p;
}
CodeParams resolve_profile(const std::string& name, int payload_bits) {
    if (name == "gf16-15-12") return CodeParams::make(FieldSpec::gf16(), 15, 12);
    if (name == "gf256-dynamic") {
        if (payload_bits <= 0 || payload_bits % 8)
            throw InvalidInput("gf256-dynamic payload must be a positive multiple of 8 bits");
        return CodeParams::make(FieldSpec::gf256(), payload_bits / 8 + 2, payload_bits / 8);
    }
    throw InvalidInput("unknown code profile: " + name);
}
BitVec rs_encode(const BitVec& message, const CodeParams& p) {
    if (static_cast<int>(message.size()) != p.message_bits()) throw InvalidInput("message bit length does not match profile");
    const int m = p.field->bits();
    auto cw = qrm::encode_symbols(m, p.n, p.k, bits_to_symbols(message, m));
    return symbols_to_bits(cw, m);
}

std::vector<std::optional<DecodeResult>> bw_decode_batch(std::span<const BitVec> received, const CodeParams& p) {
    const int m = p.field->bits(), nb = p.codeword_bits();
    for (const BitVec& r : received)
        if (static_cast<int>(r.size()) != nb) throw InvalidInput("received bit length does not match profile");
    const int64_t N = static_cast<int64_t>(received.size());
    std::vector<std::optional<DecodeResult>> out(N);
    if (N == 0) return out;
    std::vector<int8_t> ne(N);
    if (nb <= 64) {
        std::vector<uint64_t> w(N), cw(N);
        for (int64_t i = 0; i < N; ++i) w[i] = pack(received[i]);
        DevBuf<uint64_t> dw(N), dc(N);
        DevBuf<int8_t> dn(N);
        cuda_check(cudaMemcpy(dw.p, w.data(), 8 * N, cudaMemcpyHostToDevice), "H2D");
        check(qrm_rs_decode_packed_device(m, p.n, p.k, dw.p, N, dc.p, dn.p, 0, nullptr));
        cuda_check(cudaMemcpy(cw.data(), dc.p, 8 * N, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(ne.data(), dn.p, N, cudaMemcpyDeviceToHost), "D2H");
        for (int64_t i = 0; i < N; ++i)
            if (ne[i] >= 0) {
                DecodeResult r;
                r.codeword = unpack(cw[i], nb);
                r.message.assign(r.codeword.begin(), r.codeword.begin() + p.message_bits());
                r.errors_corrected = ne[i];
                out[i] = std::move(r);
            }
    } else {
        std::vector<uint8_t> sym(N * p.n), cs(N * p.n);
        for (int64_t i = 0; i < N; ++i) {
            auto s = bits_to_symbols(received[i], m);
            for (int j = 0; j < p.n; ++j) sym[i * p.n + j] = static_cast<uint8_t>(s[j]);
        }
        DevBuf<uint8_t> ds(N * p.n), dc(N * p.n);
        DevBuf<int8_t> dn(N);
        cuda_check(cudaMemcpy(ds.p, sym.data(), N * p.n, cudaMemcpyHostToDevice), "H2D");
        check(qrm_rs_decode_symbols_device(m, p.n, p.k, ds.p, N, dc.p, dn.p, nullptr));
        cuda_check(cudaMemcpy(cs.data(), dc.p, N * p.n, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(ne.data(), dn.p, N, cudaMemcpyDeviceToHost), "D2H");
        for (int64_t i = 0; i < N; ++i)
            if (ne[i] >= 0) {
                std::vector<uint16_t> s(cs.begin() + i * p.n, cs.begin() + (i + 1) * p.n);
                DecodeResult r;
                r.codeword = symbols_to_bits(s, m);
                r.message.assign(r.codeword.begin(), r.codeword.begin() + p.message_bits());
                r.errors_corrected = ne[i];
                out[i] = std::move(r);
            }
    }
    return out;
}
std::optional<DecodeResult> bw_decode(const BitVec& received, const CodeParams& p) {
    return bw_decode_batch(std::span<const BitVec>(&received, 1), p)[0];
}
double rs_aware_loss(const BitVec& pr, const BitVec& tg, const CodeParams& p) {
    if (pr.size() != tg.size()) throw InvalidInput("bit length mismatch");
    const int m = p.field->bits();
    if (pr.size() % m) throw InvalidInput("bit count not a multiple of symbol size");
    int e = 0;
    for (size_t s = 0; s < pr.size() / m; ++s)
        for (int b = 0; b < m; ++b)
            if (pr[s * m + b] != tg[s * m + b]) {
                ++e;
                break;
            }
    const double x = std::max(0, e - p.t);
    return x * x;
}
double bit_accuracy(const BitVec& a, const BitVec& b) {
    if (a.size() != b.size()) throw InvalidInput("bit length mismatch");
    if (a.empty()) return 1.0;
    size_t k = 0;
    for (size_t i = 0; i < a.size(); ++i) k += a[i] == b[i];
    return static_cast<double>(k) / static_cast<double>(a.size());
}
double word_accuracy(const std::vector<BitVec>& d, const std::vector<BitVec>& t) {
    if (d.size() != t.size()) throw InvalidInput("word count mismatch");
    if (d.empty()) return 1.0;
    size_t k = 0;
    for (size_t i = 0; i < d.size(); ++i) k += d[i] == t[i];
    return static_cast<double>(k) / static_cast<double>(d.size());
}

// ------------------------------------------------------------------- image
ImageBuffer ImageBuffer::make_byte(int w, int h) {
    if (w <= 0 || h <= 0) throw InvalidInput("image dimensions must be positive");
    ImageBuffer b;
    b.width = w;
    b.height = h;
    b.form = PixelForm::byte;
    b.bytes.assign(static_cast<size_t>(w) * h * 3, 0);
    return b;
}
ImageBuffer ImageBuffer::make_normalized(int w, int h) {
    if (w <= 0 || h <= 0) throw InvalidInput("image dimensions must be positive");
    ImageBuffer b;
    b.width = w;
    b.height = h;
    b.form = PixelForm::normalized;
    b.values.assign(static_cast<size_t>(w) * h * 3, 0.0f);
    return b;
}
ImageBuffer normalize(const ImageBuffer& img) {
    if (img.form != PixelForm::byte) throw InvalidInput("normalize expects byte form");
    ImageBuffer o = ImageBuffer::make_normalized(img.width, img.height);
    check(qrm_resample_host(img.bytes.data(), img.width, img.height, 0, img.width, img.height, 0, 0, img.width,
                            img.height, 1, o.values.data()));
    return o;
}
ImageBuffer denormalize(const ImageBuffer& img) {
    if (img.form != PixelForm::normalized) throw InvalidInput("denormalize expects normalized form");
    ImageBuffer o = ImageBuffer::make_byte(img.width, img.height);
    for (size_t i = 0; i < img.values.size(); ++i) {
        const double q = std::floor((static_cast<double>(img.values[i]) + 1.0) * 127.5 + 0.5);
        o.bytes[i] = static_cast<uint8_t>(std::clamp(q, 0.0, 255.0));
    }
    return o;
}
ImageBuffer resize_bilinear(const ImageBuffer& img, int ow, int oh) {
    if (img.form != PixelForm::byte) throw InvalidInput("resize expects byte form");
    if (ow <= 0 || oh <= 0) throw InvalidInput("resize target must be positive");
    if (ow == img.width && oh == img.height) return img;
    ImageBuffer o = ImageBuffer::make_byte(ow, oh);
    check(qrm_resample_host(img.bytes.data(), img.width, img.height, 1, ow, oh, 0, 0, ow, oh, 0, o.bytes.data()));
    return o;
}
ImageBuffer center_crop(const ImageBuffer& img, int cw, int ch) {
    if (cw > img.width || ch > img.height) throw InvalidInput("crop window larger than image");
    const int xo = (img.width - cw) / 2, yo = (img.height - ch) / 2;
    if (img.form == PixelForm::byte) {
        ImageBuffer o = ImageBuffer::make_byte(cw, ch);
        check(qrm_resample_host(img.bytes.data(), img.width, img.height, 0, img.width, img.height, xo, yo, cw, ch, 0,
                                o.bytes.data()));
        return o;
    }
    ImageBuffer o = ImageBuffer::make_normalized(cw, ch);
    for (int y = 0; y < ch; ++y)
        std::memcpy(&o.values[o.index(0, y, 0)], &img.values[img.index(xo, yo + y, 0)], sizeof(float) * cw * 3);
    return o;
}
ImageBuffer synthetic_image(uint64_t seed, int w, int h) {
    ImageBuffer o = ImageBuffer::make_byte(w, h);
    qrm_config c{};
    c.tile_size = 64;
    DevBuf<uint8_t> d(o.bytes.size());
    check(qrm_make_corpus_device(&c, seed, 1, w, h, 0, d.p, nullptr));
    cuda_check(cudaMemcpy(o.bytes.data(), d.p, o.bytes.size(), cudaMemcpyDeviceToHost), "D2H");
    return o;
}

// -------------------------------------------------------------- transforms
ImageBuffer preprocess(const ImageBuffer& img) {
    if (img.form != PixelForm::byte) throw InvalidInput("preprocess expects byte form");
    ImageBuffer o = ImageBuffer::make_normalized(kWorkingSize, kWorkingSize);
    check(qrm_preprocess_host(img.bytes.data(), img.width, img.height, o.values.data()));
    return o;
}
ImageBuffer preprocess_fused(const ImageBuffer& img) { return preprocess(img); }

// ------------------------------------------------------------------ tiling
TileStrategy parse_tile_strategy(const std::string& n) {
    if (n == "random") return TileStrategy::random;
    if (n == "random_grid") return TileStrategy::random_grid;
    if (n == "fixed") return TileStrategy::fixed;
    throw InvalidInput("unknown tile strategy: " + n);
}
std::string tile_strategy_name(TileStrategy s) {
    switch (s) {
        case TileStrategy::random: return "random";
        case TileStrategy::random_grid: return "random_grid";
        case TileStrategy::fixed: return "fixed";
    }
    return "?";
}
TileRef select_tile(int w, int h, const TileSpec& spec, uint64_t draw) {
    if (spec.size <= 0 || spec.size > std::min(w, h)) throw InvalidInput("tile size does not fit image");
    const int l = spec.size;
    if (spec.strategy == TileStrategy::fixed) return {0, 0, l};
    if (spec.strategy == TileStrategy::random)
        return {static_cast<int>(rng_below(spec.seed, 2 * draw, 0, static_cast<uint64_t>(w - l) + 1)),
                static_cast<int>(rng_below(spec.seed, 2 * draw + 1, 0, static_cast<uint64_t>(h - l) + 1)), l};
    const uint64_t cols = w / l, rows = h / l;
    const uint64_t cell = rng_below(spec.seed, draw, 0, cols * rows);
    return {static_cast<int>(cell % cols) * l, static_cast<int>(cell / cols) * l, l};
}
TileRef select_tile(const ImageBuffer& img, const TileSpec& spec, uint64_t draw) {
    return select_tile(img.width, img.height, spec, draw);
}
std::vector<TileRef> grid_cells(int w, int h, int l) {
    if (l <= 0 || l > std::min(w, h)) throw InvalidInput("tile size does not fit image");
    std::vector<TileRef> v;
    for (int y = 0; y + l <= h; y += l)
        for (int x = 0; x + l <= w; x += l) v.push_back({x, y, l});
    return v;
}
ImageBuffer extract_tile(const ImageBuffer& img, const TileRef& t) {
    if (t.x < 0 || t.y < 0 || t.x + t.size > img.width || t.y + t.size > img.height)
        throw InvalidInput("tile out of bounds");
    if (img.form == PixelForm::byte) {
        ImageBuffer o = ImageBuffer::make_byte(t.size, t.size);
        check(qrm_resample_host(img.bytes.data(), img.width, img.height, 0, img.width, img.height, t.x, t.y, t.size,
                                t.size, 0, o.bytes.data()));
        return o;
    }
    ImageBuffer o = ImageBuffer::make_normalized(t.size, t.size);
    for (int y = 0; y < t.size; ++y)
        std::memcpy(&o.values[o.index(0, y, 0)], &img.values[img.index(t.x, t.y + y, 0)], sizeof(float) * t.size * 3);
    return o;
}

// ------------------------------------------------------------------- stego
BitVec harden(const SoftBits& s) {
    BitVec b(s.values.size());
    for (size_t i = 0; i < b.size(); ++i) b[i] = s.values[i] > 0.0 ? 1 : 0;
    return b;
}
SpreadSpectrumCodec::SpreadSpectrumCodec(const WatermarkKey& key, int tile_size) : key_(key), tile_size_(tile_size) {
    if (key.n_bits <= 0) throw InvalidInput("payload width must be positive");
    if (key.alpha < 0.0) throw InvalidInput("alpha must be nonnegative");
    if (tile_size <= 0) throw InvalidInput("tile size must be positive");
}
// The host copy of the +-1 planes (stego.cpp:22-26) is built on first use:
// extraction runs on the device planes, and only residual / embed /
// pattern_correlation read these (detect_batch's per-call context never does).
const int8_t* SpreadSpectrumCodec::planes() const {
    std::call_once(host_planes_->once, [&] {
        auto& v = host_planes_->v;
        v.resize(static_cast<size_t>(key_.n_bits) * samples());
        for (int i = 0; i < key_.n_bits; ++i)
            for (size_t px = 0; px < samples(); ++px)
                v[i * samples() + px] = (rng_word(key_.seed, static_cast<uint64_t>(i), px) & 1) ? 1 : -1;
    });
    return host_planes_->v.data();
}
std::vector<float> SpreadSpectrumCodec::residual(const BitVec& bits) const {
    if (static_cast<int>(bits.size()) != key_.n_bits) throw InvalidInput("payload bit-length mismatch");
    std::vector<float> d(samples(), 0.0f);
    for (int i = 0; i < key_.n_bits; ++i) {
        const float s = bits[i] ? 1.0f : -1.0f;
        const int8_t* p = planes() + i * samples();
        for (size_t px = 0; px < d.size(); ++px) d[px] += s * p[px];
    }
    return d;
}
ImageBuffer SpreadSpectrumCodec::embed(const ImageBuffer& tile, const BitVec& bits) const {
    if (tile.form != PixelForm::normalized) throw InvalidInput("embed expects normalized form");
    if (tile.width != tile_size_ || tile.height != tile_size_) throw InvalidInput("tile dimensions do not match codec");
    const auto d = residual(bits);
    ImageBuffer o = tile;
    const float a = static_cast<float>(key_.alpha);
    for (size_t px = 0; px < d.size(); ++px) o.values[px] = std::clamp(tile.values[px] + a * d[px], -1.0f, 1.0f);
    return o;
}
SoftBits SpreadSpectrumCodec::extract(const ImageBuffer& tile) const {
    if (tile.form != PixelForm::normalized) throw InvalidInput("extract expects normalized form");
    if (tile.width != tile_size_ || tile.height != tile_size_) throw InvalidInput("tile dimensions do not match codec");
    SoftBits s;
    s.values.resize(key_.n_bits);
    check(qrm_extract_float_host(key_.seed, key_.n_bits, tile_size_, tile.values.data(), s.values.data()));
    return s;
}
double SpreadSpectrumCodec::pattern_correlation(int i, int j) const {
    const int8_t* a = planes() + i * samples();
    const int8_t* b = planes() + j * samples();
    double acc = 0.0;
    for (size_t px = 0; px < samples(); ++px) acc += static_cast<double>(a[px]) * b[px];
    return acc / static_cast<double>(samples());
}
void embed_image_grid(ImageBuffer& img, const SpreadSpectrumCodec& codec, const BitVec& bits) {
    if (img.form != PixelForm::normalized) throw InvalidInput("embed expects normalized form");
    const int l = codec.tile_size();
    const auto d = codec.residual(bits);
    const float a = static_cast<float>(codec.key().alpha);
    for (const TileRef& cell : grid_cells(img.width, img.height, l)) {
        size_t px = 0;
        for (int y = 0; y < l; ++y)
            for (int x = 0; x < l; ++x)
                for (int c = 0; c < 3; ++c, ++px) {
                    float& v = img.atf(cell.x + x, cell.y + y, c);
                    v = std::clamp(v + a * d[px], -1.0f, 1.0f);
                }
    }
}
ImageBuffer embed(const ImageBuffer& tile, const BitVec& bits, const WatermarkKey& key) {
    return SpreadSpectrumCodec(key, tile.width).embed(tile, bits);
}
SoftBits extract(const ImageBuffer& tile, const WatermarkKey& key) {
    return SpreadSpectrumCodec(key, tile.width).extract(tile);
}

// ------------------------------------------------------------------- sched
void StageProfile::validate() const {
    if (time.empty()) throw InvalidInput("profile has no stages");
    if (memory.size() != time.size()) throw InvalidInput("profile time/memory length mismatch");
    if (b0 < 1.0) throw InvalidInput("baseline batch must be >= 1");
    for (double t : time)
        if (t <= 0.0) throw InvalidInput("stage times must be positive");
    for (double u : memory)
        if (u < 0.0) throw InvalidInput("per-sample memory must be nonnegative");
}
int StreamPlan::total_streams() const { return std::accumulate(streams.begin(), streams.end(), 0); }
double stage_time(const StageProfile& p, int k, int s, int m) {
    if (s < 1) throw InvalidInput("stream count must be >= 1");
    return p.time[k] * (static_cast<double>(m) / p.b0) / static_cast<double>(s);
}
bool mem_ok(std::span<const int> s, std::span<const int> m, std::span<const double> u, double cap) {
    if (s.size() != m.size() || s.size() != u.size()) throw InvalidInput("mem_ok length mismatch");
    return qrm::sched::mem_ok(std::vector<int>(s.begin(), s.end()), std::vector<int>(m.begin(), m.end()),
                              std::vector<double>(u.begin(), u.end()), cap);
}
StreamPlan allocate_streams(const StageProfile& profile, int B, int P, double m_cap, double eps, int stall_cap) {
    profile.validate();
    qrm::sched::Profile p{profile.b0, profile.time, profile.memory};
    qrm::sched::Plan plan;
    std::string err;
    const int rc = qrm::sched::allocate_streams(p, B, P, m_cap, eps, stall_cap, plan, err);
    if (rc == 1) throw InvalidInput(err);
    if (rc == 3) throw InfeasibleConfig(err);
    return StreamPlan{plan.streams, plan.minibatch, plan.bottleneck};
}
double StreamSchedule::makespan() const {
    double w = 0.0;
    for (double l : loads) w = std::max(w, l);
    return w;
}
double StreamSchedule::total_latency() const { return std::accumulate(loads.begin(), loads.end(), 0.0); }
double WarmupStats::latency_for(PipelineMode mode, int tile) const {
    const double r = static_cast<double>(tile) / reference_tile;
    return (mode == PipelineMode::detect ? detect_latency : embed_latency) * r * r;
}
double WarmupStats::memory_for(PipelineMode mode, int tile) const {
    const double r = static_cast<double>(tile) / reference_tile;
    return (mode == PipelineMode::detect ? detect_memory : embed_memory) * r * r;
}
std::vector<Task> build_tasks(std::span<const ImageBuffer> images, const TileSizePredictor& pred,
                              const WarmupStats& stats, double, PipelineMode mode) {
    if (stats.reference_tile <= 0) throw InvalidInput("warm-up stats missing reference tile");
    std::vector<Task> v;
    for (size_t i = 0; i < images.size(); ++i) {
        const int tile = pred.select_tile_size(images[i]);
        if (tile <= 0) throw InvalidInput("predictor returned invalid tile size");
        Task t;
        t.id = static_cast<int>(i);
        t.tile_size = tile;
        t.latency = stats.latency_for(mode, tile);
        t.memory = stats.memory_for(mode, tile);
        if (t.latency <= 0.0) throw InvalidInput("warm-up stats predict nonpositive latency");
        v.push_back(t);
    }
    return v;
}
StreamSchedule lpt_schedule(std::vector<Task> tasks, int S, double lambda, double m_cap, int b_min, int B) {
    std::vector<qrm::sched::Task> t(tasks.size());
    for (size_t i = 0; i < tasks.size(); ++i)
        t[i] = {tasks[i].id, tasks[i].tile_size, tasks[i].latency, tasks[i].memory, tasks[i].units, tasks[i].mb};
    qrm::sched::Schedule s;
    std::string err;
    const int rc = qrm::sched::lpt_schedule(t, S, lambda, m_cap, b_min, B, s, err);
    if (rc == 1) throw InvalidInput(err);
    if (rc == 3) throw InfeasibleConfig(err);
    StreamSchedule o;
    o.loads = s.loads;
    o.m_unit = s.m_unit;
    for (auto& st : s.streams) {
        o.streams.emplace_back();
        for (auto& x : st) o.streams.back().push_back(Task{x.id, x.tile_size, x.latency, x.memory, x.units, x.mb});
    }
    return o;
}

// ------------------------------------------------------------------ detect
DetectionConfig DetectionConfig::make(const CodeParams& code, const TileSpec& tile, uint64_t key_seed, double alpha,
                                      BitVec key_message) {
    if (static_cast<int>(key_message.size()) != code.message_bits())
        throw InvalidInput("key message length does not match code profile");
    DetectionConfig c;
    c.code = code;
    c.tile = tile;
    c.key = WatermarkKey{key_seed, code.codeword_bits(), alpha};
    c.key_message = std::move(key_message);
    return c;
}
bool semantic_equal(const DetectionRecord& a, const DetectionRecord& b) {
    return a.image_index == b.image_index && a.raw_bits == b.raw_bits && a.corrected == b.corrected &&
           a.errors_corrected == b.errors_corrected && a.bit_acc == b.bit_acc && a.verified == b.verified &&
           a.error == b.error;
}
int verify_threshold(int n_bits, double fpr) {
    const int t = qrm::verify_threshold(n_bits, fpr);
    if (t < 0) throw InvalidInput("verify threshold needs n_bits > 0 and fpr in (0, 1)");
    return t;
}
bool verify(const BitVec& a, const BitVec& b, double fpr) {
    if (a.size() != b.size()) throw InvalidInput("verify inputs differ in length");
    int k = 0;
    for (size_t i = 0; i < a.size(); ++i) k += a[i] == b[i];
    return k >= verify_threshold(static_cast<int>(a.size()), fpr);
}

static std::string cache_key(const BitVec& raw) {
    std::string key((raw.size() + 7) / 8, '\0');  // LSB-first bit packing (detect.cpp:77-82)
    for (size_t i = 0; i < raw.size(); ++i)
        if (raw[i]) key[i / 8] |= static_cast<char>(1 << (i % 8));
    return key;
}
// The codebook keeps its keys in least-recently-used order (lru_), so eviction
// pops from the front instead of scanning the map twice per call as the
// reference does (detect.cpp:115-128). The evicted set is the same: entries
// past stale_after are exactly a prefix of that order (the oldest), and the
// capacity rule then removes the oldest one at a time.
bool CorrectionCache::record(const BitVec& raw, const std::optional<DecodeResult>& decoded) {
    return record(raw, [&] { return decoded; });
}
bool CorrectionCache::record(const BitVec& raw, const std::function<std::optional<DecodeResult>()>& decoded_on_miss) {
    return record_key(cache_key(raw), decoded_on_miss);
}
static std::string packed_key(uint64_t raw_word, int n_bits) {
    // the same key as cache_key(unpack(raw_word)): bit i of the BitVec is word
    // bit n-1-i, packed LSB-first into bytes
    uint64_t lsb_first = 0;
    for (int i = 0; i < n_bits; ++i) lsb_first |= ((raw_word >> (n_bits - 1 - i)) & 1ull) << i;
    std::string key(static_cast<size_t>((n_bits + 7) / 8), '\0');
    for (size_t b = 0; b < key.size(); ++b) key[b] = static_cast<char>((lsb_first >> (8 * b)) & 0xff);
    return key;
}
bool CorrectionCache::record_packed(uint64_t raw_word, int n_bits,
                                    const std::function<std::optional<DecodeResult>()>& decoded_on_miss) {
    return record_key(packed_key(raw_word, n_bits), decoded_on_miss);
}
void CorrectionCache::record_packed_batch(const uint64_t* raw_words, size_t count, size_t word_stride, int n_bits,
                                          const std::function<std::optional<DecodeResult>(size_t)>& decoded_on_miss,
                                          uint8_t* hit) {
    std::lock_guard<std::mutex> lk(mu_);  // one lock for the whole batch
    uint64_t prev = 0;
    std::string key;
    for (size_t i = 0; i < count; ++i) {
        const uint64_t w = raw_words[i * word_stride];
        if (i == 0 || w != prev) key = packed_key(w, n_bits);
        prev = w;
        ++tick_;
        ++lookups_;
        evict_locked();
        auto it = map_.find(key);
        if (it != map_.end()) {
            ++hits_;
            touch_locked(it->second);
            hit[i] = 1;
            continue;
        }
        insert_locked(key, decoded_on_miss(i));
        evict_locked();
        hit[i] = 0;
    }
}
bool CorrectionCache::record_key(std::string key, const std::function<std::optional<DecodeResult>()>& decoded_on_miss) {
    // correct()'s bookkeeping with the decode already done on the GPU
    std::lock_guard<std::mutex> lk(mu_);
    ++tick_;
    ++lookups_;
    evict_locked();
    auto it = map_.find(key);
    if (it != map_.end()) {
        ++hits_;
        touch_locked(it->second);
        return true;
    }
    insert_locked(std::move(key), decoded_on_miss());
    evict_locked();
    return false;
}
std::pair<std::optional<DecodeResult>, bool> CorrectionCache::correct(const BitVec& raw, const CodeParams& params) {
    std::string key = cache_key(raw);
    {
        std::lock_guard<std::mutex> lk(mu_);
        ++tick_;
        ++lookups_;
        evict_locked();
        auto it = map_.find(key);
        if (it != map_.end()) {
            ++hits_;
            touch_locked(it->second);
            return {it->second.result, true};
        }
    }
    auto res = bw_decode(raw, params);
    std::lock_guard<std::mutex> lk(mu_);
    insert_locked(std::move(key), res);
    evict_locked();
    return {std::move(res), false};
}
void CorrectionCache::touch_locked(Entry& e) {
    lru_.splice(lru_.end(), lru_, e.pos);
    e.pos->last_access = tick_;
}
void CorrectionCache::insert_locked(std::string key, std::optional<DecodeResult> result) {
    auto [it, ins] = map_.try_emplace(std::move(key));
    if (ins) it->second.pos = lru_.insert(lru_.end(), LruNode{it->first, tick_});
    it->second.result = std::move(result);
    touch_locked(it->second);
}
void CorrectionCache::evict_locked() {
    // the oldest entry is at the front; no map lookup unless it goes
    while (!lru_.empty()) {
        const LruNode& old = lru_.front();
        if (tick_ - old.last_access <= cfg_.stale_after && map_.size() <= cfg_.capacity) break;
        map_.erase(old.key);
        lru_.pop_front();
    }
}
size_t CorrectionCache::size() const {
    std::lock_guard<std::mutex> lk(mu_);
    return map_.size();
}

ImageBuffer read_ppm(const std::filesystem::path& path) {
    int w = 0, h = 0;
    const std::string p = path.string();
    check(qrm_ppm_read(p.c_str(), nullptr, 0, &w, &h));
    ImageBuffer img = ImageBuffer::make_byte(w, h);
    check(qrm_ppm_read(p.c_str(), img.bytes.data(), static_cast<int64_t>(img.bytes.size()), &w, &h));
    return img;
}
void write_ppm(const ImageBuffer& img, const std::filesystem::path& path) {
    if (img.form != PixelForm::byte) throw InvalidInput("write_ppm expects byte form");
    check(qrm_ppm_write(path.string().c_str(), img.bytes.data(), img.width, img.height));
}

static qrm_config gpu_config(const DetectionConfig& cfg) {
    qrm_config c{};
    c.symbol_bits = cfg.code.field->bits();
    c.n = cfg.code.n;
    c.k = cfg.code.k;
    c.tile_size = cfg.tile.size;
    c.tile_strategy = static_cast<int>(cfg.tile.strategy);  // random 0, random_grid 1, fixed 2
    c.tile_seed = cfg.tile.seed;
    c.key_seed = cfg.key.seed;
    c.alpha = cfg.key.alpha;
    c.key_message = cfg.key_message.data();
    c.fpr_target = cfg.fpr_target;
    return c;
}

namespace {

// Process-wide pool of C-ABI contexts keyed by (device, configuration). The
// reference builds a fresh DetectionContext for every detect_batch call
// (detect.cpp:254). Its device counterpart -- pattern planes, RS tables, the
// streams, the pinned window-staging ring (~50 MB per decode slot) -- depends
// only on the configuration, so a context returned by one call is handed to
// the next call with the same key instead of being rebuilt. A context is used
// by one DetectionContext at a time. Idle contexts are bounded; the pool is
// never destroyed (tearing down CUDA state during static destruction is unsafe).
class CtxPool {
public:
    static CtxPool& get() {
        static CtxPool* p = new CtxPool;
        return *p;
    }
    static std::string key_of(const DetectionConfig& cfg, int device) {
        std::string k = std::to_string(device) + "/" + std::to_string(cfg.code.field->bits()) + "/" +
                        std::to_string(cfg.code.n) + "/" + std::to_string(cfg.code.k) + "/" +
                        std::to_string(cfg.tile.size) + "/" + std::to_string(static_cast<int>(cfg.tile.strategy)) +
                        "/" + std::to_string(cfg.tile.seed) + "/" + std::to_string(cfg.key.seed) + "/" +
                        std::to_string(cfg.key.alpha) + "/" + std::to_string(cfg.fpr_target) + "/" +
                        std::to_string(static_cast<int>(cfg.extractor)) + "/" + std::to_string(cfg.conv_weight_seed) +
                        "/";
        for (uint8_t b : cfg.key_message) k.push_back(static_cast<char>('0' + (b & 1)));
        return k;
    }
    qrm_ctx* acquire(const DetectionConfig& cfg, int device, const std::string& key) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (auto it = idle_.begin(); it != idle_.end(); ++it)
                if (it->first == key) {
                    qrm_ctx* c = it->second;
                    idle_.erase(it);
                    return c;
                }
        }
        qrm_config c = gpu_config(cfg);
        qrm_ctx* h = nullptr;
        check(qrm_ctx_create(device, &c, &h));
        if (cfg.extractor == ExtractorKind::conv) {
            const qrm_status s = qrm_ctx_set_extractor(h, QRM_EXTRACTOR_CONV, cfg.conv_weight_seed);
            if (s != QRM_OK) {
                qrm_ctx_destroy(h);
                raise(s);
            }
        }
        return h;
    }
    void release(const std::string& key, qrm_ctx* c) {
        if (!c) return;
        qrm_ctx* evict = nullptr;
        {
            std::lock_guard<std::mutex> lk(mu_);
            idle_.emplace_back(key, c);
            if (idle_.size() > kMaxIdle) {
                evict = idle_.front().second;
                idle_.erase(idle_.begin());
            }
        }
        if (evict) qrm_ctx_destroy(evict);
    }

private:
    static constexpr size_t kMaxIdle = 8;
    std::mutex mu_;
    std::vector<std::pair<std::string, qrm_ctx*>> idle_;  // oldest first
};

}  // namespace

struct GpuContext {
    std::string key;
    qrm_ctx* h = nullptr;
    // one per DetectionConfig::devices entry (multi-device batches), created on first use
    std::vector<std::string> shard_keys;
    std::vector<qrm_ctx*> shards;
    ~GpuContext() {
        for (size_t i = 0; i < shards.size(); ++i) CtxPool::get().release(shard_keys[i], shards[i]);
        CtxPool::get().release(key, h);
    }
};

DetectionContext::DetectionContext(const DetectionConfig& cfg, int device)
    : cfg_(cfg),
      codec_(cfg.key, cfg.tile.size),
      key_codeword_(rs_encode(cfg.key_message, cfg.code)),
      tau_message_(verify_threshold(cfg.code.message_bits(), cfg.fpr_target)),
      tau_raw_(verify_threshold(cfg.code.codeword_bits(), cfg.fpr_target)),
      cache_(cfg.cache),
      gpu_(nullptr) {
    // validate before any device state is taken (a throw here leaks nothing)
    if (cfg.key.n_bits != cfg.code.codeword_bits())
        throw InvalidInput("key payload width must equal the codeword width");
    if (cfg.rs_workers < 1) throw InvalidInput("rs_workers must be >= 1");
    if (cfg.fpr_target <= 0.0 || cfg.fpr_target >= 1.0) throw InvalidInput("fpr target must be in (0, 1)");
    auto g = std::make_unique<GpuContext>();
    g->key = CtxPool::key_of(cfg_, device);
    g->h = CtxPool::get().acquire(cfg_, device, g->key);
    gpu_ = g.release();
}
DetectionContext::~DetectionContext() { delete gpu_; }

// Host threads that turn device records into DetectionRecords (large batches).
static qrm::HostPool& conversion_pool() {
    static qrm::HostPool* pool = [] {
        const unsigned hc = std::thread::hardware_concurrency();
        return new qrm::HostPool(static_cast<int>(std::max(1u, std::min(hc ? hc - 2 : 1u, 15u))));
    }();
    return *pool;
}

static DetectionRecord to_record(const qrm_record& r, size_t index, const DetectionConfig& cfg) {
    DetectionRecord d;
    const int nb = cfg.code.codeword_bits(), kb = cfg.code.message_bits();
    d.image_index = index;
    d.raw_bits = unpack(r.raw, nb);
    if (r.status == QRM_REC_DECODED) {
        d.corrected = unpack(r.msg, kb);
        d.errors_corrected = r.errors;
    }
    d.bit_acc = static_cast<double>(r.matches) / static_cast<double>(nb);
    d.verified = r.verified != 0;
    return d;
}

// The reference's StreamPlan (sched.hpp:26-34) as the executor's plan: streams
// per stage, and the mini-batch = the largest stage mini-batch (detect_batch
// sizes its queues by the largest entry, detect.cpp:266).
static qrm_plan to_gpu_plan(const StreamPlan* plan) {
    qrm_plan pl{{1, 2, 1}, {4096, 4096, 4096}};
    if (!plan) return pl;
    if (plan->streams.size() != 3) throw InvalidInput("detect pipeline expects a 3-stage plan");
    for (int k = 0; k < 3; ++k) pl.streams[k] = std::max(1, plan->streams[k]);
    if (!plan->minibatch.empty()) {
        const int mb = std::max(1, *std::max_element(plan->minibatch.begin(), plan->minibatch.end()));
        for (int k = 0; k < 3; ++k) pl.minibatch[k] = mb;
    }
    return pl;
}

std::vector<DetectionRecord> DetectionContext::detect_many(std::span<const ImageBuffer> images, uint64_t first_draw,
                                                           const StreamPlan* plan, const SyntheticStageLoad* load,
                                                           DeskReport* report) {
    const auto wall0 = std::chrono::steady_clock::now();
    const int64_t n = static_cast<int64_t>(images.size());
    const qrm_plan pl = to_gpu_plan(plan);
    std::vector<DetectionRecord> out(n);
    if (report) {
        *report = DeskReport{};
        for (int k = 0; k < 3; ++k) report->stage_workers[k] = pl.streams[k];
    }
    if (n == 0) return out;
    bool uniform = true;
    for (const ImageBuffer& im : images) {
        if (im.form != PixelForm::byte) throw InvalidInput("preprocess expects byte form");
        uniform = uniform && im.width == images[0].width && im.height == images[0].height;
    }
    const int w = images[0].width, h = images[0].height;
    const bool direct = uniform && std::min(w, h) >= kWorkingSize;  // no bilinear upscale
    qrm_stage_load ld{{0, 0, 0}};
    if (load) {
        ld.ns[0] = load->preprocess_ns;
        ld.ns[1] = load->extract_ns;
        ld.ns[2] = load->correct_ns;
        if (!direct && (ld.ns[0] || ld.ns[1] || ld.ns[2]))
            throw InvalidInput("a synthetic stage load needs same-size images of at least 256 px (the stage pipeline)");
    }
    std::vector<qrm_record> rec(n);
    std::vector<int64_t> image_ns(direct ? 3 * n : 0, 0);
    int64_t busy[3] = {0, 0, 0};
    if (direct) {
        // Only each image's l x l window leaves its ImageBuffer: the context's host
        // workers gather the windows into its pinned staging ring (no whole-image
        // copy, no per-call pinned allocation), the copy engine moves them.
        std::vector<const uint8_t*> ptrs(n);
        for (int64_t i = 0; i < n; ++i) ptrs[i] = images[i].bytes.data();
        if (cfg_.devices.size() > 1 && gpu_->shards.empty())
            for (int dev : cfg_.devices) {
                gpu_->shard_keys.push_back(CtxPool::key_of(cfg_, dev));
                gpu_->shards.push_back(nullptr);
                gpu_->shards.back() = CtxPool::get().acquire(cfg_, dev, gpu_->shard_keys.back());
            }
        const int nctx = gpu_->shards.size() > 1 ? static_cast<int>(gpu_->shards.size()) : 1;
        // contiguous shards with global draw indices, one host thread per device
        std::vector<qrm_status> st(nctx, QRM_OK);
        std::vector<std::string> err(nctx);
        std::vector<qrm_stage_times> tm(nctx);
        auto run = [&](int i) {
            const int64_t b = n * i / nctx, e = n * (i + 1) / nctx;
            tm[i] = qrm_stage_times{0, {0, 0, 0}, image_ns.data() + 3 * b};
            qrm_ctx* c = nctx > 1 ? gpu_->shards[i] : gpu_->h;
            st[i] = qrm_detect_host_images(c, ptrs.data() + b, e - b, w, h, first_draw + static_cast<uint64_t>(b),
                                           rec.data() + b, &pl, &ld, &tm[i]);
            if (st[i] != QRM_OK) err[i] = qrm_last_error();
        };
        std::vector<std::thread> th;
        for (int i = 1; i < nctx; ++i) th.emplace_back(run, i);
        run(0);
        for (auto& t : th) t.join();
        for (int i = 0; i < nctx; ++i) {
            if (st[i] != QRM_OK) {
                const std::string msg = (nctx > 1 ? "shard " + std::to_string(i) + ": " : std::string()) + err[i];
                if (st[i] == QRM_INVALID_INPUT) throw InvalidInput(msg);
                if (st[i] == QRM_INFEASIBLE) throw InfeasibleConfig(msg);
                throw CudaUnavailable(msg);
            }
            for (int k = 0; k < 3; ++k) busy[k] += tm[i].busy_ns[k];
        }
    } else {
        std::vector<const uint8_t*> ptrs(n);
        std::vector<int> ws(n), hs(n);
        for (int64_t i = 0; i < n; ++i) {
            ptrs[i] = images[i].bytes.data();
            ws[i] = images[i].width;
            hs[i] = images[i].height;
        }
        const auto r0 = std::chrono::steady_clock::now();
        check(qrm_detect_ragged(gpu_->h, ptrs.data(), ws.data(), hs.data(), n, first_draw, rec.data()));
        // one fused gather + decode + correct call: the whole span is the decode stage's
        busy[1] = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - r0).count();
    }
    // Records -> DetectionRecords on the conversion pool while this thread
    // replays the codebook (index order, as the reference's cache sees the words
    // with one correct worker; it reads only the packed words).
    auto convert = [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            out[i] = to_record(rec[i], first_draw + i, cfg_);
            if (direct) out[i].stage_ns = StageLatencies{image_ns[3 * i], image_ns[3 * i + 1], image_ns[3 * i + 2]};
        }
    };
    std::vector<uint8_t> hit(cfg_.cache.enabled ? n : 0, 0);
    auto replay = [&] {
        const int kb = cfg_.code.message_bits();
        cache_.record_packed_batch(
            &rec[0].raw, static_cast<size_t>(n), sizeof(qrm_record) / sizeof(uint64_t), cfg_.code.codeword_bits(),
            [&](size_t i) -> std::optional<DecodeResult> {
                if (rec[i].status != QRM_REC_DECODED) return std::nullopt;  // stored only on a miss
                BitVec m = unpack(rec[i].msg, kb);
                BitVec cw = rs_encode(m, cfg_.code);
                return DecodeResult{std::move(m), std::move(cw), rec[i].errors};
            },
            hit.data());
    };
    if (n >= 1024) {
        std::thread rt;
        if (cfg_.cache.enabled) rt = std::thread(replay);
        conversion_pool().parallel_for(n, 256, convert);
        if (rt.joinable()) rt.join();
    } else {
        convert(0, n);
        if (cfg_.cache.enabled) replay();
    }
    if (cfg_.cache.enabled)
        for (int64_t i = 0; i < n; ++i) out[i].cache_hit = hit[i] != 0;
    if (report) {
        report->wall_ns =
            std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - wall0).count();
        for (int k = 0; k < 3; ++k) report->stage_busy_ns[k] = busy[k];
        report->items = static_cast<size_t>(n);
    }
    return out;
}

DetectionRecord DetectionContext::detect_one(const ImageBuffer& img, uint64_t draw_index) {
    return detect_many(std::span<const ImageBuffer>(&img, 1), draw_index)[0];
}
DetectionRecord detect_one(const ImageBuffer& img, const DetectionConfig& cfg) {
    DetectionContext ctx(cfg);
    return ctx.detect_one(img, 0);
}

std::vector<DetectionRecord> detect_batch(std::span<const ImageBuffer> images, const DetectionConfig& cfg,
                                          const StreamPlan* plan, const SyntheticStageLoad* load, DeskReport* report) {
    DetectionContext ctx(cfg);
    if (images.empty()) {  // as the reference: no plan check for an empty batch (detect.cpp:256-260)
        if (report) *report = DeskReport{};
        return {};
    }
    return ctx.detect_many(images, 0, plan, load, report);
}

// --------------------------------------------------------------------- sim
StageProfile measure_stages(std::span<StageBench> stages, int iters, double b0, const std::function<int64_t()>& now_ns) {
    if (iters < 1) throw InvalidInput("need at least one warm-up iteration");
    if (stages.empty()) throw InvalidInput("no stages to measure");
    std::vector<std::function<void()>> runs;
    for (auto& s : stages) runs.push_back(s.run_batch);
    const auto med = qrm::sched::measure_stages(runs, iters, now_ns);
    StageProfile p;
    p.b0 = b0;
    for (size_t k = 0; k < stages.size(); ++k) {
        p.time.push_back(med[k]);
        p.memory.push_back(stages[k].mem_per_sample);
        p.prep.push_back(med[k] * stages[k].prep_share);
        p.names.push_back(stages[k].name);
    }
    return p;
}
StageProfile warmup_profile(std::span<const ImageBuffer> images, int iters, const DetectionConfig& cfg) {
    if (images.empty()) throw InvalidInput("warm-up needs at least one image");
    const int64_t b0 = std::min<int64_t>(static_cast<int64_t>(images.size()), 16);
    const int w = images[0].width, h = images[0].height;
    const size_t bytes = static_cast<size_t>(w) * h * 3;
    std::vector<uint8_t> packed(bytes * b0);
    for (int64_t i = 0; i < b0; ++i) {
        if (images[i].form != PixelForm::byte || images[i].width != w || images[i].height != h)
            throw InvalidInput("warm-up images must share one byte-form size");
        std::memcpy(packed.data() + i * bytes, images[i].bytes.data(), bytes);
    }
    DetectionContext ctx(cfg);
    double t[3], m[3];
    check(qrm_warmup_profile(ctx.gpu()->h, packed.data(), b0, w, h, static_cast<int64_t>(bytes), iters,
                             static_cast<int>(b0), t, m));
    StageProfile p;
    p.b0 = static_cast<double>(b0);
    p.time.assign(t, t + 3);
    p.memory.assign(m, m + 3);
    p.prep.assign(3, 0.0);
    p.names = {"transfer", "decode", "correct"};
    return p;
}
std::pair<std::vector<DetectionRecord>, DeskReport> run_desk(const StreamPlan& plan, std::span<const ImageBuffer> images,
                                                             const DetectionConfig& cfg, const SyntheticStageLoad* load) {
    DeskReport rep;
    auto recs = detect_batch(images, cfg, &plan, load, &rep);
    return {std::move(recs), rep};
}

}  // namespace qrmark
