#include "host_code.hpp"

#include <cmath>
#include <cstring>
#include <mutex>

namespace qrm {

HostField::HostField(int m_) : m(m_), q1((1 << m_) - 1), poly(m_ == 4 ? 0x13u : 0x11Du) {
    // alpha = 2 generates the multiplicative group (gf.cpp:7-18 builds the same tables).
    exp.assign(q1, 0);
    log.assign(q1 + 1, 0);
    uint32_t v = 1;
    for (int i = 0; i < q1; ++i) {
        exp[i] = static_cast<uint16_t>(v);
        log[v] = static_cast<uint16_t>(i);
        v <<= 1;
        if (v >> m) v ^= poly;
    }
}

uint16_t HostField::mul(uint16_t a, uint16_t b) const {
    if (!a || !b) return 0;
    return exp[(log[a] + log[b]) % q1];
}

uint16_t HostField::inv(uint16_t a) const { return exp[(q1 - log[a]) % q1]; }

const HostField& host_field(int m) {
    static const HostField f4(4), f8(8);
    return m == 4 ? f4 : f8;
}

std::string check_code(int m, int n, int k) {
    if (m != 4 && m != 8) return "symbol size must be 4 (GF(16)) or 8 (GF(256))";
    const int q1 = (1 << m) - 1;
    if (n > q1) return "codeword length exceeds field bound";
    if (k <= 0 || k >= n) return "message length must satisfy 0 < k < n";
    return "";
}

namespace {

std::vector<uint16_t> eval_points(const HostField& f, int n) {
    std::vector<uint16_t> X(n);
    for (int i = 0; i < n; ++i) X[i] = f.exp[i % f.q1];  // X_i = alpha^i (rs.cpp:60)
    return X;
}

// G[i][l] = L_i(X_l): the Lagrange basis of the first k points evaluated at X_l.
std::vector<std::vector<uint16_t>> generator(const HostField& f, int n, int k) {
    auto X = eval_points(f, n);
    std::vector<std::vector<uint16_t>> G(k, std::vector<uint16_t>(n, 0));
    for (int i = 0; i < k; ++i) {
        uint16_t den = 1;
        for (int j = 0; j < k; ++j)
            if (j != i) den = f.mul(den, X[i] ^ X[j]);
        const uint16_t dinv = f.inv(den);
        for (int l = 0; l < n; ++l) {
            uint16_t num = 1;
            for (int j = 0; j < k; ++j)
                if (j != i) num = f.mul(num, X[l] ^ X[j]);
            G[i][l] = f.mul(num, dinv);
        }
    }
    return G;
}

}  // namespace

std::vector<uint16_t> encode_symbols(int m, int n, int k, const std::vector<uint16_t>& msg) {
    const HostField& f = host_field(m);
    auto G = generator(f, n, k);
    std::vector<uint16_t> cw(n, 0);
    for (int l = 0; l < n; ++l)
        for (int i = 0; i < k; ++i) cw[l] ^= f.mul(msg[i], G[i][l]);
    return cw;
}

uint64_t encode_packed(int m, int n, int k, uint64_t message) {
    std::vector<uint16_t> msg(k);
    const uint64_t smask = (1ull << m) - 1;
    for (int i = 0; i < k; ++i) msg[i] = static_cast<uint16_t>((message >> (m * (k - 1 - i))) & smask);
    auto cw = encode_symbols(m, n, k, msg);
    uint64_t w = 0;
    for (int i = 0; i < n; ++i) w = (w << m) | cw[i];
    return w;
}

std::vector<uint64_t> build_encoder_masks(int m, int n, int k) {
    const int rb = (n - k) * m, kb = k * m;
    std::vector<uint64_t> masks(rb, 0);
    for (int b = 0; b < kb; ++b) {
        const uint64_t cw = encode_packed(m, n, k, 1ull << b);
        const uint64_t par = rb == 64 ? cw : (cw & ((1ull << rb) - 1));
        for (int pb = 0; pb < rb; ++pb)
            if ((par >> pb) & 1) masks[pb] |= 1ull << b;
    }
    return masks;
}

void build_rs_tables(int m, int n, int k, RsTables& T) {
    std::memset(&T, 0, sizeof T);
    const HostField& f = host_field(m);
    T.m = m;
    T.n = n;
    T.k = k;
    T.t = (n - k) / 2;
    T.r = n - k;
    T.q1 = f.q1;
    T.packed_ok = n * m <= 64;
    for (int i = 0; i < 2 * f.q1 && i < 512; ++i) T.exp2[i] = static_cast<uint8_t>(f.exp[i % f.q1]);
    for (int v = 1; v <= f.q1; ++v) T.log[v] = static_cast<uint8_t>(f.log[v]);
    auto X = eval_points(f, n);
    // GRS column multipliers v_i = 1 / prod_{l != i} (X_i - X_l).
    for (int i = 0; i < n; ++i) {
        uint16_t p = 1;
        for (int l = 0; l < n; ++l)
            if (l != i) p = f.mul(p, X[i] ^ X[l]);
        T.logv[i] = static_cast<uint8_t>(f.log[f.inv(p)]);
    }
    // Packed syndrome masks (only when a word fits 64 bits and n-k small).
    T.nmask = 0;
    if (T.packed_ok && T.r * m <= 64) {
        T.nmask = T.r * m;
        const int nb = n * m;
        for (int w = 0; w < nb; ++w) {
            const int b = nb - 1 - w;  // BitVec index of word bit w
            const int i = b / m;
            const uint16_t ri = static_cast<uint16_t>(1u << (m - 1 - b % m));
            const uint16_t vi = f.exp[T.logv[i]];
            uint16_t h = f.mul(ri, vi);  // r_i v_i X_i^j, j = 0..r-1
            for (int j = 0; j < T.r; ++j) {
                for (int e = 0; e < m; ++e)
                    if ((h >> e) & 1) T.synd_mask[j * m + e] |= 1ull << w;
                h = f.mul(h, X[i]);
            }
        }
    }
}

int verify_threshold(int n_bits, double fpr) {
    // Smallest tau with sum_{j >= tau} C(N, j) 2^-N <= fpr; exact integer tail for
    // N <= 64, log-gamma tail above (detect.cpp:31-66).
    if (n_bits <= 0 || !(fpr > 0.0) || !(fpr < 1.0)) return -1;
    int tau = n_bits + 1;
    if (n_bits <= 64) {
        const long double bound = static_cast<long double>(fpr) * std::pow(2.0L, static_cast<long double>(n_bits));
        unsigned __int128 binom = 1, tail = 0;
        for (int j = n_bits; j >= 0; --j) {
            tail += binom;
            if (static_cast<long double>(tail) > bound) break;
            tau = j;
            if (j > 0) binom = binom * static_cast<unsigned>(j) / static_cast<unsigned>(n_bits - j + 1);
        }
        return tau;
    }
    const long double ln2 = std::log(2.0L);
    long double tail = 0.0L;
    for (int j = n_bits; j >= 0; --j) {
        tail += std::exp(lgammal(n_bits + 1.0L) - lgammal(j + 1.0L) - lgammal(n_bits - j + 1.0L) - n_bits * ln2);
        if (tail > static_cast<long double>(fpr)) break;
        tau = j;
    }
    return tau;
}

}  // namespace qrm
