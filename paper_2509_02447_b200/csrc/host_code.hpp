// Host-side code construction for the device decoders: GF(2^m) tables,
// GRS column multipliers, packed-syndrome masks, systematic encoder and the
// verification threshold. Pure host C++ (no CUDA types).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "qrm_types.h"

namespace qrm {

struct HostField {
    int m = 0, q1 = 0;
    uint32_t poly = 0;
    std::vector<uint16_t> exp;  // alpha^i, i < q1
    std::vector<uint16_t> log;  // log(v), v in [1, q1]
    explicit HostField(int m_);
    uint16_t mul(uint16_t a, uint16_t b) const;
    uint16_t inv(uint16_t a) const;
};

const HostField& host_field(int m);

// Validates (m, n, k) like CodeParams::make (rs.cpp:52-56). Returns "" or the
// InvalidInput message.
std::string check_code(int m, int n, int k);

// Fills the device table image for code (m, n, k).
void build_rs_tables(int m, int n, int k, RsTables& out);

// Systematic encoder masks for packed words: parity bit b (LSB-indexed within
// the (n-k)*m parity field) = parity(message & enc_mask[b]).
std::vector<uint64_t> build_encoder_masks(int m, int n, int k);

// rs_encode (rs.cpp:78-91) of a packed message (k*m <= 64 bits, n*m <= 64).
uint64_t encode_packed(int m, int n, int k, uint64_t message);

// rs_encode on symbol arrays (any n).
std::vector<uint16_t> encode_symbols(int m, int n, int k, const std::vector<uint16_t>& msg);

// verify_threshold (detect.cpp:31-66). Returns -1 for invalid arguments.
int verify_threshold(int n_bits, double fpr);

// Sets qrm_last_error() for this thread and returns s (defined in capi.cpp).
qrm_status report_error(qrm_status s, const std::string& msg);

}  // namespace qrm
