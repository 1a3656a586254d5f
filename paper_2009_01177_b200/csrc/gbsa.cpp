// GBSA instance files at the C ABI: the reference's two formats
// (matrix_io.cpp:92-263, README.md:93-103), restated so that a caller can hand the engine the
// same files the reference's CLI and tests read and write.
//
//   binary  "GBSA" | u16 version = 1 | u32 N | u8 bits (16 or 32) | A00 then A01 upper
//           triangles, each entry (re, im) as signed little-endian `bits`-bit integers on the
//           lattice x * 2^(bits-1) (round half away from zero, clamped to +-(2^(bits-1) - 1))
//   text    "GBSA text 1" / "modes N" / one "re im" line per entry (%.17g: lossless);
//           empty lines are skipped, a trailing CR is ignored, |re|, |im| < 1
//
// Errors carry the reference's codes; ParseError positions (byte offset for binary, 1-based
// line number for text) go to tor_error.pivot_row.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/tor_capi.h"
#include "host.hpp"

namespace tor {

namespace {

constexpr char kTextMagic[] = "GBSA text 1";
constexpr uint16_t kVersion = 1;

HostError parse_error(const char* code, const char* msg, uint64_t pos) {
    HostError h(TOR_E_PARSE, code, msg);
    h.pivot_row = static_cast<int64_t>(pos);
    return h;
}

void check_bits(int bits) {
    if (bits != 16 && bits != 32) throw HostError(TOR_E_INVALID, "matrixio/bits", "quantization width must be 16 or 32");
}

size_t tri_entries(int n) { return static_cast<size_t>(n) * (n + 1) / 2; }

Input load_binary(const uint8_t* b, size_t len) {
    if (len < 6) throw parse_error("matrixio/truncated", "file ends inside the version field", 4);
    if (static_cast<uint16_t>(b[4] | (b[5] << 8)) != kVersion)
        throw parse_error("matrixio/version", "unsupported format version", 4);
    if (len < 11) throw parse_error("matrixio/truncated", "file ends inside the header", len);
    uint32_t n = 0;
    for (int i = 0; i < 4; ++i) n |= static_cast<uint32_t>(b[6 + i]) << (8 * i);
    const int bits = b[10];
    if (bits != 16 && bits != 32) throw parse_error("matrixio/format", "entry width must be 16 or 32 bits", 10);
    if (n < 1 || n > 4096) throw parse_error("matrixio/dim", "mode count out of range", 6);
    const size_t tri = tri_entries(static_cast<int>(n)), nb = static_cast<size_t>(bits / 8);
    if (len < 11 + tri * 4 * nb) throw parse_error("matrixio/truncated", "file ends inside the entry data", len);
    Input a;
    a.n = static_cast<int>(n);
    const double unit = quant_unit(bits);
    size_t pos = 11;
    auto get = [&]() {
        uint64_t u = 0;
        for (size_t i = 0; i < nb; ++i) u |= static_cast<uint64_t>(b[pos + i]) << (8 * i);
        pos += nb;
        const int64_t v = bits == 16 ? static_cast<int16_t>(u) : static_cast<int32_t>(u);
        return static_cast<double>(v) * unit;
    };
    for (auto* t : {&a.a00, &a.a01}) {
        t->resize(tri);
        for (auto& v : *t) {
            const double re = get();
            v = {re, get()};
        }
    }
    return a;
}

Input load_text(const uint8_t* b, size_t len) {
    size_t off = 0, lineno = 0;
    std::string line;
    auto next_line = [&]() {  // next non-empty line (CR stripped); lineno counts every line
        while (off < len) {
            const size_t e = static_cast<size_t>(std::find(b + off, b + len, '\n') - b);
            line.assign(reinterpret_cast<const char*>(b) + off, e - off);
            off = e < len ? e + 1 : len;
            ++lineno;
            if (!line.empty() && line.back() == '\r') line.pop_back();
            if (!line.empty()) return true;
        }
        return false;
    };
    if (!next_line() || line != kTextMagic) throw parse_error("matrixio/magic", "first line must be 'GBSA text 1'", 1);
    if (!next_line()) throw parse_error("matrixio/truncated", "missing 'modes N' line", lineno + 1);
    int n = 0;
    if (std::sscanf(line.c_str(), "modes %d", &n) != 1 || n < 1 || n > 4096)
        throw parse_error("matrixio/dim", "expected 'modes N' with 1 <= N <= 4096", lineno);
    Input a;
    a.n = n;
    for (auto* t : {&a.a00, &a.a01}) {
        t->resize(tri_entries(n));
        for (auto& v : *t) {
            if (!next_line()) throw parse_error("matrixio/truncated", "file ends inside the entry list", lineno + 1);
            double re = 0, im = 0;
            if (std::sscanf(line.c_str(), "%lf %lf", &re, &im) != 2)
                throw parse_error("matrixio/entry", "expected 're im' pair", lineno);
            if (!(std::fabs(re) < 1.0) || !(std::fabs(im) < 1.0))
                throw parse_error("matrixio/range", "entry magnitudes must be < 1", lineno);
            v = {re, im};
        }
    }
    return a;
}

}  // namespace

double quant_unit(int bits) { return std::ldexp(1.0, -(bits - 1)); }

int64_t quantize(double x, int bits) {
    check_bits(bits);
    if (!(std::fabs(x) < 1.0)) throw HostError(TOR_E_INVALID, "matrixio/range", "quantization requires |x| < 1");
    const double scale = std::ldexp(1.0, bits - 1);
    const int64_t q = std::llround(x * scale);  // half away from zero
    const int64_t lim = static_cast<int64_t>(scale) - 1;
    return q < -lim ? -lim : (q > lim ? lim : q);
}

Input load_gbsa(const uint8_t* bytes, size_t len, int* quant_bits) {
    const bool binary = len >= 4 && std::memcmp(bytes, "GBSA", 4) == 0 && !(len >= 5 && bytes[4] == ' ');
    Input a = binary ? load_binary(bytes, len) : load_text(bytes, len);
    if (quant_bits) *quant_bits = binary ? bytes[10] : 0;
    return a;
}

std::string save_gbsa(const Input& a, bool binary, int quant_bits) {
    if (a.n < 1) throw HostError(TOR_E_INVALID, "matrixio/dim", "matrix has no modes");
    const size_t tri = tri_entries(a.n);
    if (a.a00.size() != tri || a.a01.size() != tri)
        throw HostError(TOR_E_INVALID, "matrixio/dim", "triangle storage size mismatch");
    std::string s;
    if (!binary) {
        s = std::string(kTextMagic) + "\nmodes " + std::to_string(a.n) + "\n";
        char buf[64];
        for (const auto* t : {&a.a00, &a.a01})
            for (const auto& v : *t) {
                std::snprintf(buf, sizeof buf, "%.17g %.17g\n", v.real(), v.imag());
                s += buf;
            }
        return s;
    }
    check_bits(quant_bits);
    s = "GBSA";
    s += static_cast<char>(kVersion & 0xff);
    s += static_cast<char>(kVersion >> 8);
    for (int i = 0; i < 4; ++i) s += static_cast<char>((static_cast<uint32_t>(a.n) >> (8 * i)) & 0xff);
    s += static_cast<char>(quant_bits);
    for (const auto* t : {&a.a00, &a.a01})
        for (const auto& v : *t)
            for (const double x : {v.real(), v.imag()}) {
                const uint64_t q = static_cast<uint64_t>(quantize(x, quant_bits));
                for (int i = 0; i < quant_bits / 8; ++i) s += static_cast<char>((q >> (8 * i)) & 0xff);
            }
    return s;
}

}  // namespace tor
