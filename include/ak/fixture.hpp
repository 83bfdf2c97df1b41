// ak/fixture.hpp -- SIHS per-rank input fixtures (reference proj/include/ak/fixture.hpp,
// format of src/fixture.cpp:24-95), B200 build. Byte-identical layout, little-endian:
// "SIHS" | version u32 (=1) | dtype code u32 | rank u32 | count u64 | count raw elements.
// Codes 1-6 round-trip with the reference in both directions (tests/test_fixture_csv.py
// checks both against the reference compiled in place). The u64 / u32 codes 7 and 8 are this
// build's additions: the reference reader rejects them (it accepts codes 1-6 only).
#pragma once

#include <bit>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ak/dtype.hpp"

namespace ak {

static_assert(std::endian::native == std::endian::little, "SIHS fixtures are little-endian");

struct fixture_header {
    std::uint32_t version = 1;
    dtype_code dtype = dtype_code::i32;
    std::uint32_t rank = 0;
    std::uint64_t count = 0;
};

inline constexpr std::uint32_t fixture_version = 1;

namespace detail {
[[noreturn]] inline void fixture_fail(const std::filesystem::path& p, const std::string& what) {
    throw std::runtime_error("fixture " + p.string() + ": " + what);
}
}  // namespace detail

inline fixture_header read_fixture_header(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) detail::fixture_fail(path, "cannot open for reading");
    unsigned char raw[24];
    in.read(reinterpret_cast<char*>(raw), sizeof raw);
    if (!in) detail::fixture_fail(path, "truncated header");
    if (std::memcmp(raw, "SIHS", 4) != 0) detail::fixture_fail(path, "bad magic (expected SIHS)");
    fixture_header h;
    std::uint32_t code = 0;
    std::memcpy(&h.version, raw + 4, 4);
    std::memcpy(&code, raw + 8, 4);
    std::memcpy(&h.rank, raw + 12, 4);
    std::memcpy(&h.count, raw + 16, 8);
    if (h.version != fixture_version) detail::fixture_fail(path, "unsupported version " + std::to_string(h.version));
    if (code < 1 || code > 8) detail::fixture_fail(path, "unknown dtype code " + std::to_string(code));
    h.dtype = static_cast<dtype_code>(code);
    return h;
}

template <typename T>
void write_fixture(const std::filesystem::path& path, std::uint32_t rank, std::span<const T> elements) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) detail::fixture_fail(path, "cannot open for writing");
    unsigned char raw[24];
    const std::uint32_t version = fixture_version, code = static_cast<std::uint32_t>(dtype_of<T>());
    const std::uint64_t count = elements.size();
    std::memcpy(raw, "SIHS", 4);
    std::memcpy(raw + 4, &version, 4);
    std::memcpy(raw + 8, &code, 4);
    std::memcpy(raw + 12, &rank, 4);
    std::memcpy(raw + 16, &count, 8);
    out.write(reinterpret_cast<const char*>(raw), sizeof raw);
    if (count) out.write(reinterpret_cast<const char*>(elements.data()), static_cast<std::streamsize>(elements.size_bytes()));
    if (!out) detail::fixture_fail(path, "write failed");
}

/// Reads a fixture whose dtype must match T; the header's rank goes to rank_out.
template <typename T>
std::vector<T> read_fixture(const std::filesystem::path& path, std::uint32_t* rank_out = nullptr) {
    const fixture_header h = read_fixture_header(path);
    if (h.dtype != dtype_of<T>())
        detail::fixture_fail(path, std::string("dtype mismatch: file holds ") + dtype_name(h.dtype) + ", expected " +
                                       dtype_name(dtype_of<T>()));
    std::ifstream in(path, std::ios::binary);
    in.seekg(24);
    std::vector<T> out(h.count);
    if (h.count) in.read(reinterpret_cast<char*>(out.data()), static_cast<std::streamsize>(h.count * sizeof(T)));
    if (!in) detail::fixture_fail(path, "truncated payload");
    if (rank_out) *rank_out = h.rank;
    return out;
}

}  // namespace ak
