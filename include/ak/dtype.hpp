// ak/dtype.hpp -- element-type codes (reference proj/include/ak/dtype.hpp:14-35), B200 build.
//
// Codes 1-6 are the reference's and are part of the SIHS fixture format. This build sorts
// i32/u32/i64/u64/f32/f64 on the device and adds two codes the reference lacks (SURVEY.md
// §8(d) config 5 sorts UInt64): u64 = 7, u32 = 8. i16 and i128 (codes 1 and 4) have the
// device sort family (csrc/wide_keys.cu) but not sihsort / reduce / scan.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <string_view>

namespace ak {

enum class dtype_code : std::uint32_t {
    i16 = 1,
    i32 = 2,
    i64 = 3,
    i128 = 4,
    f32 = 5,
    f64 = 6,
    u64 = 7,  // new in the B200 build
    u32 = 8,  // new in the B200 build
};

inline const char* dtype_name(dtype_code code) {
    switch (code) {
        case dtype_code::i16: return "i16";
        case dtype_code::i32: return "i32";
        case dtype_code::i64: return "i64";
        case dtype_code::i128: return "i128";
        case dtype_code::f32: return "f32";
        case dtype_code::f64: return "f64";
        case dtype_code::u64: return "u64";
        case dtype_code::u32: return "u32";
    }
    return "unknown";
}

inline std::optional<dtype_code> dtype_from_name(std::string_view name) {
    for (std::uint32_t c = 1; c <= 8; ++c) {
        const auto code = static_cast<dtype_code>(c);
        if (name == dtype_name(code)) return code;
    }
    return std::nullopt;
}

inline std::size_t dtype_width(dtype_code code) {
    switch (code) {
        case dtype_code::i16: return 2;
        case dtype_code::i32:
        case dtype_code::u32:
        case dtype_code::f32: return 4;
        case dtype_code::i64:
        case dtype_code::u64:
        case dtype_code::f64: return 8;
        case dtype_code::i128: return 16;
    }
    return 0;
}

template <typename T>
constexpr dtype_code dtype_of();
template <> constexpr dtype_code dtype_of<std::int16_t>() { return dtype_code::i16; }
template <> constexpr dtype_code dtype_of<std::int32_t>() { return dtype_code::i32; }
template <> constexpr dtype_code dtype_of<std::int64_t>() { return dtype_code::i64; }
template <> constexpr dtype_code dtype_of<float>() { return dtype_code::f32; }
template <> constexpr dtype_code dtype_of<double>() { return dtype_code::f64; }
template <> constexpr dtype_code dtype_of<std::uint64_t>() { return dtype_code::u64; }
template <> constexpr dtype_code dtype_of<std::uint32_t>() { return dtype_code::u32; }

}  // namespace ak
