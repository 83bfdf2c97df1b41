// wide_keys.cuh -- int16 and int128 sort keys (the reference's dtype.hpp:14-21 list).
#pragma once

#include <cstdint>

#include "ak_common.cuh"
#include "ctx.cuh"

namespace akb {

// T = std::int16_t or __int128; V / I = unsigned 32/64-bit payload / index words.
template <typename T>
void wide_merge_sort(ak_ctx* c, T* data, std::uint64_t n, bool desc);
template <typename T, typename V>
void wide_by_key(ak_ctx* c, T* keys, V* payload, std::uint64_t n, bool desc);
template <typename T, typename I>
void wide_sortperm(ak_ctx* c, const T* data, std::uint64_t n, I* out, bool desc);

}  // namespace akb
