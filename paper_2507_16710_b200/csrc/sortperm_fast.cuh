// sortperm_fast.cuh -- sortperm of 32-bit keys as a sort of unique 64-bit composite keys.
#pragma once

#include <cstdint>

#include "ak_common.cuh"
#include "ctx.cuh"

namespace akb {

// out[i] = index of the i-th smallest key (ties by ascending index = the stable sortperm of
// sort.hpp:238-262). Returns false (nothing done) when the path does not apply (n outside
// [2^20, 2^32), or the 16 B/element work arena cannot be allocated).
template <typename T, typename I>
bool sortperm_composite(ak_ctx* c, const T* data, std::uint64_t n, I* out, bool desc);

}  // namespace akb
