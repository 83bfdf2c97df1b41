// reduce_scan.cuh -- single-pass reduce / mapreduce and decoupled look-back scan.
#pragma once

#include <cstdint>

#include "ak_common.cuh"
#include "ctx.cuh"

namespace akb {

enum red_op : int { OP_SUM = 0, OP_MIN = 1, OP_MAX = 2 };
enum red_map : int { MAP_IDENTITY = 0, MAP_ABS = 1, MAP_SQUARE = 2 };

// Accumulator type: floats accumulate in double (the f32 oracle contract,
// SURVEY.md §8(a9)); integers in their own width with wrap-around.
template <typename T>
struct acc_of {
    using type = T;
};
template <>
struct acc_of<float> {
    using type = double;
};

// reduce.hpp:24-75 -- result written to *d_result (device) as T.
template <typename T>
void reduce(ak_ctx* c, const T* x, std::uint64_t n, int op, int map, T init, T* d_result);

// scan.hpp:29-79 -- out may alias x (in-place).
template <typename T>
void scan(ak_ctx* c, const T* x, T* out, std::uint64_t n, int op, int inclusive, T init);

}  // namespace akb
