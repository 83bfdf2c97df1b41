// predicates.cuh -- any_pred / all_pred (reference include/ak/predicates.hpp:16-78).
#pragma once

#include <cstdint>

#include "ak_common.cuh"
#include "ctx.cuh"

namespace akb {

// Enumerated element predicates x OP v (callables cannot cross the C ABI).
enum pred_op : int { PRED_LT = 0, PRED_LE = 1, PRED_GT = 2, PRED_GE = 3, PRED_EQ = 4, PRED_NE = 5 };

// True iff some element has (x OP v) == want: any_pred = find(want=true),
// all_pred = !find(want=false) (predicates.hpp:24-52). early = poll-and-stop variant.
template <typename T>
bool find_decider(ak_ctx* c, const T* x, std::uint64_t n, int op, T v, bool want, bool early);

}  // namespace akb
