// search_merge.cuh -- searchsorted (K5), sample gather (K6), stable 2-way merge (K8).
#pragma once

#include <cstdint>

#include "ak_common.cuh"
#include "ctx.cuh"

namespace akb {

// search.hpp:16-50: out[i] = #hay < needle (first) or #hay <= needle (last).
template <typename T>
void searchsorted(ak_ctx* c, const T* hay, std::uint64_t n, const T* needles, std::uint64_t m,
                  int side_last, int desc, std::uint64_t* d_out);

// sample_local positions of sihsort.hpp:264-282 computed on the device, plus
// data[0] and data[n-1]: out = [data[0], data[n-1], samples...]. Returns k.
template <typename T>
std::uint64_t gather_samples(ak_ctx* c, const T* sorted, std::uint64_t n, std::uint64_t k, T* d_out);

// Stable merge of a (na) and b (nb) into dst (na+nb); a wins ties
// (sort.hpp:92-117 semantics, merge-path partitioned, co_rank sort.hpp:75-88).
template <typename T>
void merge2(ak_ctx* c, const T* a, std::uint64_t na, const T* b, std::uint64_t nb, T* dst,
            bool desc);

// Stable P-way merge of sorted runs (run order breaks ties: the stable sort of their
// concatenation); scratch: >= total elements of device memory.
constexpr int MW_MAXP = 4096;  // runs per merge_runs call (C ABI bound)
template <typename T>
void merge_runs(ak_ctx* c, int P, const T* const* runs, const std::uint64_t* lens, T* dst, T* scratch, bool desc);

// Is the device array nondecreasing under the comparator? (search.hpp:40-43 validate)
template <typename T>
bool is_sorted(ak_ctx* c, const T* x, std::uint64_t n, bool desc);

}  // namespace akb
