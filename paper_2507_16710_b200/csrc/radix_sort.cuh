// radix_sort.cuh -- stable onesweep LSD radix sort for sm_100a.
//
// Replaces the reference's bottom-up merge sort (sort.hpp:123-170): both are
// stable, so for every (keys, payload) input the output is identical.
//
// Per sort: one upfront pass computes all D digit histograms (D = key bits / 8),
// then D onesweep passes each read the keys once and write them once:
//   * tiles are claimed in launch order through an atomic tile counter, so a
//     tile's predecessors are always resident (forward progress),
//   * each warp ranks its keys with ballot-based match + per-warp smem digit
//     counters (stable: order = warp, item, lane = input order),
//   * tile digit counts are published to a decoupled look-back chain (one
//     64-bit self-contained word per (tile, digit), epoch tagged),
//   * keys are staged in shared memory in digit order and written out as
//     contiguous per-digit runs (coalesced segments).
#pragma once

#include <cstdint>

#include "ak_common.cuh"
#include "ctx.cuh"

namespace akb {

enum sort_mode : int {
    SORT_KEYS = 0,     // keys only
    SORT_PAIRS = 1,    // keys + payload co-moving (merge_sort_by_key)
    SORT_IOTA = 2,     // keys + index payload synthesised in pass 0 (sortperm)
    SORT_LOWMEM = 3,   // index array only, keys gathered through data[index] (sortperm_lowmem)
};

// Sort n keys from kin into kout (kin may equal kout). kalt: n-element scratch.
// Payload (modes 1-3): vin -> vout with valt scratch (vin ignored for IOTA/LOWMEM).
// For SORT_LOWMEM, kin is the (unmodified) data array; kout/kalt are unused.
// keys_out=false skips the key write of the last pass (sortperm).
template <typename T, typename V>
void radix_sort(ak_ctx* c, int mode, const T* kin, T* kout, T* kalt, const V* vin, V* vout,
                V* valt, std::uint64_t n, bool desc, bool keys_out);

// Scratch the caller must provide for a sort of n keys (beyond kout/kalt/valt):
// none -- look-back and histograms live in the ctx. Exposed for documentation.
std::uint64_t radix_tile_items(int key_bytes, int mode);

// Keys-only 64-bit integer P-way merge (6 <= P <= 16, >= 2^22 keys) by value tiles sorted on
// chip; returns false (nothing done) when it does not apply. Used by merge_runs.
template <typename T>
bool merge_runs_counting(ak_ctx* c, int P, const T* const* runs, const std::uint64_t* lens, T* dst, bool desc);

}  // namespace akb
