// radix_sort.cuh -- the radix sort family for sm_100a.
//
// Replaces the reference's bottom-up merge sort (sort.hpp:123-170). The stable path (payload
// modes, float keys): one upfront pass computes all D digit histograms (D = key bits / 8),
// then D onesweep passes each read the keys once and write them once -- tiles claimed in
// launch order through an atomic ticket (forward progress), stable half-warp ranking, tile
// digit counts on a decoupled look-back chain (one 64-bit epoch-tagged word per (tile,
// digit)), digit-ordered staging and contiguous per-digit runs. Keys-only 64-bit integers
// take the hybrid (two unstable MSD partition passes + an on-chip counting stage per bucket
// range): equal integer keys are identical bit patterns, so the result equals the stable
// sort's.
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
