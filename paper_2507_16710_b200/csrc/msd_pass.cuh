// msd_pass.cuh -- unstable MSD top-digit partition passes (keys-only 64-bit integers).
#pragma once

#include <cstdint>

#include "ak_common.cuh"
#include "ctx.cuh"

namespace akb {

// One read of the keys: g_hist rows 5..7 (+=, top three 8-bit digits of the ordered key),
// g_joint[0 .. 65536) = the histogram of the top 16 bits, and its exclusive scans:
// g_joint[65536 + b] = start of 16-bit bucket b, g_joint[131072 + d] = start of 8-bit bucket d.
// digit5 = false skips row 5 (the plan then reads it from a separate full histogram if needed).
template <typename T>
void msd_hist(ak_ctx* c, const T* kin, std::uint64_t n, bool desc, std::uint64_t* g_hist, std::uint64_t* g_joint,
              bool digit5);

// Exclusive scan of a 65536-bin histogram g_joint[0 .. 65536) laid out as ctx_msd (16-bit
// bucket starts at +65536, 8-bit bucket starts at +131072); g_hist rows 6 and 7 += the 8-bit
// marginals (g_hist: 8 x 256 u64).
void msd_joint_scan(ak_ctx* c, std::uint64_t* g_joint, std::uint64_t* g_hist);

// Two partition passes (kin -> kmid by the top 8 bits, kmid -> kout by the top 16 bits);
// afterwards kout is ordered by its top 16 bits (order inside a 16-bit bucket arbitrary).
// plan (device, optional): plan[0] != 0 -> both passes return without writing.
template <typename T>
void msd_top16(ak_ctx* c, const T* kin, T* kmid, T* kout, std::uint64_t n, bool desc, const std::uint64_t* g_joint,
               std::uint64_t* cur16, std::uint64_t* cur8, const int* plan = nullptr);

// The largest 16-bit bucket of the last msd_hist (device slot, filled by its joint scan).
inline std::uint64_t* msd_joint_max_slot(std::uint64_t* g_joint) { return g_joint + 2 * 65536 + 256 + 1; }

// Third partition level (n >= 2^29): kin (ordered by its top 16 bits) -> kout ordered by
// its top 24 bits; the 24-bit histogram is built by an extra read of kin (tiles span few
// 16-bit buckets, so it is counted in shared memory), then scanned into 2^24 cursors.
template <typename T>
void msd_level3(ak_ctx* c, const T* kin, T* kout, std::uint64_t n, bool desc);

// One unstable partition pass by the 8-bit digit at plan[1] (device plan, no-op when
// plan[0] != 0); cursors = the digit's exclusive offsets (consumed).
template <typename T>
void msd_digit_pass(ak_ctx* c, const T* kin, T* kout, std::uint64_t n, bool desc, std::uint64_t* cursors,
                    const int* plan);

// Largest bucket after the MSD levels (level 2: 16-bit buckets, 3: 24-bit), on the host.
std::uint64_t msd_max_bucket(ak_ctx* c, int level);

}  // namespace akb
