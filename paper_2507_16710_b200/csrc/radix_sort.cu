// radix_sort.cu -- the sort kernels (see radix_sort.cuh).
//
// 1. Stable onesweep LSD pass (every payload mode, float keys, small / skewed inputs). Per
//    tile: thread 0 prefetches the launch-order tile into L2 and takes a ticket (tiles are
//    claimed in launch order, so a tile's predecessors are resident); keys (and payload) load
//    warp-striped and their 8-bit digits are packed 4 per register; stable half-warp ranking
//    (count and peer mask in one shared word per digit); the tile's digit counts are
//    published to the decoupled look-back chain after ranking; digit-ordered staging in shared
//    memory (a 4 + 4-byte (key, payload) pair as one 8-byte slot); windowed look-back (4
//    predecessors per round trip); contiguous per-digit runs written out. Tile shapes per
//    (key, payload) size: the AKB_OS_* knobs below.
// 2. Keys-only 64-bit integers (hybrid_sort_keys): a device-planned two-level unstable MSD
//    partition (msd_pass.cu), then a counting stage sorts every bucket range on chip --
//    local_count3_kernel (ranges <= 4608 keys, 2 CTAs per SM, TMA double-buffered) or
//    local_big_kernel (<= 18432 keys, one CTA per SM, n ~2^29..2^30); the rare clustered
//    range falls back to the stable on-chip radix (local_redo_kernel), oversized ranges to a
//    segment LSD. Small sorts (n <= 2^21) run a device-planned one-pass variant as a CUDA graph.
// 3. merge_runs_counting: SIHSort's P-way merge of 64-bit integer runs by value tiles sorted
//    with the counting stage.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "radix_sort.cuh"
#include "tma.cuh"
#include "msd_pass.cuh"
#include "search_merge.cuh"

namespace akb {

namespace {

constexpr int RADIX = 256;
constexpr std::uint32_t FULL = 0xffffffffu;

#ifndef AKB_OS_MINB
#define AKB_OS_MINB 2  // resident pass CTAs per SM the register budget is sized for
#endif
#ifndef AKB_OS_ITEMS
#define AKB_OS_ITEMS 16  // keys per thread of a keys-only pass tile
#endif
// 4 + 4-byte (key, payload) pass tiles: 256 threads x 28 pairs (7168), 2 CTAs/SM, 128
// registers. r02 sweep, sortperm 1e8 f32: 384 x 16 2.52 ms, 256 x 24 2.43, 256 x 28 2.36,
// 256 x 32 2.36 (56 B of spills), 512 x 12 2.71, 256 x 16 (3 CTAs/SM) 2.57
// Keys-only pass tiles (r02 sweeps, 2^27 keys): 4-byte keys 256 threads x 40 keys (f32 sort
// onesweep 2.75 -> 2.26 ms; 384 x 16 before, 256 x 32 2.33, 256 x 48 2.26 with spills);
// 8-byte keys 256 x 32 (f64 merge_sort 6.97 -> 6.25 ms; 256 x 24 6.52, 256 x 28 6.35)
#ifndef AKB_OS_KEY4_ITEMS
#define AKB_OS_KEY4_ITEMS 40
#endif
#ifndef AKB_OS_KEY4_BLOCK
#define AKB_OS_KEY4_BLOCK 256
#endif
// 4 + 8 / 8 + 4-byte pairs: 256 x 24 (1e8 sortperm f32 -> int64 3.21 -> 2.83 ms, int64 -> int32
// 6.20 -> 5.56 ms; 384 x 12 before, 256 x 20 2.96 / 5.77); 8 + 8-byte pairs: 256 x 16 (int64 ->
// int64 7.26 -> 6.86 ms; 384 x 10 before, 256 x 20 6.84 with spills)
#ifndef AKB_OS_PAIR12_ITEMS
#define AKB_OS_PAIR12_ITEMS 24
#endif
#ifndef AKB_OS_PAIR12_BLOCK
#define AKB_OS_PAIR12_BLOCK 256
#endif
#ifndef AKB_OS_PAIR16_ITEMS
#define AKB_OS_PAIR16_ITEMS 16
#endif
#ifndef AKB_OS_PAIR16_BLOCK
#define AKB_OS_PAIR16_BLOCK 256
#endif
#ifndef AKB_OS_KEY8_ITEMS
#define AKB_OS_KEY8_ITEMS 32
#endif
#ifndef AKB_OS_KEY8_BLOCK
#define AKB_OS_KEY8_BLOCK 256
#endif
#ifndef AKB_OS_PAIR_ITEMS
#define AKB_OS_PAIR_ITEMS 28
#endif
#ifndef AKB_OS_PAIR_BLOCK
#define AKB_OS_PAIR_BLOCK 256
#endif
#ifndef AKB_OS_BLOCK
#define AKB_OS_BLOCK 384  // threads per pass CTA (>= RADIX)
#endif
#ifndef AKB_HYB_K
#define AKB_HYB_K 3  // MATCH_HYBRID: every K-th item ranks by ballots, the rest by the peer table
#endif
#ifndef AKB_LB_WIN
#define AKB_LB_WIN 4  // predecessors read per look-back round trip (r01 sweep: 2/4/8/16 -> 4 best)
#endif
// Tile counts are published to the look-back chain right after ranking (from the
// per-warp histograms the ranking builds anyway) instead of with a separate early
// shared-atomic count: one shared atomic per key less (r01: -5.5% per pass).
#ifndef AKB_EARLY_COUNTS
#define AKB_EXPERIMENT_LATE_COUNTS
#endif

#ifdef AKB_PHASES
// Phase-timing build (tools/phases.py): thread 0 of every tile stamps %globaltimer
// at each phase boundary of the pass kernel into g_phase[tile * 8 + k].
__device__ std::uint64_t* g_phase = nullptr;
#define AKB_PHASE(k)                                                                         \
    do {                                                                                     \
        if (tid == 0 && g_phase) {                                                           \
            std::uint64_t t_;                                                                \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
            g_phase[static_cast<std::uint64_t>(tile) * 8 + (k)] = t_;                        \
        }                                                                                    \
    } while (0)
#else
#define AKB_PHASE(k) \
    do {             \
    } while (0)
#endif

template <typename T, typename V, int MODE>
struct tile_cfg {
    static constexpr bool HAS_VALS = MODE != SORT_KEYS;
    static constexpr bool PAIR8 = HAS_VALS && sizeof(T) + sizeof(V) <= 8;  // 4-byte key + 4-byte payload
    static constexpr bool KEY4 = !HAS_VALS && sizeof(T) <= 4;              // keys-only, 4-byte keys
    static constexpr bool KEY8 = !HAS_VALS && sizeof(T) == 8;              // keys-only, 8-byte keys
    static constexpr bool PAIR12 = HAS_VALS && sizeof(T) + sizeof(V) == 12;
    static constexpr bool PAIR16 = HAS_VALS && sizeof(T) + sizeof(V) == 16;
    static constexpr int BLOCK =
        PAIR8 ? AKB_OS_PAIR_BLOCK
              : (PAIR12 ? AKB_OS_PAIR12_BLOCK
                        : (PAIR16 ? AKB_OS_PAIR16_BLOCK
                                  : (KEY4 ? AKB_OS_KEY4_BLOCK : (KEY8 ? AKB_OS_KEY8_BLOCK : AKB_OS_BLOCK))));
    static constexpr int ITEMS =
        !HAS_VALS ? (KEY4 ? AKB_OS_KEY4_ITEMS : (KEY8 ? AKB_OS_KEY8_ITEMS : AKB_OS_ITEMS))
                  : (sizeof(T) + sizeof(V) <= 8 ? AKB_OS_PAIR_ITEMS
                                                 : (sizeof(T) + sizeof(V) <= 12 ? AKB_OS_PAIR12_ITEMS : AKB_OS_PAIR16_ITEMS));
    static constexpr int TILE = BLOCK * ITEMS;
    static constexpr int MIN_BLOCKS = AKB_OS_MINB;
};

template <typename T>
__device__ __forceinline__ std::uint32_t digit_of(T key, int shift, bool desc) {
    const auto o = ordered(key, desc);
    if constexpr (sizeof(o) == 8) {
        const std::uint32_t w = shift >= 32 ? static_cast<std::uint32_t>(o >> 32) : static_cast<std::uint32_t>(o);
        return (w >> (shift & 31)) & 0xffu;
    } else {
        return (o >> shift) & 0xffu;
    }
}

// Predicated shared-memory ops: keep the per-item ranking loop free of divergent
// branches (BSSY/BRA/BSYNC run on the ADU pipe, which is the first to saturate).
__device__ __forceinline__ std::uint32_t atom_add_shared_if(bool p, std::uint32_t* addr, std::uint32_t v) {
    std::uint32_t old = 0;
    const std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(addr));
    asm volatile(
        "{ .reg .pred q; setp.ne.u32 q, %2, 0; @q atom.shared.add.u32 %0, [%1], %3; }"
        : "+r"(old)
        : "r"(a), "r"(static_cast<std::uint32_t>(p)), "r"(v)
        : "memory");
    return old;
}
__device__ __forceinline__ void st_shared_if(bool p, std::uint32_t* addr, std::uint32_t v) {
    const std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(addr));
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %1, 0; @q st.shared.u32 [%0], %2; }" ::"r"(a),
                 "r"(static_cast<std::uint32_t>(p)), "r"(v)
                 : "memory");
}
__device__ __forceinline__ std::uint32_t ld_shared_u32(const std::uint32_t* addr) {
    std::uint32_t v;
    const std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(addr));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void red_or_shared_if(bool p, std::uint32_t* addr, std::uint32_t v) {
    const std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(addr));
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q red.shared.or.b32 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"(static_cast<std::uint32_t>(p))
                 : "memory");
}
__device__ __forceinline__ std::uint32_t ld_shared_u32_if(bool p, const std::uint32_t* addr) {
    std::uint32_t v = 0;
    const std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(addr));
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.shared.u32 %0, [%1]; }"
                 : "+r"(v)
                 : "r"(a), "r"(static_cast<std::uint32_t>(p))
                 : "memory");
    return v;
}
__device__ __forceinline__ void red_or_shared(std::uint32_t* addr, std::uint32_t v) {
    const std::uint32_t a = static_cast<std::uint32_t>(__cvta_generic_to_shared(addr));
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// TMA bulk copies (cp.async.bulk, non-tensor) completing on an mbarrier.
// Peer-lane discovery for the warp ranking (AKB_MATCH selects at run time):
enum match_kind : int { MATCH_BALLOT = 0, MATCH_HW = 1, MATCH_SMEM = 2, MATCH_HYBRID = 3, MATCH_HALF = 4 };

// Lanes holding the same 8-bit digit (register variants).
template <int HW>
__device__ __forceinline__ std::uint32_t match_digit(std::uint32_t d) {
    if constexpr (HW == MATCH_HW) {
        return __match_any_sync(FULL, d);
    } else {
        std::uint32_t m = FULL;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const std::uint32_t bal = __ballot_sync(FULL, (d >> b) & 1u);
            // all-ones when bit b of d is clear -> keep lanes whose bit is clear too
            const std::uint32_t flip = 0u - (((d >> b) & 1u) ^ 1u);
            m &= bal ^ flip;
        }
        return m;
    }
}

// ---------------------------------------------------------------------------
#ifndef AKB_HIST_PARTS4
#define AKB_HIST_PARTS4 8  // sub-histograms per digit for 4-byte keys (r02: 4 -> 8, f32 2^28 0.41 -> 0.37 ms)
#endif
// Upfront histogram: one read of the keys, all D digit histograms.
// PARTS sub-histograms per digit spread same-digit lanes over banks.
// ---------------------------------------------------------------------------
// Digits [FIRST, PASSES) are counted (the hybrid sort only needs its top digits).
template <typename T, int PASSES, int FIRST = 0>
__global__ void __launch_bounds__(256) hist_kernel(const T* __restrict__ keys, std::uint64_t n,
                                                   int desc, std::uint64_t* __restrict__ g_hist) {
    constexpr int PARTS = AKB_HIST_PARTS4 && sizeof(T) <= 4 ? AKB_HIST_PARTS4 : 4;
    constexpr int CNT = PASSES - FIRST;
    __shared__ std::uint32_t sh[CNT * RADIX * PARTS];
    for (int i = threadIdx.x; i < CNT * RADIX * PARTS; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int part = threadIdx.x % PARTS;
    auto count = [&](T k) {
        const auto o = ordered(k, desc != 0);
#pragma unroll
        for (int p = FIRST; p < PASSES; ++p) {
            const std::uint32_t d = static_cast<std::uint32_t>((o >> (8 * p)) & 0xffu);
            atomicAdd(&sh[((p - FIRST) * RADIX + d) * PARTS + part], 1u);
        }
    };
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    const std::uint64_t tid = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    constexpr int VEC = 16 / sizeof(T);
    const bool aligned = (reinterpret_cast<std::uintptr_t>(keys) & 15) == 0;
    std::uint64_t done = 0;
    if (aligned) {
        const std::uint64_t nv = n / VEC;
        const uint4* kv = reinterpret_cast<const uint4*>(keys);
        std::uint64_t i = tid;
        for (; i + 3 * stride < nv; i += 4 * stride) {
            uint4 a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = __ldg(kv + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const T* e = reinterpret_cast<const T*>(&a[u]);
#pragma unroll
                for (int v = 0; v < VEC; ++v) count(e[v]);
            }
        }
        for (; i < nv; i += stride) {
            const uint4 a = __ldg(kv + i);
            const T* e = reinterpret_cast<const T*>(&a);
#pragma unroll
            for (int v = 0; v < VEC; ++v) count(e[v]);
        }
        done = nv * VEC;
    }
    for (std::uint64_t i = done + tid; i < n; i += stride) count(keys[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < CNT * RADIX; i += blockDim.x) {
        std::uint32_t s = 0;
#pragma unroll
        for (int q = 0; q < PARTS; ++q) s += sh[i * PARTS + q];
        if (s)
            atomicAdd(reinterpret_cast<unsigned long long*>(g_hist + FIRST * RADIX + i),
                      static_cast<unsigned long long>(s));
    }
}

// Exclusive scan of each pass's 256 digit counts -> global digit offsets.
__global__ void __launch_bounds__(RADIX) hist_scan_kernel(const std::uint64_t* __restrict__ g_hist,
                                                          std::uint64_t* __restrict__ g_offs) {
    __shared__ std::uint64_t s_warp[RADIX / 32];
    const int p = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const std::uint64_t v = g_hist[p * RADIX + t];
    std::uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint64_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    std::uint64_t base = 0;
    for (int i = 0; i < w; ++i) base += s_warp[i];
    g_offs[p * RADIX + t] = base + inc - v;
}

// ---------------------------------------------------------------------------
// One onesweep digit pass.
// ---------------------------------------------------------------------------
template <typename T, typename V, int MODE>
struct pass_smem {
    using C = tile_cfg<T, V, MODE>;
    static constexpr int BLOCK = C::BLOCK;
    static constexpr int TILE = C::TILE;
    static constexpr int WARPS = BLOCK / 32;
    static constexpr bool HAS_KEYS_SMEM = MODE != SORT_LOWMEM;
    static constexpr bool HAS_VALS = C::HAS_VALS;
    static constexpr std::size_t keys_off = 0;
    static constexpr std::size_t keys_bytes = HAS_KEYS_SMEM ? sizeof(T) * TILE : 0;
    static constexpr std::size_t vals_off = keys_off + keys_bytes;
    static constexpr std::size_t vals_bytes = HAS_VALS ? sizeof(V) * TILE : 0;
    // MATCH_SMEM peer tables (two for MATCH_SMEM2): alias the staging area, which is dead
    // until ranking is over
    static constexpr std::size_t match_off = 0;
    static constexpr std::size_t match_bytes = sizeof(std::uint32_t) * WARPS * RADIX;
    static constexpr std::size_t stage_bytes =
        keys_bytes + vals_bytes > 2 * match_bytes ? keys_bytes + vals_bytes : 2 * match_bytes;
    static constexpr std::size_t whist_off = (stage_bytes + 15) & ~std::size_t(15);
    // per ranking group (warp, or half-warp for MATCH_HALF) running digit counts
    static constexpr std::size_t whist_bytes = sizeof(std::uint32_t) * 2 * WARPS * RADIX;
    static constexpr std::size_t hist_off = whist_off + whist_bytes;
    static constexpr std::size_t hist_bytes = sizeof(std::uint32_t) * RADIX;
    static constexpr std::size_t gofs_off = hist_off + hist_bytes;
    static constexpr std::size_t gofs_bytes = sizeof(std::uint64_t) * RADIX;
    static constexpr std::size_t gofs32_off = gofs_off + gofs_bytes;  // low words, used when n <= 2^32
    static constexpr std::size_t gofs32_bytes = sizeof(std::uint32_t) * RADIX;
    static constexpr std::size_t misc_off = gofs32_off + gofs32_bytes;
    static constexpr std::size_t misc_bytes = sizeof(std::uint32_t) * 16;
    static constexpr std::size_t total = misc_off + misc_bytes;
};

template <typename T, typename V, int MODE, int HW_MATCH>
__global__ void __launch_bounds__(tile_cfg<T, V, MODE>::BLOCK, tile_cfg<T, V, MODE>::MIN_BLOCKS)
    onesweep_kernel(const T* __restrict__ kin, T* __restrict__ kout, const V* __restrict__ vin,
                    V* __restrict__ vout, std::uint64_t n, int shift, int desc, int pass_index,
                    const std::uint64_t* __restrict__ goffs, std::uint64_t* lookback,
                    std::uint32_t* tile_counter, std::uint32_t tag, int write_keys,
                    const int* __restrict__ plan) {
    // device-planned pass (small keys-only sorts): plan[0] != 0 = not applicable, plan[1] = shift
    if (plan != nullptr) {
        if (plan[0] != 0) return;
        shift = plan[1];
    }
    using L = pass_smem<T, V, MODE>;
    constexpr int BLOCK = L::BLOCK;
    constexpr int ITEMS = tile_cfg<T, V, MODE>::ITEMS;
    constexpr int TILE = L::TILE;
    constexpr int WARPS = L::WARPS;
    constexpr int DW = (ITEMS + 3) / 4;  // packed digit words
    extern __shared__ __align__(16) unsigned char smem[];
    T* s_keys = reinterpret_cast<T*>(smem + L::keys_off);
    V* s_vals = reinterpret_cast<V*>(smem + L::vals_off);
    std::uint32_t* s_whist = reinterpret_cast<std::uint32_t*>(smem + L::whist_off);
    std::uint32_t* s_hist = reinterpret_cast<std::uint32_t*>(smem + L::hist_off);
    std::uint64_t* s_gofs = reinterpret_cast<std::uint64_t*>(smem + L::gofs_off);
    std::uint32_t* s_gofs32 = reinterpret_cast<std::uint32_t*>(smem + L::gofs32_off);
    std::uint32_t* s_misc = reinterpret_cast<std::uint32_t*>(smem + L::misc_off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // ranking groups: warps, or half-warps (MATCH_HALF: 16 lanes, each group owning a
    // contiguous run of 16*ITEMS keys, count and peer mask packed in one shared word)
    constexpr bool HALF = HW_MATCH == MATCH_HALF;
    constexpr int VW = HALF ? 2 * WARPS : WARPS;
    constexpr int GL = HALF ? 16 : 32;
    const int vw = HALF ? warp * 2 + (lane >> 4) : warp;
    const int gl = HALF ? (lane & 15) : lane;
    const bool dsc = desc != 0;
    if (tid == 0) {
        // tile ids come from the ticket (look-back order) and follow the launch order closely:
        // the tile this CTA's index names is fetched into L2 while the ticket is in flight
        const std::uint64_t pb = static_cast<std::uint64_t>(blockIdx.x) * TILE;
        if (MODE != SORT_LOWMEM && pb + TILE <= n) {
            if ((reinterpret_cast<std::uintptr_t>(kin + pb) & 15) == 0 && (TILE * sizeof(T)) % 16 == 0)
                bulk_prefetch_l2(kin + pb, static_cast<std::uint32_t>(TILE * sizeof(T)));
            if (MODE == SORT_PAIRS || (MODE == SORT_IOTA && pass_index != 0))
                if ((reinterpret_cast<std::uintptr_t>(vin + pb) & 15) == 0 && (TILE * sizeof(V)) % 16 == 0)
                    bulk_prefetch_l2(vin + pb, static_cast<std::uint32_t>(TILE * sizeof(V)));
        }
        s_misc[0] = atomicAdd(tile_counter, 1u);
    }
    for (int i = tid; i < VW * RADIX; i += BLOCK) s_whist[i] = 0;
    if constexpr (HW_MATCH == MATCH_SMEM || HW_MATCH == MATCH_HYBRID) {
        std::uint32_t* s_match = reinterpret_cast<std::uint32_t*>(smem + L::match_off);
        constexpr int TABLES = 1;
        for (int i = tid; i < TABLES * WARPS * RADIX; i += BLOCK) s_match[i] = 0;
    }
    if (tid < RADIX) s_hist[tid] = 0;
    __syncthreads();
    const std::uint32_t tile = s_misc[0];
    AKB_PHASE(0);
    const std::uint64_t tile_base = static_cast<std::uint64_t>(tile) * TILE;
    const std::uint64_t remaining = n - tile_base;
    const std::uint32_t valid = remaining < TILE ? static_cast<std::uint32_t>(remaining) : TILE;
    const bool full = valid == TILE;
    const std::uint32_t wofs = static_cast<std::uint32_t>(vw) * GL * ITEMS + gl;  // tile-local index of item 0

    // ---- load (warp-striped: item i of lane l is tile-local wofs + 32 i) ----
    T k[ITEMS];
    V v[ITEMS];
    std::uint32_t dg[DW];
#pragma unroll
    for (int w = 0; w < DW; ++w) dg[w] = 0;
    // Branch-free per item: one uniform full/partial decision per tile; padded
    // slots load from a clamped in-bounds address and get digit 255 (sorted last,
    // never counted, never scattered).
    auto load_and_count = [&](auto full_c) {
        constexpr bool F = decltype(full_c)::value;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const std::uint32_t li = wofs + i * GL;
            const bool ok = F || li < valid;
            const std::uint64_t idx = tile_base + (ok ? li : 0u);
            if constexpr (MODE == SORT_LOWMEM) {
                const V ix = pass_index == 0 ? static_cast<V>(idx) : vin[idx];
                v[i] = ix;
                k[i] = kin[ix];
            } else {
                k[i] = kin[idx];
                if constexpr (MODE == SORT_PAIRS) v[i] = vin[idx];
                if constexpr (MODE == SORT_IOTA) v[i] = pass_index == 0 ? static_cast<V>(idx) : vin[idx];
            }
        }
        // ---- digits + early counts ----
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const std::uint32_t li = wofs + i * GL;
            const bool ok = F || li < valid;
            const std::uint32_t d = ok ? digit_of(k[i], shift, dsc) : 255u;  // padding sorts last
            dg[i / 4] |= d << (8 * (i % 4));
#ifndef AKB_EXPERIMENT_LATE_COUNTS
            if constexpr (F) atomicAdd(s_hist + d, 1u);
            else atomicAdd(s_hist + d, ok ? 1u : 0u);
#endif
        }
    };
    if (full) load_and_count(std::true_type{});
    else load_and_count(std::false_type{});
    __syncthreads();
    AKB_PHASE(1);
    std::uint64_t* my_lb = lookback + static_cast<std::uint64_t>(tile) * RADIX + tid;
    const std::uint64_t tagbits = static_cast<std::uint64_t>(tag) << LB_TAG_SHIFT;
    std::uint32_t count = 0;
    if (tid < RADIX) {
#ifndef AKB_EXPERIMENT_LATE_COUNTS
        count = s_hist[tid];
        st_relaxed_u64(my_lb, (tile == 0 ? LB_INC : LB_AGG) | tagbits | count);
#endif
    }

    // ---- warp-level stable ranking ----
    std::uint32_t rk[(ITEMS + 1) / 2];  // warp-local ranks (< 32*ITEMS), two 16-bit per word
#pragma unroll
    for (int w = 0; w < (ITEMS + 1) / 2; ++w) rk[w] = 0;
    std::uint32_t* wh = s_whist + vw * RADIX;
    if constexpr (HALF) {
        // word = running count << 16 | peer mask of this item (16 lanes)
        const std::uint32_t bit = 1u << gl;
        const std::uint32_t lt16 = bit - 1u;
        const std::uint32_t ge16 = 0xffffu & ~lt16;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
            red_or_shared(wh + d, bit);
            __syncwarp();
            const std::uint32_t w = ld_shared_u32(wh + d);
            __syncwarp();
            const std::uint32_t peers = w & 0xffffu, base = w >> 16;
            const bool lead = (peers & ge16) == bit;  // highest lane of the group
            st_shared_if(lead, wh + d, (base + __popc(peers)) << 16);
            rk[i / 2] |= (base + __popc(peers & lt16)) << (16 * (i % 2));
        }
        __syncwarp();
    } else if constexpr (HW_MATCH == MATCH_HYBRID) {
        // Split the peer discovery between two pipes: every AKB_HYB_K-th item finds its
        // peers with 8 ballots (ALU/vote), the others through the shared peer table
        // (LSU). Both read and bump the same per-warp running digit counts.
        std::uint32_t* mt = reinterpret_cast<std::uint32_t*>(smem + L::match_off) + warp * RADIX;
        const std::uint32_t lanebit = 1u << lane;
        const std::uint32_t lt = lanemask_lt();
        const std::uint32_t ge = ~lt;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
            constexpr int K = AKB_HYB_K;
            const bool by_vote = (i % K) == K - 1;
            std::uint32_t peers;
            if (by_vote) {
                peers = match_digit<MATCH_BALLOT>(d);
                __syncwarp();
            } else {
                red_or_shared(mt + d, lanebit);
                __syncwarp();
                peers = ld_shared_u32(mt + d);
            }
            const std::uint32_t base = ld_shared_u32(wh + d);
            __syncwarp();
            const bool lead = (peers & ge) == lanebit;
            st_shared_if(lead, wh + d, base + __popc(peers));
            if (!by_vote) st_shared_if(lead, mt + d, 0u);
            rk[i / 2] |= (base + __popc(peers & lt)) << (16 * (i % 2));
        }
        __syncwarp();
    } else if constexpr (HW_MATCH == MATCH_SMEM) {
        // peers via a per-warp digit -> lane-bitmask table: OR in, read back, leader clears
        std::uint32_t* mt = reinterpret_cast<std::uint32_t*>(smem + L::match_off) + warp * RADIX;
        const std::uint32_t lanebit = 1u << lane;
        const std::uint32_t lt = lanemask_lt();
        const std::uint32_t ge = ~lt;  // lanes >= me
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
            red_or_shared(mt + d, lanebit);
            __syncwarp();
            const std::uint32_t peers = ld_shared_u32(mt + d);
            const std::uint32_t base = ld_shared_u32(wh + d);  // group-uniform (broadcast)
            __syncwarp();
            const bool lead = (peers & ge) == lanebit;  // highest lane of the group
            st_shared_if(lead, wh + d, base + __popc(peers));
            st_shared_if(lead, mt + d, 0u);
            rk[i / 2] |= (base + __popc(peers & lt)) << (16 * (i % 2));
        }
        __syncwarp();
    } else {
        const std::uint32_t lt = lanemask_lt();
        const std::uint32_t ge = ~lt;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
            const std::uint32_t peers = match_digit<HW_MATCH>(d);
            const int leader = 31 - __clz(peers);
            const bool lead = (peers & ge) == (1u << lane);
            std::uint32_t base = atom_add_shared_if(lead, wh + d, static_cast<std::uint32_t>(__popc(peers)));
            base = __shfl_sync(FULL, base, leader);
            rk[i / 2] |= (base + __popc(peers & lt)) << (16 * (i % 2));
        }
    }
    __syncthreads();
    AKB_PHASE(2);

    // ---- tile digit totals (incl. padding), warp-exclusive offsets, block scan ----
    std::uint32_t total = 0;
    std::uint32_t incl = 0;
    if (tid < RADIX) {
#pragma unroll
        for (int w = 0; w < VW; ++w) {
            const std::uint32_t c = HALF ? (s_whist[w * RADIX + tid] >> 16) : s_whist[w * RADIX + tid];
            s_whist[w * RADIX + tid] = total;
            total += c;
        }
#ifdef AKB_EXPERIMENT_LATE_COUNTS  // publish the aggregate only after ranking (no early counts)
        count = total - (tid == RADIX - 1 ? TILE - valid : 0u);
        st_relaxed_u64(my_lb, (tile == 0 ? LB_INC : LB_AGG) | tagbits | count);
#endif
        incl = total;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_misc[4 + warp] = incl;
    }
    __syncthreads();
    std::uint32_t dstart = 0;
    if (tid < RADIX) {
        std::uint32_t wp = 0;
#pragma unroll
        for (int w = 0; w < RADIX / 32; ++w)
            if (w < warp) wp += s_misc[4 + w];
        dstart = wp + incl - total;
#pragma unroll
        for (int w = 0; w < VW; ++w) s_whist[w * RADIX + tid] += dstart;
    }
    __syncthreads();
    AKB_PHASE(3);

    // ---- stage keys (and payload) in shared memory in digit order ----
    // 4-byte keys with 4-byte payload: one packed 8-byte pair per slot (one store and one load
    // per element instead of two each)
    constexpr bool PACK = L::HAS_KEYS_SMEM && L::HAS_VALS && sizeof(T) == 4 && sizeof(V) == 4;
    uint2* s_pairs = reinterpret_cast<uint2*>(smem + L::keys_off);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
        const std::uint32_t pos = wh[d] + ((rk[i / 2] >> (16 * (i % 2))) & 0xffffu);
        if constexpr (PACK) {
            s_pairs[pos] = make_uint2(__builtin_bit_cast(std::uint32_t, k[i]), static_cast<std::uint32_t>(v[i]));
        } else {
            if constexpr (L::HAS_KEYS_SMEM) s_keys[pos] = k[i];
            if constexpr (L::HAS_VALS) s_vals[pos] = v[i];
        }
    }

    // ---- windowed decoupled look-back for this tile's per-digit exclusive prefix ----
    if (tid < RADIX) {
        std::uint64_t excl = 0;
#ifdef AKB_EXPERIMENT_NO_LOOKBACK  // timing experiment only: wrong output
        if (false) {
#else
        if (tile > 0) {
#endif
            std::int64_t p = static_cast<std::int64_t>(tile) - 1;
            bool done = false;
            while (!done) {
                constexpr int WIN = AKB_LB_WIN;
                std::uint64_t w[WIN];
#pragma unroll
                for (int q = 0; q < WIN; ++q)
                    w[q] = p - q >= 0 ? ld_relaxed_u64(lookback + (p - q) * RADIX + tid) : (LB_INC | tagbits);
                int consumed = 0;
#pragma unroll
                for (int q = 0; q < WIN; ++q) {
                    if (done || consumed < q) break;
                    const std::uint32_t wtag = static_cast<std::uint32_t>(w[q] >> LB_TAG_SHIFT) & LB_TAG_MASK;
                    const std::uint64_t flag = w[q] & (3ull << 62);
                    if (wtag != tag || flag == 0) break;  // not published yet: reload from here
                    excl += w[q] & LB_COUNT_MASK;
                    consumed = q + 1;
                    if (flag == LB_INC) done = true;
                }
                p -= consumed;
            }
            st_relaxed_u64(my_lb, LB_INC | tagbits | (excl + count));
        }
        const std::uint64_t g = goffs[tid] + excl - dstart;  // modular: g + j is the output index
        s_gofs[tid] = g;
        s_gofs32[tid] = static_cast<std::uint32_t>(g);
    }
    __syncthreads();
    AKB_PHASE(4);

    // ---- scatter contiguous digit runs ----
    auto scatter = [&](auto full_c, auto wk_c, auto narrow_c) {
        constexpr bool F = decltype(full_c)::value;
        constexpr bool WK = decltype(wk_c)::value;
        constexpr bool NARROW = decltype(narrow_c)::value;  // n <= 2^32: 32-bit offset math
        auto dst = [&](std::uint32_t d, std::uint32_t j) -> std::uint64_t {
            if constexpr (NARROW) return static_cast<std::uint32_t>(s_gofs32[d] + j);
            else return s_gofs[d] + j;
        };
        if constexpr (PACK) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const std::uint32_t j = i * BLOCK + tid;
                if (F || j < valid) {
                    const uint2 pr = s_pairs[j];
                    const T key = __builtin_bit_cast(T, pr.x);
                    const std::uint64_t o = dst(digit_of(key, shift, dsc), j);
                    if constexpr (WK) kout[o] = key;
                    vout[o] = static_cast<V>(pr.y);
                }
            }
        } else if constexpr (MODE == SORT_LOWMEM) {
            // only the index array moves; the digit of staged slot j is recomputed
            // from data[index] (L1/L2 hit: just gathered by this tile)
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const std::uint32_t j = i * BLOCK + tid;
                if (F || j < valid) {
                    const V ix = s_vals[j];
                    const std::uint32_t d = digit_of(kin[ix], shift, dsc);
                    vout[dst(d, j)] = ix;
                }
            }
        } else {
            std::uint32_t dj[DW];
#pragma unroll
            for (int w = 0; w < DW; ++w) dj[w] = 0;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const std::uint32_t j = i * BLOCK + tid;
                if (F || j < valid) {
                    const T key = s_keys[j];
                    const std::uint32_t d = digit_of(key, shift, dsc);
                    dj[i / 4] |= d << (8 * (i % 4));
                    if constexpr (WK) kout[dst(d, j)] = key;
                }
            }
            if constexpr (L::HAS_VALS) {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const std::uint32_t j = i * BLOCK + tid;
                    if (F || j < valid) {
                        const std::uint32_t d = (dj[i / 4] >> (8 * (i % 4))) & 0xffu;
                        vout[dst(d, j)] = s_vals[j];
                    }
                }
            }
        }
    };
    if (n <= 0xffffffffull) {
        if (full) {
            if (write_keys) scatter(std::true_type{}, std::true_type{}, std::true_type{});
            else scatter(std::true_type{}, std::false_type{}, std::true_type{});
        } else {
            if (write_keys) scatter(std::false_type{}, std::true_type{}, std::true_type{});
            else scatter(std::false_type{}, std::false_type{}, std::true_type{});
        }
    } else {
        if (write_keys) scatter(std::false_type{}, std::true_type{}, std::false_type{});
        else scatter(std::false_type{}, std::false_type{}, std::false_type{});
    }
    AKB_PHASE(5);
}

// Ranking variant of the onesweep pass (experiment builds: -DAKB_CFG_MATCH=...). r01 sweep,
// 2^28 int64 full sort: half 12.97 / hybrid 13.12 / smem 13.35 / ballot 14.5 / hw 18.6 ms.
#ifndef AKB_CFG_MATCH
#define AKB_CFG_MATCH MATCH_HALF
#endif

template <typename T, typename V, int MODE, int HW>
void launch_pass_impl(ak_ctx* c, const T* kin, T* kout, const V* vin, V* vout, std::uint64_t n, int shift,
                      bool desc, int pass_index, const std::uint64_t* goffs, std::uint32_t* tile_counter,
                      bool write_keys, const int* plan = nullptr) {
    using L = pass_smem<T, V, MODE>;
    auto kern = onesweep_kernel<T, V, MODE, HW>;
    smem_attr(c, kern, L::total);
    const std::uint64_t tiles = ceil_div(n, L::TILE);
    const std::uint32_t tag = ctx_lookback_pass(c, tiles);
    const int tok = ctx_prof_begin(c, KF_ONESWEEP);
    kern<<<static_cast<unsigned>(tiles), L::BLOCK, L::total, c->stream>>>(
        kin, kout, vin, vout, n, shift, desc ? 1 : 0, pass_index, goffs, c->lookback, tile_counter, tag,
        write_keys ? 1 : 0, plan);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 1;
}

template <typename T, typename V, int MODE>
void launch_pass(ak_ctx* c, const T* kin, T* kout, const V* vin, V* vout, std::uint64_t n, int shift, bool desc,
                 int pass_index, const std::uint64_t* goffs, std::uint32_t* tile_counter, bool write_keys,
                 const int* plan = nullptr) {
    launch_pass_impl<T, V, MODE, AKB_CFG_MATCH>(c, kin, kout, vin, vout, n, shift, desc, pass_index, goffs,
                                                tile_counter, write_keys, plan);
}

template <typename T, typename V, int MODE>
void radix_sort_impl(ak_ctx* c, const T* kin, T* kout, T* kalt, const V* vin, V* vout, V* valt,
                     std::uint64_t n, bool desc, bool keys_out) {
    constexpr int PASSES = key_traits<T>::nbits / 8;
    static_assert(PASSES % 2 == 0, "even pass count keeps the result in the output buffer");
    if (n == 0) return;
    // small region: hist | offs | tile counters
    std::uint64_t* g_hist = static_cast<std::uint64_t*>(c->small);
    std::uint64_t* g_offs = g_hist + PASSES * RADIX;
    std::uint32_t* counters = reinterpret_cast<std::uint32_t*>(g_offs + PASSES * RADIX);
    AKB_CUDA(cudaMemsetAsync(c->small, 0, (2 * PASSES * RADIX) * 8 + PASSES * 4, c->stream));

    // upfront histogram (for LOWMEM the keys are the data array itself)
    {
        const int blocks = c->sm_count * 4;
        const int tok = ctx_prof_begin(c, KF_HIST);
        hist_kernel<T, PASSES><<<blocks, 256, 0, c->stream>>>(kin, n, desc ? 1 : 0, g_hist);
        AKB_CUDA(cudaGetLastError());
        ctx_prof_end(c, tok);
        hist_scan_kernel<<<PASSES, RADIX, 0, c->stream>>>(g_hist, g_offs);
        AKB_CUDA(cudaGetLastError());
        c->kernel_launches += 2;
    }

    if constexpr (MODE == SORT_LOWMEM) {
        // indices ping-pong valt <-> vout; pass 0 synthesises iota
        for (int p = 0; p < PASSES; ++p) {
            V* dst = (p % 2 == 0) ? valt : vout;
            const V* src = (p % 2 == 0) ? vout : valt;  // unused at p == 0
            launch_pass<T, V, MODE>(c, kin, nullptr, src, dst, n, 8 * p, desc, p, g_offs + p * RADIX, counters + p,
                                    false);
        }
    } else {
        // keys: pass p reads src, writes dst; even passes -> kalt, odd -> kout
        for (int p = 0; p < PASSES; ++p) {
            const bool to_alt = (p % 2 == 0);
            const T* ksrc = p == 0 ? kin : (to_alt ? kout : kalt);
            T* kdst = to_alt ? kalt : kout;
            const V* vsrc = nullptr;
            V* vdst = nullptr;
            if constexpr (MODE != SORT_KEYS) {
                vsrc = p == 0 ? vin : (to_alt ? vout : valt);
                vdst = to_alt ? valt : vout;
            }
            const bool wk = keys_out || (p + 1 < PASSES);
            launch_pass<T, V, MODE>(c, ksrc, kdst, vsrc, vdst, n, 8 * p, desc, p, g_offs + p * RADIX, counters + p,
                                    wk);
        }
    }
}


// ---------------------------------------------------------------------------
// Hybrid MSD/LSD sort (keys only).
//   1. m global onesweep passes over the TOP m digits (LSD order among them) leave the
//      array stably ordered by its top 8m bits ("buckets");
//   2. the array is cut at bucket starts into ranges of at most LOCAL_TILE keys
//      (cut j = start of the bucket holding position j*step);
//   3. one CTA per range sorts it completely on chip: keys stay in registers, each
//      local pass ranks them (half-warp peer/count words, as the global pass) and
//      exchanges them through shared memory; only digits that vary inside the range
//      are passed over (the range's top digits are usually constant).
// Every key in range j precedes every key in range j+1 (cuts sit on bucket starts), equal
// keys share a bucket, and every pass is stable, so the result equals the stable LSD sort
// (= the reference's stable merge sort). Ranges that do not fit (skewed keys) are sorted
// afterwards by the plain onesweep LSD on their segment. Global traffic: m passes + one
// read and one write, instead of D passes.
// ---------------------------------------------------------------------------
constexpr int LOCAL_BLOCK = 384;
constexpr int LOCAL_MAX_ITEMS = 16;
constexpr int LOCAL_TILE = LOCAL_BLOCK * LOCAL_MAX_ITEMS;  // 6144 keys per range at most
constexpr int LOCAL_VW = LOCAL_BLOCK / 16;                  // half-warp ranking groups
constexpr int LOCAL_WARPS = LOCAL_BLOCK / 32;
constexpr std::uint32_t LOCAL_MAX_RUN = 64;  // longest run the insertion fix-up takes on

template <typename T, int ITEMS>
struct local_smem {
    static constexpr std::size_t stage_off = 0;
    static constexpr std::size_t stage_bytes = sizeof(T) * LOCAL_BLOCK * ITEMS;
    static constexpr std::size_t tab_off = stage_bytes;
    static constexpr std::size_t tab_bytes = sizeof(std::uint32_t) * LOCAL_VW * RADIX;
    static constexpr std::size_t wsum_off = tab_off + tab_bytes;  // 8 x u32 digit-scan warp sums
    static constexpr std::size_t red_off = wsum_off + 64;          // 2 x WARPS x u64 or/and partials
    static constexpr std::size_t total = red_off + 2 * LOCAL_WARPS * sizeof(std::uint64_t);
};

// Stable on-chip sort of range `range` (cuts[range] .. cuts[range+1]); see above.
template <typename T, int ITEMS>
__device__ __forceinline__ void local_radix_range(const T* __restrict__ in, T* __restrict__ out,
                                                  const std::uint64_t* __restrict__ cuts, std::uint64_t range,
                                                  int desc, int low, std::uint64_t* big, unsigned char* smem) {
    using L = local_smem<T, ITEMS>;
    using B = typename key_traits<T>::bits;
    constexpr int CAP = LOCAL_BLOCK * ITEMS;
    constexpr int PASSES = key_traits<T>::nbits / 8;
    T* s_stage = reinterpret_cast<T*>(smem + L::stage_off);
    std::uint32_t* s_tab = reinterpret_cast<std::uint32_t*>(smem + L::tab_off);
    std::uint32_t* s_wsum = reinterpret_cast<std::uint32_t*>(smem + L::wsum_off);
    B* s_red = reinterpret_cast<B*>(smem + L::red_off);
    std::uint32_t* s_maxrun = s_wsum + 8;

    const std::uint64_t b = cuts[range], e = cuts[range + 1];
    if (b >= e) return;
    if (e - b > static_cast<std::uint64_t>(CAP)) {  // left for the segment fallback
        if (threadIdx.x == 0) {
            const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull);
            big[1 + slot] = range;
        }
        return;
    }
    const std::uint32_t len = static_cast<std::uint32_t>(e - b);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int vw = warp * 2 + (lane >> 4), gl = lane & 15;
    const std::uint32_t base_i = static_cast<std::uint32_t>(vw) * 16 * ITEMS + gl;  // item i at base_i + 16 i
    const bool dsc = desc != 0;

    T k[ITEMS];
    B orv = 0, andv = static_cast<B>(~B(0));
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const std::uint32_t li = base_i + 16 * i;
        const bool ok = li < len;
        k[i] = in[b + (ok ? li : 0u)];
        const B o = ordered(k[i], dsc);
        orv |= ok ? o : B(0);
        andv &= ok ? o : static_cast<B>(~B(0));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        orv |= __shfl_xor_sync(FULL, orv, o);
        andv &= __shfl_xor_sync(FULL, andv, o);
    }
    if (lane == 0) {
        s_red[warp] = orv;
        s_red[LOCAL_WARPS + warp] = andv;
    }
    __syncthreads();
    B any1 = 0, all1 = static_cast<B>(~B(0));
#pragma unroll
    for (int w = 0; w < LOCAL_WARPS; ++w) {
        any1 |= s_red[w];
        all1 &= s_red[LOCAL_WARPS + w];
    }
    const B vary = any1 & ~all1;  // bits that differ between keys of this range

    std::uint32_t* wh = s_tab + vw * RADIX;
    const std::uint32_t bit = 1u << gl;
    const std::uint32_t lt16 = bit - 1u;
    const std::uint32_t ge16 = 0xffffu & ~lt16;
    // one stable local pass over digit p (p varies inside the range): rank the register
    // keys, stage them in digit order in shared memory, reload them in the new order
    auto do_pass = [&](int p) {
        const std::uint32_t vmask = static_cast<std::uint32_t>(vary >> (8 * p)) & 0xffu;
        // Narrow digits (<= 8 distinct values in this range, e.g. the bucket digit next to the
        // globally sorted ones): peers by ballots on the varying bits only -- the peer-table
        // atomics would serialise on the few shared addresses. Padding takes the largest
        // digit the range can hold, so it still sorts last.
        const bool narrow = __popc(vmask) <= 3;
        const std::uint32_t pad_digit =
            narrow ? ((static_cast<std::uint32_t>(all1 >> (8 * p)) & 0xffu & ~vmask) | vmask) : 255u;
        for (int i = tid; i < LOCAL_VW * RADIX; i += LOCAL_BLOCK) s_tab[i] = 0;
        __syncthreads();
        std::uint32_t dg[ITEMS / 4];
        std::uint32_t rk[ITEMS / 2];
#pragma unroll
        for (int w = 0; w < ITEMS / 4; ++w) dg[w] = 0;
#pragma unroll
        for (int w = 0; w < ITEMS / 2; ++w) rk[w] = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const bool ok = base_i + 16 * i < len;
            const std::uint32_t d = ok ? digit_of(k[i], 8 * p, dsc) : pad_digit;  // padding stays last
            dg[i / 4] |= d << (8 * (i % 4));
        }
        // Padding (slots >= len) takes no part in ranking: it keeps its own slot at the tail,
        // so it neither counts nor hammers one shared address.
        if (narrow) {
            const std::uint32_t half = (lane >> 4) * 16;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const bool ok = base_i + 16 * i < len;
                const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
                std::uint32_t m = __ballot_sync(FULL, ok);
#pragma unroll
                for (int bb = 0; bb < 8; ++bb) {
                    if (!((vmask >> bb) & 1u)) continue;  // block-uniform
                    const std::uint32_t bal = __ballot_sync(FULL, (d >> bb) & 1u);
                    m &= ((d >> bb) & 1u) ? bal : ~bal;
                }
                const std::uint32_t peers = (m >> half) & 0xffffu;
                __syncwarp();
                const std::uint32_t base = ld_shared_u32_if(ok, wh + d) >> 16;
                __syncwarp();
                const bool lead = ok && (peers & ge16) == bit;
                st_shared_if(lead, wh + d, (base + __popc(peers)) << 16);
                rk[i / 2] |= (base + __popc(peers & lt16)) << (16 * (i % 2));
            }
        } else {
            // stable rank inside the half-warp group: word = running count << 16 | peer mask
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const bool ok = base_i + 16 * i < len;
                const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
                red_or_shared_if(ok, wh + d, bit);
                __syncwarp();
                const std::uint32_t w = ld_shared_u32_if(ok, wh + d);
                __syncwarp();
                const std::uint32_t peers = w & 0xffffu, base = w >> 16;
                const bool lead = ok && (peers & ge16) == bit;
                st_shared_if(lead, wh + d, (base + __popc(peers)) << 16);
                rk[i / 2] |= (base + __popc(peers & lt16)) << (16 * (i % 2));
            }
        }
        __syncthreads();
        // digit starts + per-group offsets
        std::uint32_t total = 0, incl = 0;
        if (tid < RADIX) {
#pragma unroll
            for (int w = 0; w < LOCAL_VW; ++w) {
                const std::uint32_t cnt = s_tab[w * RADIX + tid] >> 16;
                s_tab[w * RADIX + tid] = total;
                total += cnt;
            }
            incl = total;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const std::uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
        }
        __syncthreads();
        if (tid < RADIX) {
            std::uint32_t wp = 0;
#pragma unroll
            for (int w = 0; w < RADIX / 32; ++w)
                if (w < warp) wp += s_wsum[w];
            const std::uint32_t dstart = wp + incl - total;
#pragma unroll
            for (int w = 0; w < LOCAL_VW; ++w) s_tab[w * RADIX + tid] += dstart;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const std::uint32_t li = base_i + 16 * i;
            const std::uint32_t d = (dg[i / 4] >> (8 * (i % 4))) & 0xffu;
            if (li < len) s_stage[wh[d] + ((rk[i / 2] >> (16 * (i % 2))) & 0xffffu)] = k[i];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
            if (base_i + 16 * i < len) k[i] = s_stage[base_i + 16 * i];
        // (the next pass re-zeroes s_tab only after a barrier; s_stage is rewritten only
        // after the next pass's ranking barrier, so this reload is complete by then)
    };

    // Radix passes only over the digits >= low (the high digits); then keys equal in all
    // bits >= 8*low form short runs (uniform keys: ~3% of keys, runs of 2-3), which one
    // thread per run finishes with a stable insertion sort on the full key. If some run is
    // long (clustered keys) the remaining low digits are radix-passed instead.
    int passes = 0;
#pragma unroll 1
    for (int p = low; p < PASSES; ++p)
        if ((vary >> (8 * p)) & 0xffu) {
            do_pass(p);
            ++passes;
        }
    if (passes == 0) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
            if (base_i + 16 * i < len) s_stage[base_i + 16 * i] = k[i];
    }
    const B lowbits = vary & (8 * low >= key_traits<T>::nbits ? static_cast<B>(~B(0))
                                                              : static_cast<B>((B(1) << (8 * low)) - 1));
    if (low > 0 && lowbits != 0) {
        const B hi_mask = static_cast<B>(~((B(1) << (8 * low)) - 1));
        if (tid == 0) *s_maxrun = 0;
        __syncthreads();
        // One scan: a thread owning a run start (first key of a run of equal high bits)
        // finds the run's end and insertion-sorts it on the full key (stable); runs longer
        // than LOCAL_MAX_RUN are only flagged. Other threads' sorts permute keys inside their
        // own runs only, so the high bits read across run borders never change.
        for (std::uint32_t j = tid; j < len; j += LOCAL_BLOCK) {
            const B hj = ordered(s_stage[j], dsc) & hi_mask;
            if (j > 0 && (ordered(s_stage[j - 1], dsc) & hi_mask) == hj) continue;  // not a run start
            std::uint32_t e2 = j + 1;
            while (e2 < len && e2 - j <= LOCAL_MAX_RUN && (ordered(s_stage[e2], dsc) & hi_mask) == hj) ++e2;
            if (e2 - j < 2) continue;
            if (e2 - j > LOCAL_MAX_RUN) {
                atomicMax(s_maxrun, e2 - j);
                continue;
            }
            for (std::uint32_t x = j + 1; x < e2; ++x) {
                const T v = s_stage[x];
                const B ov = ordered(v, dsc);
                std::uint32_t y = x;
                while (y > j && ordered(s_stage[y - 1], dsc) > ov) {
                    s_stage[y] = s_stage[y - 1];
                    --y;
                }
                s_stage[y] = v;
            }
        }
        __syncthreads();
        if (*s_maxrun > LOCAL_MAX_RUN) {
            // long runs: radix-pass the low digits too, then the high digits again
            // (every pass is stable and the registers still hold the pre-fix-up order,
            // so the result is the stable sort)
#pragma unroll 1
            for (int p = 0; p < low; ++p)
                if ((vary >> (8 * p)) & 0xffu) do_pass(p);
#pragma unroll 1
            for (int p = low; p < PASSES; ++p)
                if ((vary >> (8 * p)) & 0xffu) do_pass(p);
        }
        __syncthreads();
    } else {
        __syncthreads();
    }
    for (std::uint32_t j = tid; j < len; j += LOCAL_BLOCK) out[b + j] = s_stage[j];
}

// Persistent loop over the ranges listed in list[1 .. list[0]] (the ranges the counting
// kernel below handed back).
template <typename T, int ITEMS>
__global__ void __launch_bounds__(LOCAL_BLOCK, ITEMS <= 8 ? 4 : (ITEMS <= 12 ? 3 : 2))
    local_redo_kernel(const T* __restrict__ in, T* __restrict__ out, const std::uint64_t* __restrict__ cuts,
                      int desc, int low, std::uint64_t* big, const std::uint64_t* __restrict__ list) {
    extern __shared__ __align__(16) unsigned char smem[];
    const std::uint64_t nr = list[0];
    for (std::uint64_t r = blockIdx.x; r < nr; r += gridDim.x) {
        local_radix_range<T, ITEMS>(in, out, cuts, list[1 + r], desc, low, big, smem);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Keys-only integer ranges: on-chip COUNTING sort (stability is unobservable for
// integer keys without payload -- equal keys are identical bit patterns -- so the
// order of equal digits may be arbitrary). One CTA per range:
//   1. load the range (coalesced), OR/AND-reduce the ordered keys -> varying bits;
//   2. bin by the top nb varying bits (2^nb ~ len bins, Poisson(~1) keys per bin):
//      one shared atomic per key gives its slot inside the bin;
//   3. block scan of the bin counts -> bin starts; keys stored at start + slot;
//   4. each key ranks itself inside its (short) bin on the full key and is written
//      straight to its final global position (bins are contiguous, so a warp's
//      stores stay within a few sectors).
// A range whose fullest bin exceeds LC_MAX_BIN (clustered keys) is left untouched and
// listed in `redo` for the stable radix kernel above.
// ---------------------------------------------------------------------------
// 1 if (a, ia) < (b, ib) lexicographically (64-bit unsigned key, then 32-bit index): the
// borrow out of the 96-bit subtraction -- four integer ops, no compares or branches.
__device__ __forceinline__ std::uint32_t lex_less96(std::uint64_t a, std::uint32_t ia, std::uint64_t b,
                                                    std::uint32_t ib) {
    std::uint32_t d0, d1, d2, bor;
    asm("sub.cc.u32 %0, %4, %5;\n\t"
        "subc.cc.u32 %1, %6, %7;\n\t"
        "subc.cc.u32 %2, %8, %9;\n\t"
        "subc.u32 %3, 0, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(bor)
        : "r"(ia), "r"(ib), "r"(static_cast<std::uint32_t>(a)), "r"(static_cast<std::uint32_t>(b)),
          "r"(static_cast<std::uint32_t>(a >> 32)), "r"(static_cast<std::uint32_t>(b >> 32)));
    return bor & 1u;
}

constexpr int LC_BLOCK = 512;
constexpr int LC_WARPS = LC_BLOCK / 32;
#ifndef AKB_LC3_BLOCK
#define AKB_LC3_BLOCK 512  // threads of the TMA-fed counting stage (local_count3_kernel)
#endif
constexpr int LC3_BLOCK = AKB_LC3_BLOCK;
constexpr int LC_MAX_BITS = 13;                        // up to 8192 bins (u16 counts, 2 per word)
constexpr int LC_WORDS = (1 << LC_MAX_BITS) / 2;       // 4096 counter words = 16 KB
constexpr std::uint32_t LC_MAX_BIN = 48;
#ifndef AKB_RANK_BRANCHFREE
#define AKB_RANK_BRANCHFREE 1
#endif
#ifndef AKB_RANK_UNROLL
#define AKB_RANK_UNROLL 6  // positions of local_count3's rank loop in flight per thread (r02: 3 -> 6, -1.6%)
#endif
constexpr int RANK_UNROLL = AKB_RANK_UNROLL;
#ifndef AKB_LC_EXTRA
#define AKB_LC_EXTRA 1  // bins = 2^(ceil(log2(len)) + EXTRA): ~2 bins per key
#endif

template <typename T, int ITEMS, int NT = LC_BLOCK>
struct lc_smem {
    static constexpr int CAP = NT * ITEMS;
    // two key buffers (the range being sorted + the next range in flight), each with one
    // spare key at both ends: TMA copies the 16-byte aligned superset of a range
    static constexpr std::size_t buf_bytes = (sizeof(T) * (CAP + 2) + 15) & ~std::size_t(15);
    static constexpr std::size_t buf_off = 0;
    static constexpr std::size_t cnt_off = 2 * buf_bytes;
    static constexpr std::size_t cnt_bytes = sizeof(std::uint32_t) * (LC_WORDS + 4);
    static constexpr std::size_t red_off = cnt_off + cnt_bytes;  // 2 x WARPS x u64 or/and partials
    static constexpr std::size_t wsum_off = red_off + 2 * LC_WARPS * sizeof(std::uint64_t);
    static constexpr std::size_t bar_off = wsum_off + 2 * LC_WARPS * sizeof(std::uint32_t);
    static constexpr std::size_t total = bar_off + 2 * sizeof(std::uint64_t);
    static constexpr int MINB = total + 1024 <= 114 * 1024 ? 2 : 1;  // CTAs per SM that fit
};

// local_count3_kernel: as lc_smem plus a second counter table (the rank loop of range i still
// reads its table while a faster warp zeroes the other one for range i + 1: no end barrier).
template <typename T, int ITEMS, int NT = LC_BLOCK>
struct lc3_smem : lc_smem<T, ITEMS, NT> {
    using B = lc_smem<T, ITEMS, NT>;
    static constexpr std::size_t cnt2_off = B::total;
    static constexpr std::size_t total = cnt2_off + B::cnt_bytes;
    static constexpr int MINB = total + 1024 <= 114 * 1024 ? 2 : 1;
};

// The counting stage of one range whose keys are in registers (k[i] = key i*LC_BLOCK + tid;
// padding repeats a valid key) and whose per-warp min / max partials of the ordered keys are
// in s_red[0..15] / s_red[16..31] (written before the caller's barrier): bins, ranks, and stores key j of the sorted range to out[j]. Returns 1
// (nothing stored) when a bin overflows LC_MAX_BIN. Ends with a barrier; block-uniform.
template <typename T, int ITEMS, bool DESC, bool MINMAX>
__device__ __forceinline__ int count_sort_store(const T (&k)[ITEMS], std::uint32_t len, int nb_want, T* __restrict__ out,
                                                bool copy_equal, T* s_stage, std::uint32_t* s_cw,
                                                typename key_traits<T>::bits* s_red, std::uint32_t* s_wsum) {
    using B = typename key_traits<T>::bits;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    std::uint16_t* s_c16 = reinterpret_cast<std::uint16_t*>(s_cw);
    // MINMAX: lanes 0-15 fold the min partials, lanes 16-31 the max partials, and bins are
    // taken from the OFFSET to the minimum, so a range straddling an aligned boundary
    // (0x0fff.. | 0x1000..) still spreads over all bins (value tiles of the P-way merge).
    // Otherwise OR / AND partials of the raw bits (bucket ranges of the sort, aligned by
    // construction; cheaper to reduce): vary = the bits that differ, kmin = 0.
    B kmin = 0, vary;
    {
        B x = s_red[lane];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const B y = __shfl_xor_sync(FULL, x, o);
            if constexpr (MINMAX) x = lane < 16 ? (y < x ? y : x) : (y > x ? y : x);
            else x = lane < 16 ? (x | y) : (x & y);
        }
        const B lo = __shfl_sync(FULL, x, 0), hi = __shfl_sync(FULL, x, 16);
        if constexpr (MINMAX) {
            kmin = lo;
            vary = hi - lo;
        } else {
            vary = lo & ~hi;
        }
    }
    if (vary == 0) {  // every key equal: the range is already sorted
        if (copy_equal)
            for (std::uint32_t j = tid; j < len; j += LC_BLOCK) out[j] = k[0];
        __syncthreads();  // s_red is rewritten by the next range
        return 0;
    }
    int hb;
    if constexpr (sizeof(B) == 8) hb = 63 - __clzll(static_cast<long long>(vary));
    else hb = 31 - __clz(static_cast<int>(vary));
    const int nb = max(1, min(nb_want, hb + 1));
    const int shift = hb + 1 - nb;
    const std::uint32_t bmask = (1u << nb) - 1u;
    const std::uint32_t nwords = 1u << (nb - 1);

    // bin | slot << 16 per key: one shared atomic per key on its bin's half of a word
    std::uint32_t pk[ITEMS];
    bool over = false;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool ok = static_cast<std::uint32_t>(i * LC_BLOCK + tid) < len;
        const std::uint32_t bn = static_cast<std::uint32_t>((ordered(k[i], DESC) - kmin) >> shift) & bmask;
        const std::uint32_t sh = (bn & 1u) * 16u;
        const std::uint32_t old = atom_add_shared_if(ok, s_cw + (bn >> 1), 1u << sh);
        const std::uint32_t slot = (old >> sh) & 0xffffu;
        over |= ok && slot >= LC_MAX_BIN;
        pk[i] = bn | (slot << 16);
    }
    if (__syncthreads_or(over)) return 1;  // clustered keys: the caller hands the range on
    // exclusive scan of the packed counts -> packed u16 bin starts. Warp w owns words
    // [w*WPW, (w+1)*WPW), lane l the uint4 quads q*128 + 4l (conflict-free), order (q, lane).
    {
        const std::uint32_t wpw = nwords / LC_WARPS;  // words per warp (0 when nwords < 16)
        const std::uint32_t nq = wpw / 128;           // full quads per lane
        std::uint32_t* wbase = s_cw + warp * wpw + 4 * lane;
        if (nq >= 1) {
            // up to 2 quads per lane (LC_WORDS / LC_WARPS = 256 words = 2 x 128)
            uint4 u[2];
            std::uint32_t cs[2] = {0, 0};
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (q < static_cast<int>(nq)) {
                    u[q] = *reinterpret_cast<const uint4*>(wbase + q * 128);
                    const std::uint32_t S = u[q].x + u[q].y + u[q].z + u[q].w;
                    cs[q] = (S & 0xffffu) + (S >> 16);
                }
            std::uint32_t p = cs[0] | (cs[1] << 16);  // both quads' sums scanned at once
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const std::uint32_t y = __shfl_up_sync(FULL, p, o);
                if (lane >= o) p += y;
            }
            const std::uint32_t t = __shfl_sync(FULL, p, 31);
            const std::uint32_t T0 = t & 0xffffu, T1 = t >> 16;
            if (lane == 0) s_wsum[warp] = T0 + T1;
            __syncthreads();
            std::uint32_t wp = lane < warp ? s_wsum[lane] : 0u;  // lane-parallel warp prefix
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wp += __shfl_xor_sync(FULL, wp, o);
            const std::uint32_t exq[2] = {wp + (p & 0xffffu) - cs[0], wp + T0 + (p >> 16) - cs[1]};
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (q < static_cast<int>(nq)) {
                    std::uint32_t run = exq[q];
                    std::uint32_t* wv = reinterpret_cast<std::uint32_t*>(&u[q]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const std::uint32_t lo = wv[j] & 0xffffu, hi = wv[j] >> 16;
                        wv[j] = run | ((run + lo) << 16);
                        run += lo + hi;
                    }
                    *reinterpret_cast<uint4*>(wbase + q * 128) = u[q];
                }
        } else {
            // small tables (<= 1024 words): thread t owns words [wpt*t, wpt*t + wpt), wpt <= 2
            const std::uint32_t wpt = nwords > LC_BLOCK ? 2u : 1u;
            const std::uint32_t w0 = static_cast<std::uint32_t>(tid) * wpt;
            const std::uint32_t c0 = w0 < nwords ? s_cw[w0] : 0u;
            const std::uint32_t c1 = (wpt == 2 && w0 + 1 < nwords) ? s_cw[w0 + 1] : 0u;
            const std::uint32_t S = c0 + c1;
            const std::uint32_t sum = (S & 0xffffu) + (S >> 16);
            std::uint32_t inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const std::uint32_t y = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            std::uint32_t wp = 0;
#pragma unroll
            for (int w = 0; w < LC_WARPS; ++w) wp += w < warp ? s_wsum[w] : 0u;
            std::uint32_t run = wp + inc - sum;
            if (w0 < nwords) {
                const std::uint32_t lo = c0 & 0xffffu, hi = c0 >> 16;
                s_cw[w0] = run | ((run + lo) << 16);
                run += lo + hi;
            }
            if (wpt == 2 && w0 + 1 < nwords) s_cw[w0 + 1] = run | ((run + (c1 & 0xffffu)) << 16);
        }
        if (tid == 0) s_c16[2 * nwords] = static_cast<std::uint16_t>(len);  // end of the last bin
    }
    __syncthreads();
    // scatter into bin order (ordered bits: ranked as unsigned)
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
        if (static_cast<std::uint32_t>(i * LC_BLOCK + tid) < len)
            reinterpret_cast<B*>(s_stage)[s_c16[pk[i] & 0xffffu] + (pk[i] >> 16)] = ordered(k[i], DESC);
    __syncthreads();
    // each staged position ranks its key inside its (short) bin on the full key:
    // final slot = bin start + #(key, staged slot) lexicographically smaller
    B* s_ord = reinterpret_cast<B*>(s_stage);
#pragma unroll 1
    for (std::uint32_t x = tid; x < len; x += LC_BLOCK) {
        const B v = s_ord[x];
        // bin extent: consecutive positions have nondecreasing bins, so a warp's counter
        // reads fall in a few words
        const std::uint32_t bn = static_cast<std::uint32_t>((v - kmin) >> shift) & bmask;
        const std::uint32_t st = s_c16[bn], cnt = s_c16[bn + 1] - st;
        std::uint32_t rk = x;
        if (cnt > 1) {
            rk = st + lex_less96(s_ord[st], st, v, x) + lex_less96(s_ord[st + 1], st + 1, v, x);
#pragma unroll 1
            for (std::uint32_t y = st + 2; y < st + cnt; ++y) rk += lex_less96(s_ord[y], y, v, x);
        }
        const B o = DESC ? static_cast<B>(~v) : v;
        out[rk] = static_cast<T>(std::is_signed_v<T> ? (o ^ (B(1) << (8 * sizeof(B) - 1))) : o);
    }
    __syncthreads();  // the counters are read above and zeroed by the next range
    return 0;
}

// Keys-only 64-bit integer ranges: on-chip COUNTING sort. Stability is unobservable for
// integer keys without payload (equal keys are identical bit patterns), so the order in
// which equal bins fill may be arbitrary. Persistent CTAs walk the ranges; a range's keys
// arrive by one TMA bulk copy (cp.async.bulk + mbarrier) issued while the previous range is
// being sorted. Per range:
//   1. OR/AND-reduce the keys -> varying bits; bin = the top nb varying bits (~2 bins per key);
//   2. one shared atomic per key on its bin's packed u16 counter gives its slot in the bin;
//   3. scan of the counters -> bin starts; keys stored at start + slot (bin order);
//   4. each staged position ranks its key inside its (short) bin on the full key and stores
//      it to out[b + rank] (nearly coalesced: rank stays inside the bin).
// A range whose fullest bin exceeds LC_MAX_BIN (clustered keys) is left untouched and listed
// in `redo` for the stable radix kernel; ranges above CAP go to `big` (segment fallback).
template <typename T, int ITEMS, bool DESC>
__global__ void __launch_bounds__(LC_BLOCK, lc_smem<T, ITEMS>::MINB)
    local_count_kernel(const T* __restrict__ in, T* __restrict__ out, const std::uint64_t* __restrict__ cuts,
                       std::uint64_t J, std::uint64_t* big, std::uint64_t* redo) {
    using L = lc_smem<T, ITEMS>;
    using B = typename key_traits<T>::bits;
    constexpr int CAP = L::CAP;
    static_assert(sizeof(T) == 8, "TMA alignment math assumes 8-byte keys");
    extern __shared__ __align__(16) unsigned char smem[];
    std::uint32_t* s_cw = reinterpret_cast<std::uint32_t*>(smem + L::cnt_off);  // packed u16 counts
    std::uint16_t* s_c16 = reinterpret_cast<std::uint16_t*>(smem + L::cnt_off);
    B* s_red = reinterpret_cast<B*>(smem + L::red_off);
    std::uint32_t* s_wsum = reinterpret_cast<std::uint32_t*>(smem + L::wsum_off);
    std::uint64_t* s_bar = reinterpret_cast<std::uint64_t*>(smem + L::bar_off);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // TMA needs a 16-byte aligned source; the copy is the 16-byte aligned superset of the
    // range, which never leaves the allocation's last 16-byte granule
    const bool tma = (reinterpret_cast<std::uintptr_t>(in) & 15) == 0;
    auto fits = [&](std::uint64_t rb, std::uint64_t re) {
        return re > rb && re - rb <= static_cast<std::uint64_t>(CAP);
    };
    auto issue = [&](std::uint64_t r, int q) {  // one thread
        const std::uint64_t rb = cuts[r], re = cuts[r + 1];
        if (!tma || !fits(rb, re)) return;
        const std::uint64_t a0 = rb & ~std::uint64_t(1), a1 = (re + 1) & ~std::uint64_t(1);
        const std::uint32_t bytes = static_cast<std::uint32_t>((a1 - a0) * sizeof(T));
        mbar_arrive_expect_tx(s_bar + q, bytes);
        bulk_g2s(smem + L::buf_off + q * L::buf_bytes, in + a0, bytes, s_bar + q);
    };
    if (tid == 0) {
        mbar_init(s_bar, 1);
        mbar_init(s_bar + 1, 1);
        mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x < J) issue(blockIdx.x, 0);
    std::uint32_t ph0 = 0, ph1 = 0;  // parity of each buffer's next completion

#pragma unroll 1
    for (std::uint64_t r = blockIdx.x, it = 0; r < J; r += gridDim.x, ++it) {
        const int cur = static_cast<int>(it & 1);
        T* s_stage = reinterpret_cast<T*>(smem + L::buf_off + cur * L::buf_bytes);
        const std::uint64_t b = cuts[r], e = cuts[r + 1];
        const bool ok_range = fits(b, e);
        const std::uint32_t len = ok_range ? static_cast<std::uint32_t>(e - b) : 0u;
        const std::uint32_t off = static_cast<std::uint32_t>(b & 1);
        if (ok_range && tma) {
            if (cur) {
                mbar_wait(s_bar + 1, ph1);
                ph1 ^= 1u;
            } else {
                mbar_wait(s_bar, ph0);
                ph0 ^= 1u;
            }
        }

        // keys -> registers; varying bits. XOR with a constant (sign flip, descending
        // complement) flips a bit in every key alike, so OR & ~AND of the raw bits equals
        // that of the ordered bits. Padding repeats key 0 (neutral for OR/AND).
        T k[ITEMS];
        B orv = 0, andv = static_cast<B>(~B(0));
        if (len) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const std::uint32_t li = static_cast<std::uint32_t>(i * LC_BLOCK + tid);
                const std::uint32_t lj = li < len ? li : 0u;
                k[i] = tma ? s_stage[lj + off] : in[b + lj];
                orv |= static_cast<B>(k[i]);
                andv &= static_cast<B>(k[i]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            orv |= __shfl_xor_sync(FULL, orv, o);
            andv &= __shfl_xor_sync(FULL, andv, o);
        }
        if (lane == 0) {
            s_red[warp] = orv;
            s_red[LC_WARPS + warp] = andv;
        }
        const int nb_want = min(LC_MAX_BITS, (len <= 1 ? 0 : 32 - __clz(len - 1)) + AKB_LC_EXTRA);
        const int nwords_w = nb_want >= 1 ? (1 << (nb_want - 1)) : 1;
        if (nwords_w >= 4) {
            for (int i = tid; i < nwords_w / 4; i += LC_BLOCK)
                reinterpret_cast<uint4*>(s_cw)[i] = make_uint4(0, 0, 0, 0);
        } else if (tid < nwords_w) {
            s_cw[tid] = 0;
        }
        fence_proxy_async_smem();  // generic accesses to the other buffer precede its next TMA write
        __syncthreads();
        // every thread is past the previous range: its buffer may take the next one
        if (tid == 0 && r + gridDim.x < J) issue(r + gridDim.x, cur ^ 1);
        if (!ok_range) {
            if (e - b > static_cast<std::uint64_t>(CAP) && tid == 0) {  // left for the segment fallback
                const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull);
                big[1 + slot] = r;
            }
            __syncthreads();  // s_red is rewritten by the next range
            continue;
        }
        const int st_ = count_sort_store<T, ITEMS, DESC, false>(k, len, nb_want, out + b, in != out, s_stage, s_cw, s_red,
                                                         s_wsum);
        if (st_ == 1 && tid == 0) {  // clustered keys: hand the range to the radix kernel
            const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(redo), 1ull);
            redo[1 + slot] = r;
        }
    }  // ranges
}

// Counting local stage, lean variant (TMA-fed input only): local_count_kernel's algorithm --
// bins = the top nb varying bits (~2 bins per key), one shared atomic per key, keys staged in
// bin order, then every staged position ranks its key inside its (short) bin and stores it to
// its final place -- with the per-key instruction overhead cut: keys stay in ordered bits in
// registers, varying bits = OR of key ^ first key (one 64-bit reduction instead of OR + AND),
// no global-load fallback path (unaligned input takes local_count_kernel), 32-bit shared
// addressing, 32-bit range loop, double-buffered reduction slots.
// profiles/r02: local_count_kernel issued ~150 instructions per key (63% issue-busy, IPC 2.5).
// Measured and dropped (r02): settling only the keys that share a bin (random in-bin reads +
// an in-place rewrite) 2.10 ms, and coarse 16-key bins ranked by warp shuffles 5.2 ms, vs
// 1.78 ms for the per-position rank below (at 2^28 int64).
// ---- helpers of the counting local stages (one CTA of NT threads; call from all threads) ----

// Exclusive scan of nwords packed u16 bin counts (two per word) into packed u16 bin starts;
// s_c16[2 * nwords] = len afterwards (the end of the last bin). Contains __syncthreads().
template <int NT = LC_BLOCK>
__device__ __forceinline__ void lc_scan_counts(std::uint32_t* s_cw, std::uint32_t nwords, std::uint32_t len,
                                               std::uint32_t* s_wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const std::uint32_t wpw = nwords / (NT / 32);
    const std::uint32_t nq = wpw / 128;
    std::uint32_t* wbase = s_cw + warp * wpw + 4 * lane;
    if (nq >= 1) {
        uint4 u[2];
        std::uint32_t cs[2] = {0, 0};
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (q < static_cast<int>(nq)) {
                u[q] = *reinterpret_cast<const uint4*>(wbase + q * 128);
                const std::uint32_t S = u[q].x + u[q].y + u[q].z + u[q].w;
                cs[q] = (S & 0xffffu) + (S >> 16);
            }
        std::uint32_t p = cs[0] | (cs[1] << 16);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t y = __shfl_up_sync(FULL, p, o);
            if (lane >= o) p += y;
        }
        const std::uint32_t t = __shfl_sync(FULL, p, 31);
        const std::uint32_t T0 = t & 0xffffu, T1 = t >> 16;
        if (lane == 0) s_wsum[warp] = T0 + T1;
        __syncthreads();
        std::uint32_t wp = lane < warp ? s_wsum[lane] : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wp += __shfl_xor_sync(FULL, wp, o);
        const std::uint32_t exq[2] = {wp + (p & 0xffffu) - cs[0], wp + T0 + (p >> 16) - cs[1]};
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (q < static_cast<int>(nq)) {
                std::uint32_t run = exq[q];
                std::uint32_t* wv = reinterpret_cast<std::uint32_t*>(&u[q]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const std::uint32_t lo = wv[j] & 0xffffu, hi = wv[j] >> 16;
                    wv[j] = run | ((run + lo) << 16);
                    run += lo + hi;
                }
                *reinterpret_cast<uint4*>(wbase + q * 128) = u[q];
            }
    } else {
        const std::uint32_t wpt = nwords > NT ? 2u : 1u;
        const std::uint32_t w0 = static_cast<std::uint32_t>(tid) * wpt;
        const std::uint32_t c0 = w0 < nwords ? s_cw[w0] : 0u;
        const std::uint32_t c1 = (wpt == 2 && w0 + 1 < nwords) ? s_cw[w0 + 1] : 0u;
        const std::uint32_t S = c0 + c1;
        const std::uint32_t sum = (S & 0xffffu) + (S >> 16);
        std::uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        std::uint32_t wp = lane < warp ? s_wsum[lane] : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wp += __shfl_xor_sync(FULL, wp, o);
        std::uint32_t run = wp + inc - sum;
        if (w0 < nwords) {
            const std::uint32_t lo = c0 & 0xffffu, hi = c0 >> 16;
            s_cw[w0] = run | ((run + lo) << 16);
            run += lo + hi;
        }
        if (wpt == 2 && w0 + 1 < nwords) s_cw[w0 + 1] = run | ((run + (c1 & 0xffffu)) << 16);
    }
    if (tid == 0) reinterpret_cast<std::uint16_t*>(s_cw)[2 * nwords] = static_cast<std::uint16_t>(len);
}

// Each staged position x ranks its key inside its bin (bins = ((v - kmin) >> shift) & bmask,
// starts in s_c16, staged keys in sb, bin order): final slot = bin start + #(key, position)
// lexicographically smaller; store(rank, key) is called once per position.
template <typename B, int NT = LC_BLOCK, int U = 3, typename Store>
__device__ __forceinline__ void lc_rank_store(const B* sb, const std::uint16_t* s_c16, std::uint32_t len, B kmin,
                                              int shift, std::uint32_t bmask, Store&& store) {
#pragma unroll U
    for (std::uint32_t x = threadIdx.x; x < len; x += NT) {
        const B v = sb[x];
        const std::uint32_t bn = static_cast<std::uint32_t>((v - kmin) >> shift) & bmask;
        const std::uint32_t st = s_c16[bn], cnt = s_c16[bn + 1] - st;
#if AKB_RANK_BRANCHFREE
        // the first two members are compared without a branch: for a one-key bin st == x (the
        // self-compare counts 0) and slot st + 1 is the next bin's first key or a spare slot of
        // the buffer, masked out; lanes of a warp read near-consecutive slots
        const B a0 = sb[st], a1 = sb[st + 1];
        std::uint32_t rk = st + lex_less96(a0, st, v, x) + (cnt > 1 ? lex_less96(a1, st + 1, v, x) : 0u);
        if (cnt > 2) {
#pragma unroll 1
            for (std::uint32_t y = st + 2; y < st + cnt; ++y) rk += lex_less96(sb[y], y, v, x);
        }
#else
        std::uint32_t rk = x;
        if (cnt > 1) {
            rk = st + lex_less96(sb[st], st, v, x) + lex_less96(sb[st + 1], st + 1, v, x);
#pragma unroll 1
            for (std::uint32_t y = st + 2; y < st + cnt; ++y) rk += lex_less96(sb[y], y, v, x);
        }
#endif
        store(rk, v);
    }
}

// Exclusive scan of nwords (a power of two) packed u16 counts into packed u16 starts, any
// table size (NT threads): warp w owns words [w * wpw, (w + 1) * wpw); within it, row q of
// 128 words is read as one 16-byte quad per lane (conflict-free); more than two rows per
// warp are scanned in two reads (totals, then starts). Contains __syncthreads().
template <int NT>
__device__ __forceinline__ void wide_scan_counts(std::uint32_t* s_cw, std::uint32_t nwords, std::uint32_t len,
                                               std::uint32_t* s_wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const std::uint32_t wpw = nwords / (NT / 32);
    if (wpw <= 2 * 128) {  // up to two quads per lane: held in registers by the one-read scan
        lc_scan_counts<NT>(s_cw, nwords, len, s_wsum);
        return;
    }
    const std::uint32_t nq = wpw / 128;
    std::uint32_t* wbase = s_cw + warp * wpw + 4 * lane;
    // pass 1: the warp's total; pass 2: per row, a warp scan of the quad sums (recomputed
    // rather than kept: registers hold the range's keys)
    std::uint32_t tot = 0;
#pragma unroll 4
    for (std::uint32_t q = 0; q < nq; ++q) {
        const uint4 u = *reinterpret_cast<const uint4*>(wbase + q * 128);
        const std::uint32_t S = u.x + u.y + u.z + u.w;
        tot += (S & 0xffffu) + (S >> 16);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0) s_wsum[warp] = tot;
    __syncthreads();
    std::uint32_t run = lane < warp ? s_wsum[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) run += __shfl_xor_sync(FULL, run, o);
#pragma unroll 1
    for (std::uint32_t q = 0; q < nq; ++q) {
        uint4 u = *reinterpret_cast<const uint4*>(wbase + q * 128);
        const std::uint32_t S = u.x + u.y + u.z + u.w;
        const std::uint32_t c = (S & 0xffffu) + (S >> 16);
        std::uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        std::uint32_t r = run + inc - c;
        run += __shfl_sync(FULL, inc, 31);
        std::uint32_t* wv = reinterpret_cast<std::uint32_t*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const std::uint32_t lo = wv[j] & 0xffffu, hi = wv[j] >> 16;
            wv[j] = r | ((r + lo) << 16);
            r += lo + hi;
        }
        *reinterpret_cast<uint4*>(wbase + q * 128) = u;
    }
    if (tid == 0) reinterpret_cast<std::uint16_t*>(s_cw)[2 * nwords] = static_cast<std::uint16_t>(len);
}

template <typename T, int ITEMS, bool DESC, int NT = LC_BLOCK>
__global__ void __launch_bounds__(NT, lc3_smem<T, ITEMS, NT>::MINB)
    local_count3_kernel(const T* __restrict__ in, T* __restrict__ out, const std::uint64_t* __restrict__ cuts,
                        std::uint64_t J, std::uint64_t* big, std::uint64_t* redo,
                        const std::uint64_t* __restrict__ dplan) {
    using L = lc3_smem<T, ITEMS, NT>;
    constexpr int W = NT / 32;
    using B = typename key_traits<T>::bits;
    constexpr int CAP = L::CAP;
    static_assert(sizeof(T) == 8, "8-byte keys");
    constexpr B X = (std::is_signed_v<T> ? (B(1) << 63) : B(0)) ^ (DESC ? ~B(0) : B(0));  // raw <-> ordered
    extern __shared__ __align__(16) unsigned char smem[];
    B* s_red = reinterpret_cast<B*>(smem + L::red_off);  // [2][WARPS] OR partials
    std::uint32_t* s_wsum = reinterpret_cast<std::uint32_t*>(smem + L::wsum_off);
    std::uint64_t* s_bar = reinterpret_cast<std::uint64_t*>(smem + L::bar_off);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto fits = [&](std::uint64_t rb, std::uint64_t re) {
        return re > rb && re - rb <= static_cast<std::uint64_t>(CAP);
    };
    auto issue_at = [&](std::uint64_t rb, std::uint64_t re, int q) {  // one thread
        if (!fits(rb, re)) return;
        const std::uint64_t a0 = rb & ~std::uint64_t(1), a1 = (re + 1) & ~std::uint64_t(1);
        const std::uint32_t bytes = static_cast<std::uint32_t>((a1 - a0) * sizeof(T));
        mbar_arrive_expect_tx(s_bar + q, bytes);
        bulk_g2s(smem + L::buf_off + q * L::buf_bytes, in + a0, bytes, s_bar + q);
    };
    auto issue = [&](std::uint64_t r, int q) { issue_at(cuts[r], cuts[r + 1], q); };
    if (tid == 0) {
        mbar_init(s_bar, 1);
        mbar_init(s_bar + 1, 1);
        mbar_init_fence();
    }
    __syncthreads();
    // ranges < 2^32 (n / 256 at most); a device plan (dplan: {mode, group, J}) overrides J
    const std::uint32_t nr = static_cast<std::uint32_t>(dplan ? (dplan[0] ? 0 : dplan[2]) : J);
    if (tid == 0 && blockIdx.x < nr) issue(blockIdx.x, 0);
    std::uint32_t phase = 0;  // bit q = parity of buffer q's next completion
    const bool copy_equal = in != out;

    std::uint64_t nb_ = 0, ne_ = 0;  // the range bounds, loaded one range ahead
    if (blockIdx.x < nr) {
        nb_ = cuts[blockIdx.x];
        ne_ = cuts[blockIdx.x + 1];
    }
#pragma unroll 1
    for (std::uint32_t r = blockIdx.x, it = 0; r < nr; r += gridDim.x, ++it) {
        const int cur = static_cast<int>(it & 1);
        const std::uint64_t b = nb_, e = ne_;
        if (r + gridDim.x < nr) {
            nb_ = cuts[r + gridDim.x];
            ne_ = cuts[r + gridDim.x + 1];
        }
        const bool ok_range = fits(b, e);
        const std::uint32_t len = ok_range ? static_cast<std::uint32_t>(e - b) : 0u;
        B* sb = reinterpret_cast<B*>(smem + L::buf_off + cur * L::buf_bytes) + static_cast<std::uint32_t>(b & 1);
        B* red = s_red + cur * W;
        // packed u16 counts / starts, one table per parity of the range
        std::uint32_t* s_cw = reinterpret_cast<std::uint32_t*>(smem + (cur ? L::cnt2_off : L::cnt_off));
        const std::uint16_t* s_c16 = reinterpret_cast<const std::uint16_t*>(s_cw);
        B k[ITEMS];
        B orx = 0;
        if (ok_range) {
            mbar_wait(s_bar + cur, (phase >> cur) & 1u);
            phase ^= 1u << cur;
            const B k0 = sb[0];
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                if (static_cast<std::uint32_t>(i * NT) >= len) break;  // rows past len stay unused
                const std::uint32_t li = static_cast<std::uint32_t>(i * NT + tid);
                const B v = li < len ? sb[li] : k0;  // padding repeats key 0 (neutral below)
                orx |= v ^ k0;
                k[i] = v ^ X;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) orx |= __shfl_xor_sync(FULL, orx, o);
        if (lane == 0) red[warp] = orx;
        const int nb_want = min(LC_MAX_BITS, (len <= 1 ? 0 : 32 - __clz(len - 1)) + AKB_LC_EXTRA);
        const int nwords_w = nb_want >= 1 ? (1 << (nb_want - 1)) : 1;
        if (nwords_w >= 4) {
            for (int i = tid; i < nwords_w / 4; i += NT)
                reinterpret_cast<uint4*>(s_cw)[i] = make_uint4(0, 0, 0, 0);
        } else if (tid < nwords_w) {
            s_cw[tid] = 0;
        }
        fence_proxy_async_smem();  // generic accesses to the other buffer precede its next TMA write
        __syncthreads();
        if (tid == 0 && r + gridDim.x < nr) issue_at(nb_, ne_, cur ^ 1);  // the bounds loaded ahead
        if (!ok_range) {
            if (e - b > static_cast<std::uint64_t>(CAP) && tid == 0) {  // left for the segment fallback
                const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull);
                big[1 + slot] = r;
            }
            continue;
        }
        B vary = lane < W ? red[lane] : B(0);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) vary |= __shfl_xor_sync(FULL, vary, o);
        vary = __shfl_sync(FULL, vary, 0);
        if (vary == 0) {  // every key equal: the range is already sorted
            if (copy_equal)
                for (std::uint32_t j = tid; j < len; j += NT) out[b + j] = static_cast<T>(k[0] ^ X);
            continue;
        }
        const int hb = 63 - __clzll(static_cast<long long>(vary));
        const int nb = max(1, min(nb_want, hb + 1));
        const int shift = hb + 1 - nb;
        const std::uint32_t bmask = (1u << nb) - 1u;
        const std::uint32_t nwords = 1u << (nb - 1);

        // ---- counting: one shared atomic per key on its bin's half word -> slot in the bin ----
        // slots (< LC_MAX_BIN = 48: 6 bits) packed five per word; bins are recomputed from the keys
        constexpr int SW = (ITEMS + 4) / 5;
        std::uint32_t sl[SW];
#pragma unroll
        for (int w = 0; w < SW; ++w) sl[w] = 0;
        bool over = false;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (static_cast<std::uint32_t>(i * NT) >= len) break;
            const bool ok = static_cast<std::uint32_t>(i * NT + tid) < len;
            const std::uint32_t bn = static_cast<std::uint32_t>(k[i] >> shift) & bmask;
            const std::uint32_t sh = (bn & 1u) << 4;
            const std::uint32_t old = atom_add_shared_if(ok, s_cw + (bn >> 1), 1u << sh);
            const std::uint32_t slot = (old >> sh) & 0xffffu;
            over |= ok && slot >= LC_MAX_BIN;
            sl[i / 5] |= (slot & 0x3fu) << (6 * (i % 5));
        }
        if (__syncthreads_or(over)) {  // clustered keys: the stable radix kernel takes the range
            if (tid == 0) {
                const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(redo), 1ull);
                redo[1 + slot] = r;
            }
            continue;
        }
        // ---- exclusive scan of the packed counts -> packed u16 bin starts (as local_count) ----
        wide_scan_counts<NT>(s_cw, nwords, len, s_wsum);
        __syncthreads();
        // ---- keys into bin order (the range's own TMA buffer is free: keys are in registers) ----
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (static_cast<std::uint32_t>(i * NT) >= len) break;
            if (static_cast<std::uint32_t>(i * NT + tid) < len)
                sb[s_c16[static_cast<std::uint32_t>(k[i] >> shift) & bmask] + ((sl[i / 5] >> (6 * (i % 5))) & 0x3fu)] = k[i];
        }
        __syncthreads();
        // ---- each position ranks its key inside its bin: final slot = bin start + #(key, pos) smaller ----
        lc_rank_store<B, NT, RANK_UNROLL>(sb, s_c16, len, B(0), shift, bmask, [&](std::uint32_t rk, B v) { out[b + rk] = static_cast<T>(v ^ X); });
    }  // ranges
}

// Big-range counting stage (n >= 2^29 after two MSD levels): ranges of up to LB_CAP = 18432
// keys -- a whole 16-bit bucket of a 2^30-key sort -- in ONE CTA per SM (the key buffer takes
// 144 KB of shared memory; 18 keys per thread of 1024 in registers), so two partition levels suffice
// where the 4608-key stage needed a third level and its 24-bit histogram. The algorithm is
// local_count3's (up to 2^15 packed u16 bins, one shared atomic per key, scan, bin-order
// scatter, per-position rank; ranges = aligned groups of 1, 2, 4 or 8 16-bit buckets, so the
// OR-reduced varying bits are exact -- a range cut at arbitrary bucket boundaries could
// straddle an aligned boundary and crowd a few bins); the differences: the single buffer (the
// next range's TMA copy is issued once this range's rank loop is done) and the scan over up
// to 16384 counter words. A bin over LC_MAX_BIN keys sends the range to the segment fallback
// (big list: the stable redo kernel holds only 6144 keys).
#ifndef AKB_LB_BLOCK
#define AKB_LB_BLOCK 1024
#endif
constexpr int LB_BLOCK = AKB_LB_BLOCK;
constexpr int LB_WARPS = LB_BLOCK / 32;
constexpr int LB_ITEMS = 18432 / LB_BLOCK;
constexpr int LB_CAP = LB_BLOCK * LB_ITEMS;  // 18432 keys
#ifndef AKB_LB_MAX_BITS
#define AKB_LB_MAX_BITS 14  // r02: 13 / 14 / 15 bits -> 7.23 / 6.58 / 6.94 ms at 2^30 (one bin per key wins here)
#endif
constexpr int LB_MAX_BITS = AKB_LB_MAX_BITS;
constexpr int LB_WORDS = (1 << LB_MAX_BITS) / 2;  // 16384 counter words = 64 KB

template <typename T>
struct lb_smem {
    static constexpr std::size_t buf_bytes = (sizeof(T) * (LB_CAP + 2) + 15) & ~std::size_t(15);
    static constexpr std::size_t buf_off = 0;
    static constexpr std::size_t cnt_off = buf_bytes;
    static constexpr std::size_t cnt_bytes = sizeof(std::uint32_t) * (LB_WORDS + 4);
    static constexpr std::size_t red_off = cnt_off + cnt_bytes;                 // WARPS x u64 (+ spare)
    static constexpr std::size_t wsum_off = red_off + 2 * LB_WARPS * sizeof(std::uint64_t);
    static constexpr std::size_t bar_off = wsum_off + LB_WARPS * sizeof(std::uint32_t);
    static constexpr std::size_t total = bar_off + sizeof(std::uint64_t);
};


template <typename T, bool DESC>
__global__ void __launch_bounds__(LB_BLOCK, 1)
    local_big_kernel(const T* __restrict__ in, T* out, const std::uint64_t* __restrict__ cuts, std::uint64_t J,
                     std::uint64_t* big, const std::uint64_t* __restrict__ dplan) {
    using L = lb_smem<T>;
    using B = typename key_traits<T>::bits;
    constexpr int ITEMS = LB_ITEMS;
    static_assert(sizeof(T) == 8, "8-byte keys");
    constexpr B X = (std::is_signed_v<T> ? (B(1) << 63) : B(0)) ^ (DESC ? ~B(0) : B(0));  // raw <-> ordered
    extern __shared__ __align__(16) unsigned char smem[];
    B* s_red = reinterpret_cast<B*>(smem + L::red_off);
    std::uint32_t* s_wsum = reinterpret_cast<std::uint32_t*>(smem + L::wsum_off);
    std::uint64_t* s_bar = reinterpret_cast<std::uint64_t*>(smem + L::bar_off);
    std::uint32_t* s_cw = reinterpret_cast<std::uint32_t*>(smem + L::cnt_off);
    const std::uint16_t* s_c16 = reinterpret_cast<const std::uint16_t*>(s_cw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto fits = [&](std::uint64_t rb, std::uint64_t re) {
        return re > rb && re - rb <= static_cast<std::uint64_t>(LB_CAP);
    };
    auto issue_at = [&](std::uint64_t rb, std::uint64_t re) {  // one thread; the buffer is idle
        if (!fits(rb, re)) return;
        const std::uint64_t a0 = rb & ~std::uint64_t(1), a1 = (re + 1) & ~std::uint64_t(1);
        const std::uint32_t bytes = static_cast<std::uint32_t>((a1 - a0) * sizeof(T));
        mbar_arrive_expect_tx(s_bar, bytes);
        bulk_g2s(smem + L::buf_off, in + a0, bytes, s_bar);
    };
    if (tid == 0) {
        mbar_init(s_bar, 1);
        mbar_init_fence();
    }
    __syncthreads();
    const std::uint32_t nr = static_cast<std::uint32_t>(dplan ? (dplan[0] ? 0 : dplan[2]) : J);
    if (tid == 0 && blockIdx.x < nr) issue_at(cuts[blockIdx.x], cuts[blockIdx.x + 1]);
    std::uint32_t phase = 0;
    const bool copy_equal = in != out;

    // the range bounds are loaded one range ahead (one CTA per SM: a cold global load per
    // range would sit on the critical path)
    std::uint64_t nb_ = 0, ne_ = 0;
    if (blockIdx.x < nr) {
        nb_ = cuts[blockIdx.x];
        ne_ = cuts[blockIdx.x + 1];
    }
#pragma unroll 1
    for (std::uint32_t r = blockIdx.x; r < nr; r += gridDim.x) {
        const std::uint64_t b = nb_, e = ne_;
        if (r + gridDim.x < nr) {
            nb_ = cuts[r + gridDim.x];
            ne_ = cuts[r + gridDim.x + 1];
        }
        const bool ok_range = fits(b, e);
        const std::uint32_t len = ok_range ? static_cast<std::uint32_t>(e - b) : 0u;
        B* sb = reinterpret_cast<B*>(smem + L::buf_off) + static_cast<std::uint32_t>(b & 1);
        B k[ITEMS];
        B mx = 0;  // OR of the bits that differ from the first key
        if (ok_range) {
            mbar_wait(s_bar, phase);
            phase ^= 1u;
            const B k0 = sb[0];
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                if (static_cast<std::uint32_t>(i * LB_BLOCK) >= len) break;  // rows past len stay unused
                const std::uint32_t li = static_cast<std::uint32_t>(i * LB_BLOCK + tid);
                const B v = (li < len ? sb[li] : k0) ^ X;  // padding repeats key 0 (neutral)
                k[i] = v;
                mx |= v ^ (k0 ^ X);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx |= __shfl_xor_sync(FULL, mx, o);
        if (lane == 0) s_red[warp] = mx;
        const int nb_want = min(LB_MAX_BITS, (len <= 1 ? 0 : 32 - __clz(len - 1)) + AKB_LC_EXTRA);
        const int nwords_w = nb_want >= 1 ? (1 << (nb_want - 1)) : 1;
        if (nwords_w >= 4) {
            for (int i = tid; i < nwords_w / 4; i += LB_BLOCK) reinterpret_cast<uint4*>(s_cw)[i] = make_uint4(0, 0, 0, 0);
        } else if (tid < nwords_w) {
            s_cw[tid] = 0;
        }
        __syncthreads();
        bool done = !ok_range;
        if (!ok_range && e - b > static_cast<std::uint64_t>(LB_CAP) && tid == 0) {
            const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull);
            big[1 + slot] = r;
        }
        B vary = 0;
        if (!done) {  // ranges are aligned groups of buckets: the OR of the differing bits is exact
            vary = lane < LB_WARPS ? s_red[lane] : B(0);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) vary |= __shfl_xor_sync(FULL, vary, o);
            if (vary == 0) {  // every key equal
                if (copy_equal)
                    for (std::uint32_t j = tid; j < len; j += LB_BLOCK) out[b + j] = static_cast<T>(k[0] ^ X);
                done = true;
            }
        }
        if (!done) {
            const int hb = 63 - __clzll(static_cast<long long>(vary));
            const int nb = max(1, min(nb_want, hb + 1));
            const int shift = hb + 1 - nb;
            const std::uint32_t bmask = (1u << nb) - 1u;
            const std::uint32_t nwords = 1u << (nb - 1);
            constexpr int SW = (ITEMS + 4) / 5;
            std::uint32_t sl[SW];
#pragma unroll
            for (int w = 0; w < SW; ++w) sl[w] = 0;
            bool over = false;
            // item rows past len are skipped by block-uniform branches
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                if (static_cast<std::uint32_t>(i * LB_BLOCK) >= len) break;
                const bool ok = static_cast<std::uint32_t>(i * LB_BLOCK + tid) < len;
                const std::uint32_t bn = static_cast<std::uint32_t>(k[i] >> shift) & bmask;
                const std::uint32_t sh = (bn & 1u) << 4;
                const std::uint32_t old = atom_add_shared_if(ok, s_cw + (bn >> 1), 1u << sh);
                const std::uint32_t slot = (old >> sh) & 0xffffu;
                over |= ok && slot >= LC_MAX_BIN;
                sl[i / 5] |= (slot & 0x3fu) << (6 * (i % 5));
            }
            if (__syncthreads_or(over)) {  // clustered keys: the segment fallback sorts the range
                if (tid == 0) {
                    const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull);
                    big[1 + slot] = r;
                }
            } else {
                wide_scan_counts<LB_BLOCK>(s_cw, nwords, len, s_wsum);
                __syncthreads();
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    if (static_cast<std::uint32_t>(i * LB_BLOCK) >= len) break;
                    if (static_cast<std::uint32_t>(i * LB_BLOCK + tid) < len)
                        sb[s_c16[static_cast<std::uint32_t>(k[i] >> shift) & bmask] + ((sl[i / 5] >> (6 * (i % 5))) & 0x3fu)] =
                            k[i];
                }
                __syncthreads();
                lc_rank_store<B, LB_BLOCK>(sb, s_c16, len, B(0), shift, bmask,
                                 [&](std::uint32_t rk, B v) { out[b + rk] = static_cast<T>(v ^ X); });
            }
        }
        // the buffer and the counters are idle once every thread is here: next range's copy
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0 && r + gridDim.x < nr) issue_at(nb_, ne_);  // the bounds loaded ahead
    }  // ranges
}

// Device plan of a small keys-only sort (no host round trip): among the top three digits
// (histograms in g_hist), the highest one that is not constant partitions the keys into 256
// buckets by one onesweep pass. Writes plan = {mode, shift} (mode 0 = go; 1 = its largest
// bucket exceeds cap: the host plan takes over after the call's one synchronisation), that
// digit's exclusive offsets (the pass's bucket starts) and the range cuts (the bucket
// starts; all zero when mode != 0, so the local stage finds only empty ranges).
__global__ void __launch_bounds__(RADIX) small_plan_kernel(const std::uint64_t* __restrict__ g_hist, std::uint64_t n,
                                                           std::uint64_t cap, int* __restrict__ plan,
                                                           std::uint64_t* __restrict__ offs,
                                                           std::uint64_t* __restrict__ cuts,
                                                           std::uint64_t* __restrict__ big,
                                                           std::uint64_t* __restrict__ redo) {
    __shared__ std::uint64_t s_w[RADIX / 32];
    __shared__ int s_d;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) s_d = -1;
    __syncthreads();
    std::uint64_t mx = 0;
    for (int d = 7; d >= 5; --d) {  // block-uniform loop
        std::uint64_t m = g_hist[d * RADIX + t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const std::uint64_t y = __shfl_xor_sync(FULL, m, o);
            m = m > y ? m : y;
        }
        if (lane == 0) s_w[w] = m;
        __syncthreads();
        mx = 0;
        for (int i = 0; i < RADIX / 32; ++i) mx = mx > s_w[i] ? mx : s_w[i];
        __syncthreads();
        if (mx < n) {
            if (t == 0) s_d = d;
            break;
        }
    }
    __syncthreads();
    const int d = s_d;
    const int mode = (d < 0 || mx > cap) ? 1 : 0;
    const std::uint64_t v = d >= 0 ? g_hist[d * RADIX + t] : 0;
    std::uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint64_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    std::uint64_t base = 0;
    for (int i = 0; i < w; ++i) base += s_w[i];
    const std::uint64_t ex = base + inc - v;
    offs[t] = ex;
    cuts[t] = mode == 0 ? ex : 0;
    if (t == 0) {
        cuts[RADIX] = mode == 0 ? n : 0;
        plan[0] = mode;
        plan[1] = 8 * (d < 0 ? 0 : d);
        big[0] = 0;  // the local stage's oversized / clustered range lists
        redo[0] = 0;
    }
}

// cut j = first index of the bucket (top bits) holding position j*step; cuts[J] = n.
template <typename T>
__global__ void range_cuts_kernel(const T* __restrict__ keys, std::uint64_t n, int top_shift, int desc,
                                  std::uint64_t step, std::uint64_t J, std::uint64_t* __restrict__ cuts) {
    using B = typename key_traits<T>::bits;
    const std::uint64_t j = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j > J) return;
    if (j == 0 || j == J) {
        cuts[j] = j == 0 ? 0 : n;
        return;
    }
    const bool dsc = desc != 0;
    const std::uint64_t p = j * step;
    const B t = static_cast<B>(ordered(keys[p], dsc) >> top_shift);
    std::uint64_t lo = 0, hi = p;
    while (lo < hi) {
        const std::uint64_t mid = lo + (hi - lo) / 2;
        if (static_cast<B>(ordered(keys[mid], dsc) >> top_shift) < t) lo = mid + 1;
        else hi = mid;
    }
    cuts[j] = lo;
}

// cuts[0] = 0, cuts[j] = ends[j - 1] (the MSD cursors after the last pass = bucket ends), cuts[J] = n.
__global__ void cuts_from_ends_kernel(const std::uint64_t* __restrict__ ends, std::uint64_t J, std::uint64_t n,
                                      std::uint64_t group, const std::uint64_t* __restrict__ dplan,
                                      std::uint64_t* __restrict__ cuts) {
    if (dplan) {  // device plan {mode, group, J}: nothing to cut when the plan does not apply
        if (dplan[0]) return;
        group = dplan[1];
        J = dplan[2];
    }
    const std::uint64_t j = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j > J) return;
    cuts[j] = j == 0 ? 0 : (j == J ? n : ends[j * group - 1]);
}

// cut b = first index whose top bits are >= b (bucket starts), b in [0, J); cuts[J] = n.
template <typename T>
__global__ void bucket_cuts_kernel(const T* __restrict__ keys, std::uint64_t n, int top_shift, int desc,
                                   std::uint64_t J, std::uint64_t base_id, std::uint64_t* __restrict__ cuts) {
    using B = typename key_traits<T>::bits;
    const std::uint64_t j = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j > J) return;
    if (j == J) {
        cuts[j] = n;
        return;
    }
    const bool dsc = desc != 0;
    std::uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const std::uint64_t mid = lo + (hi - lo) / 2;
        if (static_cast<std::uint64_t>(ordered(keys[mid], dsc) >> top_shift) < base_id + j) lo = mid + 1;
        else hi = mid;
    }
    cuts[j] = lo;
}

// 0: stable onesweep top-digit passes instead of the MSD partition (experiment builds: make variant DEFS=-DAKB_CFG_MSD=...)
#ifndef AKB_CFG_MSD
#define AKB_CFG_MSD 1
#endif
constexpr int msd_env() { return AKB_CFG_MSD; }

// 0: plain LSD; m > 0: force m top passes; -1: planned from the data (experiment builds: make variant DEFS=-DAKB_CFG_HYBRID=...)
#ifndef AKB_CFG_HYBRID
#define AKB_CFG_HYBRID -1
#endif
constexpr int hybrid_env() { return AKB_CFG_HYBRID; }

// ---------------------------------------------------------------------------
// Keys-only 64-bit integer P-way merge (SIHSort's second local step): the output is cut
// into value tiles [b_j, b_{j+1}) (b_j from a sorted sample of every run); tile j is the
// union of one contiguous piece per run (lower_bound of b_j, b_{j+1} in each run), so it is
// sorted on chip by the counting stage above and stored at its output offset (the number of
// keys below b_j). Equal integer keys are indistinguishable, so this equals the stable merge.
// ---------------------------------------------------------------------------
constexpr int MC_MAXP = 16;

template <typename T, int ITEMS>
struct mc_smem {
    static constexpr int CAP = LC_BLOCK * ITEMS;
    static constexpr std::size_t stage_off = 0;
    static constexpr std::size_t cnt_off = sizeof(T) * CAP;
    static constexpr std::size_t red_off = cnt_off + sizeof(std::uint32_t) * (LC_WORDS + 4);
    static constexpr std::size_t wsum_off = red_off + 2 * LC_WARPS * sizeof(std::uint64_t);
    static constexpr std::size_t piece_off = wsum_off + 2 * LC_WARPS * sizeof(std::uint32_t);
    static constexpr std::size_t total = piece_off + 3 * (MC_MAXP + 1) * sizeof(std::uint64_t);
};

template <typename T, int ITEMS, bool DESC>
__global__ void __launch_bounds__(LC_BLOCK, 2)
    merge_count_kernel(const T* const* __restrict__ runs, int P, const std::uint64_t* __restrict__ pos, T* __restrict__ dst,
                       std::uint64_t* big) {
    using L = mc_smem<T, ITEMS>;
    using B = typename key_traits<T>::bits;
    constexpr int CAP = L::CAP;
    extern __shared__ __align__(16) unsigned char smem[];
    T* s_stage = reinterpret_cast<T*>(smem + L::stage_off);
    std::uint32_t* s_cw = reinterpret_cast<std::uint32_t*>(smem + L::cnt_off);
    B* s_red = reinterpret_cast<B*>(smem + L::red_off);
    std::uint32_t* s_wsum = reinterpret_cast<std::uint32_t*>(smem + L::wsum_off);
    std::uint64_t* s_lo = reinterpret_cast<std::uint64_t*>(smem + L::piece_off);  // piece start in its run
    std::uint64_t* s_pre = s_lo + (MC_MAXP + 1);                                   // prefix of piece lengths
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const std::uint64_t j = blockIdx.x;
    if (tid == 0) {
        std::uint64_t acc = 0, off = 0;
        for (int r = 0; r < P; ++r) {
            const std::uint64_t lo = pos[j * P + r], hi = pos[(j + 1) * P + r];
            s_lo[r] = lo;
            s_pre[r] = acc;
            acc += hi - lo;
            off += lo;
        }
        s_pre[P] = acc;
        s_pre[MC_MAXP + 1 + 0] = off;  // output offset of the tile
    }
    __syncthreads();
    const std::uint64_t total = s_pre[P], off = s_pre[MC_MAXP + 1];
    if (total == 0) return;
    if (total > static_cast<std::uint64_t>(CAP)) {
        if (tid == 0) {
            const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull);
            big[1 + slot] = j;
        }
        return;
    }
    const std::uint32_t len = static_cast<std::uint32_t>(total);
    T k[ITEMS];
    B orv = static_cast<B>(~B(0)), andv = 0;  // min / max of the ordered keys
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const std::uint32_t li = static_cast<std::uint32_t>(i * LC_BLOCK + tid);
        const std::uint32_t lj = li < len ? li : 0u;
        int r = 0;
        for (int q = 1; q < P; ++q) r += (s_pre[q] <= lj) ? 1 : 0;
        k[i] = runs[r][s_lo[r] + (lj - s_pre[r])];
        const B o = ordered(k[i], DESC);
        orv = o < orv ? o : orv;
        andv = o > andv ? o : andv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const B y0 = __shfl_xor_sync(FULL, orv, o), y1 = __shfl_xor_sync(FULL, andv, o);
        orv = y0 < orv ? y0 : orv;
        andv = y1 > andv ? y1 : andv;
    }
    if (lane == 0) {
        s_red[warp] = orv;
        s_red[LC_WARPS + warp] = andv;
    }
    const int nb_want = min(LC_MAX_BITS, (len <= 1 ? 0 : 32 - __clz(len - 1)) + AKB_LC_EXTRA);
    const int nwords_w = nb_want >= 1 ? (1 << (nb_want - 1)) : 1;
    if (nwords_w >= 4) {
        for (int i = tid; i < nwords_w / 4; i += LC_BLOCK) reinterpret_cast<uint4*>(s_cw)[i] = make_uint4(0, 0, 0, 0);
    } else if (tid < nwords_w) {
        s_cw[tid] = 0;
    }
    __syncthreads();
    if (count_sort_store<T, ITEMS, DESC, true>(k, len, nb_want, dst + off, true, s_stage, s_cw, s_red, s_wsum) == 1 &&
        tid == 0) {
        const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull);
        big[1 + slot] = j;
    }
}

// samples[so[r] + i] = run r at i * S (the run's first key included)
template <typename T>
__global__ void mc_sample_kernel(const T* const* __restrict__ runs, const std::uint64_t* __restrict__ so, int P,
                                 std::uint32_t S, T* __restrict__ samples) {
    const std::uint64_t M = so[P];
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t x = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < M; x += stride) {
        int r = 0;
        while (r + 1 < P && so[r + 1] <= x) ++r;
        samples[x] = runs[r][(x - so[r]) * S];
    }
}

// pos[j * P + r] = lower_bound(run r, b_j) with b_j = sorted[j * K]; row 0 = 0, row J = lens;
// mx = largest tile.
template <typename T>
__global__ void mc_bounds_kernel(const T* const* __restrict__ runs, const std::uint64_t* __restrict__ lens, int P,
                                 const T* __restrict__ sorted, std::uint64_t J, std::uint32_t K, int desc,
                                 std::uint64_t* __restrict__ pos) {
    const std::uint64_t x = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (x >= (J + 1) * P) return;
    const std::uint64_t j = x / P;
    const int r = static_cast<int>(x % P);
    const std::uint64_t n = lens[r];
    if (j == 0 || j == J) {
        pos[x] = j == 0 ? 0 : n;
        return;
    }
    const T v = sorted[j * K];
    const T* h = runs[r];
    std::uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const std::uint64_t mid = lo + (hi - lo) / 2;
        if (key_less(h[mid], v, desc != 0)) lo = mid + 1;
        else hi = mid;
    }
    pos[x] = lo;
}

__global__ void mc_maxtile_kernel(const std::uint64_t* __restrict__ pos, int P, std::uint64_t J,
                                  unsigned long long* __restrict__ mx) {
    const std::uint64_t j = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    std::uint64_t t = 0;
    if (j < J)
        for (int r = 0; r < P; ++r) t += pos[(j + 1) * P + r] - pos[j * P + r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const std::uint64_t y = __shfl_xor_sync(FULL, t, o);
        t = t > y ? t : y;
    }
    if ((threadIdx.x & 31) == 0 && t) atomicMax(mx, static_cast<unsigned long long>(t));
}

// Counting local stage (integer keys only), then the stable radix kernel over the ranges
// it handed back (persistent loop over redo[1 .. redo[0]]; no host round trip).
template <typename T, int ITEMS>
void launch_local_count(ak_ctx* c, const T* G, T* kout, const std::uint64_t* cuts, std::uint64_t J, std::uint64_t n,
                        bool desc, int low, std::uint64_t* big, std::uint64_t* redo, bool redo_zeroed = false,
                        const std::uint64_t* dplan = nullptr) {
    constexpr int CITEMS = ITEMS * LOCAL_BLOCK / LC_BLOCK;
    static_assert(CITEMS * LC_BLOCK == ITEMS * LOCAL_BLOCK, "same range capacity");
    using CS = lc_smem<T, CITEMS>;
    using LS = local_smem<T, ITEMS>;
    smem_attr(c, local_redo_kernel<T, ITEMS>, LS::total);
    if (!redo_zeroed) AKB_CUDA(cudaMemsetAsync(redo, 0, sizeof(std::uint64_t), c->stream));
    const int tok = ctx_prof_begin(c, KF_LOCAL);
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(J, static_cast<std::uint64_t>(c->sm_count) * CS::MINB));
    if ((reinterpret_cast<std::uintptr_t>(G) & 15) == 0) {  // TMA-fed lean kernel
        constexpr int NT3 = LC3_BLOCK;
        constexpr int CITEMS3 = ITEMS * LOCAL_BLOCK / NT3;
        static_assert(CITEMS3 * NT3 == ITEMS * LOCAL_BLOCK, "same range capacity");
        using C3 = lc3_smem<T, CITEMS3, NT3>;
        const unsigned grid3 =
            static_cast<unsigned>(std::min<std::uint64_t>(J, static_cast<std::uint64_t>(c->sm_count) * C3::MINB));
        auto kern = desc ? local_count3_kernel<T, CITEMS3, true, NT3> : local_count3_kernel<T, CITEMS3, false, NT3>;
        smem_attr(c, kern, C3::total);
        kern<<<grid3, NT3, C3::total, c->stream>>>(G, kout, cuts, J, big, redo, dplan);
    } else {
        auto kern = desc ? local_count_kernel<T, CITEMS, true> : local_count_kernel<T, CITEMS, false>;
        smem_attr(c, kern, CS::total);
        kern<<<grid, LC_BLOCK, CS::total, c->stream>>>(G, kout, cuts, J, big, redo);
    }
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    local_redo_kernel<T, ITEMS><<<static_cast<unsigned>(c->sm_count * 2), LOCAL_BLOCK, LS::total, c->stream>>>(
        G, kout, cuts, desc ? 1 : 0, low, big, redo);
    AKB_CUDA(cudaGetLastError());
    c->kernel_launches += 2;
}

// Returns false when the plain LSD should be used instead.
//
// The plan is read off the data: one histogram pass over the top three digits (plus all
// eight when those are constant) gives, per digit, its largest bin. Constant leading digits
// are skipped; the bucket size after m global passes over the next digits is estimated as
// n * prod(max bin / n) (exact for m = 1, independence otherwise), and the smallest m whose
// buckets fit a CTA is taken. Skewed inputs thus get more global digits instead of
// oversized ranges; a mis-estimate only costs the (bounded) segment fallback.
// Ranges the local stage left in `big` (oversized buckets of skewed keys): plain LSD on each
// segment, or on the whole array when there are many. Needs the big count on the host.
template <typename T>
void sort_oversized(ak_ctx* c, const T* G, T* kout, T* kalt, std::uint64_t n, bool desc, const std::uint64_t* cuts,
                    const std::uint64_t* big, std::uint64_t J, std::uint64_t nbig) {
    if (!nbig) return;
    std::vector<std::uint64_t> hc(J + 1), hl(nbig);
    AKB_CUDA(cudaMemcpy(hc.data(), cuts, (J + 1) * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
    AKB_CUDA(cudaMemcpy(hl.data(), big + 1, nbig * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
    const bool whole = nbig > 32;
    for (std::uint64_t r : hl) {
        const std::uint64_t b = hc[r], len = hc[r + 1] - hc[r];
        if (G != kout) AKB_CUDA(cudaMemcpyAsync(kout + b, G + b, len * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
        if (whole) continue;
        T* scratch = (G == kout) ? kalt + b : const_cast<T*>(G) + b;
        radix_sort_impl<T, std::uint32_t, SORT_KEYS>(c, kout + b, kout + b, scratch, nullptr, nullptr, nullptr, len,
                                                     desc, true);
    }
    if (whole) {
        T* scratch = (G == kout) ? kalt : const_cast<T*>(G);
        radix_sort_impl<T, std::uint32_t, SORT_KEYS>(c, kout, kout, scratch, nullptr, nullptr, nullptr, n, desc, true);
    }
}

// 1: two MSD levels + the big-range stage at n >= 2^29; 0: three MSD levels + the 4608-key
// stage (experiment builds: make variant DEFS=-DAKB_CFG_BIG_LOCAL=0)
#ifndef AKB_CFG_BIG_LOCAL
#define AKB_CFG_BIG_LOCAL 1
#endif

template <typename T>
void launch_local_big(ak_ctx* c, const T* G, T* kout, const std::uint64_t* cuts, std::uint64_t J, bool desc,
                      std::uint64_t* big, const std::uint64_t* dplan = nullptr) {
    using LB = lb_smem<T>;
    auto kern = desc ? local_big_kernel<T, true> : local_big_kernel<T, false>;
    smem_attr(c, kern, LB::total);
    const int tok = ctx_prof_begin(c, KF_LOCAL);
    kern<<<static_cast<unsigned>(std::min<std::uint64_t>(J, static_cast<std::uint64_t>(c->sm_count))), LB_BLOCK,
           LB::total, c->stream>>>(G, kout, cuts, J, big, dplan);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 1;
}

// device-planned one-level path up to here: its 8-bit buckets must fit a 4608-key CTA (uniform
// keys: ~n / 256 + 4 sigma), so at 2^21 it was always rejected after its round trip (r02)
constexpr std::uint64_t SMALL_DEVICE_MAX = std::uint64_t(1) << 20;
#ifndef AKB_SMALL_HIST_KEYS
#define AKB_SMALL_HIST_KEYS 4096  // keys per histogram CTA of a small sort (r02: 16384 / 8192 / 4096 / 2048 -> 55 / 53 / 52 / 54 us per 1e6 sort)
#endif

// Small keys-only 64-bit integer sorts with NO host round trip before the last kernel: the top
// three digits' histograms -> device plan (small_plan_kernel) -> one unstable partition pass
// by the chosen digit (msd_pass_kernel<0>: per-bin atomic cursors, no look-back state) ->
// bucket cuts = its offsets -> counting local stage. The sequence is replayed as one CUDA
// graph once the same buffers come back (every launch parameter lives in the ctx), and the
// call's only synchronisation at the end reads {plan mode, oversized-range count}; only
// skewed inputs then take the host-planned path. Returns false when that path must run.
template <typename T>
bool small_sort_device(ak_ctx* c, const T* kin, T* kout, T* kalt, std::uint64_t n, bool desc) {
    constexpr int PASSES = 8;
    constexpr int ITEMS = 12;  // 4608-key ranges, two counting CTAs per SM
    constexpr std::uint64_t CAPK = LC_BLOCK * (ITEMS * LOCAL_BLOCK / LC_BLOCK);
    std::uint64_t* g_hist = static_cast<std::uint64_t*>(c->small);  // rows 5..7 used
    std::uint64_t* curs = g_hist + PASSES * RADIX;  // the chosen digit's offsets: the partition's cursors
    const std::uint64_t J = RADIX;
    // [cuts J+1][plan {mode, shift}][big count + list J][redo count + list J]: plan and the big
    // count are adjacent, so one 16-byte read back gives both
    std::uint64_t* cuts = ctx_cuts(c, 3 * J + 6);
    int* plan = reinterpret_cast<int*>(cuts + J + 1);
    std::uint64_t* big = cuts + J + 2;
    std::uint64_t* redo = big + J + 1;
    auto* h = static_cast<std::uint64_t*>(ctx_pinned(c, 2 * sizeof(std::uint64_t)));
    // one histogram CTA per 4096 keys (at most 4 per SM): each flushes 3 x 256 global atomics,
    // so fewer, fatter CTAs flush less but read with less parallelism
    const unsigned hist_grid = static_cast<unsigned>(
        std::max<std::uint64_t>(1, std::min<std::uint64_t>(static_cast<std::uint64_t>(c->sm_count) * 4,
                                                            ceil_div(n, AKB_SMALL_HIST_KEYS))));
    auto enqueue = [&] {
        AKB_CUDA(cudaMemsetAsync(g_hist + (PASSES - 3) * RADIX, 0, 3 * RADIX * sizeof(std::uint64_t), c->stream));
        const int tok = ctx_prof_begin(c, KF_HIST);
        hist_kernel<T, PASSES, PASSES - 3><<<hist_grid, 256, 0, c->stream>>>(kin, n, desc ? 1 : 0, g_hist);
        AKB_CUDA(cudaGetLastError());
        ctx_prof_end(c, tok);
        small_plan_kernel<<<1, RADIX, 0, c->stream>>>(g_hist, n, CAPK - 64, plan, curs, cuts, big, redo);
        AKB_CUDA(cudaGetLastError());
        msd_digit_pass<T>(c, kin, kalt, n, desc, curs, plan);
        launch_local_count<T, ITEMS>(c, kalt, kout, cuts, J, n, desc, 0, big, redo, true);
        c->kernel_launches += 2;
        AKB_CUDA(cudaMemcpyAsync(h, plan, 2 * sizeof(std::uint64_t), cudaMemcpyDeviceToHost, c->stream));
    };
    const ak_ctx::small_graph key{kin, kout, kalt, n, desc ? 1 : 0, static_cast<int>(sizeof(T)), cuts, h, nullptr, 0};
    auto same = [&](const ak_ctx::small_graph& g) {
        return g.kin == key.kin && g.kout == key.kout && g.kalt == key.kalt && g.n == key.n && g.desc == key.desc &&
               g.width == key.width && g.cuts == key.cuts && g.pinned == key.pinned;
    };
    cudaGraphExec_t exec = nullptr;
    if (!c->profiling) {
        for (auto& g : c->graphs)
            if (same(g)) {
                exec = g.exec;
                c->kernel_launches += g.launches;
            }
        if (!exec && same(c->last_small)) {  // the same buffers again: capture once, replay from now on
            const std::uint64_t before = c->kernel_launches;
            cudaGraph_t graph = nullptr;
            AKB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue();
            } catch (...) {
                cudaStreamEndCapture(c->stream, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            AKB_CUDA(cudaStreamEndCapture(c->stream, &graph));
            AKB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
            AKB_CUDA(cudaGraphDestroy(graph));
            ak_ctx::small_graph g = key;
            g.exec = exec;
            g.launches = c->kernel_launches - before;
            if (c->graphs.size() >= 4) {
                AKB_CUDA(cudaGraphExecDestroy(c->graphs.front().exec));
                c->graphs.erase(c->graphs.begin());
            }
            c->graphs.push_back(g);
        }
    }
    if (exec) AKB_CUDA(cudaGraphLaunch(exec, c->stream));
    else enqueue();
    c->last_small = key;
    AKB_CUDA(cudaStreamSynchronize(c->stream));  // the call's one synchronisation
    const int mode = static_cast<int>(h[0] & 0xffffffffu);
    const std::uint64_t nbig = h[1];
    if (mode != 0) return false;  // nothing was written: the host plan starts from kin
    sort_oversized<T>(c, kalt, kout, kalt, n, desc, cuts, big, J, nbig);
    return true;
}

// Device plan of a two-level sort (2^24 <= n <= ~2^30; no host round trip before the last
// kernel): the largest 16-bit bucket (filled by the joint scan) picks how many aligned
// buckets form one range of the predicted counting stage, or rejects the plan (mode 1: the
// partition passes, the cuts and the counting stage then do nothing, and the host plan runs
// from the same histograms). dplan = {mode, group, J}.
__global__ void two_level_plan_kernel(const std::uint64_t* __restrict__ maxslot, std::uint64_t fit_cap,
                                      std::uint64_t group_cap, std::uint64_t max_group,
                                      std::uint64_t* __restrict__ dplan) {
    const std::uint64_t maxb = *maxslot;
    std::uint64_t mode = 1, g = 1;
    if (maxb > 0 && maxb <= fit_cap) {
        mode = 0;
        while (g < max_group && 2 * g * maxb <= group_cap) g *= 2;
    }
    dplan[0] = mode;
    dplan[1] = g;
    dplan[2] = 65536 / g;
}

// The device-planned two-level sort: joint histogram -> plan -> two unstable partition passes
// -> bucket-group cuts -> counting stage (4608-key, or the big-range stage above ~2^28 keys),
// then ONE synchronisation reading {plan, oversized-range count}. Returns false when the plan
// was rejected (skewed keys): nothing was written, and the histograms in g_hist / msdbuf are
// those the host plan starts from.
#ifndef AKB_TWO_LEVEL_MIN_LOG
#define AKB_TWO_LEVEL_MIN_LOG 20  // r02: 2^22 / 2^23 int64 0.241 / 0.314 -> 0.191 / 0.252 ms (was 24)
#endif

template <typename T>
bool two_level_device(ak_ctx* c, const T* kin, T* kout, T* kalt, std::uint64_t n, bool desc, std::uint64_t* g_hist,
                      std::uint64_t* msdbuf) {
    constexpr std::uint64_t JM = 65536;
    const bool big = AKB_CFG_BIG_LOCAL && n > (std::uint64_t(1) << 28) + (std::uint64_t(1) << 23);
    std::uint64_t* cuts = ctx_cuts(c, 4 * (JM + 1) + 8);
    std::uint64_t* bigl = cuts + JM + 1;
    std::uint64_t* redo = bigl + JM + 1;
    std::uint64_t* dplan = redo + JM + 1;
    constexpr int ITEMS = 12;  // the 4608-key stage: 2 CTAs per SM
    const std::uint64_t cap = big ? static_cast<std::uint64_t>(LB_CAP) : static_cast<std::uint64_t>(LOCAL_BLOCK) * ITEMS;
    AKB_CUDA(cudaMemsetAsync(c->small, 0, (2 * 8 * RADIX) * 8 + 8 * 4, c->stream));
    msd_hist<T>(c, kin, n, desc, g_hist, msdbuf, false);
    two_level_plan_kernel<<<1, 1, 0, c->stream>>>(msd_joint_max_slot(msdbuf), big ? cap - 256 : cap, cap,
                                                  big ? 8 : 256, dplan);
    AKB_CUDA(cudaGetLastError());
    msd_top16<T>(c, kin, kalt, kout, n, desc, msdbuf, msdbuf + JM, msdbuf + 2 * JM, reinterpret_cast<const int*>(dplan));
    cuts_from_ends_kernel<<<static_cast<unsigned>(ceil_div(JM + 1, 256)), 256, 0, c->stream>>>(msdbuf + JM, JM, n, 1,
                                                                                              dplan, cuts);
    AKB_CUDA(cudaGetLastError());
    AKB_CUDA(cudaMemsetAsync(bigl, 0, sizeof(std::uint64_t), c->stream));
    if (big) launch_local_big<T>(c, kout, kout, cuts, JM, desc, bigl, dplan);
    else launch_local_count<T, ITEMS>(c, kout, kout, cuts, JM, n, desc, 0, bigl, redo, false, dplan);
    c->kernel_launches += 2;
    auto* h = static_cast<std::uint64_t*>(ctx_pinned(c, 4 * sizeof(std::uint64_t)));
    AKB_CUDA(cudaMemcpyAsync(h, dplan, 3 * sizeof(std::uint64_t), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaMemcpyAsync(h + 3, bigl, sizeof(std::uint64_t), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));  // the call's one synchronisation
    if (h[0] != 0) return false;
    const std::uint64_t J = h[2], nbig = h[3];
    sort_oversized<T>(c, kout, kout, kalt, n, desc, cuts, bigl, J, nbig);
    return true;
}

template <typename T>
bool hybrid_sort_keys_impl(ak_ctx* c, const T* kin, T* kout, T* kalt, std::uint64_t n, bool desc) {
    constexpr int PASSES = key_traits<T>::nbits / 8;
    const int env = hybrid_env();
    if (env < 0 && c->blocking && n > static_cast<std::uint64_t>(LOCAL_TILE) && n <= SMALL_DEVICE_MAX &&
        ((reinterpret_cast<std::uintptr_t>(kalt) & 15) == 0) && small_sort_device<T>(c, kin, kout, kalt, n, desc))
        return true;
    // 64-bit integer keys. Float keys concentrate their top digits in the exponent (uniform
    // floats of [-1e6, 1e6) use ~40 of 256 top-digit values), which breaks the bucket-size
    // estimate and sends most ranges to the fallback (measured r01: f32 2^27 6.6 ms hybrid
    // vs 3.1 ms plain), so they keep the plain D-pass LSD.
    if (env == 0 || PASSES != 8 || !std::is_integral_v<T>) return false;
    if (n == 0) return true;
    std::uint64_t* g_hist = static_cast<std::uint64_t*>(c->small);
    // two MSD levels planned on the device (the common case of 2^24 .. ~2^30 keys); a rejected
    // plan leaves the histograms for the host plan below
    bool hist_ready = false;
    if (env < 0 && msd_env() != 0 && n >= (std::uint64_t(1) << AKB_TWO_LEVEL_MIN_LOG) &&
        n <= (std::uint64_t(1) << 30) + (std::uint64_t(1) << 26) &&
        ((reinterpret_cast<std::uintptr_t>(kin) | reinterpret_cast<std::uintptr_t>(kalt) |
          reinterpret_cast<std::uintptr_t>(kout)) & 15) == 0) {
        if (two_level_device<T>(c, kin, kout, kalt, n, desc, g_hist, ctx_msd(c))) return true;
        // the host plan below reuses the joint read where it would have made it itself
        // (n >= 2^24); smaller sorts plan from their own top-three-digit histogram
        hist_ready = n >= (std::uint64_t(1) << 24);
    }
    std::uint64_t* g_offs = g_hist + PASSES * RADIX;
    std::uint32_t* counters = reinterpret_cast<std::uint32_t*>(g_offs + PASSES * RADIX);
    int m = 0, top = PASSES, items = LOCAL_MAX_ITEMS;
    bool bucket_mode = false, big_local = false;
    std::uint64_t group = 1;  // big-range stage: 16-bit buckets per range
    std::uint64_t step = n, J = 1, base_id = 0;
    const T* G = kin;  // buffer holding the bucket-ordered keys
    std::uint64_t* msdbuf = nullptr;
    bool used_msd = false;
    if (n > static_cast<std::uint64_t>(LOCAL_TILE)) {
        const int blocks = c->sm_count * 4;
        if (!hist_ready) AKB_CUDA(cudaMemsetAsync(c->small, 0, (2 * PASSES * RADIX) * 8 + PASSES * 4, c->stream));
        int first = PASSES - 3;
        // 64-bit integer keys: the first read also builds the 16-bit joint histogram that
        // the unstable MSD passes start their cursors from
        const bool msd_ok = msd_env() != 0 && std::is_integral_v<T> && sizeof(T) == 8 && env <= 0 &&
                            n >= (std::uint64_t(1) << 24);  // below: the joint-histogram flush dominates
        msdbuf = msd_ok ? ctx_msd(c) : nullptr;
        bool joint_valid = false;
        // up to ~2^30 keys the plan needs only digits 7 and 6 (the joint histogram's marginals:
        // two MSD levels, then the 4608-key or the big-range stage): the joint read skips digit
        // 5, and a plan that does reach it re-reads (skewed keys). Above, uniform keys need a
        // third level, so the first read counts digit 5 too.
        const bool d5 = AKB_CFG_BIG_LOCAL ? n > (std::uint64_t(1) << 30) + (std::uint64_t(1) << 26)
                                          : n >= (std::uint64_t(1) << 29);
        if (msd_ok && !d5) first = PASSES - 2;
        auto run_hist = [&](int f) {
            if (f != 0 && msd_ok) {
                msd_hist<T>(c, kin, n, desc, g_hist, msdbuf, d5);
                joint_valid = true;
                return;
            }
            const int tok = ctx_prof_begin(c, KF_HIST);
            if (f == PASSES - 3) hist_kernel<T, PASSES, PASSES - 3><<<blocks, 256, 0, c->stream>>>(kin, n, desc, g_hist);
            else hist_kernel<T, PASSES, 0><<<blocks, 256, 0, c->stream>>>(kin, n, desc, g_hist);
            AKB_CUDA(cudaGetLastError());
            ctx_prof_end(c, tok);
            c->kernel_launches += 1;
        };
        if (hist_ready) joint_valid = msd_ok && !d5;  // the device plan's read (digit 5 not counted)
        else run_hist(first);
        std::vector<std::uint64_t> h(PASSES * RADIX);
        auto fetch = [&] {
            std::uint64_t* hp = static_cast<std::uint64_t*>(ctx_pinned(c, PASSES * RADIX * sizeof(std::uint64_t)));
            AKB_CUDA(cudaMemcpyAsync(hp, g_hist, PASSES * RADIX * sizeof(std::uint64_t), cudaMemcpyDeviceToHost,
                                     c->stream));
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            std::copy(hp, hp + PASSES * RADIX, h.begin());
        };
        fetch();
        auto maxbin = [&](int d, int* which) {
            std::uint64_t mx = 0;
            for (int i = 0; i < RADIX; ++i)
                if (h[d * RADIX + i] > mx) {
                    mx = h[d * RADIX + i];
                    if (which) *which = i;
                }
            return mx;
        };
        // skip constant leading digits (their value becomes the bucket-id prefix)
        std::uint64_t prefix = 0;
        for (;;) {
            if (top == first) {
                if (first == 0) break;
                AKB_CUDA(cudaMemsetAsync(g_hist, 0, PASSES * RADIX * 8, c->stream));
                first = 0;
                run_hist(0);
                fetch();
            }
            int v = 0;
            if (maxbin(top - 1, &v) != n) break;
            prefix = (prefix << 8) | static_cast<std::uint64_t>(v);
            --top;
            if (top == 0) break;
        }
        if (top == 0) {  // every key equal
            if (kin != kout) AKB_CUDA(cudaMemcpyAsync(kout, kin, n * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
            return true;
        }
        double est = static_cast<double>(n);
        for (m = 1; m <= 3 && m <= top; ++m) {
            if (top - m < first) {  // need the histogram of a lower digit
                AKB_CUDA(cudaMemsetAsync(g_hist, 0, PASSES * RADIX * 8, c->stream));
                first = 0;
                run_hist(0);
                fetch();
            }
            est *= static_cast<double>(maxbin(top - m, nullptr)) / static_cast<double>(n);
            const double need = est + 6.0 * std::sqrt(est) + 64.0;
            if (AKB_CFG_BIG_LOCAL && m == 2 && env < 0 && need > LOCAL_TILE && need + 256.0 <= LB_CAP && msd_ok &&
                top == PASSES && n < (std::uint64_t(1) << 32) && ((reinterpret_cast<std::uintptr_t>(kin) & 15) == 0) &&
                ((reinterpret_cast<std::uintptr_t>(kalt) & 15) == 0)) {
                // 16-bit buckets over the 4608-key stage but within LB_CAP: two MSD levels + the
                // big-range stage instead of a third level (see local_big_kernel)
                big_local = true;
                bucket_mode = true;  // groups of 2^g buckets per range, g from the exact largest bucket
                break;
            }
            if (need > LOCAL_TILE) continue;
            if (env > 0 && env != m) continue;
            const int ib = need <= LOCAL_BLOCK * 8 ? 8 : (need <= LOCAL_BLOCK * 12 ? 12 : 16);
            if (est >= 0.55 * LOCAL_BLOCK * ib) {  // one bucket fills most of an ib-item CTA
                bucket_mode = true;
                items = ib;
            } else {
                // ranges of several buckets: cap them at 12-item CTAs (4608 keys), whose
                // counting kernel keeps two CTAs per SM (16-item ones fit only one)
                const bool counting = need <= LOCAL_BLOCK * 6;
                if (counting) items = 12;
                step = static_cast<std::uint64_t>((counting ? LOCAL_BLOCK * 12 : LOCAL_TILE) - need);
                if (step < 256) step = 256;
            }
            break;
        }
        if (m > 3 || m > top) return false;
        J = bucket_mode ? (1ull << (8 * m)) : ceil_div(n, step);
        base_id = prefix << (8 * m);
        const T* cur = kin;
        const bool tma_ok = (reinterpret_cast<std::uintptr_t>(kin) & 15) == 0 &&
                            (reinterpret_cast<std::uintptr_t>(kalt) & 15) == 0;  // TMA-fed passes
        const bool msd_path = joint_valid && (m == 2 || m == 3) && top == PASSES && tma_ok && n < (std::uint64_t(1) << 32);
        if (!msd_path) {  // the onesweep passes and the one-pass bucket cuts read the digit offsets
            hist_scan_kernel<<<PASSES, RADIX, 0, c->stream>>>(g_hist, g_offs);
            AKB_CUDA(cudaGetLastError());
            c->kernel_launches += 1;
        }
        if (msd_path) {
            // unstable MSD partition by the top 16 (24) bits (keys-only integers: order among
            // equal keys is unobservable). Measured and dropped (r02): two levels of 11 + 9 bits
            // instead of three 8-bit ones at n >= 2^29 -- 2^30 int64 MSD 11.9 ms vs 12.1 ms: the
            // finer digits' 4- and 16-key runs per tile cost what the saved level saved.
            msd_top16<T>(c, kin, kalt, kout, n, desc, msdbuf, msdbuf + 65536, msdbuf + 2 * 65536);
            cur = kout;
            used_msd = true;
            if (m == 3) {
                msd_level3<T>(c, kout, kalt, n, desc);
                cur = kalt;
            }
            if (big_local) {
                // ranges = groups of `group` consecutive 16-bit buckets (aligned: OR-reduced
                // varying bits stay exact), group * largest bucket <= LB_CAP
                const std::uint64_t maxb = msd_max_bucket(c, m);
                if (maxb + 256 <= static_cast<std::uint64_t>(LB_CAP)) {
                    while (group < 8 && 2 * group * maxb <= static_cast<std::uint64_t>(LB_CAP)) group *= 2;
                    J = 65536 / group;
                } else {  // a bucket over the big-range stage (skewed keys): a third level instead
                    big_local = false;
                    bucket_mode = false;
                    msd_level3<T>(c, kout, kalt, n, desc);
                    cur = kalt;
                    m = 3;
                    items = 12;
                    const std::uint64_t cap = static_cast<std::uint64_t>(LOCAL_BLOCK) * items;
                    const std::uint64_t maxb3 = msd_max_bucket(c, 3);
                    step = maxb3 + 256 <= cap ? cap - maxb3 : 256;
                    J = ceil_div(n, step);
                }
            } else if (!bucket_mode) {
                // ranges of several buckets, sized from the exact largest bucket (the plan's
                // estimate assumes independent digits, which skewed keys -- e.g. the
                // exponent-heavy top bits of composite float keys -- violate). Two levels:
                // aligned groups of 2^g 16-bit buckets (2^g x largest bucket <= the CTA's
                // capacity), so the counting stage's OR-reduced varying bits stay exact and
                // ranges stay nearly full; three levels: step-cut ranges of several buckets.
                const std::uint64_t maxb = msd_max_bucket(c, m);
                const std::uint64_t cap = static_cast<std::uint64_t>(LOCAL_BLOCK) * items;
                if (m == 2 && maxb > 0 && maxb <= cap) {
                    while (group < 256 && 2 * group * maxb <= cap) group *= 2;
                    bucket_mode = true;
                    J = 65536 / group;
                } else if (maxb + 256 <= cap) {
                    step = cap - maxb;
                    J = ceil_div(n, step);
                }
            }
        } else {
            for (int q = 0; q < m; ++q) {
                const int p = top - m + q;
                T* dst = (q % 2 == 0) ? kalt : kout;
                launch_pass<T, std::uint32_t, SORT_KEYS>(c, cur, dst, nullptr, nullptr, n, 8 * p, desc, p,
                                                         g_offs + p * RADIX, counters + p, true);
                cur = dst;
            }
        }
        G = cur;
    }
    std::uint64_t* cuts = ctx_cuts(c, 3 * J + 4);
    std::uint64_t* big = cuts + J + 1;
    std::uint64_t* redo = big + J + 1;
    AKB_CUDA(cudaMemsetAsync(big, 0, sizeof(std::uint64_t), c->stream));
    const int top_shift = 8 * (top - (m > 0 ? m : 1));
    if (bucket_mode && used_msd && m == 2 && J * group == 65536)
        // the MSD cursors end at the bucket ends: cuts[j] = end of bucket j * group - 1 (no search)
        cuts_from_ends_kernel<<<static_cast<unsigned>(ceil_div(J + 1, 256)), 256, 0, c->stream>>>(msdbuf + 65536, J, n,
                                                                                                 group, nullptr, cuts);
    else if (bucket_mode && !used_msd && m == 1 && J == RADIX)
        // one onesweep pass over digit top - 1: bucket j starts at that digit's exclusive
        // global offset j (hist_scan_kernel), so cuts[j] = offs[j] (no search)
        cuts_from_ends_kernel<<<static_cast<unsigned>(ceil_div(J + 1, 256)), 256, 0, c->stream>>>(
            g_offs + (top - 1) * RADIX + 1, J, n, 1, nullptr, cuts);
    else if (bucket_mode)
        bucket_cuts_kernel<T><<<static_cast<unsigned>(ceil_div(J + 1, 256)), 256, 0, c->stream>>>(
            G, n, top_shift, desc ? 1 : 0, J, base_id, cuts);
    else
        range_cuts_kernel<T><<<static_cast<unsigned>(ceil_div(J + 1, 256)), 256, 0, c->stream>>>(
            G, n, top_shift, desc ? 1 : 0, step, J, cuts);
    AKB_CUDA(cudaGetLastError());
    c->kernel_launches += 1;
    // local radix passes cover the two digits under the bucket digits; the rest is the
    // run fix-up (experiment builds: -DAKB_CFG_LOCAL_LOW=0 radix-passes every varying digit)
    int low = top - m - 2;
    if (low < 0) low = 0;
#ifdef AKB_CFG_LOCAL_LOW
    low = AKB_CFG_LOCAL_LOW;
#endif
    // the counting stages (64-bit integer keys are the only ones that reach here, see above);
    // ranges they hand back run the stable on-chip radix (local_redo_kernel)
    if (big_local) launch_local_big<T>(c, G, kout, cuts, J, desc, big);
    else if (items == 8) launch_local_count<T, 8>(c, G, kout, cuts, J, n, desc, low, big, redo);
    else if (items == 12) launch_local_count<T, 12>(c, G, kout, cuts, J, n, desc, low, big, redo);
    else launch_local_count<T, 16>(c, G, kout, cuts, J, n, desc, low, big, redo);
    if (m == 0) return true;  // a single range of <= LOCAL_TILE keys always fits
    // oversized ranges (skewed keys): plain LSD on each such segment, or on the whole
    // array when there are many (every range is a stable permutation of its keys, equal
    // keys never straddle ranges, so a stable sort of the partial result is the answer)
    std::uint64_t* hb = static_cast<std::uint64_t*>(ctx_pinned(c, sizeof(std::uint64_t)));
    AKB_CUDA(cudaMemcpyAsync(hb, big, sizeof(std::uint64_t), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    sort_oversized<T>(c, G, kout, kalt, n, desc, cuts, big, J, hb[0]);
    return true;
}

template <typename T>
bool hybrid_sort_keys(ak_ctx* c, const T* kin, T* kout, T* kalt, std::uint64_t n, bool desc) {
    if constexpr (std::is_integral_v<T> && sizeof(T) == 8) return hybrid_sort_keys_impl<T>(c, kin, kout, kalt, n, desc);
    else return false;
}

// 0: always the merge-path tree (experiment builds: make variant DEFS=-DAKB_CFG_MERGE_COUNT=...)
#ifndef AKB_CFG_MERGE_COUNT
#define AKB_CFG_MERGE_COUNT 1
#endif
constexpr int merge_count_env() { return AKB_CFG_MERGE_COUNT; }

template <typename T>
bool merge_runs_counting_impl(ak_ctx* c, int P, const T* const* runs, const std::uint64_t* lens, T* dst, bool desc) {
    constexpr int ITEMS = 9;  // 4608-key tiles, two CTAs per SM
    using MS = mc_smem<T, ITEMS>;
    constexpr std::uint32_t CAPK = MS::CAP;
    std::uint64_t n = 0;
    for (int r = 0; r < P; ++r) n += lens[r];
    // P = 8, 2^28 int64: 3.70 -> 2.83 ms; P = 4: break-even with the 2-level tree (2.44 ms)
    if (merge_count_env() == 0 || P < 6 || P > MC_MAXP || n < (std::uint64_t(1) << 22)) return false;
    // sample stride S with (K + P) * S <= CAP (the largest possible tile without heavy ties)
    // sample stride S and tile width K (samples): a tile holds at most (K + P) * S keys (each
    // run adds at most one partial sample block), expected K * S
    const std::uint32_t S = 128;
    const std::uint32_t K = CAPK / S - static_cast<std::uint32_t>(P);
    std::vector<std::uint64_t> so(P + 1, 0);
    for (int r = 0; r < P; ++r) so[r + 1] = so[r] + (lens[r] + S - 1) / S;
    const std::uint64_t M = so[P];
    const std::uint64_t J = (M + K - 1) / K;
    // arena: [P run ptrs][P lens][P+1 sample offsets][M samples][M scratch][(J+1)P pos][1 max]
    //        [CAP tile scratch for the clustered-tile fallback]
    const std::size_t words = 3 * P + 1 + 2 * M + (J + 1) * P + 1 + CAPK;
    auto* w = static_cast<std::uint64_t*>(ctx_work(c, words * sizeof(std::uint64_t)));
    if (!w) return false;
    auto* d_runs = reinterpret_cast<const T**>(w);
    std::uint64_t* d_lens = w + P;
    std::uint64_t* d_so = w + 2 * P;
    T* samples = reinterpret_cast<T*>(w + 3 * P + 1);
    T* sscr = samples + M;
    std::uint64_t* pos = w + 3 * P + 1 + 2 * M;
    std::uint64_t* mx = pos + (J + 1) * P;
    auto* h = static_cast<std::uint64_t*>(ctx_pinned(c, (3 * P + 1) * sizeof(std::uint64_t)));
    for (int r = 0; r < P; ++r) {
        h[r] = reinterpret_cast<std::uint64_t>(runs[r]);
        h[P + r] = lens[r];
    }
    for (int r = 0; r <= P; ++r) h[2 * P + r] = so[r];
    AKB_CUDA(cudaMemcpyAsync(w, h, (3 * P + 1) * sizeof(std::uint64_t), cudaMemcpyHostToDevice, c->stream));
    mc_sample_kernel<T><<<c->sm_count * 4, 256, 0, c->stream>>>(d_runs, d_so, P, S, samples);
    AKB_CUDA(cudaGetLastError());
    radix_sort<T, std::uint32_t>(c, SORT_KEYS, samples, samples, sscr, nullptr, nullptr, nullptr, M, desc, true);
    mc_bounds_kernel<T><<<static_cast<unsigned>(ceil_div((J + 1) * P, 256)), 256, 0, c->stream>>>(
        d_runs, d_lens, P, samples, J, K, desc ? 1 : 0, pos);
    AKB_CUDA(cudaMemsetAsync(mx, 0, sizeof(std::uint64_t), c->stream));
    mc_maxtile_kernel<<<static_cast<unsigned>(ceil_div(J, 256)), 256, 0, c->stream>>>(
        pos, P, J, reinterpret_cast<unsigned long long*>(mx));
    AKB_CUDA(cudaGetLastError());
    AKB_CUDA(cudaMemcpyAsync(h, mx, sizeof(std::uint64_t), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    if (h[0] > CAPK) return false;  // heavy ties: the merge-path tree
    std::uint64_t* big = ctx_cuts(c, J + 2);
    AKB_CUDA(cudaMemsetAsync(big, 0, sizeof(std::uint64_t), c->stream));
    smem_attr(c, merge_count_kernel<T, ITEMS, false>, MS::total);
    smem_attr(c, merge_count_kernel<T, ITEMS, true>, MS::total);
    const int tok = ctx_prof_begin(c, KF_MERGE);
    if (desc)
        merge_count_kernel<T, ITEMS, true><<<static_cast<unsigned>(J), LC_BLOCK, MS::total, c->stream>>>(d_runs, P, pos,
                                                                                                      dst, big);
    else
        merge_count_kernel<T, ITEMS, false><<<static_cast<unsigned>(J), LC_BLOCK, MS::total, c->stream>>>(d_runs, P,
                                                                                                       pos, dst, big);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 5;
    // clustered tiles (a bin over LC_MAX_BIN): the caller's tree merges them piece-wise
    AKB_CUDA(cudaMemcpyAsync(h, big, sizeof(std::uint64_t), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    const std::uint64_t nbig = h[0];
    if (nbig) {
        std::vector<std::uint64_t> ids(nbig), hp((J + 1) * P);
        AKB_CUDA(cudaMemcpy(ids.data(), big + 1, nbig * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
        AKB_CUDA(cudaMemcpy(hp.data(), pos, hp.size() * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
        T* tscr = reinterpret_cast<T*>(mx + 1);  // tiles here hold <= CAP keys
        for (std::uint64_t j : ids) {
            std::vector<const T*> pp(P);
            std::vector<std::uint64_t> pl(P);
            std::uint64_t off = 0, tot = 0;
            for (int r = 0; r < P; ++r) {
                pp[r] = runs[r] + hp[j * P + r];
                pl[r] = hp[(j + 1) * P + r] - hp[j * P + r];
                off += hp[j * P + r];
                tot += pl[r];
            }
            merge_runs<T>(c, P, pp.data(), pl.data(), dst + off, tscr, desc);
        }
    }
    return true;
}

}  // namespace

template <typename T>
bool merge_runs_counting(ak_ctx* c, int P, const T* const* runs, const std::uint64_t* lens, T* dst, bool desc) {
    if constexpr (std::is_integral_v<T> && sizeof(T) == 8) return merge_runs_counting_impl<T>(c, P, runs, lens, dst, desc);
    else return false;
}

template <typename T, typename V>
void radix_sort(ak_ctx* c, int mode, const T* kin, T* kout, T* kalt, const V* vin, V* vout, V* valt,
                std::uint64_t n, bool desc, bool keys_out) {
    switch (mode) {
        case SORT_KEYS:
            if (!hybrid_sort_keys<T>(c, kin, kout, kalt, n, desc))
                radix_sort_impl<T, V, SORT_KEYS>(c, kin, kout, kalt, nullptr, nullptr, nullptr, n, desc, true);
            break;
        case SORT_PAIRS:
            radix_sort_impl<T, V, SORT_PAIRS>(c, kin, kout, kalt, vin, vout, valt, n, desc, true);
            break;
        case SORT_IOTA:
            radix_sort_impl<T, V, SORT_IOTA>(c, kin, kout, kalt, nullptr, vout, valt, n, desc, keys_out);
            break;
        case SORT_LOWMEM:
            radix_sort_impl<T, V, SORT_LOWMEM>(c, kin, nullptr, nullptr, nullptr, vout, valt, n, desc, false);
            break;
        default:
            throw invalid_argument("radix_sort: unknown mode");
    }
}

#ifdef AKB_PHASES
extern "C" int ak_debug_set_phase_buffer(void* p) {
    return cudaMemcpyToSymbol(g_phase, &p, sizeof(p)) == cudaSuccess ? 0 : 4;
}
#endif

std::uint64_t radix_tile_items(int key_bytes, int) {
    return key_bytes == 8 ? tile_cfg<std::uint64_t, std::uint32_t, SORT_KEYS>::TILE
                          : tile_cfg<std::uint32_t, std::uint32_t, SORT_KEYS>::TILE;
}

// Keys-only sorts never touch the payload type: instantiate them once (V = u32)
// and route the other payload types of SORT_KEYS there.
#define AKB_INST(T, V)                                                                                        \
    template void radix_sort<T, V>(ak_ctx*, int, const T*, T*, T*, const V*, V*, V*, std::uint64_t, bool, bool);
#define AKB_INST_K(T)          \
    AKB_INST(T, std::uint32_t) \
    AKB_INST(T, std::uint64_t)

template bool merge_runs_counting<std::int64_t>(ak_ctx*, int, const std::int64_t* const*, const std::uint64_t*, std::int64_t*, bool);
template bool merge_runs_counting<std::uint64_t>(ak_ctx*, int, const std::uint64_t* const*, const std::uint64_t*, std::uint64_t*, bool);

AKB_INST_K(std::int32_t)
AKB_INST_K(std::uint32_t)
AKB_INST_K(std::int64_t)
AKB_INST_K(std::uint64_t)
AKB_INST_K(float)
AKB_INST_K(double)

}  // namespace akb
