// msd_pass.cu -- unstable MSD partition passes for keys-only 64-bit integer sorts.
//
// For keys without payload, stability is unobservable (equal integer keys are identical
// bit patterns), so the global top-digit passes of the hybrid sort need no look-back
// chain: a tile claims its output space per bin with one global atomicAdd on that bin's
// cursor, whose start comes from a histogram computed in the single upfront read.
//
//   hist_joint_kernel: one read of the keys -> the 256-bin histograms of the top three
//       digits (the plan) and the 65536-bin histogram of the top 16 bits (the cursors);
//   joint_scan_{a,b}_kernel: exclusive scan of the 65536 counts -> 16-bit bucket starts and the
//       8-bit bucket starts (the cursors of both passes);
//   msd_pass_kernel<LEVEL>: LEVEL 1 partitions by the top 8 bits, LEVEL 2 partitions each
//       top-8 bucket by the next 8 bits (a tile of the LEVEL-1 output spans few top
//       buckets). Per tile: load (128-bit, coalesced) -> shared-atomic slots per bin ->
//       bin starts + one global atomicAdd per non-empty bin -> keys staged in bin order
//       in shared memory -> contiguous per-bin runs written out.
// After the two passes the array is ordered by its top 16 bits, exactly as the stable
// top-digit onesweep passes leave it up to the order inside each 16-bit bucket, which the
// local stage sorts anyway.
#include <algorithm>
#include <cstdint>

#include "msd_pass.cuh"

namespace akb {

namespace {

constexpr std::uint32_t FULLM = 0xffffffffu;
constexpr int JOINT_BITS = 16;
constexpr int JOINT_BINS = 1 << JOINT_BITS;
constexpr int JH_BLOCK = 1024;
constexpr int JH_PARTS = 4;
constexpr std::uint32_t JH_FLUSH = 0x4000;  // u16 half-counter spill threshold
#ifndef AKB_JH_KEYS_LOG
#define AKB_JH_KEYS_LOG 17
#endif
#ifndef AKB_JH_UNROLL
#define AKB_JH_UNROLL 8  // r02: 2 / 4 / 8 / 16 -> 0.394 / 0.355 / 0.344 / 0.344 ms at 2^28
#endif

template <typename T>
__device__ __forceinline__ std::uint64_t ord64(T v, bool desc) {
    return static_cast<std::uint64_t>(ordered(v, desc));
}

// Joint histogram: 65536 u16 counters packed two per shared word (128 KB). A counter that
// reaches JH_FLUSH is moved to the global histogram by the thread whose increment reached
// it (at most JH_BLOCK increments can be in flight, far below the 0x10000 - JH_FLUSH of
// headroom, so a half never carries into its neighbour).
template <typename T, bool D5>
__global__ void __launch_bounds__(JH_BLOCK, 1)
    hist_joint_kernel(const T* __restrict__ keys, std::uint64_t n, int desc, std::uint64_t* __restrict__ g_hist,
                      std::uint64_t* __restrict__ g_joint) {
    extern __shared__ __align__(16) unsigned char smem[];
    std::uint32_t* s_joint = reinterpret_cast<std::uint32_t*>(smem);                    // 32768 words
    std::uint32_t* s_dig = reinterpret_cast<std::uint32_t*>(smem + JOINT_BINS * 2);      // 256 x PARTS
    for (int i = threadIdx.x; i < JOINT_BINS / 2; i += JH_BLOCK) s_joint[i] = 0;
    for (int i = threadIdx.x; i < 256 * JH_PARTS; i += JH_BLOCK) s_dig[i] = 0;
    __syncthreads();
    const bool dsc = desc != 0;
    const int part = threadIdx.x % JH_PARTS;
    auto count = [&](T k) {
        const std::uint64_t o = ord64(k, dsc);
        const std::uint32_t hi = static_cast<std::uint32_t>(o >> 32);
        if constexpr (D5) atomicAdd(&s_dig[((hi >> 8) & 0xffu) * JH_PARTS + part], 1u);  // digit 5 (6, 7: marginals)
        const std::uint32_t bin = hi >> 16;
        const std::uint32_t sh = (bin & 1u) * 16u;
        const std::uint32_t old = atomicAdd(&s_joint[bin >> 1], 1u << sh);
        if (((old >> sh) & 0xffffu) == JH_FLUSH - 1) {
            atomicSub(&s_joint[bin >> 1], JH_FLUSH << sh);
            atomicAdd(reinterpret_cast<unsigned long long*>(g_joint + bin), static_cast<unsigned long long>(JH_FLUSH));
        }
    };
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * JH_BLOCK;
    const std::uint64_t tid = static_cast<std::uint64_t>(blockIdx.x) * JH_BLOCK + threadIdx.x;
    std::uint64_t done = 0;
    if ((reinterpret_cast<std::uintptr_t>(keys) & 15) == 0) {
        const std::uint64_t nv = n / 2;
        const uint4* kv = reinterpret_cast<const uint4*>(keys);
        std::uint64_t i = tid;
        constexpr int U = AKB_JH_UNROLL;  // 16-byte loads in flight per thread
        for (; i + (U - 1) * stride < nv; i += U * stride) {
            uint4 a[U];
#pragma unroll
            for (int u = 0; u < U; ++u) a[u] = __ldg(kv + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                count(reinterpret_cast<const T*>(&a[u])[0]);
                count(reinterpret_cast<const T*>(&a[u])[1]);
            }
        }
        for (; i < nv; i += stride) {
            const uint4 a = __ldg(kv + i);
            const T* e = reinterpret_cast<const T*>(&a);
            count(e[0]);
            count(e[1]);
        }
        done = nv * 2;
    }
    for (std::uint64_t i = done + tid; i < n; i += stride) count(keys[i]);
    __syncthreads();
    for (int w = threadIdx.x; w < JOINT_BINS / 2; w += JH_BLOCK) {
        const std::uint32_t v = s_joint[w];
        if (v & 0xffffu)
            atomicAdd(reinterpret_cast<unsigned long long*>(g_joint + 2 * w), static_cast<unsigned long long>(v & 0xffffu));
        if (v >> 16)
            atomicAdd(reinterpret_cast<unsigned long long*>(g_joint + 2 * w + 1), static_cast<unsigned long long>(v >> 16));
    }
    for (int i = threadIdx.x; D5 && i < 256; i += JH_BLOCK) {
        std::uint32_t s = 0;
#pragma unroll
        for (int q = 0; q < JH_PARTS; ++q) s += s_dig[i * JH_PARTS + q];
        if (s) atomicAdd(reinterpret_cast<unsigned long long*>(g_hist + 5 * 256 + i), static_cast<unsigned long long>(s));
    }
}

// Exclusive scan of the 65536 joint counts in two launches of 64 CTAs (CTA b owns bins
// [1024 b, 1024 b + 1024) = rows 4b .. 4b+3 of the (digit 7, digit 6) table):
//   A: CTA-local exclusive scan -> cur16, CTA total -> sums[b], row sums -> digit-7 histogram,
//      the CTA's column partials -> colpart[b][256];
//   B: cur16 += sum of the earlier CTAs' totals, cur8 = row starts; CTA 0 folds the column
//      partials into the digit-6 histogram.
constexpr int JS_CTAS = JOINT_BINS / 1024;
__global__ void __launch_bounds__(1024) joint_scan_a_kernel(const std::uint64_t* __restrict__ g_joint,
                                                            std::uint64_t* __restrict__ cur16,
                                                            std::uint64_t* __restrict__ sums,
                                                            std::uint64_t* __restrict__ colpart,
                                                            std::uint64_t* __restrict__ g_hist,
                                                            unsigned long long* __restrict__ maxslot) {
    __shared__ std::uint64_t s_w[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int i = blockIdx.x * 1024 + t;
    const std::uint64_t v = g_joint[i];
    {  // the largest 16-bit bucket (device plans): warp max, one atomic per warp
        std::uint64_t m = v;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const std::uint64_t y = __shfl_xor_sync(FULLM, m, o);
            m = m > y ? m : y;
        }
        if (lane == 0 && m) atomicMax(maxslot, static_cast<unsigned long long>(m));
    }
    std::uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint64_t y = __shfl_up_sync(FULLM, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    std::uint64_t wp = 0;
    for (int k = 0; k < w; ++k) wp += s_w[k];
    cur16[i] = wp + inc - v;
    if (t == 1023) sums[blockIdx.x] = wp + inc;
    if ((t & 255) == 255) {  // a row of 256 bins ends here: its sum = prefix difference
        std::uint64_t row_start = 0;
        const int r0 = t - 255;  // first bin of the row (block-local)
        for (int k = 0; k < (r0 >> 5); ++k) row_start += s_w[k];
        g_hist[7 * 256 + (i >> 8)] += (wp + inc) - row_start;
    }
    if (t < 256) {
        const std::uint64_t* b = g_joint + blockIdx.x * 1024;
        colpart[blockIdx.x * 256 + t] = b[t] + b[256 + t] + b[512 + t] + b[768 + t];
    }
}
__global__ void __launch_bounds__(1024) joint_scan_b_kernel(std::uint64_t* __restrict__ cur16,
                                                            std::uint64_t* __restrict__ cur8,
                                                            const std::uint64_t* __restrict__ sums,
                                                            const std::uint64_t* __restrict__ colpart,
                                                            std::uint64_t* __restrict__ g_hist) {
    __shared__ std::uint64_t s_off;
    const int t = threadIdx.x;
    if (t < 32) {
        std::uint64_t x = 0;
        for (int k = t; k < static_cast<int>(blockIdx.x); k += 32) x += sums[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULLM, x, o);
        if (t == 0) s_off = x;
    }
    __syncthreads();
    const int i = blockIdx.x * 1024 + t;
    const std::uint64_t c = cur16[i] + s_off;
    cur16[i] = c;
    if ((i & 0xff) == 0) cur8[i >> 8] = c;
    if (blockIdx.x == 0) {  // column sums: 4 threads per column, 16 partials each (no long serial chain)
        const int col = t & 255, q = t >> 8;
        std::uint64_t x = 0;
#pragma unroll
        for (int k = q; k < JS_CTAS; k += 4) x += colpart[k * 256 + col];
        __shared__ std::uint64_t s_col[3][256];
        if (q) s_col[q - 1][col] = x;
        __syncthreads();
        if (q == 0) g_hist[6 * 256 + col] += x + s_col[0][col] + s_col[1][col] + s_col[2][col];
    }
}

// 256 threads x 20 keys (5120-key tiles), 3 CTAs per SM: r02 sweep at 2^28 int64, ms per
// pass: 512x16 (2 CTAs/SM) 0.954, 256x16 (4) 0.914, 256x18 (3) 0.922, 256x20 (3) 0.891,
// 256x22 (3) 0.916, 256x24 (3) 0.942, 288x18 (3) 0.898, 320x16 (3) 0.904, 256x12 (5) 1.01,
// 192x16 (5) 1.62 -- more, smaller CTAs overlap one another's load / claim latencies better
#ifndef AKB_MP_BLOCK
#define AKB_MP_BLOCK 256
#endif
constexpr int MP_BLOCK = AKB_MP_BLOCK;
#ifndef AKB_MP_ITEMS
#define AKB_MP_ITEMS 20
#endif
#ifndef AKB_MP_MINB
#define AKB_MP_MINB 3
#endif
constexpr int MP_ITEMS = AKB_MP_ITEMS;
constexpr int MP_TILE = MP_BLOCK * MP_ITEMS;  // 5120 keys
constexpr int MP_SPAN = 4;                    // LEVEL 2: top buckets a tile may span on chip
constexpr int MP_BINS = 256 * MP_SPAN;
#ifndef AKB_MP_PARTS
#define AKB_MP_PARTS 1
#endif
// sub-counters per bin (lane & (PARTS-1) picks one): spreads a warp's same-bin atomics
constexpr int MP_PARTS = AKB_MP_PARTS;

struct mp_smem {
    static constexpr std::size_t stage_off = 0;
    static constexpr std::size_t stage_bytes = 8 * MP_TILE;
    static constexpr std::size_t cnt_off = stage_bytes;  // u32 counts, then local starts
    static constexpr std::size_t gofs_off = cnt_off + 4 * MP_BINS * MP_PARTS;
    static constexpr std::size_t wsum_off = gofs_off + 8 * MP_BINS;
    static constexpr std::size_t misc_off = wsum_off + 4 * (MP_BLOCK / 32);
    static constexpr std::size_t total = misc_off + 16;
};

// Digit geometry of a partition level: the keys are already ordered by their top PB bits
// (PB = 0: first level) and are partitioned by the next DB bits; cursor index = the top
// PB + DB bits. LEVEL 1/2/3: 8-bit digits (8-, 16- and 24-bit buckets); LEVEL 0: one 8-bit
// digit chosen on the device (plan = {mode, shift}: mode != 0 -> no-op; small sorts).
template <int LEVEL>
struct mp_level {
    static constexpr int PB = LEVEL == 2 ? 8 : LEVEL == 3 ? 16 : 0;
    static constexpr int DB = 8;
    static constexpr int TOP = 64 - PB - DB;
};

template <typename T, int LEVEL>
__global__ void __launch_bounds__(MP_BLOCK, AKB_MP_MINB)
    msd_pass_kernel(const T* __restrict__ in, T* __restrict__ out, std::uint64_t n, int desc,
                    std::uint64_t* __restrict__ cursors, const int* __restrict__ plan = nullptr) {
    using L = mp_smem;
    extern __shared__ __align__(16) unsigned char smem[];
    T* s_stage = reinterpret_cast<T*>(smem + L::stage_off);
    std::uint32_t* s_cnt = reinterpret_cast<std::uint32_t*>(smem + L::cnt_off);
    std::uint64_t* s_gofs = reinterpret_cast<std::uint64_t*>(smem + L::gofs_off);
    std::uint32_t* s_wsum = reinterpret_cast<std::uint32_t*>(smem + L::wsum_off);
    std::uint32_t* s_misc = reinterpret_cast<std::uint32_t*>(smem + L::misc_off);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool dsc = desc != 0;
    const std::uint64_t t0 = static_cast<std::uint64_t>(blockIdx.x) * MP_TILE;
    const std::uint32_t len = static_cast<std::uint32_t>(n - t0 < MP_TILE ? n - t0 : MP_TILE);

    // load first: 128-bit vectors when the tile is full and aligned; the plan / span reads
    // below are then in flight together with the tile instead of ahead of it
    T k[MP_ITEMS];
    const bool vec = len == MP_TILE && (reinterpret_cast<std::uintptr_t>(in + t0) & 15) == 0;
    if (vec) {
        const uint4* v = reinterpret_cast<const uint4*>(in + t0);
#pragma unroll
        for (int i = 0; i < MP_ITEMS / 2; ++i) {
            const uint4 a = __ldg(v + i * MP_BLOCK + tid);
            k[2 * i] = reinterpret_cast<const T*>(&a)[0];
            k[2 * i + 1] = reinterpret_cast<const T*>(&a)[1];
        }
    } else {
#pragma unroll
        for (int i = 0; i < MP_ITEMS / 2; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const std::uint32_t li = 2 * (i * MP_BLOCK + tid) + h;
                k[2 * i + h] = li < len ? in[t0 + li] : T(0);
            }
    }

    // bin range of this tile: LEVEL 1 = the 256 top digits; LEVEL L > 1 = the 8L-bit prefixes
    // of the (already 8(L-1)-bit partitioned) tile, relative to its first key's 8(L-1)-bit
    // prefix (cursor index = the 8L-bit prefix)
    if (plan != nullptr && plan[0] != 0) return;  // device plan: not applicable, nothing written
    using G = mp_level<LEVEL>;
    constexpr int DB = G::DB;
    const int TOP = LEVEL == 0 ? plan[1] : G::TOP;  // shift of the digit (cursor index = key >> TOP)
    constexpr std::uint32_t DMASK = LEVEL == 0 ? 0xffu : 0xffffffffu;
    std::uint32_t lo16 = 0, span = 1;
    if constexpr (G::PB > 0) {
        const std::uint32_t f = static_cast<std::uint32_t>(ord64(in[t0], dsc) >> (TOP + DB));
        const std::uint32_t l = static_cast<std::uint32_t>(ord64(in[t0 + len - 1], dsc) >> (TOP + DB));
        lo16 = f << DB;
        span = l - f + 1;
    }
    const std::uint32_t nbins = span << DB;
    if (G::PB > 0 && span > MP_SPAN) {
        // tiny buckets (skewed keys): per-key cursor claims, written straight out
        for (std::uint32_t j = tid; j < len; j += MP_BLOCK) {
            const T key = in[t0 + j];
            const std::uint32_t bp = static_cast<std::uint32_t>(ord64(key, dsc) >> TOP);
            const unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(cursors + bp), 1ull);
            out[p] = key;
        }
        return;
    }
    for (std::uint32_t i = tid; i < nbins * MP_PARTS; i += MP_BLOCK) s_cnt[i] = 0;

    auto item_ok = [&](int i) { return 2 * ((i / 2) * MP_BLOCK + tid) + (i & 1) < static_cast<int>(len); };
    auto bin_of = [&](T key) {
        const std::uint64_t o = ord64(key, dsc);
        return (static_cast<std::uint32_t>(o >> TOP) & DMASK) - lo16;
    };
    __syncthreads();
    // slots inside the bins (arbitrary order): one shared atomic per key
    std::uint32_t sl[MP_ITEMS / 2];
#pragma unroll
    for (int i = 0; i < MP_ITEMS / 2; ++i) sl[i] = 0;
#pragma unroll
    const std::uint32_t part = static_cast<std::uint32_t>(lane) & (MP_PARTS - 1);
    for (int i = 0; i < MP_ITEMS; ++i)
        if (item_ok(i)) sl[i / 2] |= atomicAdd(&s_cnt[bin_of(k[i]) * MP_PARTS + part], 1u) << (16 * (i & 1));
    __syncthreads();
    // bin starts: thread t owns whole bins [t*BPT, t*BPT + BPT) (BPT <= 2) and their PARTS
    // sub-counters; exclusive scan in (bin, part) order + one global claim per non-empty bin
    {
        constexpr int BPTMAX = MP_BLOCK >= MP_BINS ? 1 : (2 * MP_BLOCK >= MP_BINS ? 2 : 4);  // bins per thread
        constexpr int MAXC = BPTMAX * MP_PARTS;
        const std::uint32_t bpt = nbins > 2 * MP_BLOCK ? 4u : nbins > MP_BLOCK ? 2u : 1u;
        const std::uint32_t fs = static_cast<std::uint32_t>(tid) * bpt * MP_PARTS;  // first sub-counter
        const std::uint32_t nsub = nbins * MP_PARTS;
        std::uint32_t c[MAXC];
        std::uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < MAXC; ++q) {
            c[q] = (static_cast<std::uint32_t>(q) < bpt * MP_PARTS && fs + q < nsub) ? s_cnt[fs + q] : 0u;
            sum += c[q];
        }
        // global position of staged slot j in bin b = gofs[b] + j. The cursor claims are issued
        // as soon as the counts are read and consumed only after the keys are staged: the
        // global atomic round trip overlaps the scan, the start rewrite and the staging stores
        std::uint64_t gclaim[BPTMAX];
        std::uint32_t tot[BPTMAX];
#pragma unroll
        for (int bi = 0; bi < BPTMAX; ++bi) {
            const std::uint32_t bin = fs / MP_PARTS + bi;
            tot[bi] = 0;
#pragma unroll
            for (int q = 0; q < MP_PARTS; ++q) tot[bi] += c[bi * MP_PARTS + q];
            gclaim[bi] = 0;
            if (static_cast<std::uint32_t>(bi) < bpt && bin < nbins && tot[bi])
                gclaim[bi] = atomicAdd(reinterpret_cast<unsigned long long*>(cursors + lo16 + bin),
                                       static_cast<unsigned long long>(tot[bi]));
        }
        std::uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t y = __shfl_up_sync(FULLM, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        std::uint32_t wp = 0;
#pragma unroll
        for (int w = 0; w < MP_BLOCK / 32; ++w) wp += w < warp ? s_wsum[w] : 0u;
        std::uint32_t run = wp + inc - sum;
        std::uint32_t gbase[BPTMAX];
        {
            std::uint32_t r2 = run;
#pragma unroll
            for (int bi = 0; bi < BPTMAX; ++bi) {
                const std::uint32_t bin = fs / MP_PARTS + bi;
                gbase[bi] = (static_cast<std::uint32_t>(bi) < bpt && bin < nbins && tot[bi]) ? r2 : 0xffffffffu;
                r2 += tot[bi];
            }
        }
        // (each thread rewrites only the counters it read: no barrier before the rewrite)
#pragma unroll
        for (int q = 0; q < MAXC; ++q)
            if (static_cast<std::uint32_t>(q) < bpt * MP_PARTS && fs + q < nsub) {
                s_cnt[fs + q] = run;
                run += c[q];
            }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < MP_ITEMS; ++i)
            if (item_ok(i)) s_stage[s_cnt[bin_of(k[i]) * MP_PARTS + part] + ((sl[i / 2] >> (16 * (i & 1))) & 0xffffu)] = k[i];
#pragma unroll
        for (int bi = 0; bi < BPTMAX; ++bi)
            if (gbase[bi] != 0xffffffffu) s_gofs[fs / MP_PARTS + bi] = gclaim[bi] - gbase[bi];
    }
    __syncthreads();
    // contiguous per-bin runs: consecutive staged slots of one bin go to consecutive addresses
#pragma unroll 4
    for (std::uint32_t j = tid; j < len; j += MP_BLOCK) {
        const T key = s_stage[j];
        out[s_gofs[bin_of(key)] + j] = key;
    }
    (void)s_misc;
}

// Histogram of the prefixes one DB-bit digit below an existing partition: the array is ordered
// by its top (64 - PS) bits; counts of the prefixes key >> (PS - DB). A tile spans few buckets
// of the existing partition (relative bins in shared memory), flushed with one global atomic
// per non-empty bin into hist[2^(64 - PS + DB)] (u32 counts; n < 2^32 per sort).
// PS = 48, DB = 8: the 24-bit prefixes under 16-bit buckets; PS = 53, DB = 9: the 20-bit
// prefixes under 11-bit buckets.
template <typename T, int PS, int DB = 8>
__global__ void __launch_bounds__(MP_BLOCK) hist_sub_kernel(const T* __restrict__ in, std::uint64_t n, int desc,
                                                          std::uint32_t* __restrict__ hist) {
    constexpr int SH = PS - DB;
    __shared__ std::uint32_t s_cnt[(1 << DB) * MP_SPAN];
    const int tid = threadIdx.x;
    const bool dsc = desc != 0;
    const std::uint64_t t0 = static_cast<std::uint64_t>(blockIdx.x) * MP_TILE;
    const std::uint32_t len = static_cast<std::uint32_t>(n - t0 < MP_TILE ? n - t0 : MP_TILE);
    const std::uint32_t f = static_cast<std::uint32_t>(ord64(in[t0], dsc) >> PS);
    const std::uint32_t l = static_cast<std::uint32_t>(ord64(in[t0 + len - 1], dsc) >> PS);
    const std::uint32_t lo = f << DB, span = l - f + 1;
    if (span > MP_SPAN) {
        for (std::uint32_t j = tid; j < len; j += MP_BLOCK)
            atomicAdd(hist + static_cast<std::uint32_t>(ord64(in[t0 + j], dsc) >> SH), 1u);
        return;
    }
    for (int i = tid; i < (1 << DB) * MP_SPAN; i += MP_BLOCK) s_cnt[i] = 0;
    __syncthreads();
    if (len == MP_TILE && (reinterpret_cast<std::uintptr_t>(in + t0) & 15) == 0) {
        const uint4* v = reinterpret_cast<const uint4*>(in + t0);
#pragma unroll 4
        for (int i = tid; i < MP_TILE / 2; i += MP_BLOCK) {
            const uint4 a = __ldg(v + i);
            atomicAdd(&s_cnt[static_cast<std::uint32_t>(ord64(reinterpret_cast<const T*>(&a)[0], dsc) >> SH) - lo], 1u);
            atomicAdd(&s_cnt[static_cast<std::uint32_t>(ord64(reinterpret_cast<const T*>(&a)[1], dsc) >> SH) - lo], 1u);
        }
    } else {
        for (std::uint32_t j = tid; j < len; j += MP_BLOCK)
            atomicAdd(&s_cnt[static_cast<std::uint32_t>(ord64(in[t0 + j], dsc) >> SH) - lo], 1u);
    }
    __syncthreads();
    for (std::uint32_t i = tid; i < (span << DB); i += MP_BLOCK)
        if (s_cnt[i]) atomicAdd(hist + lo + i, s_cnt[i]);
}

// Exclusive scan of hist24 (2^24 u32) into cur24 (u64), three launches: chunk sums,
// one-CTA scan of the 4096 chunk sums, chunk-local scans.
constexpr int S24_CHUNK = 4096;
__global__ void __launch_bounds__(1024) scan24_sums_kernel(const std::uint32_t* __restrict__ h,
                                                           std::uint64_t* __restrict__ sums) {
    __shared__ std::uint64_t s_w[32];
    const int t = threadIdx.x;
    const uint4 v = reinterpret_cast<const uint4*>(h + static_cast<std::size_t>(blockIdx.x) * S24_CHUNK)[t];
    std::uint64_t x = static_cast<std::uint64_t>(v.x) + v.y + v.z + v.w;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULLM, x, o);
    if ((t & 31) == 0) s_w[t >> 5] = x;
    __syncthreads();
    if (t < 32) {
        std::uint64_t y = s_w[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULLM, y, o);
        if (t == 0) sums[blockIdx.x] = y;
    }
}
__global__ void __launch_bounds__(1024) scan24_top_kernel(std::uint64_t* __restrict__ sums, int nchunks) {
    __shared__ std::uint64_t s_w[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    constexpr int PER = 4;  // 4096 chunks max
    std::uint64_t v[PER], tot = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        v[q] = t * PER + q < nchunks ? sums[t * PER + q] : 0;
        tot += v[q];
    }
    std::uint64_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint64_t y = __shfl_up_sync(FULLM, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    std::uint64_t base = 0;
    for (int i = 0; i < w; ++i) base += s_w[i];
    std::uint64_t run = base + inc - tot;
#pragma unroll
    for (int q = 0; q < PER; ++q)
        if (t * PER + q < nchunks) {
            sums[t * PER + q] = run;
            run += v[q];
        }
}
__global__ void __launch_bounds__(1024) scan24_chunk_kernel(const std::uint32_t* __restrict__ h,
                                                            const std::uint64_t* __restrict__ sums,
                                                            std::uint64_t* __restrict__ cur) {
    __shared__ std::uint64_t s_w[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const std::size_t base = static_cast<std::size_t>(blockIdx.x) * S24_CHUNK;
    const uint4 v = reinterpret_cast<const uint4*>(h + base)[t];
    const std::uint64_t tot = static_cast<std::uint64_t>(v.x) + v.y + v.z + v.w;
    std::uint64_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint64_t y = __shfl_up_sync(FULLM, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    std::uint64_t run = sums[blockIdx.x] + inc - tot;
    for (int i = 0; i < w; ++i) run += s_w[i];
    std::uint64_t* o = cur + base + 4 * t;
    o[0] = run;
    o[1] = run + v.x;
    o[2] = run + v.x + v.y;
    o[3] = run + v.x + v.y + v.z;
}

}  // namespace

template <typename T>
void msd_hist(ak_ctx* c, const T* kin, std::uint64_t n, bool desc, std::uint64_t* g_hist, std::uint64_t* g_joint,
              bool digit5) {
    constexpr std::size_t smem = JOINT_BINS * 2 + 256 * JH_PARTS * 4;
    smem_attr(c, hist_joint_kernel<T, true>, smem);
    smem_attr(c, hist_joint_kernel<T, false>, smem);
    AKB_CUDA(cudaMemsetAsync(g_joint, 0, JOINT_BINS * sizeof(std::uint64_t), c->stream));
    // every CTA flushes its whole 65536-bin table into the global one: at small n fewer,
    // fatter CTAs (one per 2^JH_KEYS_LOG keys, at least 16)
    const unsigned grid = static_cast<unsigned>(std::max<std::uint64_t>(
        16, std::min<std::uint64_t>(static_cast<std::uint64_t>(c->sm_count), n >> AKB_JH_KEYS_LOG)));
    const int tok = ctx_prof_begin(c, KF_HIST);
    if (digit5)
        hist_joint_kernel<T, true><<<grid, JH_BLOCK, smem, c->stream>>>(kin, n, desc ? 1 : 0, g_hist, g_joint);
    else
        hist_joint_kernel<T, false><<<grid, JH_BLOCK, smem, c->stream>>>(kin, n, desc ? 1 : 0, g_hist, g_joint);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    msd_joint_scan(c, g_joint, g_hist);
    c->kernel_launches += 1;
}

void msd_joint_scan(ak_ctx* c, std::uint64_t* g_joint, std::uint64_t* g_hist) {
    std::uint64_t* sums = g_joint + 2 * JOINT_BINS + 256 + 8;  // ctx_msd tail
    std::uint64_t* colpart = sums + JS_CTAS;
    auto* maxslot = reinterpret_cast<unsigned long long*>(g_joint + 2 * JOINT_BINS + 256 + 1);
    AKB_CUDA(cudaMemsetAsync(maxslot, 0, sizeof(std::uint64_t), c->stream));
    joint_scan_a_kernel<<<JS_CTAS, 1024, 0, c->stream>>>(g_joint, g_joint + JOINT_BINS, sums, colpart, g_hist, maxslot);
    joint_scan_b_kernel<<<JS_CTAS, 1024, 0, c->stream>>>(g_joint + JOINT_BINS, g_joint + 2 * JOINT_BINS, sums, colpart,
                                                         g_hist);
    AKB_CUDA(cudaGetLastError());
    c->kernel_launches += 2;
}

template <typename T>
void msd_top16(ak_ctx* c, const T* kin, T* kmid, T* kout, std::uint64_t n, bool desc, const std::uint64_t* g_joint,
               std::uint64_t* cur16, std::uint64_t* cur8, const int* plan) {
    smem_attr(c, msd_pass_kernel<T, 1>, mp_smem::total);
    smem_attr(c, msd_pass_kernel<T, 2>, mp_smem::total);
    const unsigned tiles = static_cast<unsigned>(ceil_div(n, MP_TILE));
    int tok = ctx_prof_begin(c, KF_MSD);
    msd_pass_kernel<T, 1><<<tiles, MP_BLOCK, mp_smem::total, c->stream>>>(kin, kmid, n, desc ? 1 : 0, cur8, plan);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    tok = ctx_prof_begin(c, KF_MSD);
    msd_pass_kernel<T, 2><<<tiles, MP_BLOCK, mp_smem::total, c->stream>>>(kmid, kout, n, desc ? 1 : 0, cur16, plan);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 2;
}

template <typename T>
void msd_digit_pass(ak_ctx* c, const T* kin, T* kout, std::uint64_t n, bool desc, std::uint64_t* cursors,
                    const int* plan) {
    smem_attr(c, msd_pass_kernel<T, 0>, mp_smem::total);
    const unsigned tiles = static_cast<unsigned>(ceil_div(n, MP_TILE));
    const int tok = ctx_prof_begin(c, KF_MSD);
    msd_pass_kernel<T, 0><<<tiles, MP_BLOCK, mp_smem::total, c->stream>>>(kin, kout, n, desc ? 1 : 0, cursors, plan);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 1;
}

template <typename T>
void msd_level3(ak_ctx* c, const T* kin, T* kout, std::uint64_t n, bool desc) {
    smem_attr(c, msd_pass_kernel<T, 3>, mp_smem::total);
    std::uint64_t* cur24 = ctx_msd3(c);                                   // 2^24 u64 cursors
    std::uint32_t* hist24 = reinterpret_cast<std::uint32_t*>(cur24 + (1u << 24));  // 2^24 u32 counts
    std::uint64_t* sums = cur24 + (1u << 24) + (1u << 23);               // 4096 chunk sums
    AKB_CUDA(cudaMemsetAsync(hist24, 0, (std::size_t(1) << 24) * sizeof(std::uint32_t), c->stream));
    const unsigned tiles = static_cast<unsigned>(ceil_div(n, MP_TILE));
    int tok = ctx_prof_begin(c, KF_HIST);
    hist_sub_kernel<T, 48><<<tiles, MP_BLOCK, 0, c->stream>>>(kin, n, desc ? 1 : 0, hist24);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    constexpr int nchunks = (1 << 24) / S24_CHUNK;
    scan24_sums_kernel<<<nchunks, 1024, 0, c->stream>>>(hist24, sums);
    scan24_top_kernel<<<1, 1024, 0, c->stream>>>(sums, nchunks);
    scan24_chunk_kernel<<<nchunks, 1024, 0, c->stream>>>(hist24, sums, cur24);
    AKB_CUDA(cudaGetLastError());
    tok = ctx_prof_begin(c, KF_MSD);
    msd_pass_kernel<T, 3><<<tiles, MP_BLOCK, mp_smem::total, c->stream>>>(kin, kout, n, desc ? 1 : 0, cur24);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 5;
}

template <typename C>
__global__ void bucket_max_kernel(const C* __restrict__ h, std::uint64_t cnt, unsigned long long* __restrict__ out) {
    std::uint64_t m = 0;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt; i += stride)
        m = m > h[i] ? m : static_cast<std::uint64_t>(h[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const std::uint64_t y = __shfl_xor_sync(FULLM, m, o);
        m = m > y ? m : y;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, static_cast<unsigned long long>(m));
}

std::uint64_t msd_max_bucket(ak_ctx* c, int level) {
    std::uint64_t* slot = ctx_msd(c) + 2 * JOINT_BINS + 256;
    AKB_CUDA(cudaMemsetAsync(slot, 0, sizeof(std::uint64_t), c->stream));
    if (level == 3) {
        const std::uint32_t* hist24 = reinterpret_cast<const std::uint32_t*>(ctx_msd3(c) + (1u << 24));
        bucket_max_kernel<std::uint32_t><<<c->sm_count * 4, 256, 0, c->stream>>>(
            hist24, std::uint64_t(1) << 24, reinterpret_cast<unsigned long long*>(slot));
    } else {
        bucket_max_kernel<std::uint64_t><<<64, 256, 0, c->stream>>>(ctx_msd(c), JOINT_BINS,
                                                                    reinterpret_cast<unsigned long long*>(slot));
    }
    AKB_CUDA(cudaGetLastError());
    auto* h = static_cast<std::uint64_t*>(ctx_pinned(c, sizeof(std::uint64_t)));
    AKB_CUDA(cudaMemcpyAsync(h, slot, sizeof(std::uint64_t), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    c->kernel_launches += 1;
    return *h;
}

template void msd_digit_pass<std::int64_t>(ak_ctx*, const std::int64_t*, std::int64_t*, std::uint64_t, bool,
                                           std::uint64_t*, const int*);
template void msd_digit_pass<std::uint64_t>(ak_ctx*, const std::uint64_t*, std::uint64_t*, std::uint64_t, bool,
                                            std::uint64_t*, const int*);
template void msd_level3<std::int64_t>(ak_ctx*, const std::int64_t*, std::int64_t*, std::uint64_t, bool);
template void msd_level3<std::uint64_t>(ak_ctx*, const std::uint64_t*, std::uint64_t*, std::uint64_t, bool);
template void msd_hist<std::int64_t>(ak_ctx*, const std::int64_t*, std::uint64_t, bool, std::uint64_t*,
                                     std::uint64_t*, bool);
template void msd_hist<std::uint64_t>(ak_ctx*, const std::uint64_t*, std::uint64_t, bool, std::uint64_t*,
                                      std::uint64_t*, bool);
template void msd_top16<std::int64_t>(ak_ctx*, const std::int64_t*, std::int64_t*, std::int64_t*, std::uint64_t,
                                      bool, const std::uint64_t*, std::uint64_t*, std::uint64_t*, const int*);
template void msd_top16<std::uint64_t>(ak_ctx*, const std::uint64_t*, std::uint64_t*, std::uint64_t*, std::uint64_t,
                                       bool, const std::uint64_t*, std::uint64_t*, std::uint64_t*, const int*);

}  // namespace akb
