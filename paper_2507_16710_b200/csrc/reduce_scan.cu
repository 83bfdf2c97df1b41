// reduce_scan.cu -- reduce / mapreduce (K1) and single-pass scan (K2).
#include <limits>
#include <type_traits>

#include "reduce_scan.cuh"
#include "tma.cuh"

namespace akb {

namespace {

constexpr std::uint32_t FULL = 0xffffffffu;

template <typename A, int OP>
struct opf {
    __device__ __forceinline__ static A apply(A a, A b) {
        if constexpr (OP == OP_SUM) {
            if constexpr (std::is_integral_v<A>) {
                using U = std::make_unsigned_t<A>;
                return static_cast<A>(static_cast<U>(a) + static_cast<U>(b));
            } else {
                return a + b;
            }
        } else if constexpr (OP == OP_MIN) {
            return b < a ? b : a;
        } else {
            return a < b ? b : a;
        }
    }
    __device__ __forceinline__ static A identity() {
        if constexpr (OP == OP_SUM) {
            return A(0);
        } else if constexpr (OP == OP_MIN) {
            if constexpr (std::is_floating_point_v<A>) return A(INFINITY);
            else return std::numeric_limits<A>::max();
        } else {
            if constexpr (std::is_floating_point_v<A>) return A(-INFINITY);
            else return std::numeric_limits<A>::lowest();
        }
    }
};

template <typename A, int MAP>
__device__ __forceinline__ A map_apply(A v) {
    if constexpr (MAP == MAP_ABS) {
        if constexpr (std::is_unsigned_v<A>) return v;
        else if constexpr (std::is_integral_v<A>) {
            using U = std::make_unsigned_t<A>;
            return v < 0 ? static_cast<A>(U(0) - static_cast<U>(v)) : v;
        } else return v < A(0) ? -v : v;
    } else if constexpr (MAP == MAP_SQUARE) {
        if constexpr (std::is_integral_v<A>) {
            using U = std::make_unsigned_t<A>;
            return static_cast<A>(static_cast<U>(v) * static_cast<U>(v));
        } else return v * v;
    } else {
        return v;
    }
}

template <typename A>
__device__ __forceinline__ A shfl_xor_any(A v, int m) {
    return __shfl_xor_sync(FULL, v, m);
}
template <typename A>
__device__ __forceinline__ A shfl_up_any(A v, int m) {
    return __shfl_up_sync(FULL, v, m);
}
template <typename A>
__device__ __forceinline__ A shfl_any(A v, int src) {
    return __shfl_sync(FULL, v, src);
}

template <typename A>
__device__ __forceinline__ std::uint64_t to_bits(A v) {
    std::uint64_t b = 0;
    memcpy(&b, &v, sizeof(A));
    return b;
}
template <typename A>
__device__ __forceinline__ A from_bits(std::uint64_t b) {
    A v;
    memcpy(&v, &b, sizeof(A));
    return v;
}

// ---------------------------------------------------------------------------
// K1: grid-stride vectorised reduce, block partials, last-block fold.
// ---------------------------------------------------------------------------
constexpr int RED_BLOCK = 512;

template <typename T, int OP, int MAP>
__global__ void __launch_bounds__(RED_BLOCK)
    reduce_kernel(const T* __restrict__ x, std::uint64_t n, typename acc_of<T>::type* partials,
                  std::uint32_t* ticket, T init, T* result) {
    using A = typename acc_of<T>::type;
    using F = opf<A, OP>;
    constexpr int VEC = 16 / sizeof(T);
    A acc = F::identity();
    const std::uint64_t g = static_cast<std::uint64_t>(blockIdx.x) * RED_BLOCK + threadIdx.x;
    const std::uint64_t S = static_cast<std::uint64_t>(gridDim.x) * RED_BLOCK;
    const std::uintptr_t addr = reinterpret_cast<std::uintptr_t>(x);
    std::uint64_t head = ((16 - (addr & 15)) & 15) / sizeof(T);
    if (head > n) head = n;
    if (g < head) acc = F::apply(acc, map_apply<A, MAP>(static_cast<A>(x[g])));
    const uint4* v = reinterpret_cast<const uint4*>(x + head);
    const std::uint64_t nv = (n - head) / VEC;
    std::uint64_t i = g;
    for (; i + 3 * S < nv; i += 4 * S) {
        uint4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = __ldg(v + i + u * S);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const T* e = reinterpret_cast<const T*>(&q[u]);
#pragma unroll
            for (int k = 0; k < VEC; ++k) acc = F::apply(acc, map_apply<A, MAP>(static_cast<A>(e[k])));
        }
    }
    for (; i < nv; i += S) {
        const uint4 q = __ldg(v + i);
        const T* e = reinterpret_cast<const T*>(&q);
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc = F::apply(acc, map_apply<A, MAP>(static_cast<A>(e[k])));
    }
    for (std::uint64_t j = head + nv * VEC + g; j < n; j += S)
        acc = F::apply(acc, map_apply<A, MAP>(static_cast<A>(x[j])));

    __shared__ A s_w[RED_BLOCK / 32];
    __shared__ bool s_last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = F::apply(acc, shfl_xor_any(acc, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) s_w[w] = acc;
    __syncthreads();
    if (w == 0) {
        acc = lane < RED_BLOCK / 32 ? s_w[lane] : F::identity();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = F::apply(acc, shfl_xor_any(acc, o));
        if (lane == 0) {
            partials[blockIdx.x] = acc;
            __threadfence();
            s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        A t = F::identity();
        for (unsigned b = threadIdx.x; b < gridDim.x; b += RED_BLOCK) {
            t = F::apply(t, *reinterpret_cast<volatile A*>(partials + b));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = F::apply(t, shfl_xor_any(t, o));
        if (lane == 0) s_w[w] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            A r = F::identity();
            for (int k = 0; k < RED_BLOCK / 32; ++k) r = F::apply(r, s_w[k]);
            r = F::apply(static_cast<A>(init), r);  // init folded exactly once
            *result = static_cast<T>(r);
            *ticket = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// K2: single-pass scan, dynamic tiles, decoupled look-back (Merrill & Garland;
// the "opportunistic look-back" of PAPER.md:161).
//   load   : coalesced 16-byte loads, transposed through a shared tile whose 16-byte
//            chunks are XOR-swizzled per thread run (conflict-free 16-byte accesses
//            in both the coalesced and the per-run order);
//   local  : each thread scans its 16 contiguous elements serially, warp shuffle
//            scan of thread totals, block scan of 8 warp totals;
//   chain  : warp 0 publishes the tile aggregate, looks back 32 tiles per round
//            trip, publishes the inclusive prefix;
//   store  : results back through the same shared slots, coalesced 16-byte stores.
// Floats accumulate in double (acc_of), so carries over ~2^18 tiles stay exact
// enough for the 1e-5 contract.
// ---------------------------------------------------------------------------
template <typename T>
struct scan_cfg {
    // 256 threads and 32 KB tiles for every element size (16 x 8 B or 32 x 4 B per thread);
    // 6 tiles in flight per SM (runs are re-read from shared memory, not held in registers)
    // hide the look-back round trips.
    static constexpr int BLOCK = 256;
    static constexpr int ITEMS = 32 / sizeof(T) * 4;
    static constexpr int TILE = BLOCK * ITEMS;
    static constexpr int VEC = 16 / sizeof(T);
    static constexpr int CHUNKS = ITEMS / VEC;  // 16-byte chunks per thread run (8)
};

// 16-byte chunk g of the tile (thread run t = g / 8, chunk j = g % 8 of the run) lives at
// chunk t * 8 + (j ^ (t & 7)): eight consecutive threads reading chunk j of their runs hit
// eight different 16-byte bank groups, and so do eight consecutive coalesced chunks.
__device__ __forceinline__ int scan_chunk(int g) { return (g & ~7) | ((g ^ (g >> 3)) & 7); }
template <int VEC>
__device__ __forceinline__ int scan_slot(int e) { return scan_chunk(e / VEC) * VEC + e % VEC; }

// In-thread accumulation type: floats scan their 32-element run in float (error ~1e-7 of
// the run) and carry everything beyond the run in double (acc_of).
template <typename T>
struct local_acc_of {
    using type = T;
};

// Scan of one tile already staged in the swizzled shared tile: thread-serial runs -> warp /
// block scan -> decoupled look-back -> results written back into the same shared slots.
// Ends with a __syncthreads (the tile is ready to store).
template <typename T, int OP>
__device__ __forceinline__ void scan_tile_core(T* s_tile, typename acc_of<T>::type* s_warp,
                                               typename acc_of<T>::type& s_excl, std::uint32_t tile,
                                               std::uint64_t rem, bool full, T init, int inclusive,
                                               std::uint64_t* vals, std::uint32_t tag) {
    using A = typename acc_of<T>::type;
    using F = opf<A, OP>;
    using LA = typename local_acc_of<T>::type;
    using FL = opf<LA, OP>;
    using Cfg = scan_cfg<T>;
    constexpr int ITEMS = Cfg::ITEMS;
    constexpr int SCAN_BLOCK = Cfg::BLOCK;
    constexpr int WARPS = SCAN_BLOCK / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // ---- thread-serial scan of ITEMS contiguous elements (16 x 8 B or 32 x 4 B) ----
    // (pass 1 only totals the run; pass 2 below re-reads it from shared memory and
    // rebuilds the same prefixes, so no per-item registers live across the look-back)
    constexpr int VEC = Cfg::VEC;
    constexpr int CHUNKS = Cfg::CHUNKS;
    static_assert(CHUNKS == 8, "the chunk swizzle assumes 8 chunks per thread run");
    uint4* s4 = reinterpret_cast<uint4*>(s_tile);
    const int my0 = tid * ITEMS;
    LA run = FL::identity();
#pragma unroll
    for (int j = 0; j < CHUNKS; ++j) {
        const uint4 q = s4[tid * CHUNKS + (j ^ (tid & 7))];
        const T* e = reinterpret_cast<const T*>(&q);
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const bool ok = full || static_cast<std::uint64_t>(my0 + j * VEC + k) < rem;
            run = FL::apply(run, ok ? static_cast<LA>(e[k]) : FL::identity());
        }
    }
    // warp scan of thread totals
    A winc = static_cast<A>(run);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const A y = shfl_up_any(winc, o);
        if (lane >= o) winc = F::apply(y, winc);
    }
    A texcl = shfl_up_any(winc, 1);  // exclusive prefix of this thread within its warp
    if (lane == 0) texcl = F::identity();
    if (lane == 31) s_warp[warp] = winc;
    __syncthreads();
    A wexcl = F::identity();
    A tile_total = F::identity();
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        if (w == warp) wexcl = tile_total;
        tile_total = F::apply(tile_total, s_warp[w]);
    }

    // ---- decoupled look-back (warp 0). Descriptor per tile, published with one
    // relaxed store: 4-byte accumulators pack {status|tag : value} into one 64-bit
    // word; 8-byte accumulators use two such words (one per 32-bit value half),
    // stored together and accepted only when both halves carry the same status,
    // so correctness needs only 64-bit single-copy atomicity ----
    if (warp == 0) {
        A excl = F::identity();
        constexpr bool NARROW = sizeof(A) == 4;
        std::uint64_t* my = vals + (NARROW ? 1 : 2) * static_cast<std::uint64_t>(tile);
        auto publish = [&](A v, std::uint32_t status) {
            const std::uint64_t b = to_bits(v);
            const std::uint64_t hi_status = static_cast<std::uint64_t>(status) << 32;
            if constexpr (NARROW) st_relaxed_u64(my, hi_status | b);
            else st_relaxed_desc(my, hi_status | (b & 0xffffffffull), hi_status | (b >> 32));
        };
        if (tile == 0) {
            if (lane == 0) publish(tile_total, SC_INC | tag);
        } else {
            if (lane == 0) publish(tile_total, SC_AGG | tag);
            std::int64_t pbase = static_cast<std::int64_t>(tile) - 1;
            while (true) {
                const std::int64_t p = pbase - lane;
                std::uint64_t vb = 0;
                std::uint32_t f = SC_INC | tag;
                if (p >= 0) {
                    if constexpr (NARROW) {
                        const std::uint64_t w = ld_relaxed_u64(vals + p);
                        vb = w & 0xffffffffull;
                        f = static_cast<std::uint32_t>(w >> 32);
                    } else {
                        // each 64-bit half carries the status word; a read that straddles a
                        // republication sees two different statuses and is treated as not ready
                        std::uint64_t w0, w1;
                        ld_relaxed_desc(vals + 2 * static_cast<std::uint64_t>(p), w0, w1);
                        vb = (w0 & 0xffffffffull) | (w1 << 32);
                        const std::uint32_t f0 = static_cast<std::uint32_t>(w0 >> 32);
                        f = f0 == static_cast<std::uint32_t>(w1 >> 32) ? f0 : 0u;
                    }
                }
                const bool ready = (f & SC_TAG_MASK) == tag && (f & ~SC_TAG_MASK) != 0;
                const std::uint32_t ready_mask = __ballot_sync(FULL, ready);
                const std::uint32_t inc_mask = __ballot_sync(FULL, ready && (f & ~SC_TAG_MASK) == SC_INC);
                const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
                const int first_nr = ~ready_mask ? __ffs(~ready_mask) - 1 : 32;
                if (first_nr <= first_inc && first_nr < 32) continue;  // a needed tile is not published yet
                const int lim = first_inc < 32 ? first_inc : 31;
                A a = (p >= 0 && lane <= lim) ? from_bits<A>(vb) : F::identity();
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a = F::apply(a, shfl_xor_any(a, o));
                excl = F::apply(a, excl);
                if (inc_mask) break;
                pbase -= 32;
            }
            if (lane == 0) publish(F::apply(excl, tile_total), SC_INC | tag);
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();

    // ---- results back into this thread's own shared slots ----
    const A pre = F::apply(F::apply(F::apply(static_cast<A>(init), s_excl), wexcl), texcl);
    LA r = FL::identity();
#pragma unroll
    for (int j = 0; j < CHUNKS; ++j) {
        uint4& qr = s4[tid * CHUNKS + (j ^ (tid & 7))];
        uint4 q = qr;
        T* e = reinterpret_cast<T*>(&q);
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const bool ok = full || static_cast<std::uint64_t>(my0 + j * VEC + k) < rem;
            const LA before = r;
            r = FL::apply(r, ok ? static_cast<LA>(e[k]) : FL::identity());  // as in pass 1
            e[k] = static_cast<T>(F::apply(pre, static_cast<A>(inclusive ? r : before)));
        }
        qr = q;
    }
    __syncthreads();

}

template <typename T, int OP, bool VECIO>
__global__ void __launch_bounds__(scan_cfg<T>::BLOCK, 6)
    scan_kernel(const T* x, T* out, std::uint64_t n, T init, int inclusive, std::uint32_t* flags,
                std::uint64_t* vals, std::uint32_t tag, std::uint32_t* tile_counter) {
    using A = typename acc_of<T>::type;
    using F = opf<A, OP>;
    using LA = typename local_acc_of<T>::type;
    using FL = opf<LA, OP>;
    using Cfg = scan_cfg<T>;
    constexpr int TILE = Cfg::TILE;
    constexpr int VEC = Cfg::VEC;
    constexpr int SCAN_BLOCK = Cfg::BLOCK;
    constexpr int WARPS = SCAN_BLOCK / 32;
    __shared__ __align__(16) T s_tile[TILE];
    __shared__ A s_warp[WARPS];
    __shared__ A s_excl;
    __shared__ std::uint32_t s_tile_id;
    const int tid = threadIdx.x;
    if (tid == 0) {
        // the tile id comes from the ticket below (look-back order); tickets follow the launch
        // order closely, so the tile this CTA's index names -- read by this or a neighbouring
        // CTA -- is fetched into L2 while the ticket round trip is in flight
        const std::uint64_t pb = static_cast<std::uint64_t>(blockIdx.x) * TILE;
        if (VECIO && pb + TILE <= n) bulk_prefetch_l2(x + pb, static_cast<std::uint32_t>(TILE * sizeof(T)));
        s_tile_id = atomicAdd(tile_counter, 1u);
    }
    __syncthreads();
    const std::uint32_t tile = s_tile_id;
    const std::uint64_t base = static_cast<std::uint64_t>(tile) * TILE;
    const std::uint64_t rem = n - base;
    const bool full = rem >= static_cast<std::uint64_t>(TILE);

    // ---- load: global (coalesced) -> swizzled shared tile ----
    if (VECIO && full) {
        const uint4* src = reinterpret_cast<const uint4*>(x + base);
        uint4 q[TILE / VEC / SCAN_BLOCK];
#pragma unroll
        for (int j = 0; j < TILE / VEC / SCAN_BLOCK; ++j) q[j] = __ldg(src + j * SCAN_BLOCK + tid);
#pragma unroll
        for (int j = 0; j < TILE / VEC / SCAN_BLOCK; ++j)
            reinterpret_cast<uint4*>(s_tile)[scan_chunk(j * SCAN_BLOCK + tid)] = q[j];
    } else {
#pragma unroll 4
        for (int e = tid; e < TILE; e += SCAN_BLOCK)
            if (static_cast<std::uint64_t>(e) < rem) s_tile[scan_slot<VEC>(e)] = x[base + e];
    }
    __syncthreads();

    scan_tile_core<T, OP>(s_tile, s_warp, s_excl, tile, rem, full, init, inclusive, vals, tag);

    // ---- store: swizzled shared tile -> global (coalesced) ----
    if (VECIO && full) {
        uint4* dst = reinterpret_cast<uint4*>(out + base);
#pragma unroll
        for (int j = 0; j < TILE / VEC / SCAN_BLOCK; ++j)
            dst[j * SCAN_BLOCK + tid] = reinterpret_cast<const uint4*>(s_tile)[scan_chunk(j * SCAN_BLOCK + tid)];
    } else {
#pragma unroll 4
        for (int e = tid; e < TILE; e += SCAN_BLOCK)
            if (static_cast<std::uint64_t>(e) < rem) out[base + e] = s_tile[scan_slot<VEC>(e)];
    }
}

}  // namespace

template <typename T>
void reduce(ak_ctx* c, const T* x, std::uint64_t n, int op, int map, T init, T* d_result) {
    using A = typename acc_of<T>::type;
    // small-region layout: [64 KiB, 128 KiB): ticket + partials
    char* base = static_cast<char*>(c->small) + 65536;
    std::uint32_t* ticket = reinterpret_cast<std::uint32_t*>(base);
    A* partials = reinterpret_cast<A*>(base + 256);
    int blocks = c->sm_count * 4;
    const std::uint64_t need = ceil_div(n, static_cast<std::uint64_t>(RED_BLOCK) * (16 / sizeof(T)) * 4);
    if (static_cast<std::uint64_t>(blocks) > need) blocks = static_cast<int>(need < 1 ? 1 : need);
    AKB_CUDA(cudaMemsetAsync(ticket, 0, 4, c->stream));
    const int tok = ctx_prof_begin(c, KF_REDUCE);
#define AKB_RED(OPV, MAPV)                                                                     \
    reduce_kernel<T, OPV, MAPV><<<blocks, RED_BLOCK, 0, c->stream>>>(x, n, partials, ticket,     \
                                                                      init, d_result)
    if (map == MAP_IDENTITY) {
        if (op == OP_SUM) AKB_RED(OP_SUM, MAP_IDENTITY);
        else if (op == OP_MIN) AKB_RED(OP_MIN, MAP_IDENTITY);
        else AKB_RED(OP_MAX, MAP_IDENTITY);
    } else if (map == MAP_ABS) {
        if (op == OP_SUM) AKB_RED(OP_SUM, MAP_ABS);
        else if (op == OP_MIN) AKB_RED(OP_MIN, MAP_ABS);
        else AKB_RED(OP_MAX, MAP_ABS);
    } else {
        if (op == OP_SUM) AKB_RED(OP_SUM, MAP_SQUARE);
        else if (op == OP_MIN) AKB_RED(OP_MIN, MAP_SQUARE);
        else AKB_RED(OP_MAX, MAP_SQUARE);
    }
#undef AKB_RED
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 1;
}

template <typename T>
void scan(ak_ctx* c, const T* x, T* out, std::uint64_t n, int op, int inclusive, T init) {
    if (n == 0) return;
    const std::uint64_t tiles = ceil_div(n, scan_cfg<T>::TILE);
    const std::uint32_t tag = ctx_scan_pass(c, tiles);
    std::uint32_t* counter = reinterpret_cast<std::uint32_t*>(static_cast<char*>(c->small) + 131072);
    AKB_CUDA(cudaMemsetAsync(counter, 0, 4, c->stream));
    const int tok = ctx_prof_begin(c, KF_SCAN);
    const bool vecio = ((reinterpret_cast<std::uintptr_t>(x) | reinterpret_cast<std::uintptr_t>(out)) & 15) == 0;
    // 6 x 32 KB tiles per SM: ask for the full shared-memory carveout (once per device)
#define AKB_SCAN(OPV, V)                                                                       \
    do {                                                                                       \
        func_attr_once(c, reinterpret_cast<const void*>(scan_kernel<T, OPV, V>),              \
                       cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared); \
        scan_kernel<T, OPV, V><<<static_cast<unsigned>(tiles), scan_cfg<T>::BLOCK, 0, c->stream>>>(     \
            x, out, n, init, inclusive, c->scan_flags, c->scan_vals, tag, counter);            \
    } while (0)
    if (vecio) {
        if (op == OP_SUM) AKB_SCAN(OP_SUM, true);
        else if (op == OP_MIN) AKB_SCAN(OP_MIN, true);
        else AKB_SCAN(OP_MAX, true);
    } else {
        if (op == OP_SUM) AKB_SCAN(OP_SUM, false);
        else if (op == OP_MIN) AKB_SCAN(OP_MIN, false);
        else AKB_SCAN(OP_MAX, false);
    }
#undef AKB_SCAN
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 1;
}

#define AKB_INST(T)                                                                             \
    template void reduce<T>(ak_ctx*, const T*, std::uint64_t, int, int, T, T*);                 \
    template void scan<T>(ak_ctx*, const T*, T*, std::uint64_t, int, int, T);

AKB_INST(std::int32_t)
AKB_INST(std::uint32_t)
AKB_INST(std::int64_t)
AKB_INST(std::uint64_t)
AKB_INST(float)
AKB_INST(double)

}  // namespace akb
