// reduce_scan.cu -- reduce / mapreduce (K1) and single-pass scan (K2).
#include <limits>
#include <type_traits>

#include "reduce_scan.cuh"

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
// K2: single-pass scan, dynamic tiles, warp-cooperative decoupled look-back.
// Tile = 256 threads x ITEMS; warp w owns a contiguous run of 32*ITEMS
// elements processed in rounds of 32 (coalesced, one element per lane).
// ---------------------------------------------------------------------------
constexpr int SCAN_BLOCK = 256;

template <typename T>
struct scan_cfg {
    static constexpr int ITEMS = sizeof(T) == 8 ? 16 : 24;
    static constexpr int TILE = SCAN_BLOCK * ITEMS;
};

template <typename T, int OP>
__global__ void __launch_bounds__(SCAN_BLOCK)
    scan_kernel(const T* x, T* out, std::uint64_t n, T init, int inclusive, std::uint32_t* flags,
                std::uint64_t* vals, std::uint32_t tag, std::uint32_t* tile_counter) {
    using A = typename acc_of<T>::type;
    using F = opf<A, OP>;
    constexpr int ITEMS = scan_cfg<T>::ITEMS;
    constexpr int TILE = scan_cfg<T>::TILE;
    constexpr int WARPS = SCAN_BLOCK / 32;
    __shared__ A s_warp[WARPS];
    __shared__ A s_excl;
    __shared__ std::uint32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const std::uint32_t tile = s_tile;
    const std::uint64_t wbase =
        static_cast<std::uint64_t>(tile) * TILE + static_cast<std::uint64_t>(warp) * 32 * ITEMS;

    A v[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const std::uint64_t idx = wbase + i * 32 + lane;
        v[i] = idx < n ? static_cast<A>(x[idx]) : F::identity();
    }
    // inclusive scan of the warp's run; v[i] becomes the run-local inclusive prefix
    A carry = F::identity();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        A s = v[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const A y = shfl_up_any(s, o);
            if (lane >= o) s = F::apply(y, s);
        }
        s = F::apply(carry, s);
        v[i] = s;
        carry = shfl_any(s, 31);
    }
    if (lane == 0) s_warp[warp] = carry;
    __syncthreads();
    A wexcl = F::identity();
    A tile_total = F::identity();
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        if (w == warp) wexcl = tile_total;
        tile_total = F::apply(tile_total, s_warp[w]);
    }

    if (warp == 0) {
        A excl = F::identity();
        if (tile == 0) {
            if (lane == 0) {
                st_relaxed_u64(vals + 1, to_bits(tile_total));
                st_release_u32(flags, SC_INC | tag);
            }
        } else {
            if (lane == 0) {
                st_relaxed_u64(vals + 2 * static_cast<std::uint64_t>(tile), to_bits(tile_total));
                st_release_u32(flags + tile, SC_AGG | tag);
            }
            std::int64_t base = static_cast<std::int64_t>(tile) - 1;
            while (true) {
                const std::int64_t p = base - lane;
                std::uint32_t f = SC_INC;
                bool ready = true;
                if (p >= 0) {
                    f = ld_acquire_u32(flags + p);
                    ready = (f & SC_TAG_MASK) == tag && (f & ~SC_TAG_MASK) != 0;
                }
                const std::uint32_t ready_mask = __ballot_sync(FULL, ready);
                const std::uint32_t inc_mask =
                    __ballot_sync(FULL, ready && (p < 0 || (f & ~SC_TAG_MASK) == SC_INC));
                const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
                const int first_nr = ~ready_mask ? __ffs(~ready_mask) - 1 : 32;
                if (first_nr <= first_inc && first_nr < 32) continue;  // a needed tile is not published yet
                const int lim = first_inc < 32 ? first_inc : 31;
                A a = F::identity();
                if (p >= 0 && lane <= lim) {
                    const bool inc = (lane == lim) && inc_mask;
                    a = from_bits<A>(ld_relaxed_u64(vals + 2 * static_cast<std::uint64_t>(p) + (inc ? 1 : 0)));
                }
                // fold in order nearest-last: reduce lanes lim..0 (commutative ops)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a = F::apply(a, shfl_xor_any(a, o));
                excl = F::apply(a, excl);
                if (inc_mask) break;
                base -= 32;
            }
            if (lane == 0) {
                st_relaxed_u64(vals + 2 * static_cast<std::uint64_t>(tile) + 1,
                               to_bits(F::apply(excl, tile_total)));
                st_release_u32(flags + tile, SC_INC | tag);
            }
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const A pre = F::apply(F::apply(static_cast<A>(init), s_excl), wexcl);
    A prev_carry = F::identity();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const std::uint64_t idx = wbase + i * 32 + lane;
        A r;
        if (inclusive) {
            r = F::apply(pre, v[i]);
        } else {
            A up = shfl_up_any(v[i], 1);
            if (lane == 0) up = prev_carry;
            r = (i == 0 && lane == 0) ? pre : F::apply(pre, up);
            prev_carry = shfl_any(v[i], 31);
        }
        if (idx < n) out[idx] = static_cast<T>(r);
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
#define AKB_SCAN(OPV)                                                                          \
    scan_kernel<T, OPV><<<static_cast<unsigned>(tiles), SCAN_BLOCK, 0, c->stream>>>(            \
        x, out, n, init, inclusive, c->scan_flags, c->scan_vals, tag, counter)
    if (op == OP_SUM) AKB_SCAN(OP_SUM);
    else if (op == OP_MIN) AKB_SCAN(OP_MIN);
    else AKB_SCAN(OP_MAX);
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
