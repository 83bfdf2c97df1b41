// search_merge.cu -- searchsorted, sample gather, merge-path 2-way merge, is_sorted.
#include "search_merge.cuh"
#include "radix_sort.cuh"

#include <vector>

namespace akb {

namespace {

template <typename T>
__device__ __forceinline__ std::uint64_t lower_bound_dev(const T* h, std::uint64_t n, T v, bool desc) {
    std::uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const std::uint64_t mid = lo + (hi - lo) / 2;
        if (key_less(h[mid], v, desc)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
template <typename T>
__device__ __forceinline__ std::uint64_t upper_bound_dev(const T* h, std::uint64_t n, T v, bool desc) {
    std::uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const std::uint64_t mid = lo + (hi - lo) / 2;
        if (!key_less(v, h[mid], desc)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename T>
__global__ void search_kernel(const T* __restrict__ hay, std::uint64_t n, const T* __restrict__ needles,
                              std::uint64_t m, int side_last, int desc, std::uint64_t* __restrict__ out) {
    const std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const T v = needles[i];
    out[i] = side_last ? upper_bound_dev(hay, n, v, desc != 0) : lower_bound_dev(hay, n, v, desc != 0);
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ x, std::uint64_t n, std::uint64_t k, T* __restrict__ out) {
    const std::uint64_t j = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j == 0) {
        out[0] = x[0];
        out[1] = x[n - 1];
    }
    if (j >= k) return;
    std::uint64_t pos;
    if (k == 1) pos = n / 2;
    else pos = (2 * j * (n - 1) + (k - 1)) / (2 * (k - 1));  // sihsort.hpp:279
    out[2 + j] = x[pos];
}

// co_rank of sort.hpp:75-88: #elements of a among the first k merged outputs.
template <typename T>
__device__ __forceinline__ std::uint64_t co_rank_dev(std::uint64_t k, const T* a, std::uint64_t na,
                                                     const T* b, std::uint64_t nb, bool desc) {
    std::uint64_t lo = k > nb ? k - nb : 0;
    std::uint64_t hi = k < na ? k : na;
    while (lo < hi) {
        const std::uint64_t i = lo + (hi - lo) / 2;
        if (key_less(b[k - i - 1], a[i], desc)) hi = i;
        else lo = i + 1;
    }
    return lo;
}

constexpr int MERGE_BLOCK = 256;
template <typename T>
struct merge_cfg {
    static constexpr int ITEMS = sizeof(T) == 8 ? 13 : 17;  // odd: no bank-aligned thread windows
    static constexpr int TILE = MERGE_BLOCK * ITEMS;
};

template <typename T>
__global__ void merge_partition_kernel(const T* __restrict__ a, std::uint64_t na, const T* __restrict__ b,
                                       std::uint64_t nb, std::uint64_t tiles, int desc,
                                       std::uint64_t* __restrict__ split) {
    const std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t > tiles) return;
    std::uint64_t diag = t * merge_cfg<T>::TILE;
    if (diag > na + nb) diag = na + nb;
    split[t] = co_rank_dev(diag, a, na, b, nb, desc != 0);
}

template <typename T>
__global__ void __launch_bounds__(MERGE_BLOCK)
    merge_kernel(const T* __restrict__ a, std::uint64_t na, const T* __restrict__ b, std::uint64_t nb,
                 const std::uint64_t* __restrict__ split, T* __restrict__ dst, int desc) {
    constexpr int ITEMS = merge_cfg<T>::ITEMS;
    constexpr int TILE = merge_cfg<T>::TILE;
#ifdef AKB_MERGE_LDG
    __shared__ T s[TILE];
#else
    // the a- and b-pieces arrive by two TMA bulk copies of their 16-byte aligned supersets
    // (global -> shared without a register or L1 round trip); each copy has <= 16 bytes of
    // slack at both ends
    constexpr int SLACK = 16 / sizeof(T);
    __shared__ __align__(16) T s[TILE + 4 * SLACK];
    __shared__ __align__(8) std::uint64_t bar;
#endif
    const bool dsc = desc != 0;
    const std::uint64_t t = blockIdx.x;
    const std::uint64_t d0 = t * TILE;
    std::uint64_t d1 = d0 + TILE;
    if (d1 > na + nb) d1 = na + nb;
    const std::uint64_t a0 = split[t], a1 = split[t + 1];
    const std::uint64_t b0 = d0 - a0, b1 = d1 - a1;
    const int la = static_cast<int>(a1 - a0), lb = static_cast<int>(b1 - b0);
#ifdef AKB_MERGE_LDG
    for (int i = threadIdx.x; i < la; i += MERGE_BLOCK) s[i] = a[a0 + i];
    for (int i = threadIdx.x; i < lb; i += MERGE_BLOCK) s[la + i] = b[b0 + i];
    __syncthreads();
    const T* sa = s;
    const T* sb = s + la;
#else
    auto span_of = [](const T* p, std::uint64_t lo, std::uint64_t hi, std::uintptr_t& g0, std::uint32_t& bytes) {
        const std::uintptr_t x0 = reinterpret_cast<std::uintptr_t>(p + lo), x1 = reinterpret_cast<std::uintptr_t>(p + hi);
        g0 = x0 & ~std::uintptr_t(15);
        bytes = static_cast<std::uint32_t>(((x1 + 15) & ~std::uintptr_t(15)) - g0);
        return static_cast<int>((x0 - g0) / sizeof(T));  // element shift inside the copy
    };
    std::uintptr_t ga = 0, gb = 0;
    std::uint32_t ba = 0, bb = 0;
    const int sha = la ? span_of(a, a0, a1, ga, ba) : 0;
    const int shb = lb ? span_of(b, b0, b1, gb, bb) : 0;
    const int offb = ((la + sha + SLACK - 1) / SLACK + 1) * SLACK;  // 16-byte aligned start of the b copy
    const std::uint32_t sbar = static_cast<std::uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(ba + bb) : "memory");
        if (ba)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             static_cast<std::uint32_t>(__cvta_generic_to_shared(s))),
                         "l"(ga), "r"(ba), "r"(sbar)
                         : "memory");
        if (bb)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             static_cast<std::uint32_t>(__cvta_generic_to_shared(s + offb))),
                         "l"(gb), "r"(bb), "r"(sbar)
                         : "memory");
    }
    __syncthreads();  // barrier initialised before anyone waits
    asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W_%=; }" ::"r"(sbar)
                 : "memory");
    const T* sa = s + sha;
    const T* sb = s + offb + shb;
#endif
    const int total = la + lb;
    T outv[ITEMS];
    const int k0 = threadIdx.x * ITEMS;
    int cnt = 0;
    if (k0 < total) {
        int ai = static_cast<int>(co_rank_dev<T>(k0, sa, la, sb, lb, dsc));
        int bi = k0 - ai;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (k0 + j < total) {
                const bool take_a = ai < la && (bi >= lb || !key_less(sb[bi], sa[ai], dsc));
                outv[j] = take_a ? sa[ai] : sb[bi];
                ai += take_a ? 1 : 0;
                bi += take_a ? 0 : 1;
                ++cnt;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
        if (j < cnt) s[k0 + j] = outv[j];
    __syncthreads();
    for (int i = threadIdx.x; i < total; i += MERGE_BLOCK) dst[d0 + i] = s[i];
}


template <typename T>
__global__ void unsorted_kernel(const T* __restrict__ x, std::uint64_t n, int desc, unsigned* flag) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    bool bad = false;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i + 1 < n;
         i += stride)
        bad |= key_less(x[i + 1], x[i], desc != 0);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

template <typename T>
void searchsorted(ak_ctx* c, const T* hay, std::uint64_t n, const T* needles, std::uint64_t m,
                  int side_last, int desc, std::uint64_t* d_out) {
    if (m == 0) return;
    const unsigned blocks = static_cast<unsigned>(ceil_div(m, 256));
    search_kernel<T><<<blocks, 256, 0, c->stream>>>(hay, n, needles, m, side_last, desc, d_out);
    AKB_CUDA(cudaGetLastError());
    c->kernel_launches += 1;
}

template <typename T>
std::uint64_t gather_samples(ak_ctx* c, const T* sorted, std::uint64_t n, std::uint64_t k, T* d_out) {
    if (n == 0) return 0;
    if (k > n) k = n;
    const unsigned blocks = static_cast<unsigned>(ceil_div(k > 0 ? k : 1, 256));
    gather_kernel<T><<<blocks, 256, 0, c->stream>>>(sorted, n, k, d_out);
    AKB_CUDA(cudaGetLastError());
    c->kernel_launches += 1;
    return k;
}

template <typename T>
void merge2(ak_ctx* c, const T* a, std::uint64_t na, const T* b, std::uint64_t nb, T* dst, bool desc) {
    const std::uint64_t total = na + nb;
    if (total == 0) return;
    if (nb == 0 || na == 0) {
        const T* src = na ? a : b;
        if (src != dst)
            AKB_CUDA(cudaMemcpyAsync(dst, src, total * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    const std::uint64_t tiles = ceil_div(total, merge_cfg<T>::TILE);
    std::uint64_t* split = ctx_split(c, tiles + 1);
    merge_partition_kernel<T><<<static_cast<unsigned>(ceil_div(tiles + 1, 256)), 256, 0, c->stream>>>(
        a, na, b, nb, tiles, desc ? 1 : 0, split);
    AKB_CUDA(cudaGetLastError());
    const int tok = ctx_prof_begin(c, KF_MERGE);
    merge_kernel<T><<<static_cast<unsigned>(tiles), MERGE_BLOCK, 0, c->stream>>>(a, na, b, nb, split, dst,
                                                                                desc ? 1 : 0);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 2;
}


// K8: stable P-way merge as a tree of merge-path 2-way merges over HBM, ceil(log2 P)
// levels ping-ponging between dst and scratch (the last level lands in dst). Measured on
// B200 (r01): a 2-way level runs at ~3.3 TB/s of key traffic, and a one-pass variant that
// merged the P pieces of value-cut tiles in shared memory was slower (its on-chip levels are
// latency-bound, ~0.7 ms per level at 2^27 keys), so the tree stays.
template <typename T>
void merge_runs(ak_ctx* c, int P, const T* const* runs, const std::uint64_t* lens, T* dst, T* scratch, bool desc) {
    if (P < 1) throw invalid_argument("merge_runs: P >= 1 runs");
    struct run {
        const T* p;
        std::uint64_t len, off;
    };
    std::vector<run> live;
    std::uint64_t off = 0;
    for (int r = 0; r < P; ++r) {
        if (lens[r]) live.push_back({runs[r], lens[r], off});
        off += lens[r];
    }
    if (live.empty()) return;
    if (live.size() == 1) {
        if (live[0].p != dst)
            AKB_CUDA(cudaMemcpyAsync(dst, live[0].p, live[0].len * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    if constexpr (std::is_integral_v<T> && sizeof(T) == 8) {
        // keys-only 64-bit integers, P >= 6: one pass over value tiles (radix_sort.cu)
        std::vector<const T*> rp;
        std::vector<std::uint64_t> rl;
        for (const run& x : live) {
            rp.push_back(x.p);
            rl.push_back(x.len);
        }
        if (merge_runs_counting<T>(c, static_cast<int>(live.size()), rp.data(), rl.data(), dst, desc)) return;
    }
    int levels = 0;
    for (std::size_t m = 1; m < live.size(); m <<= 1) ++levels;
    for (int l = 1; l <= levels; ++l) {
        T* out = ((levels - l) % 2 == 0) ? dst : scratch;
        std::vector<run> next;
        for (std::size_t i = 0; i < live.size(); i += 2) {
            if (i + 1 == live.size()) {  // odd run out: moved into this level's buffer
                const run& a = live[i];
                AKB_CUDA(cudaMemcpyAsync(out + a.off, a.p, a.len * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
                next.push_back({out + a.off, a.len, a.off});
                continue;
            }
            const run& a = live[i];
            const run& b = live[i + 1];
            merge2<T>(c, a.p, a.len, b.p, b.len, out + a.off, desc);
            next.push_back({out + a.off, a.len + b.len, a.off});
        }
        live.swap(next);
    }
}

template <typename T>
bool is_sorted(ak_ctx* c, const T* x, std::uint64_t n, bool desc) {
    if (n < 2) return true;
    unsigned* flag = reinterpret_cast<unsigned*>(static_cast<char*>(c->small) + 196608);
    AKB_CUDA(cudaMemsetAsync(flag, 0, 4, c->stream));
    unsorted_kernel<T><<<c->sm_count * 4, 256, 0, c->stream>>>(x, n, desc ? 1 : 0, flag);
    AKB_CUDA(cudaGetLastError());
    c->kernel_launches += 1;
    unsigned* h = static_cast<unsigned*>(ctx_pinned(c, 4));
    AKB_CUDA(cudaMemcpyAsync(h, flag, 4, cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    return *h == 0;
}

#define AKB_INST(T)                                                                               \
    template void searchsorted<T>(ak_ctx*, const T*, std::uint64_t, const T*, std::uint64_t, int,  \
                                  int, std::uint64_t*);                                           \
    template std::uint64_t gather_samples<T>(ak_ctx*, const T*, std::uint64_t, std::uint64_t, T*);  \
    template void merge2<T>(ak_ctx*, const T*, std::uint64_t, const T*, std::uint64_t, T*, bool);   \
    template bool is_sorted<T>(ak_ctx*, const T*, std::uint64_t, bool);                            \
    template void merge_runs<T>(ak_ctx*, int, const T* const*, const std::uint64_t*, T*, T*, bool);

AKB_INST(std::int32_t)
AKB_INST(std::uint32_t)
AKB_INST(std::int64_t)
AKB_INST(std::uint64_t)
AKB_INST(float)
AKB_INST(double)

}  // namespace akb
