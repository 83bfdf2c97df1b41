// wide_keys.cu -- the reference's remaining sort key types: int16 and int128 (dtype.hpp:14-21).
//
// int16: widened to int32 (order-preserving, equal keys stay equal), sorted by the int32
//   path (same stability), narrowed back.
// int128: stable LSD over its two 64-bit halves. perm = stable sortperm of the low halves
//   (unsigned); then a stable by-key sort of the gathered high halves (signed) carrying perm
//   as payload. Both passes are stable, so perm orders by (hi, lo) with ties in input order
//   = the stable sort of sort.hpp:92-117 under operator< on __int128; std::greater runs both
//   passes descending. Keys and payload are then gathered through perm.
// Both use a ctx-owned work arena (reused across calls); the caller's buffers are validated
// exactly as the reference requires (capi.cu).
#include "radix_sort.cuh"
#include "wide_keys.cuh"

namespace akb {

namespace {

__global__ void widen16_kernel(const std::int16_t* __restrict__ s, std::int32_t* __restrict__ d, std::uint64_t n) {
    const std::uint64_t st = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += st) d[i] = s[i];
}
__global__ void narrow16_kernel(const std::int32_t* __restrict__ s, std::int16_t* __restrict__ d, std::uint64_t n) {
    const std::uint64_t st = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += st)
        d[i] = static_cast<std::int16_t>(s[i]);
}
__global__ void split128_kernel(const __int128* __restrict__ s, std::uint64_t* __restrict__ lo,
                                std::int64_t* __restrict__ hi, std::uint64_t n) {
    const std::uint64_t st = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += st) {
        const __int128 v = s[i];
        lo[i] = static_cast<std::uint64_t>(v);
        hi[i] = static_cast<std::int64_t>(v >> 64);
    }
}
// d[i] = s[perm[i]]
template <typename T, typename P>
__global__ void gather_kernel(const T* __restrict__ s, const P* __restrict__ perm, T* __restrict__ d, std::uint64_t n) {
    const std::uint64_t st = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += st)
        d[i] = s[perm[i]];
}
template <typename I>
__global__ void convert_kernel(const std::uint64_t* __restrict__ s, I* __restrict__ d, std::uint64_t n) {
    const std::uint64_t st = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += st)
        d[i] = static_cast<I>(s[i]);
}

unsigned grid_of(ak_ctx* c) { return static_cast<unsigned>(c->sm_count * 8); }

template <typename T>
T* work_arena(ak_ctx* c, std::size_t bytes) {
    void* p = ctx_work(c, bytes);
    if (!p) throw invalid_argument("int16/int128 sort: cannot allocate the work arena");
    return static_cast<T*>(p);
}

// Stable permutation of n int128 keys (u64 indices) in w[2n .. 3n); w holds 6n words.
std::uint64_t* perm128(ak_ctx* c, const __int128* d, std::uint64_t n, bool desc, std::uint64_t* w) {
    std::uint64_t* lo = w;
    auto* hi = reinterpret_cast<std::int64_t*>(w + n);
    std::uint64_t* perm = w + 2 * n;
    std::uint64_t* k1 = w + 3 * n;
    std::uint64_t* k2 = w + 4 * n;
    std::uint64_t* pv = w + 5 * n;
    split128_kernel<<<grid_of(c), 256, 0, c->stream>>>(d, lo, hi, n);
    AKB_CUDA(cudaGetLastError());
    // pass 1: stable sortperm of the low halves
    radix_sort<std::uint64_t, std::uint64_t>(c, SORT_IOTA, lo, k1, k2, nullptr, perm, pv, n, desc, false);
    // pass 2: stable by-key sort of the high halves (gathered through perm), perm as payload
    auto* hk = reinterpret_cast<std::int64_t*>(k1);
    gather_kernel<std::int64_t, std::uint64_t><<<grid_of(c), 256, 0, c->stream>>>(hi, perm, hk, n);
    AKB_CUDA(cudaGetLastError());
    radix_sort<std::int64_t, std::uint64_t>(c, SORT_PAIRS, hk, hk, reinterpret_cast<std::int64_t*>(k2), perm, perm,
                                            pv, n, desc, true);
    c->kernel_launches += 2;
    return perm;
}

}  // namespace

template <>
void wide_merge_sort<std::int16_t>(ak_ctx* c, std::int16_t* d, std::uint64_t n, bool desc) {
    auto* w = work_arena<std::int32_t>(c, 2 * n * sizeof(std::int32_t));
    widen16_kernel<<<grid_of(c), 256, 0, c->stream>>>(d, w, n);
    AKB_CUDA(cudaGetLastError());
    radix_sort<std::int32_t, std::uint32_t>(c, SORT_KEYS, w, w, w + n, nullptr, nullptr, nullptr, n, desc, true);
    narrow16_kernel<<<grid_of(c), 256, 0, c->stream>>>(w, d, n);
    AKB_CUDA(cudaGetLastError());
    c->kernel_launches += 2;
}

template <>
void wide_merge_sort<__int128>(ak_ctx* c, __int128* d, std::uint64_t n, bool desc) {
    auto* w = work_arena<std::uint64_t>(c, 6 * n * sizeof(std::uint64_t));
    std::uint64_t* perm = perm128(c, d, n, desc, w);
    auto* tmp = reinterpret_cast<__int128*>(w);  // lo/hi are dead: 2n words = n int128
    gather_kernel<__int128, std::uint64_t><<<grid_of(c), 256, 0, c->stream>>>(d, perm, tmp, n);
    AKB_CUDA(cudaGetLastError());
    AKB_CUDA(cudaMemcpyAsync(d, tmp, n * sizeof(__int128), cudaMemcpyDeviceToDevice, c->stream));
    c->kernel_launches += 1;
}

template <typename T, typename V>
void wide_by_key(ak_ctx* c, T* k, V* v, std::uint64_t n, bool desc) {
    if constexpr (sizeof(T) == 2) {
        auto* w = work_arena<std::int32_t>(c, 2 * n * sizeof(std::int32_t) + n * sizeof(V));
        auto* vs = reinterpret_cast<V*>(w + 2 * n);
        widen16_kernel<<<grid_of(c), 256, 0, c->stream>>>(k, w, n);
        AKB_CUDA(cudaGetLastError());
        radix_sort<std::int32_t, V>(c, SORT_PAIRS, w, w, w + n, v, v, vs, n, desc, true);
        narrow16_kernel<<<grid_of(c), 256, 0, c->stream>>>(w, k, n);
        AKB_CUDA(cudaGetLastError());
        c->kernel_launches += 2;
    } else {
        auto* w = work_arena<std::uint64_t>(c, 6 * n * sizeof(std::uint64_t));
        std::uint64_t* perm = perm128(c, k, n, desc, w);
        auto* tmp = reinterpret_cast<__int128*>(w);
        gather_kernel<__int128, std::uint64_t><<<grid_of(c), 256, 0, c->stream>>>(k, perm, tmp, n);
        AKB_CUDA(cudaMemcpyAsync(k, tmp, n * sizeof(__int128), cudaMemcpyDeviceToDevice, c->stream));
        auto* vt = reinterpret_cast<V*>(w + 3 * n);  // k1/k2 are dead
        gather_kernel<V, std::uint64_t><<<grid_of(c), 256, 0, c->stream>>>(v, perm, vt, n);
        AKB_CUDA(cudaMemcpyAsync(v, vt, n * sizeof(V), cudaMemcpyDeviceToDevice, c->stream));
        AKB_CUDA(cudaGetLastError());
        c->kernel_launches += 2;
    }
}

template <typename T, typename I>
void wide_sortperm(ak_ctx* c, const T* d, std::uint64_t n, I* out, bool desc) {
    if constexpr (sizeof(T) == 2) {
        auto* w = work_arena<std::int32_t>(c, (3 * n + 2) * sizeof(std::int32_t) + n * sizeof(I));
        auto* si = reinterpret_cast<I*>(w + ((3 * n + 1) & ~std::uint64_t(1)));  // 8-byte aligned
        widen16_kernel<<<grid_of(c), 256, 0, c->stream>>>(d, w, n);
        AKB_CUDA(cudaGetLastError());
        radix_sort<std::int32_t, I>(c, SORT_IOTA, w, w + n, w + 2 * n, nullptr, out, si, n, desc, false);
        c->kernel_launches += 1;
    } else {
        auto* w = work_arena<std::uint64_t>(c, 6 * n * sizeof(std::uint64_t));
        std::uint64_t* perm = perm128(c, d, n, desc, w);
        convert_kernel<I><<<grid_of(c), 256, 0, c->stream>>>(perm, out, n);
        AKB_CUDA(cudaGetLastError());
        c->kernel_launches += 1;
    }
}

template void wide_by_key<std::int16_t, std::uint32_t>(ak_ctx*, std::int16_t*, std::uint32_t*, std::uint64_t, bool);
template void wide_by_key<std::int16_t, std::uint64_t>(ak_ctx*, std::int16_t*, std::uint64_t*, std::uint64_t, bool);
template void wide_by_key<__int128, std::uint32_t>(ak_ctx*, __int128*, std::uint32_t*, std::uint64_t, bool);
template void wide_by_key<__int128, std::uint64_t>(ak_ctx*, __int128*, std::uint64_t*, std::uint64_t, bool);
template void wide_sortperm<std::int16_t, std::uint32_t>(ak_ctx*, const std::int16_t*, std::uint64_t, std::uint32_t*, bool);
template void wide_sortperm<std::int16_t, std::uint64_t>(ak_ctx*, const std::int16_t*, std::uint64_t, std::uint64_t*, bool);
template void wide_sortperm<__int128, std::uint32_t>(ak_ctx*, const __int128*, std::uint64_t, std::uint32_t*, bool);
template void wide_sortperm<__int128, std::uint64_t>(ak_ctx*, const __int128*, std::uint64_t, std::uint64_t*, bool);

}  // namespace akb
