// ak/sort.hpp -- drop-in for proj/include/ak/sort.hpp (sort.hpp:22-290) on the B200 build.
//
// Same names, parameter orders, buffer structs and required_bytes, same exceptions thrown
// before any mutation. The sorts run in libak_cuda.so and give the reference's stable merge
// sort's output exactly (ties keep input order): 64-bit integer keys-only sorts by the hybrid
// MSD partition + on-chip counting stage (equal integer keys are indistinguishable, so any
// correct order of them is the stable one), every other key type / payload sort by the
// stable LSD onesweep radix sort.
// Spans may live in host memory (staged through HBM, blocking) or in device memory
// (sorted in place; device scratch spans are used as the radix ping-pong buffers).
// Comparators: std::less<T> / std::less<> (ascending) and std::greater<T> / std::greater<>
// (descending); anything else is a compile-time error (no CPU fallback).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "ak/exec.hpp"

namespace ak {

// ---------------------------------------------------------------------------
// Caller-owned scratch (sort.hpp:22-65): required sizes are a pure function of n.
// ---------------------------------------------------------------------------
template <typename Key>
struct sort_buffers {
    std::vector<Key> scratch_keys;
    static std::size_t required_bytes(std::size_t n) { return n * sizeof(Key); }
    static sort_buffers with_capacity(std::size_t n) { return {std::vector<Key>(n)}; }
};

template <typename Key, typename Payload>
struct sort_by_key_buffers {
    std::vector<Key> scratch_keys;
    std::vector<Payload> scratch_payload;
    static std::size_t required_bytes(std::size_t n) { return n * (sizeof(Key) + sizeof(Payload)); }
    static sort_by_key_buffers with_capacity(std::size_t n) {
        return {std::vector<Key>(n), std::vector<Payload>(n)};
    }
};

template <typename Key, typename Index = std::size_t>
struct sortperm_buffers {
    std::vector<Key> working_keys;
    std::vector<Key> scratch_keys;
    std::vector<Index> scratch_index;
    static std::size_t required_bytes(std::size_t n) { return n * (2 * sizeof(Key) + sizeof(Index)); }
    static sortperm_buffers with_capacity(std::size_t n) {
        return {std::vector<Key>(n), std::vector<Key>(n), std::vector<Index>(n)};
    }
};

template <typename Index = std::size_t>
struct sortperm_lowmem_buffers {
    std::vector<Index> scratch_index;
    static std::size_t required_bytes(std::size_t n) { return n * sizeof(Index); }
    static sortperm_lowmem_buffers with_capacity(std::size_t n) { return {std::vector<Index>(n)}; }
};

namespace detail {

template <typename T>
inline constexpr bool is_key_v =
    std::is_same_v<T, std::int32_t> || std::is_same_v<T, std::uint32_t> || std::is_same_v<T, std::int64_t> ||
    std::is_same_v<T, std::uint64_t> || std::is_same_v<T, float> || std::is_same_v<T, double> ||
    std::is_same_v<T, std::int16_t> || std::is_same_v<T, __int128>;  // dtype.hpp:14-21

template <typename T, typename Cmp>
constexpr int desc_of() {
    using C = std::remove_cvref_t<Cmp>;
    if constexpr (std::is_same_v<C, std::less<T>> || std::is_same_v<C, std::less<>>) {
        return 0;
    } else if constexpr (std::is_same_v<C, std::greater<T>> || std::is_same_v<C, std::greater<>>) {
        return 1;
    } else {
        static_assert(sizeof(C) == 0,
                      "ak (B200 build): comparator must be std::less or std::greater (no CPU fallback)");
        return 0;
    }
}

// Typed C-ABI dispatch (include/ak_cuda.h), one overload set per key type.
#define AK_SORT_DISPATCH(S, T)                                                                            \
    inline int c_merge_sort(ak_ctx* c, T* d, std::uint64_t n, T* s, std::uint64_t sn, int desc) {          \
        return ak_merge_sort_##S(c, d, n, s, sn, desc);                                                  \
    }                                                                                                     \
    inline int c_merge_sort_host(ak_ctx* c, T* h, std::uint64_t n, int desc) {                            \
        return ak_merge_sort_host_##S(c, h, n, desc);                                                    \
    }                                                                                                     \
    inline int c_by_key(ak_ctx* c, T* k, std::uint64_t nk, void* p, std::uint64_t np, T* sk,             \
                        std::uint64_t skn, void* sp, std::uint64_t spn, int desc, int pbytes) {          \
        return pbytes == 4 ? ak_merge_sort_by_key_##S##_b32(c, k, nk, p, np, sk, skn, sp, spn, desc)      \
                           : ak_merge_sort_by_key_##S##_b64(c, k, nk, p, np, sk, skn, sp, spn, desc);     \
    }                                                                                                     \
    inline int c_sortperm(ak_ctx* c, const T* d, std::uint64_t n, void* o, std::uint64_t on, T* wk,      \
                          std::uint64_t wkn, T* sk, std::uint64_t skn, void* si, std::uint64_t sin,      \
                          int desc, int ibytes) {                                                        \
        return ibytes == 4 ? ak_sortperm_##S##_i32(c, d, n, static_cast<std::int32_t*>(o), on, wk, wkn,  \
                                                   sk, skn, static_cast<std::int32_t*>(si), sin, desc)   \
                           : ak_sortperm_##S##_i64(c, d, n, static_cast<std::int64_t*>(o), on, wk, wkn,  \
                                                   sk, skn, static_cast<std::int64_t*>(si), sin, desc);  \
    }                                                                                                     \
    inline int c_sortperm_lowmem(ak_ctx* c, const T* d, std::uint64_t n, void* o, std::uint64_t on,      \
                                 void* si, std::uint64_t sin, int desc, int ibytes) {                    \
        return ibytes == 4                                                                               \
                   ? ak_sortperm_lowmem_##S##_i32(c, d, n, static_cast<std::int32_t*>(o), on,             \
                                                  static_cast<std::int32_t*>(si), sin, desc)             \
                   : ak_sortperm_lowmem_##S##_i64(c, d, n, static_cast<std::int64_t*>(o), on,             \
                                                  static_cast<std::int64_t*>(si), sin, desc);            \
    }
AK_SORT_DISPATCH(i32, std::int32_t)
AK_SORT_DISPATCH(u32, std::uint32_t)
AK_SORT_DISPATCH(i64, std::int64_t)
AK_SORT_DISPATCH(u64, std::uint64_t)
AK_SORT_DISPATCH(f32, float)
AK_SORT_DISPATCH(f64, double)
AK_SORT_DISPATCH(i16, std::int16_t)
AK_SORT_DISPATCH(i128, __int128)
#undef AK_SORT_DISPATCH

template <typename T>
void require_key() {
    static_assert(is_key_v<T>,
                  "ak (B200 build): key type must be int16/int32/uint32/int64/uint64/int128/float/double");
}
template <typename V>
void require_word() {
    static_assert(std::is_trivially_copyable_v<V> && (sizeof(V) == 4 || sizeof(V) == 8),
                  "ak (B200 build): payload / index type must be a trivially copyable 4- or 8-byte type");
}

}  // namespace detail

// ---------------------------------------------------------------------------
// merge_sort (sort.hpp:180-203)
// ---------------------------------------------------------------------------
template <typename T, typename Cmp = std::less<T>>
void merge_sort(std::span<T> data, std::span<T> scratch, const exec_backend& ex, Cmp = {}) {
    detail::require_key<T>();
    constexpr int desc = detail::desc_of<T, Cmp>();
    if (scratch.size() < data.size()) throw std::invalid_argument("merge_sort: scratch buffer too small");
    if (data.size() < 2) return;
    if (detail::on_device(data.data()) && detail::on_device(scratch.data())) {
        detail::check(detail::c_merge_sort(ex.ctx(), data.data(), data.size(), scratch.data(), scratch.size(), desc));
    } else {
        detail::check(detail::c_merge_sort_host(ex.ctx(), data.data(), data.size(), desc));
    }
}

template <typename T, typename Cmp = std::less<T>>
void merge_sort(std::span<T> data, sort_buffers<T>& buffers, const exec_backend& ex, Cmp cmp = {}) {
    merge_sort(data, std::span<T>(buffers.scratch_keys), ex, cmp);
}

/// Allocating variant: a sorted copy, data untouched (sort.hpp:197-203).
template <typename T, typename Cmp = std::less<T>>
std::vector<T> merge_sort_copy(std::span<const T> data, const exec_backend& ex, Cmp cmp = {}) {
    std::vector<T> out(data.begin(), data.end());
    auto buffers = sort_buffers<T>::with_capacity(out.size());
    merge_sort(std::span<T>(out), buffers, ex, cmp);
    return out;
}

// ---------------------------------------------------------------------------
// merge_sort_by_key (sort.hpp:211-229)
// ---------------------------------------------------------------------------
template <typename K, typename V, typename Cmp = std::less<K>>
void merge_sort_by_key(std::span<K> keys, std::span<V> payload, std::span<K> scratch_keys,
                       std::span<V> scratch_payload, const exec_backend& ex, Cmp = {}) {
    detail::require_key<K>();
    detail::require_word<V>();
    constexpr int desc = detail::desc_of<K, Cmp>();
    if (keys.size() != payload.size())
        throw std::invalid_argument("merge_sort_by_key: keys and payload lengths differ");
    if (scratch_keys.size() < keys.size() || scratch_payload.size() < keys.size())
        throw std::invalid_argument("merge_sort_by_key: scratch buffers too small");
    const std::size_t n = keys.size();
    if (n < 2) return;
    ak_ctx* c = ex.ctx();
    if (detail::on_device(keys.data()) && detail::on_device(payload.data()) &&
        detail::on_device(scratch_keys.data()) && detail::on_device(scratch_payload.data())) {
        detail::check(detail::c_by_key(c, keys.data(), n, payload.data(), n, scratch_keys.data(),
                                       scratch_keys.size(), scratch_payload.data(), scratch_payload.size(), desc,
                                       static_cast<int>(sizeof(V))));
        return;
    }
    detail::device_buffer<K> dk(c, n), dsk(c, n);
    detail::device_buffer<V> dv(c, n), dsv(c, n);
    dk.upload(keys.data(), n);
    dv.upload(payload.data(), n);
    detail::check(detail::c_by_key(c, dk.p, n, dv.p, n, dsk.p, n, dsv.p, n, desc, static_cast<int>(sizeof(V))));
    dk.download(keys.data(), n);
    dv.download(payload.data(), n);
}

template <typename K, typename V, typename Cmp = std::less<K>>
void merge_sort_by_key(std::span<K> keys, std::span<V> payload, sort_by_key_buffers<K, V>& buffers,
                       const exec_backend& ex, Cmp cmp = {}) {
    merge_sort_by_key(keys, payload, std::span<K>(buffers.scratch_keys), std::span<V>(buffers.scratch_payload), ex,
                      cmp);
}

// ---------------------------------------------------------------------------
// sortperm (sort.hpp:238-262): stable permutation, equal keys with ascending indices
// ---------------------------------------------------------------------------
template <typename T, typename I = std::size_t, typename Cmp = std::less<T>>
void sortperm(std::span<const T> data, std::span<I> out, sortperm_buffers<T, I>& buffers, const exec_backend& ex,
              Cmp = {}) {
    detail::require_key<T>();
    detail::require_word<I>();
    constexpr int desc = detail::desc_of<T, Cmp>();
    const std::size_t n = data.size();
    if (out.size() != n) throw std::invalid_argument("sortperm: output length must match input length");
    if (buffers.working_keys.size() < n || buffers.scratch_keys.size() < n || buffers.scratch_index.size() < n)
        throw std::invalid_argument("sortperm: scratch buffers too small");
    if (n == 0) return;
    ak_ctx* c = ex.ctx();
    detail::device_buffer<T> dd(c, n), dwk(c, n), dsk(c, n);
    detail::device_buffer<I> dout(c, n), dsi(c, n);
    dd.upload(data.data(), n);
    detail::check(detail::c_sortperm(c, dd.p, n, dout.p, n, dwk.p, n, dsk.p, n, dsi.p, n, desc,
                                     static_cast<int>(sizeof(I))));
    dout.download(out.data(), n);
}

/// Device-resident variant: every span in HBM, caller-owned device scratch.
template <typename T, typename I, typename Cmp = std::less<T>>
void sortperm(std::span<const T> data, std::span<I> out, std::span<T> working_keys, std::span<T> scratch_keys,
              std::span<I> scratch_index, const exec_backend& ex, Cmp = {}) {
    detail::require_key<T>();
    detail::require_word<I>();
    constexpr int desc = detail::desc_of<T, Cmp>();
    const std::size_t n = data.size();
    if (out.size() != n) throw std::invalid_argument("sortperm: output length must match input length");
    if (working_keys.size() < n || scratch_keys.size() < n || scratch_index.size() < n)
        throw std::invalid_argument("sortperm: scratch buffers too small");
    if (n == 0) return;
    detail::check(detail::c_sortperm(ex.ctx(), data.data(), n, out.data(), n, working_keys.data(),
                                     working_keys.size(), scratch_keys.data(), scratch_keys.size(),
                                     scratch_index.data(), scratch_index.size(), desc, static_cast<int>(sizeof(I))));
}

template <typename T, typename I = std::size_t, typename Cmp = std::less<T>>
std::vector<I> sortperm(std::span<const T> data, const exec_backend& ex, Cmp cmp = {}) {
    std::vector<I> out(data.size());
    auto buffers = sortperm_buffers<T, I>::with_capacity(data.size());
    sortperm(data, std::span<I>(out), buffers, ex, cmp);
    return out;
}

/// Low-memory variant (sort.hpp:267-290): scratch is one index array.
template <typename T, typename I = std::size_t, typename Cmp = std::less<T>>
void sortperm_lowmem(std::span<const T> data, std::span<I> out, sortperm_lowmem_buffers<I>& buffers,
                     const exec_backend& ex, Cmp = {}) {
    detail::require_key<T>();
    detail::require_word<I>();
    constexpr int desc = detail::desc_of<T, Cmp>();
    const std::size_t n = data.size();
    if (out.size() != n) throw std::invalid_argument("sortperm_lowmem: output length must match input length");
    if (buffers.scratch_index.size() < n) throw std::invalid_argument("sortperm_lowmem: scratch buffer too small");
    if (n == 0) return;
    ak_ctx* c = ex.ctx();
    if (detail::on_device(data.data()) && detail::on_device(out.data()) &&
        detail::on_device(buffers.scratch_index.data())) {
        detail::check(detail::c_sortperm_lowmem(c, data.data(), n, out.data(), n, buffers.scratch_index.data(),
                                                buffers.scratch_index.size(), desc, static_cast<int>(sizeof(I))));
        return;
    }
    detail::device_buffer<T> dd(c, n);
    detail::device_buffer<I> dout(c, n), dsi(c, n);
    dd.upload(data.data(), n);
    detail::check(detail::c_sortperm_lowmem(c, dd.p, n, dout.p, n, dsi.p, n, desc, static_cast<int>(sizeof(I))));
    dout.download(out.data(), n);
}

template <typename T, typename I = std::size_t, typename Cmp = std::less<T>>
std::vector<I> sortperm_lowmem(std::span<const T> data, const exec_backend& ex, Cmp cmp = {}) {
    std::vector<I> out(data.size());
    auto buffers = sortperm_lowmem_buffers<I>::with_capacity(data.size());
    sortperm_lowmem(data, std::span<I>(out), buffers, ex, cmp);
    return out;
}

}  // namespace ak
