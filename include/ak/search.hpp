// ak/search.hpp -- drop-in for proj/include/ak/search.hpp (search.hpp:16-50), B200 build.
//
// searchsorted runs libak_cuda.so's batched binary search (K5): one insertion index per
// needle, first = #elements < v, last = #elements <= v. validate runs the O(n) device
// sortedness check and throws std::invalid_argument before searching (search.hpp:40-43).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <vector>

#include "ak/exec.hpp"
#include "ak/sort.hpp"

namespace ak {

enum class search_side { first, last };

namespace detail {
#define AK_SEARCH_DISPATCH(S, T)                                                                           \
    inline int c_searchsorted(ak_ctx* c, const T* h, std::uint64_t n, const T* nd, std::uint64_t m, int last, \
                              int desc, int validate, std::uint64_t* out) {                                \
        return ak_searchsorted_##S(c, h, n, nd, m, last, desc, validate, out);                             \
    }
AK_SEARCH_DISPATCH(i32, std::int32_t)
AK_SEARCH_DISPATCH(u32, std::uint32_t)
AK_SEARCH_DISPATCH(i64, std::int64_t)
AK_SEARCH_DISPATCH(u64, std::uint64_t)
AK_SEARCH_DISPATCH(f32, float)
AK_SEARCH_DISPATCH(f64, double)
#undef AK_SEARCH_DISPATCH
}  // namespace detail

/// Batched binary search (search.hpp:36-50). The haystack must be nondecreasing under cmp.
template <typename T, typename Cmp = std::less<T>>
std::vector<std::size_t> searchsorted(std::span<const T> haystack, std::span<const T> needles, search_side side,
                                      const exec_backend& ex, Cmp = {}, bool validate = false) {
    detail::require_key<T>();
    constexpr int desc = detail::desc_of<T, Cmp>();
    const std::size_t n = haystack.size(), m = needles.size();
    std::vector<std::size_t> out(m);
    ak_ctx* c = ex.ctx();
    const int last = side == search_side::last ? 1 : 0;
    detail::device_buffer<std::uint64_t> dres(c, m);
    const bool dev = detail::on_device(haystack.data()) && detail::on_device(needles.data());
    if (dev || (n == 0 && m == 0)) {
        detail::check(detail::c_searchsorted(c, haystack.data(), n, needles.data(), m, last, desc, validate ? 1 : 0,
                                             dres.p));
    } else {
        detail::device_buffer<T> dh(c, n), dn(c, m);
        dh.upload(haystack.data(), n);
        dn.upload(needles.data(), m);
        detail::check(detail::c_searchsorted(c, dh.p, n, dn.p, m, last, desc, validate ? 1 : 0, dres.p));
    }
    static_assert(sizeof(std::size_t) == sizeof(std::uint64_t));
    dres.download(reinterpret_cast<std::uint64_t*>(out.data()), m);
    return out;
}

/// Count of elements < v (search.hpp:19-23), on the default device.
template <typename T, typename Cmp = std::less<T>>
std::size_t search_first(std::span<const T> haystack, const T& v, Cmp cmp = {}) {
    return searchsorted(haystack, std::span<const T>(&v, 1), search_side::first, detail::default_backend(), cmp)[0];
}

/// Count of elements <= v (search.hpp:26-30), on the default device.
template <typename T, typename Cmp = std::less<T>>
std::size_t search_last(std::span<const T> haystack, const T& v, Cmp cmp = {}) {
    return searchsorted(haystack, std::span<const T>(&v, 1), search_side::last, detail::default_backend(), cmp)[0];
}

}  // namespace ak
