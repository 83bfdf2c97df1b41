// ak/predicates.hpp -- drop-in for proj/include/ak/predicates.hpp (predicates.hpp:16-78), B200 build.
//
// any_pred / all_pred run one device pass (early_exit polls a device flag per block trip and
// stops once decided; via_mapreduce always scans everything -- identical results, as in the
// reference). The predicate cannot cross the C ABI as a lambda: it is one of the comparison
// functors below (x < v, x <= v, x > v, x >= v, x == v, x != v), a compile-time error otherwise.
#pragma once

#include <cstdint>
#include <span>
#include <type_traits>

#include "ak/exec.hpp"

namespace ak {

enum class predicate_algo { early_exit, via_mapreduce };

/// Comparison predicates recognised on the device: ak::pred::gt<int>{0} is x > 0.
namespace pred {
template <typename T> struct lt { T v; constexpr bool operator()(T x) const { return x < v; } };
template <typename T> struct le { T v; constexpr bool operator()(T x) const { return x <= v; } };
template <typename T> struct gt { T v; constexpr bool operator()(T x) const { return x > v; } };
template <typename T> struct ge { T v; constexpr bool operator()(T x) const { return x >= v; } };
template <typename T> struct eq { T v; constexpr bool operator()(T x) const { return x == v; } };
template <typename T> struct ne { T v; constexpr bool operator()(T x) const { return x != v; } };
}  // namespace pred

namespace detail {

template <typename P>
struct pred_code;
template <typename T> struct pred_code<pred::lt<T>> { static constexpr int op = 0; };
template <typename T> struct pred_code<pred::le<T>> { static constexpr int op = 1; };
template <typename T> struct pred_code<pred::gt<T>> { static constexpr int op = 2; };
template <typename T> struct pred_code<pred::ge<T>> { static constexpr int op = 3; };
template <typename T> struct pred_code<pred::eq<T>> { static constexpr int op = 4; };
template <typename T> struct pred_code<pred::ne<T>> { static constexpr int op = 5; };

template <typename P, typename = void>
struct is_device_pred : std::false_type {};
template <typename P>
struct is_device_pred<P, std::void_t<decltype(pred_code<P>::op)>> : std::true_type {};

#define AK_PRED_DISPATCH(S, T)                                                                             \
    inline int c_pred(bool any, ak_ctx* c, const T* x, std::uint64_t n, int op, T v, int algo, int* r) {   \
        return any ? ak_any_pred_##S(c, x, n, op, v, algo, r) : ak_all_pred_##S(c, x, n, op, v, algo, r); \
    }
AK_PRED_DISPATCH(u8, std::uint8_t)
AK_PRED_DISPATCH(i8, std::int8_t)
AK_PRED_DISPATCH(i16, std::int16_t)
AK_PRED_DISPATCH(i32, std::int32_t)
AK_PRED_DISPATCH(u32, std::uint32_t)
AK_PRED_DISPATCH(i64, std::int64_t)
AK_PRED_DISPATCH(u64, std::uint64_t)
AK_PRED_DISPATCH(f32, float)
AK_PRED_DISPATCH(f64, double)
#undef AK_PRED_DISPATCH

template <typename T, typename Pred>
bool run_pred(bool any, std::span<const T> data, const Pred& p, const exec_backend& ex, predicate_algo algo) {
    using P = std::remove_cvref_t<Pred>;
    static_assert(is_device_pred<P>::value,
                  "ak (B200 build): predicate must be ak::pred::{lt,le,gt,ge,eq,ne}<T>{value}");
    int r = 0;
    const int a = algo == predicate_algo::early_exit ? 0 : 1;
    const T v = static_cast<T>(p.v);
    if (data.empty() || on_device(data.data())) {
        check(c_pred(any, ex.ctx(), data.data(), data.size(), pred_code<P>::op, v, a, &r));
    } else {
        device_buffer<T> d(ex.ctx(), data.size());
        d.upload(data.data(), data.size());
        check(c_pred(any, ex.ctx(), d.p, data.size(), pred_code<P>::op, v, a, &r));
    }
    return r != 0;
}

}  // namespace detail

/// True iff pred holds for at least one element; empty data yields false (predicates.hpp:57).
template <typename T, typename Pred>
bool any_pred(std::span<const T> data, Pred pred, const exec_backend& ex,
              predicate_algo algo = predicate_algo::early_exit) {
    return detail::run_pred<T>(true, data, pred, ex, algo);
}

/// True iff pred holds for every element; empty data yields true (predicates.hpp:69).
template <typename T, typename Pred>
bool all_pred(std::span<const T> data, Pred pred, const exec_backend& ex,
              predicate_algo algo = predicate_algo::early_exit) {
    return detail::run_pred<T>(false, data, pred, ex, algo);
}

}  // namespace ak
