// ak/reduce.hpp -- drop-in for proj/include/ak/reduce.hpp (reduce.hpp:15-75), B200 build.
//
// reduce/mapreduce run libak_cuda.so's single-pass K1 kernel. The operator and map cannot
// cross a C ABI, so they are recognised by type: ak::plus / std::plus (sum), ak::minimum,
// ak::maximum (min/max); maps ak::identity / ak::absolute / ak::square. Any other callable
// is a compile-time error (no CPU fallback). Integers fold with two's-complement wrap
// (exact); float folds accumulate in double. init is folded exactly once; the reference's
// contract is that init is neutral (reduce.hpp:12-14), under which both agree.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <span>
#include <type_traits>
#include <vector>

#include "ak/exec.hpp"
#include "ak/sort.hpp"

namespace ak {

template <typename T>
struct reduce_config {
    T init{};
    std::size_t switch_below = 256;  // accepted for source compatibility; single-pass on the GPU
};

/// Named operators the device path recognises.
struct plus {
    template <typename A, typename B>
    constexpr auto operator()(A a, B b) const {
        return a + b;
    }
};
struct minimum {
    template <typename A>
    constexpr A operator()(A a, A b) const {
        return b < a ? b : a;
    }
};
struct maximum {
    template <typename A>
    constexpr A operator()(A a, A b) const {
        return a < b ? b : a;
    }
};
/// Named maps for mapreduce.
struct identity {
    template <typename A>
    constexpr A operator()(A a) const {
        return a;
    }
};
struct absolute {
    template <typename A>
    constexpr A operator()(A a) const {
        return a < A(0) ? -a : a;
    }
};
struct square {
    template <typename A>
    constexpr A operator()(A a) const {
        return a * a;
    }
};

namespace detail {

template <typename T, typename Op>
constexpr int op_code() {
    using O = std::remove_cvref_t<Op>;
    if constexpr (std::is_same_v<O, ak::plus> || std::is_same_v<O, std::plus<T>> || std::is_same_v<O, std::plus<>>) {
        return 0;
    } else if constexpr (std::is_same_v<O, ak::minimum>) {
        return 1;
    } else if constexpr (std::is_same_v<O, ak::maximum>) {
        return 2;
    } else {
        static_assert(sizeof(O) == 0,
                      "ak (B200 build): operator must be ak::plus/std::plus, ak::minimum or ak::maximum");
        return 0;
    }
}

template <typename F>
constexpr int map_code() {
    using M = std::remove_cvref_t<F>;
    if constexpr (std::is_same_v<M, ak::identity> || std::is_same_v<M, std::identity>) {
        return 0;
    } else if constexpr (std::is_same_v<M, ak::absolute>) {
        return 1;
    } else if constexpr (std::is_same_v<M, ak::square>) {
        return 2;
    } else {
        static_assert(sizeof(M) == 0, "ak (B200 build): map must be ak::identity, ak::absolute or ak::square");
        return 0;
    }
}

#define AK_RED_DISPATCH(S, T)                                                                         \
    inline int c_reduce(ak_ctx* c, const T* x, std::uint64_t n, int op, int map, T init, T* r) {      \
        return ak_reduce_##S(c, x, n, op, map, init, r);                                             \
    }
AK_RED_DISPATCH(i32, std::int32_t)
AK_RED_DISPATCH(u32, std::uint32_t)
AK_RED_DISPATCH(i64, std::int64_t)
AK_RED_DISPATCH(u64, std::uint64_t)
AK_RED_DISPATCH(f32, float)
AK_RED_DISPATCH(f64, double)
#undef AK_RED_DISPATCH

template <typename T>
T reduce_dispatch(int op, int map, std::span<const T> data, const T& init, const exec_backend& ex) {
    require_key<T>();
    if (data.empty()) return init;
    T result{};
    ak_ctx* c = ex.ctx();
    if (on_device(data.data())) {
        check(c_reduce(c, data.data(), data.size(), op, map, init, &result));
    } else {
        device_buffer<T> d(c, data.size());
        d.upload(data.data(), data.size());
        check(c_reduce(c, d.p, data.size(), op, map, init, &result));
    }
    return result;
}

}  // namespace detail

/// Folds init with all elements under op (reduce.hpp:62-66). Empty data returns init.
template <typename T, typename Op>
T reduce(Op, std::span<const T> data, const reduce_config<T>& cfg, const exec_backend& ex) {
    return detail::reduce_dispatch<T>(detail::op_code<T, Op>(), 0, data, cfg.init, ex);
}

/// reduce over f(element) without materialising the mapped array (reduce.hpp:70-75).
/// The mapped type R must equal the element type T on the device path.
template <typename R, typename T, typename F, typename Op>
R mapreduce(F, Op, std::span<const T> data, const reduce_config<R>& cfg, const exec_backend& ex) {
    static_assert(std::is_same_v<R, T>, "ak (B200 build): mapreduce result type must equal the element type");
    return detail::reduce_dispatch<T>(detail::op_code<T, Op>(), detail::map_code<F>(), data, cfg.init, ex);
}

}  // namespace ak
