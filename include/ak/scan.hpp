// ak/scan.hpp -- drop-in for proj/include/ak/scan.hpp (scan.hpp:12-88), B200 build.
//
// accumulate runs libak_cuda.so's single-pass decoupled look-back scan (K2). out may
// alias data (in place). Integer scans are exact (association-independent); float scans
// carry in double, so they match an f64 prefix to ~1e-7 relative and the reference's
// chunked float result within its 1e-5 contract. chunk_size is validated
// (>= 1, scan.hpp:35-37) but does not change integer results.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "ak/exec.hpp"
#include "ak/reduce.hpp"

namespace ak {

enum class scan_mode { inclusive, exclusive };

template <typename T>
struct scan_spec {
    scan_mode mode = scan_mode::inclusive;
    T init{};
    std::size_t chunk_size = 4096;
};

namespace detail {
#define AK_SCAN_DISPATCH(S, T)                                                                              \
    inline int c_accumulate(ak_ctx* c, const T* x, std::uint64_t n, T* o, std::uint64_t on, int op, int inc, \
                            T init, std::uint64_t chunk) {                                                  \
        return ak_accumulate_##S(c, x, n, o, on, op, inc, init, chunk);                                     \
    }
AK_SCAN_DISPATCH(i32, std::int32_t)
AK_SCAN_DISPATCH(u32, std::uint32_t)
AK_SCAN_DISPATCH(i64, std::int64_t)
AK_SCAN_DISPATCH(u64, std::uint64_t)
AK_SCAN_DISPATCH(f32, float)
AK_SCAN_DISPATCH(f64, double)
#undef AK_SCAN_DISPATCH
}  // namespace detail

/// Prefix scan of data into out (same length; may alias data) (scan.hpp:29-79).
template <typename T, typename Op>
void accumulate(Op, std::span<const T> data, const scan_spec<T>& spec, const exec_backend& ex, std::span<T> out) {
    detail::require_key<T>();
    constexpr int op = detail::op_code<T, Op>();
    if (out.size() != data.size()) throw std::invalid_argument("accumulate: output length must match input length");
    if (spec.chunk_size == 0) throw std::invalid_argument("accumulate: chunk_size must be >= 1");
    const std::size_t n = data.size();
    if (n == 0) return;
    const int inc = spec.mode == scan_mode::inclusive ? 1 : 0;
    ak_ctx* c = ex.ctx();
    if (detail::on_device(data.data()) && detail::on_device(out.data())) {
        detail::check(detail::c_accumulate(c, data.data(), n, out.data(), n, op, inc, spec.init, spec.chunk_size));
        return;
    }
    detail::device_buffer<T> d(c, n);
    d.upload(data.data(), n);
    detail::check(detail::c_accumulate(c, d.p, n, d.p, n, op, inc, spec.init, spec.chunk_size));
    d.download(out.data(), n);
}

/// Allocating variant (scan.hpp:82-88).
template <typename T, typename Op>
std::vector<T> accumulate(Op op, std::span<const T> data, const scan_spec<T>& spec, const exec_backend& ex) {
    std::vector<T> out(data.size());
    accumulate(op, data, spec, ex, std::span<T>(out));
    return out;
}

}  // namespace ak
