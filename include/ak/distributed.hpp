// ak/distributed.hpp -- multi-rank reduce and scan, B200 build.
//
// The reference's reduce/accumulate are single-process (reduce.hpp, scan.hpp). These run
// over the same communicators as sihsort (ak::sim::rank_comm on one GPU, ak::nccl::rank_comm
// one rank per GPU): every rank reduces its slice on the device, the P rank partials are
// allgathered and folded in rank order, and accumulate_all seeds each rank's local scan with
// init and the totals of the lower ranks -- so rank r returns its slice of the scan of the
// concatenation of all ranks' data in rank order. Collective; init must be neutral for
// reduce_all (reduce.hpp:12-14).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "ak/reduce.hpp"
#include "ak/scan.hpp"
#include "ak/sim_comm.hpp"

namespace ak {

namespace detail {
#define AK_DIST_DISPATCH(S, T)                                                                                  \
    inline int c_reduce_all(ak_ctx* c, ak_comm* cm, const T* x, std::uint64_t n, int op, int map, T init, T* r) { \
        return ak_reduce_all_##S(c, cm, x, n, op, map, init, r);                                               \
    }                                                                                                           \
    inline int c_accumulate_all(ak_ctx* c, ak_comm* cm, const T* x, std::uint64_t n, T* o, std::uint64_t on,     \
                                int op, int inc, T init) {                                                      \
        return ak_accumulate_all_##S(c, cm, x, n, o, on, op, inc, init);                                       \
    }
AK_DIST_DISPATCH(i32, std::int32_t)
AK_DIST_DISPATCH(u32, std::uint32_t)
AK_DIST_DISPATCH(i64, std::int64_t)
AK_DIST_DISPATCH(u64, std::uint64_t)
AK_DIST_DISPATCH(f32, float)
AK_DIST_DISPATCH(f64, double)
#undef AK_DIST_DISPATCH
}  // namespace detail

template <typename T, typename Op, typename Comm>
T reduce_all(Op, std::span<const T> data, const reduce_config<T>& cfg, Comm& comm, const exec_backend& ex) {
    detail::require_key<T>();
    T r{};
    ak_ctx* c = ex.ctx();
    if (data.empty() || detail::on_device(data.data())) {
        detail::check(detail::c_reduce_all(c, comm.handle(), data.data(), data.size(), detail::op_code<T, Op>(), 0,
                                           cfg.init, &r));
    } else {
        detail::device_buffer<T> d(c, data.size());
        d.upload(data.data(), data.size());
        detail::check(detail::c_reduce_all(c, comm.handle(), d.p, data.size(), detail::op_code<T, Op>(), 0, cfg.init, &r));
    }
    return r;
}

template <typename T, typename Op, typename Comm>
void accumulate_all(Op, std::span<const T> data, const scan_spec<T>& spec, Comm& comm, const exec_backend& ex,
                    std::span<T> out) {
    detail::require_key<T>();
    if (out.size() != data.size()) throw std::invalid_argument("accumulate: output length must match input length");
    if (spec.chunk_size == 0) throw std::invalid_argument("accumulate: chunk_size must be >= 1");
    const int inc = spec.mode == scan_mode::inclusive ? 1 : 0;
    ak_ctx* c = ex.ctx();
    const std::size_t n = data.size();
    if (n == 0 || (detail::on_device(data.data()) && detail::on_device(out.data()))) {
        detail::check(detail::c_accumulate_all(c, comm.handle(), data.data(), n, out.data(), n,
                                               detail::op_code<T, Op>(), inc, spec.init));
        return;
    }
    detail::device_buffer<T> d(c, n);
    d.upload(data.data(), n);
    detail::check(detail::c_accumulate_all(c, comm.handle(), d.p, n, d.p, n, detail::op_code<T, Op>(), inc, spec.init));
    d.download(out.data(), n);
}

template <typename T, typename Op, typename Comm>
std::vector<T> accumulate_all(Op op, std::span<const T> data, const scan_spec<T>& spec, Comm& comm,
                              const exec_backend& ex) {
    std::vector<T> out(data.size());
    accumulate_all(op, data, spec, comm, ex, std::span<T>(out));
    return out;
}

}  // namespace ak
