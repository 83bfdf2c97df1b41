// ak/sihsort.hpp -- drop-in for proj/include/ak/sihsort.hpp (sihsort.hpp:21-569), B200 build.
//
// sihsort() runs the reference protocol rank by rank (config check, local sort, sampling,
// distributed equal-width histogram, interpolated splitters, exact-count refinement,
// redistribution, local merge) with the keys resident in HBM: libak_cuda.so radix-sorts,
// gathers samples, searches bucket bounds and merges on the device, NCCL (or the
// single-GPU loopback world) moves the slices, and the long-double splitter math runs on
// the host exactly as the reference's, so per-rank outputs and sih_stats match it.
//
// Communicators: ak::sim::rank_comm (P logical ranks on one GPU, run_ranks) or
// ak::nccl::rank_comm (one rank per GPU). The reference's pluggable Sorter overload
// (sihsort.hpp:508) accepts ak::cuda_sorter, the library's device sorter; a host callable
// cannot run inside the device pipeline and is rejected at compile time.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <type_traits>
#include <utility>
#include <vector>

#include "ak/exec.hpp"
#include "ak/search.hpp"
#include "ak/sim_comm.hpp"
#include "ak/sort.hpp"

namespace ak {

/// sihsort.hpp:21-26: zero = derive from the world size (32P samples, 8P bins).
struct sih_config {
    std::size_t sample_per_rank = 0;
    std::size_t bins = 0;
    std::size_t max_refine_rounds = 4;
    double imbalance_tol = 0.25;
};

/// sihsort.hpp:45-53 (redistribution_bytes keeps the reference's piggyback accounting).
struct sih_stats {
    std::size_t rounds_used = 0;
    bool converged = false;
    double max_deviation = 0.0;
    std::uint64_t redistribution_sends = 0;
    std::uint64_t redistribution_bytes = 0;
    std::uint64_t collective_ops = 0;
    std::uint64_t output_count = 0;
};

/// The library's device sorter, usable in the Sorter slot.
struct cuda_sorter {};

namespace detail {

#define AK_SIH_DISPATCH(S, T)                                                                                 \
    inline int c_sihsort_host(ak_ctx* c, ak_comm* cm, const T* in, std::uint64_t n, T* out, std::uint64_t cap, \
                              std::uint64_t* cnt, const ak_sih_config* cfg, ak_sih_stats* st) {               \
        return ak_sihsort_host_##S(c, cm, in, n, out, cap, cnt, cfg, st);                                     \
    }                                                                                                         \
    inline int c_sihsort(ak_ctx* c, ak_comm* cm, const T* in, std::uint64_t n, T* out, std::uint64_t cap,      \
                         std::uint64_t* cnt, const ak_sih_config* cfg, ak_sih_stats* st) {                    \
        return ak_sihsort_##S(c, cm, in, n, out, cap, cnt, cfg, st);                                          \
    }
AK_SIH_DISPATCH(i32, std::int32_t)
AK_SIH_DISPATCH(u32, std::uint32_t)
AK_SIH_DISPATCH(i64, std::int64_t)
AK_SIH_DISPATCH(u64, std::uint64_t)
AK_SIH_DISPATCH(f32, float)
AK_SIH_DISPATCH(f64, double)
#undef AK_SIH_DISPATCH

inline ak_sih_config to_c(const sih_config& c) {
    return ak_sih_config{c.sample_per_rank, c.bins, c.max_refine_rounds, c.imbalance_tol};
}
inline sih_stats from_c(const ak_sih_stats& s) {
    sih_stats o;
    o.rounds_used = s.rounds_used;
    o.converged = s.converged != 0;
    o.max_deviation = s.max_deviation;
    o.redistribution_sends = s.redistribution_sends;
    o.redistribution_bytes = s.redistribution_bytes;
    o.collective_ops = s.collective_ops;
    o.output_count = s.output_count;
    return o;
}

}  // namespace detail

/// Distributed sampling sort over the communicator's P ranks (sihsort.hpp:508-559):
/// afterwards the concatenation of the returned arrays in rank order is globally sorted
/// and the global multiset is preserved. Collective: every rank calls with the same cfg.
template <typename T, typename Comm>
std::pair<std::vector<T>, sih_stats> sihsort(std::vector<T> local_data, Comm& comm, const sih_config& cfg,
                                             const exec_backend& ex) {
    detail::require_key<T>();
    const ak_sih_config c = detail::to_c(cfg);
    ak_sih_stats st{};
    const std::uint64_t n = local_data.size();
    // keys go to HBM once; the output is sized on the device and copied back at its exact length
    detail::device_buffer<T> din(ex.ctx(), n);
    din.upload(local_data.data(), n);
    std::uint64_t cap = n + n / 4 + 4096;
    std::uint64_t count = 0;
    for (;;) {
        detail::device_buffer<T> dout(ex.ctx(), cap);
        const int rc = detail::c_sihsort(ex.ctx(), comm.handle(), din.p, n, dout.p, cap, &count, &c, &st);
        if (rc == AK_ECAPACITY) {  // raised on every rank together: all retry with room
            cap = (count > cap ? count : cap) + cap / 8 + 4096;
            continue;
        }
        detail::check(rc, count);
        std::vector<T> out(count);
        dout.download(out.data(), count);
        return {std::move(out), detail::from_c(st)};
    }
}

/// Sorter-slot overload (sihsort.hpp:508): ak::cuda_sorter selects the device pipeline.
template <typename T, typename Comm, typename Sorter>
std::pair<std::vector<T>, sih_stats> sihsort(std::vector<T> local_data, Comm& comm, const sih_config& cfg,
                                             const exec_backend& ex, Sorter&&) {
    static_assert(std::is_same_v<std::remove_cvref_t<Sorter>, cuda_sorter>,
                  "ak (B200 build): the local sorter runs on the device; pass ak::cuda_sorter{}");
    return sihsort<T>(std::move(local_data), comm, cfg, ex);
}

/// Device-resident variant: input stays in HBM, output written to a caller device buffer of
/// `capacity` elements; returns the element count (throws ak::capacity_error with the
/// required count when too small -- on every rank together).
template <typename T, typename Comm>
std::uint64_t sihsort_device(std::span<const T> local_data, std::span<T> out, Comm& comm, const sih_config& cfg,
                             const exec_backend& ex, sih_stats* stats = nullptr) {
    detail::require_key<T>();
    const ak_sih_config c = detail::to_c(cfg);
    ak_sih_stats st{};
    std::uint64_t count = 0;
    detail::check(detail::c_sihsort(ex.ctx(), comm.handle(), local_data.data(), local_data.size(), out.data(),
                                    out.size(), &count, &c, &st),
                  count);
    if (stats) *stats = detail::from_c(st);
    return count;
}

}  // namespace ak
