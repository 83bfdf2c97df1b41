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
#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <tuple>
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

/// sihsort.hpp:28-34: equal-width histogram over the sampled key range (long double edges).
struct key_histogram {
    std::vector<long double> bin_edges;  // K+1 (single bin when degenerate)
    std::vector<std::uint64_t> counts;   // K
    std::uint64_t total = 0;
};

/// sihsort.hpp:36-42: P-1 nondecreasing splitters; keys equal to a splitter go to the lower rank.
template <typename T>
struct splitter_set {
    std::vector<T> values;
};

/// sihsort.hpp:351-357.
template <typename T>
struct refine_result {
    splitter_set<T> splitters;
    std::size_t rounds_used = 0;
    bool converged = false;
    double max_deviation = 0.0;
};

namespace detail {

#define AK_STAGE_DISPATCH(S, T)                                                                                  \
    inline int c_sample_local(ak_ctx* c, const T* d, std::uint64_t n, std::uint64_t k, T* h, std::uint64_t* cnt) {  \
        return ak_sample_local_##S(c, d, n, k, h, cnt);                                                          \
    }                                                                                                            \
    inline int c_histogram(const T* smp, std::uint64_t m, std::uint64_t bins, long double* e, std::uint64_t* cts,    \
                           std::uint64_t cap, std::uint64_t* nb, std::uint64_t* tot) {                            \
        return ak_build_interpolated_histogram_##S(smp, m, bins, e, cts, cap, nb, tot);                          \
    }                                                                                                            \
    inline int c_select(const long double* e, const std::uint64_t* cts, std::uint64_t nb, std::uint64_t tot,       \
                        std::uint64_t world, T* out) {                                                           \
        return ak_select_splitters_##S(e, cts, nb, tot, world, out);                                             \
    }                                                                                                            \
    inline int c_refine(ak_ctx* c, ak_comm* cm, const T* d, std::uint64_t n, T* spl, std::uint64_t m,              \
                        const ak_sih_config* cfg, std::uint64_t* rounds, int* conv, double* dev) {               \
        return ak_refine_splitters_##S(c, cm, d, n, spl, m, cfg, rounds, conv, dev);                             \
    }                                                                                                            \
    inline int c_redistribute(ak_ctx* c, ak_comm* cm, const T* d, std::uint64_t n, const T* spl, std::uint64_t m,  \
                              std::uint64_t nt, T* out, std::uint64_t cap, std::uint64_t* oc) {                  \
        return ak_redistribute_##S(c, cm, d, n, spl, m, nt, out, cap, oc, nullptr, nullptr);                     \
    }
AK_STAGE_DISPATCH(i32, std::int32_t)
AK_STAGE_DISPATCH(u32, std::uint32_t)
AK_STAGE_DISPATCH(i64, std::int64_t)
AK_STAGE_DISPATCH(u64, std::uint64_t)
AK_STAGE_DISPATCH(f32, float)
AK_STAGE_DISPATCH(f64, double)
#undef AK_STAGE_DISPATCH

/// A span's keys in HBM: the span itself when it is device memory, else a staged copy.
template <typename T>
struct device_view {
    device_buffer<T> staged;
    const T* p;
    device_view(ak_ctx* c, std::span<const T> s) : staged(c, on_device(s.data()) ? 0 : s.size()), p(s.data()) {
        if (!on_device(s.data())) {
            staged.upload(s.data(), s.size());
            p = staged.p;
        }
    }
};

#define AK_SIH_DISPATCH(S, T)                                                                                 \
    inline int c_sihsort_host(ak_ctx* c, ak_comm* cm, const T* in, std::uint64_t n, T* out, std::uint64_t cap, \
                              std::uint64_t* cnt, const ak_sih_config* cfg, ak_sih_stats* st) {               \
        return ak_sihsort_host_##S(c, cm, in, n, out, cap, cnt, cfg, st);                                     \
    }                                                                                                         \
    inline int c_sihsort(ak_ctx* c, ak_comm* cm, const T* in, std::uint64_t n, T* out, std::uint64_t cap,      \
                         std::uint64_t* cnt, const ak_sih_config* cfg, ak_sih_stats* st) {                    \
        return ak_sihsort_##S(c, cm, in, n, out, cap, cnt, cfg, st);                                          \
    }                                                                                                         \
    inline int c_sihsort_perm(ak_ctx* c, ak_comm* cm, const T* in, std::uint64_t n, T* out,                  \
                              std::uint64_t* idx, std::uint64_t cap, std::uint64_t* cnt,                     \
                              const ak_sih_config* cfg, ak_sih_stats* st) {                                  \
        return ak_sihsort_perm_##S(c, cm, in, n, out, idx, cap, cnt, cfg, st);                                \
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

/// Distributed sortperm (an extension: the reference's sihsort is keys-only,
/// sihsort.hpp:472-501). Rank r's key i has global index (sum of the lower ranks' sizes) + i;
/// returns this rank's slice of the globally STABLE order as (keys, global indices): the
/// ranks' results concatenated are the sorted keys and the global sortperm. Collective.
template <typename T, typename Comm>
std::tuple<std::vector<T>, std::vector<std::uint64_t>, sih_stats> sihsort_perm(std::span<const T> local_data,
                                                                              Comm& comm, const sih_config& cfg,
                                                                              const exec_backend& ex) {
    detail::require_key<T>();
    const ak_sih_config c = detail::to_c(cfg);
    ak_sih_stats st{};
    const std::uint64_t n = local_data.size();
    detail::device_view<T> din(ex.ctx(), local_data);
    std::uint64_t cap = n + n / 4 + 4096;
    std::uint64_t count = 0;
    for (;;) {
        detail::device_buffer<T> dout(ex.ctx(), cap);
        detail::device_buffer<std::uint64_t> didx(ex.ctx(), cap);
        const int rc =
            detail::c_sihsort_perm(ex.ctx(), comm.handle(), din.p, n, dout.p, didx.p, cap, &count, &c, &st);
        if (rc == AK_ECAPACITY) {  // raised on every rank together: all retry with room
            cap = (count > cap ? count : cap) + cap / 8 + 4096;
            continue;
        }
        detail::check(rc, count);
        std::vector<T> keys(count);
        std::vector<std::uint64_t> idx(count);
        dout.download(keys.data(), count);
        didx.download(idx.data(), count);
        return {std::move(keys), std::move(idx), detail::from_c(st)};
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

// ---- stage functions (sihsort.hpp:264-501); sorted spans may be host or device memory ----

/// k evenly spaced order statistics of a sorted local array (sihsort.hpp:264-282): positions
/// round-half-up(j(n-1)/(k-1)), k = 1 probes n/2, k clamps to n; gathered on the device.
template <typename T>
std::vector<T> sample_local(std::span<const T> sorted_local, std::size_t k,
                            const exec_backend& ex = detail::default_backend()) {
    detail::require_key<T>();
    const std::size_t n = sorted_local.size();
    if (n == 0 || k == 0) return {};
    std::vector<T> out(std::min(k, n));
    detail::device_view<T> d(ex.ctx(), sorted_local);
    std::uint64_t cnt = 0;
    detail::check(detail::c_sample_local(ex.ctx(), d.p, n, k, out.data(), &cnt));
    out.resize(cnt);
    return out;
}

/// Equal-width histogram of gathered samples over [min, max] (sihsort.hpp:286-305); host math
/// in long double, as the reference (tiny, parity-critical).
template <typename T>
key_histogram build_interpolated_histogram(std::span<const T> all_samples, std::size_t bins) {
    detail::require_key<T>();
    const std::size_t cap = bins > 0 ? bins : 1;
    key_histogram h;
    h.bin_edges.resize(cap + 1);
    h.counts.resize(cap);
    std::uint64_t nb = 0, tot = 0;
    detail::check(detail::c_histogram(all_samples.data(), all_samples.size(), bins, h.bin_edges.data(),
                                      h.counts.data(), cap, &nb, &tot));
    h.bin_edges.resize(nb + 1);
    h.counts.resize(nb);
    h.total = tot;
    return h;
}

/// P-1 splitters at the estimated global quantiles (sihsort.hpp:310-349).
template <typename T>
splitter_set<T> select_splitters(const key_histogram& hist, std::size_t world) {
    detail::require_key<T>();
    splitter_set<T> out;
    if (world <= 1) return out;
    if (hist.counts.empty() || hist.bin_edges.size() != hist.counts.size() + 1)
        throw std::invalid_argument("select_splitters: malformed histogram");
    out.values.resize(world - 1);
    detail::check(detail::c_select(hist.bin_edges.data(), hist.counts.data(), hist.counts.size(), hist.total, world,
                                   out.values.data()));
    return out;
}

/// Exact-count splitter refinement (sihsort.hpp:364-464). Collective over comm.
template <typename T, typename Comm>
refine_result<T> refine_splitters(std::span<const T> local_sorted, splitter_set<T> splitters, Comm& comm,
                                  const sih_config& cfg, const exec_backend& ex = detail::default_backend()) {
    detail::require_key<T>();
    const ak_sih_config c = detail::to_c(cfg);
    detail::device_view<T> d(ex.ctx(), local_sorted);
    refine_result<T> r;
    std::uint64_t rounds = 0;
    int conv = 0;
    double dev = 0.0;
    detail::check(detail::c_refine(ex.ctx(), comm.handle(), d.p, local_sorted.size(), splitters.values.data(),
                                   splitters.values.size(), &c, &rounds, &conv, &dev));
    r.splitters = std::move(splitters);
    r.rounds_used = rounds;
    r.converged = conv != 0;
    r.max_deviation = dev;
    return r;
}

/// One all-to-all pass (sihsort.hpp:472-501): the received slices plus the kept local slice,
/// concatenated in SOURCE-RANK order (not merged). n_total = the agreed global count (it only
/// fixes the reference's piggyback accounting here; sizes travel in a count exchange).
template <typename T, typename Comm>
std::vector<T> redistribute(std::span<const T> local_sorted, const splitter_set<T>& splitters, Comm& comm,
                            std::uint64_t n_total, const exec_backend& ex = detail::default_backend()) {
    detail::require_key<T>();
    detail::device_view<T> d(ex.ctx(), local_sorted);
    std::uint64_t cap = local_sorted.size() + local_sorted.size() / 4 + 4096;
    for (;;) {
        detail::device_buffer<T> out(ex.ctx(), cap);
        std::uint64_t count = 0;
        const int rc = detail::c_redistribute(ex.ctx(), comm.handle(), d.p, local_sorted.size(),
                                              splitters.values.data(), splitters.values.size(), n_total, out.p, cap,
                                              &count);
        if (rc == AK_ECAPACITY) {  // every rank retries together
            cap = (count > cap ? count : cap) + cap / 8 + 4096;
            continue;
        }
        detail::check(rc, count);
        std::vector<T> h(count);
        out.download(h.data(), count);
        return h;
    }
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
