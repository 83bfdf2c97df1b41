// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library headers and sources in
// /root/reference/proj (compiled in place by oracle/Makefile into
// oracle/_ref/libakref.so; no reference source is copied into this repo).
// It lets the Python tests pin oracle/ak_oracle.c against the reference
// itself, lets tests/golden/make_golden.py record golden vectors, and is the
// "reference" CPU arm of bench.py (--impl reference, cpu_baseline.kind
// "reference"). The product path never loads it.
//
// threads == 0 selects exec_backend::sequential(); otherwise
// exec_backend::threaded(threads) (reference exec.hpp:38-46).
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <random>
#include <type_traits>
#include <span>
#include <vector>

#include "ak/csv.hpp"
#include "ak/exec.hpp"
#include "ak/fixture.hpp"
#include "ak/reduce.hpp"
#include "ak/scan.hpp"
#include "ak/search.hpp"
#include "ak/sihsort.hpp"
#include "ak/sim_comm.hpp"
#include "ak/sort.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

ak::exec_backend backend(std::uint64_t threads) {
    return threads == 0 ? ak::exec_backend::sequential() : ak::exec_backend::threaded(threads);
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const ak::sim::protocol_error&) {
        return 2;
    } catch (const ak::sim::transport_error&) {
        return 3;
    } catch (...) {
        return 9;
    }
}

template <typename T>
int merge_sort_impl(T* data, std::uint64_t n, int desc, std::uint64_t threads) {
    return guarded([&] {
        const auto ex = backend(threads);
        auto buffers = ak::sort_buffers<T>::with_capacity(n);
        if (desc) {
            ak::merge_sort(std::span<T>(data, n), buffers, ex, std::greater<T>{});
        } else {
            ak::merge_sort(std::span<T>(data, n), buffers, ex);
        }
    });
}

template <typename K, typename V>
int by_key_impl(K* keys, V* payload, std::uint64_t n, int desc, std::uint64_t threads) {
    return guarded([&] {
        const auto ex = backend(threads);
        auto buffers = ak::sort_by_key_buffers<K, V>::with_capacity(n);
        if (desc) {
            ak::merge_sort_by_key(std::span<K>(keys, n), std::span<V>(payload, n), buffers, ex,
                                  std::greater<K>{});
        } else {
            ak::merge_sort_by_key(std::span<K>(keys, n), std::span<V>(payload, n), buffers, ex);
        }
    });
}

template <typename T, typename I>
int sortperm_impl(const T* data, std::uint64_t n, I* out, int desc, int lowmem,
                  std::uint64_t threads) {
    return guarded([&] {
        const auto ex = backend(threads);
        std::span<const T> d(data, n);
        std::span<I> o(out, n);
        if (lowmem) {
            auto b = ak::sortperm_lowmem_buffers<I>::with_capacity(n);
            if (desc) ak::sortperm_lowmem<T, I>(d, o, b, ex, std::greater<T>{});
            else ak::sortperm_lowmem<T, I>(d, o, b, ex);
        } else {
            auto b = ak::sortperm_buffers<T, I>::with_capacity(n);
            if (desc) ak::sortperm<T, I>(d, o, b, ex, std::greater<T>{});
            else ak::sortperm<T, I>(d, o, b, ex);
        }
    });
}

template <typename T>
T reduce_impl(const T* x, std::uint64_t n, int op, T init, std::uint64_t threads) {
    const auto ex = backend(threads);
    std::span<const T> d(x, n);
    const ak::reduce_config<T> cfg{init, 256};
    if (op == 0) return ak::reduce<T>([](T a, T b) { return a + b; }, d, cfg, ex);
    if (op == 1) return ak::reduce<T>([](T a, T b) { return b < a ? b : a; }, d, cfg, ex);
    return ak::reduce<T>([](T a, T b) { return a < b ? b : a; }, d, cfg, ex);
}

template <typename T>
int scan_impl(const T* x, std::uint64_t n, T* out, int inclusive, T init, std::uint64_t chunk,
              std::uint64_t threads) {
    return guarded([&] {
        const auto ex = backend(threads);
        const ak::scan_spec<T> spec{inclusive ? ak::scan_mode::inclusive : ak::scan_mode::exclusive,
                                    init, chunk};
        ak::accumulate<T>([](T a, T b) { return a + b; }, std::span<const T>(x, n), spec, ex,
                          std::span<T>(out, n));
    });
}

template <typename T>
int search_impl(const T* h, std::uint64_t n, const T* needles, std::uint64_t m, int side_last,
                std::uint64_t* out, std::uint64_t threads) {
    return guarded([&] {
        const auto ex = backend(threads);
        const auto r = ak::searchsorted<T>(std::span<const T>(h, n), std::span<const T>(needles, m),
                                           side_last ? ak::search_side::last : ak::search_side::first,
                                           ex);
        for (std::uint64_t i = 0; i < m; ++i) out[i] = r[i];
    });
}

struct ref_sih_stats {
    std::uint64_t rounds_used;
    std::uint64_t converged;
    double max_deviation;
    std::uint64_t redistribution_sends;
    std::uint64_t redistribution_bytes;
    std::uint64_t collective_ops;
    std::uint64_t output_count;
};

struct ref_sih_config {
    std::uint64_t sample_per_rank;
    std::uint64_t bins;
    std::uint64_t max_refine_rounds;
    double imbalance_tol;
};

// One simulated-world sihsort (reference bench.cpp:146-162 shape). out receives
// the rank outputs concatenated in rank order; out may be null for timing runs.
template <typename T>
int sihsort_impl(std::uint64_t P, const T* const* inputs, const std::uint64_t* counts,
                 const ref_sih_config* c, std::uint64_t threads_per_rank, T* out,
                 std::uint64_t* out_counts, ref_sih_stats* stats) {
    return guarded([&] {
        ak::sih_config cfg;
        if (c) {
            cfg.sample_per_rank = c->sample_per_rank;
            cfg.bins = c->bins;
            cfg.max_refine_rounds = c->max_refine_rounds;
            cfg.imbalance_tol = c->imbalance_tol;
        }
        std::vector<std::vector<T>> results(P);
        std::vector<ak::sih_stats> st(P);
        ak::sim::world w(P);
        ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
            const std::size_t r = comm.rank();
            const auto ex = backend(threads_per_rank);
            std::vector<T> local(inputs[r], inputs[r] + counts[r]);
            auto [o, s] = ak::sihsort<T>(std::move(local), comm, cfg, ex);
            results[r] = std::move(o);
            st[r] = s;
        });
        std::uint64_t base = 0;
        for (std::uint64_t r = 0; r < P; ++r) {
            if (out) std::memcpy(out + base, results[r].data(), results[r].size() * sizeof(T));
            base += results[r].size();
            if (out_counts) out_counts[r] = results[r].size();
            if (stats) {
                stats[r].rounds_used = st[r].rounds_used;
                stats[r].converged = st[r].converged ? 1 : 0;
                stats[r].max_deviation = st[r].max_deviation;
                stats[r].redistribution_sends = st[r].redistribution_sends;
                stats[r].redistribution_bytes = st[r].redistribution_bytes;
                stats[r].collective_ops = st[r].collective_ops;
                stats[r].output_count = st[r].output_count;
            }
        }
    });
}

}  // namespace

#define REF_SORT(SUF, T)                                                                       \
    REF_API int ref_merge_sort_##SUF(T* d, std::uint64_t n, int desc, std::uint64_t th) {      \
        return merge_sort_impl<T>(d, n, desc, th);                                             \
    }                                                                                          \
    REF_API int ref_sortperm_##SUF##_u64(const T* d, std::uint64_t n, std::uint64_t* o,        \
                                         int desc, int lowmem, std::uint64_t th) {             \
        return sortperm_impl<T, std::uint64_t>(d, n, o, desc, lowmem, th);                     \
    }                                                                                          \
    REF_API int ref_sortperm_##SUF##_i32(const T* d, std::uint64_t n, std::int32_t* o,         \
                                         int desc, int lowmem, std::uint64_t th) {             \
        return sortperm_impl<T, std::int32_t>(d, n, o, desc, lowmem, th);                      \
    }                                                                                          \
    REF_API int ref_merge_sort_by_key_##SUF##_i32(T* k, std::int32_t* v, std::uint64_t n,      \
                                                  int desc, std::uint64_t th) {                \
        return by_key_impl<T, std::int32_t>(k, v, n, desc, th);                                \
    }                                                                                          \
    REF_API int ref_merge_sort_by_key_##SUF##_u64(T* k, std::uint64_t* v, std::uint64_t n,     \
                                                  int desc, std::uint64_t th) {                \
        return by_key_impl<T, std::uint64_t>(k, v, n, desc, th);                               \
    }                                                                                          \
    REF_API int ref_searchsorted_##SUF(const T* h, std::uint64_t n, const T* nd,               \
                                       std::uint64_t m, int last, std::uint64_t* o,            \
                                       std::uint64_t th) {                                     \
        return search_impl<T>(h, n, nd, m, last, o, th);                                       \
    }

REF_SORT(i32, std::int32_t)
REF_SORT(u32, std::uint32_t)
REF_SORT(i64, std::int64_t)
REF_SORT(u64, std::uint64_t)
REF_SORT(f32, float)
REF_SORT(f64, double)

#define REF_RED(SUF, T)                                                                        \
    REF_API T ref_reduce_##SUF(const T* x, std::uint64_t n, int op, T init, std::uint64_t th) { \
        return reduce_impl<T>(x, n, op, init, th);                                             \
    }                                                                                          \
    REF_API int ref_accumulate_##SUF(const T* x, std::uint64_t n, T* o, int inclusive, T init, \
                                     std::uint64_t chunk, std::uint64_t th) {                  \
        return scan_impl<T>(x, n, o, inclusive, init, chunk, th);                              \
    }

REF_RED(i32, std::int32_t)
REF_RED(i64, std::int64_t)
REF_RED(u64, std::uint64_t)
REF_RED(f32, float)
REF_RED(f64, double)

#define REF_SIH(SUF, T)                                                                        \
    REF_API int ref_sihsort_##SUF(std::uint64_t P, const T* const* in, const std::uint64_t* c, \
                                  const ref_sih_config* cfg, std::uint64_t th, T* out,         \
                                  std::uint64_t* oc, ref_sih_stats* st) {                      \
        return sihsort_impl<T>(P, in, c, cfg, th, out, oc, st);                                \
    }

REF_SIH(i32, std::int32_t)
REF_SIH(i64, std::int64_t)
REF_SIH(u64, std::uint64_t)
REF_SIH(f32, float)
REF_SIH(f64, double)

// ---- reference bench inputs (bench.cpp:44-62 random_keys, :164-173 generate_rank_inputs;
// both sit in an anonymous namespace of src/bench.cpp, so they are restated here) ----
// Lets the reference arm of bench.py make its inputs without loading the product library.
template <typename T>
void bench_keys_impl(std::uint64_t seed, std::uint64_t rank, std::uint64_t n, T* out) {
    std::mt19937_64 rng(seed + 0x9e3779b97f4a7c15ULL * (rank + 1));  // bench.cpp:168
    if constexpr (std::is_integral_v<T>) {
        for (std::uint64_t i = 0; i < n; ++i) out[i] = static_cast<T>(rng());  // bench.cpp:50-52
    } else {
        std::uniform_real_distribution<T> dist(T(-1e6), T(1e6));  // bench.cpp:55-58
        for (std::uint64_t i = 0; i < n; ++i) out[i] = dist(rng);
    }
}
#define REF_KEYS(SUF, T)                                                                                    \
    REF_API int ref_bench_keys_##SUF(std::uint64_t seed, std::uint64_t rank, std::uint64_t n, T* out) {     \
        return guarded([&] { bench_keys_impl<T>(seed, rank, n, out); });                                   \
    }
REF_KEYS(i32, std::int32_t)
REF_KEYS(u32, std::uint32_t)
REF_KEYS(i64, std::int64_t)
REF_KEYS(u64, std::uint64_t)
REF_KEYS(f32, float)
REF_KEYS(f64, double)

REF_API std::uint64_t ref_sortperm_bytes(std::uint64_t n, int key_bytes, int index_bytes, int lowmem) {
    // sort.hpp:43-65 required_bytes formulas for equal-width instantiations
    if (key_bytes == 8 && index_bytes == 8) {
        return lowmem ? ak::sortperm_lowmem_buffers<std::uint64_t>::required_bytes(n)
                      : ak::sortperm_buffers<std::uint64_t, std::uint64_t>::required_bytes(n);
    }
    if (key_bytes == 4 && index_bytes == 4) {
        return lowmem ? ak::sortperm_lowmem_buffers<std::int32_t>::required_bytes(n)
                      : ak::sortperm_buffers<float, std::int32_t>::required_bytes(n);
    }
    return 0;
}

// ---- SIHS fixtures and benchmark CSV (reference src/fixture.cpp, src/csv.cpp) ----
#define REF_FIXTURE(SUF, T)                                                                           \
    REF_API int ref_write_fixture_##SUF(const char* path, std::uint32_t rank, const T* d,             \
                                        std::uint64_t n) {                                            \
        return guarded([&] { ak::write_fixture<T>(path, rank, std::span<const T>(d, n)); });          \
    }                                                                                                 \
    REF_API int ref_read_fixture_##SUF(const char* path, std::uint32_t* rank, T* out,                 \
                                       std::uint64_t cap, std::uint64_t* n) {                         \
        return guarded([&] {                                                                          \
            auto v = ak::read_fixture<T>(path, rank);                                                 \
            *n = v.size();                                                                            \
            if (v.size() > cap) throw std::invalid_argument("capacity");                              \
            std::memcpy(out, v.data(), v.size() * sizeof(T));                                         \
        });                                                                                           \
    }
REF_FIXTURE(i32, std::int32_t)
REF_FIXTURE(i64, std::int64_t)
REF_FIXTURE(f32, float)
REF_FIXTURE(f64, double)

REF_API int ref_emit_csv(const char* path, int nrec, const char* const* case_names, const char* const* dtypes,
                         const std::uint64_t* n, const std::uint64_t* workers, const std::uint64_t* reps,
                         const double* mean_ms, const double* stddev_ms, const double* gbps, const double* norm_ms) {
    return guarded([&] {
        std::vector<ak::bench::bench_record> recs(nrec);
        for (int i = 0; i < nrec; ++i) {
            recs[i].case_name = case_names[i];
            recs[i].dtype = dtypes[i];
            recs[i].n = n[i];
            recs[i].workers = workers[i];
            recs[i].reps = reps[i];
            recs[i].mean_ms = mean_ms[i];
            recs[i].stddev_ms = stddev_ms[i];
            recs[i].throughput_gbps = gbps[i];
            recs[i].normalized_ms = norm_ms[i];
        }
        ak::bench::emit_csv(std::filesystem::path(path), recs);
    });
}
