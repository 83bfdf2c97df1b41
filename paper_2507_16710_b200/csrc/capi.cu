// capi.cu -- extern "C" entry points of libak_cuda.so (declared in include/ak_cuda.h).
#include <climits>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <limits>
#include <type_traits>
#include <vector>

#include "../../include/ak_cuda.h"
#include "ctx.cuh"
#include "radix_sort.cuh"
#include "sortperm_fast.cuh"
#include "wide_keys.cuh"
#include "predicates.cuh"
#include "reduce_scan.cuh"
#include "search_merge.cuh"
#include "sihsort.cuh"

struct ak_comm {
    std::unique_ptr<akb::comm_iface> impl;
    bool host_p2p = false;                      // loopback: messages never touch the device
    std::map<int, std::vector<char>> pending;   // received message awaiting a larger buffer
};

// sim::world (sim_comm.hpp:41-80) on one device: P logical ranks, one host thread each.
struct ak_world {
    akb::loopback_world w;
    ak_world(int ranks, std::size_t queue_capacity) : w(ranks, queue_capacity) {}
};

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return AK_OK;
    } catch (const akb::proto_capacity_error& e) {
        g_err = e.what();
        return AK_ECAPACITY;
    } catch (const akb::capacity_error& e) {
        g_err = e.what();
        return AK_ECAPACITY;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return AK_EINVAL;
    } catch (const akb::proto_protocol_error& e) {
        g_err = e.what();
        return AK_EPROTOCOL;
    } catch (const akb::protocol_error& e) {
        g_err = e.what();
        return AK_EPROTOCOL;
    } catch (const akb::transport_error& e) {
        g_err = e.what();
        return AK_ETRANSPORT;
    } catch (const akb::cuda_error& e) {
        g_err = e.what();
        return AK_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return AK_EINTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return AK_EINTERNAL;
    }
}

void need(bool ok, const char* msg) {
    if (!ok) throw akb::invalid_argument(msg);
}

struct ctx_lock {
    ak_ctx* c;
    std::lock_guard<std::mutex> lk;
    explicit ctx_lock(ak_ctx* ctx) : c(ctx), lk((need(ctx != nullptr, "ak: null ctx"), ctx->mu)) {
        AKB_CUDA(cudaSetDevice(c->device));
    }
};

// Trivial single-rank transport for comm == NULL (P = 1).
struct self_comm final : akb::comm_iface {
    int rank() const override { return 0; }
    int size() const override { return 1; }
    void allgather(const void* in, std::size_t bytes, void* out) override { std::memcpy(out, in, bytes); }
    void allreduce_sum_u64(std::uint64_t*, std::size_t) override {}
    void exchange(const void*, const std::uint64_t*, const std::uint64_t*, void*, const std::uint64_t*,
                  const std::uint64_t*, std::size_t) override {}
};

akb::sih_config_c to_cfg(const ak_sih_config* cfg) {
    akb::sih_config_c c{0, 0, 4, 0.25};
    if (cfg) {
        c.sample_per_rank = cfg->sample_per_rank;
        c.bins = cfg->bins;
        c.max_refine_rounds = cfg->max_refine_rounds;
        c.imbalance_tol = cfg->imbalance_tol;
    }
    return c;
}

void to_stats(const akb::sih_stats_c& s, ak_sih_stats* out) {
    if (!out) return;
    static_assert(sizeof(ak_sih_stats) == sizeof(akb::sih_stats_c));
    std::memcpy(out, &s, sizeof(s));
}

template <typename T>
void merge_sort_impl(ak_ctx* c, T* data, std::uint64_t n, T* scratch, std::uint64_t scratch_n, int desc) {
    ctx_lock g(c);
    need(scratch_n >= n, "merge_sort: scratch buffer too small");  // sort.hpp:182-184
    need(n == 0 || (data && scratch), "merge_sort: null buffer");
    akb::radix_sort<T, std::uint32_t>(c, akb::SORT_KEYS, data, data, scratch, nullptr, nullptr, nullptr, n,
                                      desc != 0, true);
    akb::ctx_finish(c);
}

// A caller's large pageable host array is page-locked for the duration of one in-place host
// sort (its two copies then run at the link's DMA rate instead of through the driver's
// staging buffers); arrays that are already pinned or registered, and ones under 32 MB
// (registering costs ~1 ms), are left alone. merge_sort_host of 2^24 int64: 18.7 -> 11.0 ms,
// 2^27: 147 -> 79 ms. Not used for one-way copies: the C++ headers' staging (ak_memcpy) of
// fresh 512 MB vectors got slower with it (ak_bench sort-weak 2^26 host path 545 -> 725 ms).
#ifndef AKB_HOST_PIN_MIN_MB
#define AKB_HOST_PIN_MIN_MB 32
#endif
struct host_pin {
    void* p = nullptr;
    host_pin(const void* ptr, std::size_t bytes) {
        if (!ptr || bytes < (std::size_t(AKB_HOST_PIN_MIN_MB) << 20)) return;
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) == cudaSuccess && a.type != cudaMemoryTypeUnregistered) return;
        (void)cudaGetLastError();
        if (cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterDefault) == cudaSuccess)
            p = const_cast<void*>(ptr);
        else
            (void)cudaGetLastError();  // not registrable (e.g. overlapping a registered range): pageable copies
    }
    ~host_pin() {
        if (p) (void)cudaHostUnregister(p);
    }
    host_pin(const host_pin&) = delete;
    host_pin& operator=(const host_pin&) = delete;
};

template <typename T>
void merge_sort_host_impl(ak_ctx* c, T* h, std::uint64_t n, int desc) {
    ctx_lock g(c);
    need(n == 0 || h, "merge_sort: null buffer");
    if (n < 2) return;
    host_pin pin(h, n * sizeof(T));
    T* d = static_cast<T*>(akb::ctx_stage(c, 2 * n * sizeof(T)));
    AKB_CUDA(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    akb::radix_sort<T, std::uint32_t>(c, akb::SORT_KEYS, d, d, d + n, nullptr, nullptr, nullptr, n, desc != 0,
                                      true);
    AKB_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
}

template <typename T, typename V>
void by_key_impl(ak_ctx* c, T* keys, std::uint64_t nk, void* payload, std::uint64_t np, T* sk,
                 std::uint64_t skn, void* sp, std::uint64_t spn, int desc) {
    ctx_lock g(c);
    need(nk == np, "merge_sort_by_key: keys and payload lengths differ");  // sort.hpp:214-216
    need(skn >= nk && spn >= nk, "merge_sort_by_key: scratch buffers too small");  // :217-219
    need(nk == 0 || (keys && payload && sk && sp), "merge_sort_by_key: null buffer");
    akb::radix_sort<T, V>(c, akb::SORT_PAIRS, keys, keys, sk, static_cast<const V*>(payload),
                          static_cast<V*>(payload), static_cast<V*>(sp), nk, desc != 0, true);
    akb::ctx_finish(c);
}

template <typename T, typename I>
void sortperm_impl(ak_ctx* c, const T* data, std::uint64_t n, I* out, std::uint64_t out_n, T* wk,
                   std::uint64_t wkn, T* sk, std::uint64_t skn, I* si, std::uint64_t sin_, int desc) {
    ctx_lock g(c);
    need(out_n == n, "sortperm: output length must match input length");  // sort.hpp:242-244
    need(wkn >= n && skn >= n && sin_ >= n, "sortperm: scratch buffers too small");  // :245-248
    need(n <= static_cast<std::uint64_t>(std::numeric_limits<I>::max()), "sortperm: index type too narrow");
    need(n == 0 || (data && out && wk && sk && si), "sortperm: null buffer");
    using V = std::make_unsigned_t<I>;
    if (n == 1) {
        AKB_CUDA(cudaMemsetAsync(out, 0, sizeof(I), c->stream));
    } else if (n > 1) {
        bool done = false;
        // 32-bit integer keys: composite (key, index) keys through the 64-bit hybrid sort
        // (1e8 i32: 2.31 ms vs 2.64 ms onesweep). Float keys keep the onesweep: their
        // exponent-heavy top bits need a third MSD level, which costs more than it saves
        // (1e8 f32 uniform in [-1e6, 1e6): 3.03 ms vs 2.64 ms, measured r01; r02 with the
        // current kernels 3.51 ms vs 2.72 ms: 3 MSD levels 1.11 + histograms 0.57 + compose /
        // decompose 0.52 + counting stage 0.95 ms, whose ranges span many tiny low-exponent
        // buckets).
        if constexpr (sizeof(T) == 4 && std::is_integral_v<T>)
            done = akb::sortperm_composite<T, V>(c, data, n, reinterpret_cast<V*>(out), desc != 0);
        if (!done)
            akb::radix_sort<T, V>(c, akb::SORT_IOTA, data, sk, wk, nullptr, reinterpret_cast<V*>(out),
                                  reinterpret_cast<V*>(si), n, desc != 0, false);
    }
    akb::ctx_finish(c);
}

template <typename T, typename I>
void sortperm_lowmem_impl(ak_ctx* c, const T* data, std::uint64_t n, I* out, std::uint64_t out_n, I* si,
                          std::uint64_t sin_, int desc) {
    ctx_lock g(c);
    need(out_n == n, "sortperm_lowmem: output length must match input length");  // sort.hpp:270-272
    need(sin_ >= n, "sortperm_lowmem: scratch buffer too small");  // :273-276
    need(n <= static_cast<std::uint64_t>(std::numeric_limits<I>::max()), "sortperm: index type too narrow");
    need(n == 0 || (data && out && si), "sortperm_lowmem: null buffer");
    using V = std::make_unsigned_t<I>;
    if (n == 1) {
        AKB_CUDA(cudaMemsetAsync(out, 0, sizeof(I), c->stream));
    } else if (n > 1) {
        akb::radix_sort<T, V>(c, akb::SORT_LOWMEM, data, nullptr, nullptr, nullptr, reinterpret_cast<V*>(out),
                              reinterpret_cast<V*>(si), n, desc != 0, false);
    }
    akb::ctx_finish(c);
}

template <typename T>
void reduce_impl(ak_ctx* c, const T* x, std::uint64_t n, int op, int map, T init, T* res, bool host) {
    ctx_lock g(c);
    need(op >= 0 && op <= 2, "reduce: op must be 0 (sum), 1 (min) or 2 (max)");
    need(map >= 0 && map <= 2, "mapreduce: map must be 0 (identity), 1 (abs) or 2 (square)");
    need(res != nullptr, "reduce: null result");
    need(n == 0 || x, "reduce: null buffer");
    if (n == 0) {  // reduce.hpp:28-30: empty data returns init
        if (host) *res = init;
        else AKB_CUDA(cudaMemcpyAsync(res, &init, sizeof(T), cudaMemcpyHostToDevice, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    T* d_res = host ? reinterpret_cast<T*>(static_cast<char*>(c->small) + 200704) : res;
    akb::reduce<T>(c, x, n, op, map, init, d_res);
    if (host) {
        T* h = static_cast<T*>(akb::ctx_pinned(c, sizeof(T)));
        AKB_CUDA(cudaMemcpyAsync(h, d_res, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        *res = *h;
    } else {
        akb::ctx_finish(c);
    }
}

template <typename T>
void scan_impl(ak_ctx* c, const T* x, std::uint64_t n, T* out, std::uint64_t out_n, int op, int inclusive,
               T init, std::uint64_t chunk) {
    ctx_lock g(c);
    need(out_n == n, "accumulate: output length must match input length");  // scan.hpp:32-34
    need(chunk != 0, "accumulate: chunk_size must be >= 1");                 // scan.hpp:35-37
    need(op >= 0 && op <= 2, "accumulate: op must be 0 (sum), 1 (min) or 2 (max)");
    need(n == 0 || (x && out), "accumulate: null buffer");
    akb::scan<T>(c, x, out, n, op, inclusive ? 1 : 0, init);
    akb::ctx_finish(c);
}

template <typename T>
void merge_runs_impl(ak_ctx* c, int P, const T* const* runs, const uint64_t* lens, T* dst, T* scratch, int desc) {
    ctx_lock g(c);
    need(P >= 1 && P <= akb::MW_MAXP, "merge_runs: 1 <= P <= 4096 runs");
    need(runs && lens, "merge_runs: null runs");
    std::uint64_t total = 0;
    for (int r = 0; r < P; ++r) {
        need(lens[r] == 0 || runs[r], "merge_runs: null run");
        total += lens[r];
    }
    need(total == 0 || (dst && scratch), "merge_runs: null output or scratch");
    akb::merge_runs<T>(c, P, runs, lens, dst, scratch, desc != 0);
    akb::ctx_finish(c);
}

template <typename T>
void search_impl(ak_ctx* c, const T* hay, std::uint64_t n, const T* needles, std::uint64_t m, int side_last,
                 int desc, int validate, std::uint64_t* out) {
    ctx_lock g(c);
    need((n == 0 || hay) && (m == 0 || (needles && out)), "searchsorted: null buffer");
    if (validate && !akb::is_sorted<T>(c, hay, n, desc != 0))  // search.hpp:40-43
        throw akb::invalid_argument("searchsorted: haystack is not sorted");
    akb::searchsorted<T>(c, hay, n, needles, m, side_last ? 1 : 0, desc ? 1 : 0, out);
    akb::ctx_finish(c);
}

akb::comm_iface& comm_of(ak_comm* comm, self_comm& fallback, ak_ctx* c) {
    if (!comm) return fallback;
    comm->impl->bind(c->stream, c->sm_count);
    return *comm->impl;
}

template <typename T>
void sihsort_impl(ak_ctx* c, ak_comm* comm, const T* in, std::uint64_t n, T* out, std::uint64_t cap,
                  std::uint64_t* out_count, const ak_sih_config* cfg, ak_sih_stats* stats) {
    ctx_lock g(c);
    need(out_count != nullptr, "sihsort: null out_count");
    need(n == 0 || in, "sihsort: null input");
    need(cap == 0 || out, "sihsort: null output");
    self_comm self;
    akb::comm_iface& cm = comm_of(comm, self, c);
    akb::sih_stats_c st{};
    try {
        *out_count = akb::sihsort_device<T>(c, cm, in, n, out, cap, to_cfg(cfg), st);
    } catch (const akb::proto_capacity_error& e) {
        *out_count = e.required;
        throw;
    }
    to_stats(st, stats);
    akb::ctx_finish(c);
}

template <typename T>
void sihsort_host_impl(ak_ctx* c, ak_comm* comm, const T* h_in, std::uint64_t n, T* h_out, std::uint64_t cap,
                       std::uint64_t* out_count, const ak_sih_config* cfg, ak_sih_stats* stats) {
    ctx_lock g(c);
    need(out_count != nullptr, "sihsort: null out_count");
    need(n == 0 || h_in, "sihsort: null input");
    need(cap == 0 || h_out, "sihsort: null output");
    T* d = static_cast<T*>(akb::ctx_stage(c, (n + cap + 1) * sizeof(T)));
    T* d_in = d;
    T* d_out = d + n;
    if (n) AKB_CUDA(cudaMemcpyAsync(d_in, h_in, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    self_comm self;
    akb::comm_iface& cm = comm_of(comm, self, c);
    akb::sih_stats_c st{};
    try {
        *out_count = akb::sihsort_device<T>(c, cm, d_in, n, d_out, cap, to_cfg(cfg), st);
    } catch (const akb::proto_capacity_error& e) {
        *out_count = e.required;
        throw;
    }
    if (*out_count)
        AKB_CUDA(cudaMemcpyAsync(h_out, d_out, *out_count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    to_stats(st, stats);
}

// ---- sihsort stage functions (sihsort.hpp:264-501) ----
template <typename T>
void sample_local_impl(ak_ctx* c, const T* d, uint64_t n, uint64_t k, T* h, uint64_t* cnt) {
    ctx_lock g(c);
    need(cnt != nullptr, "sample_local: null count");
    need(n == 0 || d, "sample_local: null input");
    need(k == 0 || n == 0 || h, "sample_local: null output");
    *cnt = akb::sample_local_device<T>(c, d, n, k, h);
}

template <typename T>
void histogram_impl(const T* smp, uint64_t m, uint64_t bins, long double* e, uint64_t* cts, uint64_t cap,
                    uint64_t* nb, uint64_t* tot) {
    need(nb && tot && e && cts, "build_interpolated_histogram: null argument");
    need(m == 0 || smp, "build_interpolated_histogram: null samples");
    const akb::proto::histogram h = akb::proto::build_histogram(std::vector<T>(smp, smp + m), bins);
    need(h.counts.size() <= cap, "build_interpolated_histogram: bin capacity too small");
    std::copy(h.edges.begin(), h.edges.end(), e);
    std::copy(h.counts.begin(), h.counts.end(), cts);
    *nb = h.counts.size();
    *tot = h.total;
}

template <typename T>
void select_impl(const long double* e, const uint64_t* cts, uint64_t nb, uint64_t tot, uint64_t world, T* out) {
    need(e && cts && nb >= 1, "select_splitters: empty histogram");
    need(world <= 1 || out, "select_splitters: null output");
    const auto v = akb::proto::select<T>(std::vector<long double>(e, e + nb + 1), std::vector<uint64_t>(cts, cts + nb),
                                         tot, world);
    std::copy(v.begin(), v.end(), out);
}

template <typename T>
void refine_impl(ak_ctx* c, ak_comm* comm, const T* d, uint64_t n, T* spl, uint64_t m, const ak_sih_config* cfg,
                 uint64_t* rounds, int* conv, double* dev) {
    ctx_lock g(c);
    need(n == 0 || d, "refine_splitters: null input");
    need(m == 0 || spl, "refine_splitters: null splitters");
    self_comm self;
    akb::comm_iface& cm = comm_of(comm, self, c);
    std::vector<T> v(spl, spl + m);
    const akb::refine_out r = akb::refine_device<T>(c, cm, d, n, v, to_cfg(cfg));
    std::copy(v.begin(), v.end(), spl);
    if (rounds) *rounds = r.rounds_used;
    if (conv) *conv = static_cast<int>(r.converged);
    if (dev) *dev = r.max_deviation;
}

template <typename T>
void redistribute_impl(ak_ctx* c, ak_comm* comm, const T* d, uint64_t n, const T* spl, uint64_t m, uint64_t nt,
                       T* out, uint64_t cap, uint64_t* oc, uint64_t* sends, uint64_t* bytes) {
    ctx_lock g(c);
    need(oc != nullptr, "redistribute: null out_count");
    need(n == 0 || d, "redistribute: null input");
    need(m == 0 || spl, "redistribute: null splitters");
    need(cap == 0 || out, "redistribute: null output");
    self_comm self;
    akb::comm_iface& cm = comm_of(comm, self, c);
    uint64_t s0 = 0, b0 = 0;
    try {
        *oc = akb::redistribute_device<T>(c, cm, d, n, std::vector<T>(spl, spl + m), out, cap, &s0, &b0, nt);
    } catch (const akb::proto_capacity_error& e) {
        *oc = e.required;
        throw;
    }
    if (sends) *sends = s0;
    if (bytes) *bytes = b0;
}

template <typename T>
void sihsort_perm_impl(ak_ctx* c, ak_comm* comm, const T* in, std::uint64_t n, T* out, std::uint64_t* out_idx,
                       std::uint64_t cap, std::uint64_t* out_count, const ak_sih_config* cfg, ak_sih_stats* stats) {
    ctx_lock g(c);
    need(out_count != nullptr, "sihsort_perm: null out_count");
    need(n == 0 || in, "sihsort_perm: null input");
    need(cap == 0 || (out && out_idx), "sihsort_perm: null output");
    self_comm self;
    akb::comm_iface& cm = comm_of(comm, self, c);
    akb::sih_stats_c st{};
    try {
        *out_count = akb::sihsort_perm_device<T>(c, cm, in, n, out, out_idx, cap, to_cfg(cfg), st);
    } catch (const akb::proto_capacity_error& e) {
        *out_count = e.required;
        throw;
    }
    to_stats(st, stats);
    akb::ctx_finish(c);
}

// P logical ranks of the distributed sortperm on one device (threads over the loopback world).
template <typename T>
void sihsort_perm_loopback_impl(int device, std::uint64_t P, const T* const* in, const std::uint64_t* n,
                                T* const* out, std::uint64_t* const* out_idx, const std::uint64_t* cap,
                                std::uint64_t* out_count, const ak_sih_config* cfg, ak_sih_stats* stats) {
    need(P >= 1, "world: rank count must be >= 1");
    need(in && n && out && out_idx && cap && out_count, "sihsort_perm_loopback: null argument");
    akb::loopback_world world(static_cast<int>(P));
    std::vector<std::thread> threads;
    std::mutex err_mu;
    std::exception_ptr first;
    const akb::sih_config_c c = to_cfg(cfg);
    for (std::uint64_t r = 0; r < P; ++r) {
        threads.emplace_back([&, r] {
            ak_ctx* ctx = nullptr;
            try {
                if (ak_ctx_create(device, nullptr, &ctx) != AK_OK) throw akb::cuda_error(g_err);
                akb::loopback_comm cm(&world, static_cast<int>(r), ctx->stream);
                cm.bind(ctx->stream, ctx->sm_count);
                akb::sih_stats_c st{};
                {
                    std::lock_guard<std::mutex> lk(ctx->mu);
                    AKB_CUDA(cudaSetDevice(device));
                    try {
                        out_count[r] =
                            akb::sihsort_perm_device<T>(ctx, cm, in[r], n[r], out[r], out_idx[r], cap[r], c, st);
                    } catch (const akb::proto_capacity_error& e) {
                        out_count[r] = e.required;
                        throw;
                    }
                    AKB_CUDA(cudaStreamSynchronize(ctx->stream));
                }
                to_stats(st, stats ? stats + r : nullptr);
            } catch (...) {
                {
                    std::lock_guard<std::mutex> lk(err_mu);
                    if (!first) first = std::current_exception();
                }
                world.abort();
            }
            if (ctx) ak_ctx_destroy(ctx);
        });
    }
    for (auto& t : threads) t.join();
    if (first) std::rethrow_exception(first);
}

template <typename T>
void sihsort_loopback_impl(int device, std::uint64_t P, const T* const* in, const std::uint64_t* n,
                           T* const* out, const std::uint64_t* cap, std::uint64_t* out_count,
                           const ak_sih_config* cfg, ak_sih_stats* stats) {
    need(P >= 1, "world: rank count must be >= 1");  // sim_comm.cpp:7-9
    need(in && n && out && cap && out_count, "sihsort_loopback: null argument");
    akb::loopback_world world(static_cast<int>(P));
    std::vector<std::thread> threads;
    std::mutex err_mu;
    std::exception_ptr first;
    const akb::sih_config_c c = to_cfg(cfg);
    for (std::uint64_t r = 0; r < P; ++r) {
        threads.emplace_back([&, r] {
            ak_ctx* ctx = nullptr;
            try {
                if (ak_ctx_create(device, nullptr, &ctx) != AK_OK) throw akb::cuda_error(g_err);
                akb::loopback_comm cm(&world, static_cast<int>(r), ctx->stream);
                cm.bind(ctx->stream, ctx->sm_count);
                akb::sih_stats_c st{};
                {
                    std::lock_guard<std::mutex> lk(ctx->mu);
                    AKB_CUDA(cudaSetDevice(device));
                    try {
                        out_count[r] = akb::sihsort_device<T>(ctx, cm, in[r], n[r], out[r], cap[r], c, st);
                    } catch (const akb::proto_capacity_error& e) {
                        out_count[r] = e.required;
                        throw;
                    }
                    AKB_CUDA(cudaStreamSynchronize(ctx->stream));
                }
                to_stats(st, stats ? stats + r : nullptr);
            } catch (...) {
                {
                    std::lock_guard<std::mutex> lk(err_mu);
                    if (!first) first = std::current_exception();
                }
                world.abort();  // sim_comm.hpp:203-208: abort wakes the other ranks
            }
            if (ctx) ak_ctx_destroy(ctx);
        });
    }
    for (auto& t : threads) t.join();
    if (first) std::rethrow_exception(first);
}

template <typename T>
void pred_impl(ak_ctx* c, const T* x, uint64_t n, int op, T v, int any, int algo, int* result) {
    ctx_lock g(c);
    need(result != nullptr, "predicate: null result");
    need(n == 0 || x, "predicate: null input");
    need(op >= akb::PRED_LT && op <= akb::PRED_NE, "predicate: unknown comparison");
    const bool found = akb::find_decider<T>(c, x, n, op, v, any != 0, algo == 0);
    *result = any ? (found ? 1 : 0) : (found ? 0 : 1);  // all(p) = !exists(!p) (predicates.hpp:69-78)
}

// identity of op for the rank fold (the reference requires a neutral init, reduce.hpp:12-14)
template <typename T>
T op_identity(int op) {
    if (op == akb::OP_SUM) return T(0);
    if constexpr (std::is_floating_point_v<T>) return op == akb::OP_MIN ? std::numeric_limits<T>::infinity()
                                                                       : -std::numeric_limits<T>::infinity();
    else return op == akb::OP_MIN ? std::numeric_limits<T>::max() : std::numeric_limits<T>::lowest();
}
template <typename T>
T op_apply(int op, T a, T b) {
    if (op == akb::OP_SUM) {
        if constexpr (std::is_integral_v<T>) {
            using U = std::make_unsigned_t<T>;
            return static_cast<T>(static_cast<U>(a) + static_cast<U>(b));
        } else {
            return a + b;
        }
    }
    if (op == akb::OP_MIN) return b < a ? b : a;
    return a < b ? b : a;
}

// Rank partials: local reduce on the device (identity init), then an allgather.
template <typename T>
std::vector<T> rank_partials(ak_ctx* c, akb::comm_iface& cm, const T* x, uint64_t n, int op, int map) {
    T* dres = reinterpret_cast<T*>(static_cast<char*>(c->small) + 196608 + 128);
    T local = op_identity<T>(op);
    if (n) {
        akb::reduce<T>(c, x, n, op, map, op_identity<T>(op), dres);
        AKB_CUDA(cudaMemcpyAsync(&local, dres, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
    }
    std::vector<T> all(cm.size());
    cm.allgather(&local, sizeof(T), all.data());
    return all;
}

template <typename T>
void reduce_all_impl(ak_ctx* c, ak_comm* comm, const T* x, uint64_t n, int op, int map, T init, T* result) {
    ctx_lock g(c);
    need(result != nullptr, "reduce_all: null result");
    need(n == 0 || x, "reduce_all: null input");
    need(op >= akb::OP_SUM && op <= akb::OP_MAX, "reduce_all: unknown op");
    self_comm self;
    akb::comm_iface& cm = comm_of(comm, self, c);
    const std::vector<T> parts = rank_partials<T>(c, cm, x, n, op, map);
    T r = init;
    for (const T& p : parts) r = op_apply<T>(op, r, p);
    *result = r;
}

template <typename T>
void accumulate_all_impl(ak_ctx* c, ak_comm* comm, const T* x, uint64_t n, T* out, uint64_t out_n, int op,
                         int inclusive, T init) {
    ctx_lock g(c);
    need(out_n == n, "accumulate: output length must match input length");  // scan.hpp:32-34
    need(n == 0 || (x && out), "accumulate_all: null input or output");
    need(op >= akb::OP_SUM && op <= akb::OP_MAX, "accumulate_all: unknown op");
    self_comm self;
    akb::comm_iface& cm = comm_of(comm, self, c);
    const std::vector<T> parts = rank_partials<T>(c, cm, x, n, op, akb::MAP_IDENTITY);
    T carry = init;  // init folded with the totals of every lower rank
    for (int q = 0; q < cm.rank(); ++q) carry = op_apply<T>(op, carry, parts[q]);
    if (n) akb::scan<T>(c, x, out, n, op, inclusive, carry);
    akb::ctx_finish(c);
}

}  // namespace

// ---- int16 / int128 keys (dtype.hpp:14-21): sort family only, same argument checks ----
template <typename T>
void wide_merge_sort_impl(ak_ctx* c, T* data, std::uint64_t n, T* scratch, std::uint64_t scratch_n, int desc) {
    ctx_lock g(c);
    need(scratch_n >= n, "merge_sort: scratch buffer too small");  // sort.hpp:182-184
    need(n == 0 || (data && scratch), "merge_sort: null buffer");
    if (n >= 2) akb::wide_merge_sort<T>(c, data, n, desc != 0);
    akb::ctx_finish(c);
}
template <typename T>
void wide_merge_sort_host_impl(ak_ctx* c, T* h, std::uint64_t n, int desc) {
    ctx_lock g(c);
    need(n == 0 || h, "merge_sort: null buffer");
    if (n < 2) return;
    host_pin pin(h, n * sizeof(T));
    T* d = static_cast<T*>(akb::ctx_stage(c, n * sizeof(T)));
    AKB_CUDA(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    akb::wide_merge_sort<T>(c, d, n, desc != 0);
    AKB_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
}
template <typename T, typename V>
void wide_by_key_impl(ak_ctx* c, T* keys, std::uint64_t nk, void* payload, std::uint64_t np, T* sk,
                      std::uint64_t skn, void* sp, std::uint64_t spn, int desc) {
    ctx_lock g(c);
    need(nk == np, "merge_sort_by_key: keys and payload lengths differ");            // sort.hpp:214-216
    need(skn >= nk && spn >= nk, "merge_sort_by_key: scratch buffers too small");  // :217-219
    need(nk == 0 || (keys && payload && sk && sp), "merge_sort_by_key: null buffer");
    if (nk >= 2) akb::wide_by_key<T, V>(c, keys, static_cast<V*>(payload), nk, desc != 0);
    akb::ctx_finish(c);
}
template <typename T, typename I>
void wide_sortperm_impl(ak_ctx* c, const T* data, std::uint64_t n, I* out, std::uint64_t out_n, std::uint64_t wkn,
                        std::uint64_t skn, std::uint64_t sin_, bool lowmem, int desc) {
    ctx_lock g(c);
    need(out_n == n, lowmem ? "sortperm_lowmem: output length must match input length"
                            : "sortperm: output length must match input length");  // sort.hpp:242-244, :270-272
    need(lowmem ? sin_ >= n : (wkn >= n && skn >= n && sin_ >= n),
         lowmem ? "sortperm_lowmem: scratch buffer too small" : "sortperm: scratch buffers too small");
    need(n <= static_cast<std::uint64_t>(std::numeric_limits<I>::max()), "sortperm: index type too narrow");
    need(n == 0 || (data && out), "sortperm: null buffer");
    using V = std::make_unsigned_t<I>;
    if (n == 1) AKB_CUDA(cudaMemsetAsync(out, 0, sizeof(I), c->stream));
    else if (n > 1) akb::wide_sortperm<T, V>(c, data, n, reinterpret_cast<V*>(out), desc != 0);
    akb::ctx_finish(c);
}

extern "C" {

const char* ak_last_error(void) { return g_err.c_str(); }
const char* ak_version(void) { return "ak-b200 0.1 (sm_100a)"; }

int ak_ctx_create(int device, void* stream, ak_ctx** out) {
    return guard([&] {
        need(out != nullptr, "ak_ctx_create: null out");
        AKB_CUDA(cudaSetDevice(device));
        auto c = std::make_unique<ak_ctx>();
        c->device = device;
        if (stream) {
            c->stream = static_cast<cudaStream_t>(stream);
        } else {
            AKB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        AKB_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        AKB_CUDA(cudaMalloc(&c->small, akb::SMALL_BYTES));
        c->small_bytes = akb::SMALL_BYTES;
        AKB_CUDA(cudaMemsetAsync(c->small, 0, akb::SMALL_BYTES, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        *out = c.release();
    });
}

int ak_ctx_destroy(ak_ctx* c) {
    return guard([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        for (auto& g : c->graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        if (c->aux) cudaFree(c->aux);
        if (c->lookback) cudaFree(c->lookback);
        if (c->scan_flags) cudaFree(c->scan_flags);
        if (c->scan_vals) cudaFree(c->scan_vals);
        if (c->small) cudaFree(c->small);
        if (c->split) cudaFree(c->split);
        if (c->cuts) cudaFree(c->cuts);
        if (c->msd) cudaFree(c->msd);
        if (c->msd3) cudaFree(c->msd3);
        if (c->stage) cudaFree(c->stage);
        if (c->work) cudaFree(c->work);
        if (c->pinned) cudaFreeHost(c->pinned);
        for (auto& b : c->free_blocks) cudaFree(b.second);
        for (auto& t : c->pending) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        for (auto& e : c->event_pool) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

int ak_ctx_set_blocking(ak_ctx* c, int blocking) {
    return guard([&] {
        ctx_lock g(c);
        c->blocking = blocking ? 1 : 0;
    });
}

int ak_ctx_synchronize(ak_ctx* c) {
    return guard([&] {
        ctx_lock g(c);
        AKB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ak_ctx_reserve(ak_ctx* c, uint64_t bytes) {
    return guard([&] {
        ctx_lock g(c);
        akb::ctx_reserve_aux(c, bytes);
    });
}

int ak_ctx_set_profiling(ak_ctx* c, int on) {
    return guard([&] {
        ctx_lock g(c);
        c->profiling = on ? 1 : 0;
    });
}

int ak_ctx_kernel_time(ak_ctx* c, int family, double* ms, uint64_t* launches) {
    return guard([&] {
        ctx_lock g(c);
        need(family >= 0 && family < 10, "ak_ctx_kernel_time: bad family");
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        akb::ctx_prof_resolve(c);
        if (ms) *ms = c->family_ms[family];
        if (launches) *launches = c->family_count[family];
    });
}

int ak_ctx_reset_kernel_time(ak_ctx* c) {
    return guard([&] {
        ctx_lock g(c);
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        akb::ctx_prof_resolve(c);
        for (int i = 0; i < 16; ++i) {
            c->family_ms[i] = 0;
            c->family_count[i] = 0;
        }
    });
}

uint64_t ak_ctx_kernel_launches(const ak_ctx* c) { return c ? c->kernel_launches : 0; }
void* ak_ctx_stream(const ak_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

// ak_malloc / ak_free keep freed blocks on the ctx and hand them out again (smallest block
// that fits and is at most twice the request), so a caller that stages through fresh device
// buffers on every call -- the C++ headers with host spans, ak_bench without
// --device-resident -- does not pay a GiB-sized cudaMalloc / cudaFree per call. At most
// 1/4 of the device memory (or 16 GiB) is held; ak_ctx_destroy releases everything.
namespace {
std::size_t free_cap(ak_ctx* c) {
    std::size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        (void)cudaGetLastError();
        tot = std::size_t(64) << 30;
    }
    (void)c;
    return std::min<std::size_t>(tot / 4, std::size_t(16) << 30);
}
}  // namespace

int ak_malloc(ak_ctx* c, uint64_t bytes, void** out) {
    return guard([&] {
        ctx_lock g(c);
        need(out != nullptr, "ak_malloc: null out");
        const std::size_t want = bytes ? bytes : 1;
        std::size_t best = c->free_blocks.size();
        for (std::size_t i = 0; i < c->free_blocks.size(); ++i) {
            const std::size_t sz = c->free_blocks[i].first;
            if (sz >= want && sz <= 2 * want && (best == c->free_blocks.size() || sz < c->free_blocks[best].first))
                best = i;
        }
        if (best < c->free_blocks.size()) {
            *out = c->free_blocks[best].second;
            c->live_blocks.emplace_back(*out, c->free_blocks[best].first);
            c->free_bytes -= c->free_blocks[best].first;
            c->free_blocks.erase(c->free_blocks.begin() + static_cast<std::ptrdiff_t>(best));
            return;
        }
        AKB_CUDA(cudaMalloc(out, want));
        c->live_blocks.emplace_back(*out, want);
    });
}
int ak_free(ak_ctx* c, void* p) {
    return guard([&] {
        ctx_lock g(c);
        if (!p) return;
        AKB_CUDA(cudaStreamSynchronize(c->stream));  // the block may still be read by queued work
        std::size_t sz = 0;
        for (std::size_t i = 0; i < c->live_blocks.size(); ++i)
            if (c->live_blocks[i].first == p) {
                sz = c->live_blocks[i].second;
                c->live_blocks.erase(c->live_blocks.begin() + static_cast<std::ptrdiff_t>(i));
                break;
            }
        if (sz == 0) {  // not ours (or unknown): release it
            AKB_CUDA(cudaFree(p));
            return;
        }
        c->free_blocks.emplace_back(sz, p);
        c->free_bytes += sz;
        const std::size_t cap = free_cap(c);
        while (c->free_bytes > cap && !c->free_blocks.empty()) {  // oldest first
            AKB_CUDA(cudaFree(c->free_blocks.front().second));
            c->free_bytes -= c->free_blocks.front().first;
            c->free_blocks.erase(c->free_blocks.begin());
        }
    });
}
int ak_memcpy(ak_ctx* c, void* dst, const void* src, uint64_t bytes) {
    return guard([&] {
        ctx_lock g(c);
        if (bytes == 0) return;
        AKB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

uint64_t ak_sort_scratch_bytes(uint64_t n, int kb) { return n * static_cast<uint64_t>(kb); }
uint64_t ak_sort_by_key_scratch_bytes(uint64_t n, int kb, int vb) { return n * static_cast<uint64_t>(kb + vb); }
uint64_t ak_sortperm_scratch_bytes(uint64_t n, int kb, int ib) { return n * static_cast<uint64_t>(2 * kb + ib); }
uint64_t ak_sortperm_lowmem_scratch_bytes(uint64_t n, int ib) { return n * static_cast<uint64_t>(ib); }
uint64_t ak_sort_ctx_bytes(uint64_t n, int kb) {
    const uint64_t tile = akb::radix_tile_items(kb, 0);
    return ((n + tile - 1) / tile) * 256 * 8 + akb::SMALL_BYTES;
}

#define AK_DEFINE(S, T)                                                                                 \
    int ak_merge_sort_##S(ak_ctx* c, T* d, uint64_t n, T* s, uint64_t sn, int desc) {                   \
        return guard([&] { merge_sort_impl<T>(c, d, n, s, sn, desc); });                                \
    }                                                                                                    \
    int ak_merge_sort_host_##S(ak_ctx* c, T* h, uint64_t n, int desc) {                                 \
        return guard([&] { merge_sort_host_impl<T>(c, h, n, desc); });                                   \
    }                                                                                                    \
    int ak_merge_sort_by_key_##S##_b32(ak_ctx* c, T* k, uint64_t nk, void* p, uint64_t np, T* sk,       \
                                       uint64_t skn, void* sp, uint64_t spn, int desc) {                \
        return guard([&] { by_key_impl<T, std::uint32_t>(c, k, nk, p, np, sk, skn, sp, spn, desc); });  \
    }                                                                                                    \
    int ak_merge_sort_by_key_##S##_b64(ak_ctx* c, T* k, uint64_t nk, void* p, uint64_t np, T* sk,       \
                                       uint64_t skn, void* sp, uint64_t spn, int desc) {                \
        return guard([&] { by_key_impl<T, std::uint64_t>(c, k, nk, p, np, sk, skn, sp, spn, desc); });  \
    }                                                                                                    \
    int ak_sortperm_##S##_i32(ak_ctx* c, const T* d, uint64_t n, int32_t* o, uint64_t on, T* wk,        \
                              uint64_t wkn, T* sk, uint64_t skn, int32_t* si, uint64_t sin_, int desc) { \
        return guard([&] { sortperm_impl<T, std::int32_t>(c, d, n, o, on, wk, wkn, sk, skn, si, sin_, desc); }); \
    }                                                                                                    \
    int ak_sortperm_##S##_i64(ak_ctx* c, const T* d, uint64_t n, int64_t* o, uint64_t on, T* wk,        \
                              uint64_t wkn, T* sk, uint64_t skn, int64_t* si, uint64_t sin_, int desc) { \
        return guard([&] { sortperm_impl<T, std::int64_t>(c, d, n, o, on, wk, wkn, sk, skn, si, sin_, desc); }); \
    }                                                                                                    \
    int ak_sortperm_lowmem_##S##_i32(ak_ctx* c, const T* d, uint64_t n, int32_t* o, uint64_t on,        \
                                     int32_t* si, uint64_t sin_, int desc) {                            \
        return guard([&] { sortperm_lowmem_impl<T, std::int32_t>(c, d, n, o, on, si, sin_, desc); });   \
    }                                                                                                    \
    int ak_sortperm_lowmem_##S##_i64(ak_ctx* c, const T* d, uint64_t n, int64_t* o, uint64_t on,        \
                                     int64_t* si, uint64_t sin_, int desc) {                            \
        return guard([&] { sortperm_lowmem_impl<T, std::int64_t>(c, d, n, o, on, si, sin_, desc); });   \
    }                                                                                                    \
    int ak_reduce_##S(ak_ctx* c, const T* x, uint64_t n, int op, int map, T init, T* r) {               \
        return guard([&] { reduce_impl<T>(c, x, n, op, map, init, r, true); });                          \
    }                                                                                                    \
    int ak_reduce_device_##S(ak_ctx* c, const T* x, uint64_t n, int op, int map, T init, T* r) {        \
        return guard([&] { reduce_impl<T>(c, x, n, op, map, init, r, false); });                         \
    }                                                                                                    \
    int ak_accumulate_##S(ak_ctx* c, const T* x, uint64_t n, T* o, uint64_t on, int op, int inc,        \
                          T init, uint64_t chunk) {                                                      \
        return guard([&] { scan_impl<T>(c, x, n, o, on, op, inc, init, chunk); });                       \
    }                                                                                                    \
    int ak_merge_runs_##S(ak_ctx* c, int P, const T* const* runs, const uint64_t* lens, T* dst, T* scratch,  \
                          int desc) {                                                                  \
        return guard([&] { merge_runs_impl<T>(c, P, runs, lens, dst, scratch, desc); });               \
    }                                                                                                   \
    int ak_searchsorted_##S(ak_ctx* c, const T* h, uint64_t n, const T* nd, uint64_t m, int last,       \
                            int desc, int validate, uint64_t* o) {                                      \
        return guard([&] { search_impl<T>(c, h, n, nd, m, last, desc, validate, o); });                  \
    }                                                                                                    \
    int ak_sihsort_##S(ak_ctx* c, ak_comm* cm, const T* in, uint64_t n, T* out, uint64_t cap,           \
                       uint64_t* oc, const ak_sih_config* cfg, ak_sih_stats* st) {                      \
        return guard([&] { sihsort_impl<T>(c, cm, in, n, out, cap, oc, cfg, st); });                     \
    }                                                                                                    \
    int ak_sihsort_host_##S(ak_ctx* c, ak_comm* cm, const T* in, uint64_t n, T* out, uint64_t cap,      \
                            uint64_t* oc, const ak_sih_config* cfg, ak_sih_stats* st) {                 \
        return guard([&] { sihsort_host_impl<T>(c, cm, in, n, out, cap, oc, cfg, st); });                \
    }                                                                                                    \
    int ak_sihsort_loopback_##S(int dev, uint64_t P, const T* const* in, const uint64_t* n,             \
                                T* const* out, const uint64_t* cap, uint64_t* oc,                       \
                                const ak_sih_config* cfg, ak_sih_stats* st) {                           \
        return guard([&] { sihsort_loopback_impl<T>(dev, P, in, n, out, cap, oc, cfg, st); });           \
    }                                                                                                    \
    int ak_sihsort_perm_##S(ak_ctx* c, ak_comm* cm, const T* in, uint64_t n, T* out, uint64_t* idx,      \
                            uint64_t cap, uint64_t* oc, const ak_sih_config* cfg, ak_sih_stats* st) {   \
        return guard([&] { sihsort_perm_impl<T>(c, cm, in, n, out, idx, cap, oc, cfg, st); });           \
    }                                                                                                    \
    int ak_sihsort_perm_loopback_##S(int dev, uint64_t P, const T* const* in, const uint64_t* n,        \
                                     T* const* out, uint64_t* const* idx, const uint64_t* cap,          \
                                     uint64_t* oc, const ak_sih_config* cfg, ak_sih_stats* st) {        \
        return guard([&] { sihsort_perm_loopback_impl<T>(dev, P, in, n, out, idx, cap, oc, cfg, st); }); \
    }                                                                                                    \
    int ak_sample_local_##S(ak_ctx* c, const T* d, uint64_t n, uint64_t k, T* h, uint64_t* cnt) {        \
        return guard([&] { sample_local_impl<T>(c, d, n, k, h, cnt); });                                \
    }                                                                                                    \
    int ak_build_interpolated_histogram_##S(const T* smp, uint64_t m, uint64_t bins, long double* e,     \
                                            uint64_t* cts, uint64_t cap, uint64_t* nb, uint64_t* tot) {  \
        return guard([&] { histogram_impl<T>(smp, m, bins, e, cts, cap, nb, tot); });                   \
    }                                                                                                    \
    int ak_select_splitters_##S(const long double* e, const uint64_t* cts, uint64_t nb, uint64_t tot,    \
                                uint64_t world, T* out) {                                                \
        return guard([&] { select_impl<T>(e, cts, nb, tot, world, out); });                              \
    }                                                                                                    \
    int ak_refine_splitters_##S(ak_ctx* c, ak_comm* cm, const T* d, uint64_t n, T* spl, uint64_t m,      \
                                const ak_sih_config* cfg, uint64_t* rounds, int* conv, double* dev) {    \
        return guard([&] { refine_impl<T>(c, cm, d, n, spl, m, cfg, rounds, conv, dev); });              \
    }                                                                                                    \
    int ak_redistribute_##S(ak_ctx* c, ak_comm* cm, const T* d, uint64_t n, const T* spl, uint64_t m,    \
                            uint64_t nt, T* out, uint64_t cap, uint64_t* oc, uint64_t* sends,            \
                            uint64_t* bytes) {                                                           \
        return guard([&] { redistribute_impl<T>(c, cm, d, n, spl, m, nt, out, cap, oc, sends, bytes); }); \
    }

AK_DEFINE(i32, int32_t)
AK_DEFINE(u32, uint32_t)
AK_DEFINE(i64, int64_t)
AK_DEFINE(u64, uint64_t)
AK_DEFINE(f32, float)
AK_DEFINE(f64, double)

#define AK_DEFINE_WIDE(S, T)                                                                            \
    int ak_merge_sort_##S(ak_ctx* c, T* d, uint64_t n, T* s, uint64_t sn, int desc) {                   \
        return guard([&] { wide_merge_sort_impl<T>(c, d, n, s, sn, desc); });                           \
    }                                                                                                    \
    int ak_merge_sort_host_##S(ak_ctx* c, T* h, uint64_t n, int desc) {                                 \
        return guard([&] { wide_merge_sort_host_impl<T>(c, h, n, desc); });                              \
    }                                                                                                    \
    int ak_merge_sort_by_key_##S##_b32(ak_ctx* c, T* k, uint64_t nk, void* p, uint64_t np, T* sk,       \
                                       uint64_t skn, void* sp, uint64_t spn, int desc) {                \
        return guard([&] { wide_by_key_impl<T, std::uint32_t>(c, k, nk, p, np, sk, skn, sp, spn, desc); }); \
    }                                                                                                    \
    int ak_merge_sort_by_key_##S##_b64(ak_ctx* c, T* k, uint64_t nk, void* p, uint64_t np, T* sk,       \
                                       uint64_t skn, void* sp, uint64_t spn, int desc) {                \
        return guard([&] { wide_by_key_impl<T, std::uint64_t>(c, k, nk, p, np, sk, skn, sp, spn, desc); }); \
    }                                                                                                    \
    int ak_sortperm_##S##_i32(ak_ctx* c, const T* d, uint64_t n, int32_t* o, uint64_t on, T*,           \
                              uint64_t wkn, T*, uint64_t skn, int32_t*, uint64_t sin_, int desc) {       \
        return guard([&] { wide_sortperm_impl<T, std::int32_t>(c, d, n, o, on, wkn, skn, sin_, false, desc); }); \
    }                                                                                                    \
    int ak_sortperm_##S##_i64(ak_ctx* c, const T* d, uint64_t n, int64_t* o, uint64_t on, T*,           \
                              uint64_t wkn, T*, uint64_t skn, int64_t*, uint64_t sin_, int desc) {       \
        return guard([&] { wide_sortperm_impl<T, std::int64_t>(c, d, n, o, on, wkn, skn, sin_, false, desc); }); \
    }                                                                                                    \
    int ak_sortperm_lowmem_##S##_i32(ak_ctx* c, const T* d, uint64_t n, int32_t* o, uint64_t on,        \
                                     int32_t*, uint64_t sin_, int desc) {                               \
        return guard([&] { wide_sortperm_impl<T, std::int32_t>(c, d, n, o, on, 0, 0, sin_, true, desc); }); \
    }                                                                                                    \
    int ak_sortperm_lowmem_##S##_i64(ak_ctx* c, const T* d, uint64_t n, int64_t* o, uint64_t on,        \
                                     int64_t*, uint64_t sin_, int desc) {                               \
        return guard([&] { wide_sortperm_impl<T, std::int64_t>(c, d, n, o, on, 0, 0, sin_, true, desc); }); \
    }

AK_DEFINE_WIDE(i16, int16_t)
AK_DEFINE_WIDE(i128, ak_int128)

#define AK_DEFINE_DIST(S, T)                                                                               \
    int ak_reduce_all_##S(ak_ctx* c, ak_comm* cm, const T* x, uint64_t n, int op, int map, T init, T* r) {    \
        return guard([&] { reduce_all_impl<T>(c, cm, x, n, op, map, init, r); });                           \
    }                                                                                                       \
    int ak_accumulate_all_##S(ak_ctx* c, ak_comm* cm, const T* x, uint64_t n, T* o, uint64_t on, int op,     \
                              int inc, T init) {                                                            \
        return guard([&] { accumulate_all_impl<T>(c, cm, x, n, o, on, op, inc, init); });                   \
    }
AK_DEFINE_DIST(i32, int32_t)
AK_DEFINE_DIST(u32, uint32_t)
AK_DEFINE_DIST(i64, int64_t)
AK_DEFINE_DIST(u64, uint64_t)
AK_DEFINE_DIST(f32, float)
AK_DEFINE_DIST(f64, double)

#define AK_DEFINE_PRED(S, T)                                                                               \
    int ak_any_pred_##S(ak_ctx* c, const T* x, uint64_t n, int op, T v, int algo, int* r) {                  \
        return guard([&] { pred_impl<T>(c, x, n, op, v, 1, algo, r); });                                    \
    }                                                                                                       \
    int ak_all_pred_##S(ak_ctx* c, const T* x, uint64_t n, int op, T v, int algo, int* r) {                  \
        return guard([&] { pred_impl<T>(c, x, n, op, v, 0, algo, r); });                                    \
    }
AK_DEFINE_PRED(u8, uint8_t)
AK_DEFINE_PRED(i8, int8_t)
AK_DEFINE_PRED(i16, int16_t)
AK_DEFINE_PRED(i32, int32_t)
AK_DEFINE_PRED(u32, uint32_t)
AK_DEFINE_PRED(i64, int64_t)
AK_DEFINE_PRED(u64, uint64_t)
AK_DEFINE_PRED(f32, float)
AK_DEFINE_PRED(f64, double)

int ak_nccl_unique_id(void* out, uint64_t bytes) {
    return guard([&] {
        need(out && bytes >= sizeof(ncclUniqueId), "ak_nccl_unique_id: buffer too small");
        ncclUniqueId id;
        const ncclResult_t r = ncclGetUniqueId(&id);
        if (r != ncclSuccess) throw akb::transport_error(ncclGetErrorString(r));
        std::memcpy(out, &id, sizeof(id));
    });
}

int ak_comm_nccl_create(const void* uid, int nranks, int rank, int device, ak_comm** out) {
    return guard([&] {
        need(uid && out, "ak_comm_nccl_create: null argument");
        need(nranks >= 1 && rank >= 0 && rank < nranks, "ak_comm_nccl_create: bad rank");
        AKB_CUDA(cudaSetDevice(device));
        auto impl = std::make_unique<akb::nccl_comm>();
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof(id));
        const ncclResult_t r = ncclCommInitRank(&impl->comm, nranks, id, rank);
        if (r != ncclSuccess) throw akb::transport_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        impl->r = rank;
        impl->p = nranks;
        impl->device = device;
        auto c = std::make_unique<ak_comm>();
        c->impl = std::move(impl);
        *out = c.release();
    });
}

int ak_comm_callbacks_create(int nranks, int rank, void* user, ak_allgather_fn ag, ak_allreduce_u64_fn ar,
                             ak_exchange_fn ex, ak_comm** out) {
    return guard([&] {
        need(out && ag && ar && ex, "ak_comm_callbacks_create: null argument");
        need(nranks >= 1 && rank >= 0 && rank < nranks, "ak_comm_callbacks_create: bad rank");
        auto c = std::make_unique<ak_comm>();
        c->impl = std::make_unique<akb::callback_comm>(rank, nranks, user, ag, ar, ex);
        *out = c.release();
    });
}

int ak_comm_ipc_create(int nranks, int rank, int device, void* user, ak_allgather_fn ag, ak_allreduce_u64_fn ar,
                       ak_comm** out) {
    return guard([&] {
        need(out && ag && ar, "ak_comm_ipc_create: null argument");
        need(nranks >= 1 && rank >= 0 && rank < nranks, "ak_comm_ipc_create: bad rank");
        int ndev = 0;
        AKB_CUDA(cudaGetDeviceCount(&ndev));
        need(device >= 0 && device < ndev, "ak_comm_ipc_create: bad device");
        auto c = std::make_unique<ak_comm>();
        c->impl = std::make_unique<akb::ipc_comm>(rank, nranks, device, user, ag, ar);
        *out = c.release();
    });
}

int ak_comm_bytes_sent(const ak_comm* comm, uint64_t* out) {
    return guard([&] {
        need(comm && out, "ak_comm_bytes_sent: null argument");
        *out = comm->impl->payload_bytes_sent();
    });
}

int ak_world_create(int ranks, ak_world** out) { return ak_world_create_ex(ranks, 64, out); }

int ak_world_create_ex(int ranks, uint64_t queue_capacity, ak_world** out) {
    return guard([&] {
        need(out != nullptr, "ak_world_create: null output");
        need(ranks >= 1, "world: rank count must be >= 1");              // sim_comm.cpp:7-9
        need(queue_capacity >= 1, "world: queue capacity must be >= 1");  // sim_comm.cpp:10-12
        *out = new ak_world(ranks, queue_capacity);
    });
}

int ak_comm_send(ak_comm* comm, ak_ctx* c, int dest, const void* bytes, uint64_t n, int control) {
    return guard([&] {
        need(comm != nullptr, "send: null communicator");
        need(n == 0 || bytes, "send: null message");
        if (comm->host_p2p) {
            comm->impl->send_bytes(dest, bytes, n, control != 0);
            return;
        }
        ctx_lock g(c);
        self_comm self;
        comm_of(comm, self, c).send_bytes(dest, bytes, n, control != 0);
    });
}

int ak_comm_recv(ak_comm* comm, ak_ctx* c, int src, void* buf, uint64_t cap, uint64_t* n) {
    return guard([&] {
        need(comm && n, "recv: null argument");
        auto it = comm->pending.find(src);
        if (it == comm->pending.end()) {
            std::vector<char> m;
            if (comm->host_p2p) {
                m = comm->impl->recv_bytes(src);
            } else {
                ctx_lock g(c);
                self_comm self;
                m = comm_of(comm, self, c).recv_bytes(src);
            }
            it = comm->pending.emplace(src, std::move(m)).first;
        }
        *n = it->second.size();
        if (it->second.size() > cap) throw akb::capacity_error("recv: message larger than the buffer", *n);
        if (*n) std::memcpy(buf, it->second.data(), *n);
        comm->pending.erase(it);
    });
}

int ak_comm_allgather(ak_comm* comm, ak_ctx* c, const void* in, uint64_t bytes, void* out) {
    return guard([&] {
        need(bytes == 0 || (in && out), "allgather: null argument");
        if (comm && comm->host_p2p) {  // host-level collective: no ctx lock (ranks share no device state)
            comm->impl->allgather(in, bytes, out);
            comm->impl->count_collective();
            return;
        }
        ctx_lock g(c);
        self_comm self;
        akb::comm_iface& cm = comm_of(comm, self, c);
        cm.allgather(in, bytes, out);
        cm.count_collective();
    });
}

int ak_comm_counters(const ak_comm* comm, ak_rank_counters* out) {
    return guard([&] {
        need(comm && out, "counters: null argument");
        const auto k = comm->impl->counters();
        out->p2p_sends = k.p2p_sends;
        out->p2p_bytes = k.p2p_bytes;
        out->collective_ops = k.collective_ops;
        out->collective_sends = k.collective_sends;
        out->control_bytes_peak = k.control_bytes_peak;
    });
}

int ak_world_size(const ak_world* w) { return w ? w->w.P : 0; }

int ak_world_abort(ak_world* w) {
    return guard([&] {
        need(w != nullptr, "ak_world_abort: null world");
        w->w.abort();
    });
}

int ak_world_destroy(ak_world* w) {
    return guard([&] { delete w; });
}

int ak_comm_loopback_create(ak_world* w, int rank, ak_comm** out) {
    return guard([&] {
        need(w && out, "ak_comm_loopback_create: null argument");
        need(rank >= 0 && rank < w->w.P, "rank_comm: rank out of range");  // sim_comm.cpp:11-13
        auto impl = std::make_unique<akb::loopback_comm>(&w->w, rank, nullptr);
        auto c = std::make_unique<ak_comm>();
        c->host_p2p = true;
        c->impl = std::move(impl);
        *out = c.release();
    });
}

int ak_pointer_is_device(const void* p) {
    if (!p) return 0;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? 1 : 0;
}

int ak_comm_rank(const ak_comm* c) { return c ? c->impl->rank() : 0; }
int ak_comm_size(const ak_comm* c) { return c ? c->impl->size() : 1; }

int ak_comm_allreduce_sum_u64(ak_comm* comm, ak_ctx* c, uint64_t* v, uint64_t n) {
    return guard([&] {
        ctx_lock g(c);
        self_comm self;
        comm_of(comm, self, c).allreduce_sum_u64(v, n);
    });
}

int ak_comm_allreduce_max_f64(ak_comm* comm, ak_ctx* c, double* v, uint64_t n) {
    return guard([&] {
        ctx_lock g(c);
        self_comm self;
        akb::comm_iface& cm = comm_of(comm, self, c);
        std::vector<double> all(n * cm.size());
        cm.allgather(v, n * sizeof(double), all.data());
        for (uint64_t i = 0; i < n; ++i)
            for (int q = 0; q < cm.size(); ++q) v[i] = all[q * n + i] > v[i] ? all[q * n + i] : v[i];
    });
}

int ak_comm_barrier(ak_comm* comm, ak_ctx* c) {
    uint64_t one = 1;
    return ak_comm_allreduce_sum_u64(comm, c, &one, 1);
}

int ak_comm_destroy(ak_comm* c) {
    return guard([&] { delete c; });
}

int ak_bench_keys(uint64_t seed, uint64_t rank, uint64_t n, int code, void* out) {
    return guard([&] {
        need(n == 0 || out, "ak_bench_keys: null output");
        std::mt19937_64 rng(seed + 0x9e3779b97f4a7c15ULL * (rank + 1));  // bench.cpp:168
        auto ints = [&](auto* p) {
            using T = std::remove_pointer_t<decltype(p)>;
            for (uint64_t i = 0; i < n; ++i) p[i] = static_cast<T>(rng());  // bench.cpp:50-52
        };
        auto reals = [&](auto* p) {
            using T = std::remove_pointer_t<decltype(p)>;
            std::uniform_real_distribution<T> dist(T(-1e6), T(1e6));  // bench.cpp:55-58
            for (uint64_t i = 0; i < n; ++i) p[i] = dist(rng);
        };
        switch (code) {  // dtype codes of dtype.hpp:14-21, + u64 = 7, u32 = 8
            case 2: ints(static_cast<int32_t*>(out)); break;
            case 3: ints(static_cast<int64_t*>(out)); break;
            case 5: reals(static_cast<float*>(out)); break;
            case 6: reals(static_cast<double*>(out)); break;
            case 7: ints(static_cast<uint64_t*>(out)); break;
            case 8: ints(static_cast<uint32_t*>(out)); break;
            default: throw akb::invalid_argument("ak_bench_keys: unsupported dtype code");
        }
    });
}

}  // extern "C"
