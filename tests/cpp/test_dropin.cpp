// test_dropin.cpp -- the reference's own test cases (proj/tests/test_primitives.cpp:36-204 and
// the SPEC.md known answers for sorting/sihsort) written against the B200
// drop-in headers include/ak/*.hpp. Only the operator spellings change (ak::plus instead of a
// generic lambda: callables cannot cross the C ABI). Sort results are checked against
// std::stable_sort (the reference merge sort is stable with identical tie order).
//
// Built by tests/test_dropin.py (g++ -std=c++20, linked to libak_cuda.so); runs on a GPU.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <numeric>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ak/distributed.hpp"
#include "ak/predicates.hpp"
#include "ak/reduce.hpp"
#include "ak/scan.hpp"
#include "ak/search.hpp"
#include "ak/sihsort.hpp"
#include "ak/sort.hpp"

namespace {

int g_checks = 0, g_fail = 0;
#define CHECK(...)                                                                   \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(__VA_ARGS__)) {                                                             \
            ++g_fail;                                                                \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, E)                                                     \
    do {                                                                             \
        ++g_checks;                                                                  \
        bool caught_ = false;                                                        \
        try {                                                                        \
            expr;                                                                    \
        } catch (const E&) {                                                         \
            caught_ = true;                                                          \
        } catch (...) {                                                              \
        }                                                                            \
        if (!caught_) {                                                              \
            ++g_fail;                                                                \
            std::fprintf(stderr, "%s:%d: expected %s from %s\n", __FILE__, __LINE__, #E, #expr); \
        }                                                                            \
    } while (0)

template <typename T>
std::vector<T> random_ints(std::mt19937_64& rng, std::size_t n, T lo, T hi) {
    std::uniform_int_distribution<T> d(lo, hi);
    std::vector<T> v(n);
    for (auto& x : v) x = d(rng);
    return v;
}

bool approx_rel(double a, double b, double tol) {  // test_utils.hpp:109-112
    const double scale = std::max({1.0, std::fabs(a), std::fabs(b)});
    return std::fabs(a - b) <= tol * scale;
}

const ak::exec_backend ex = ak::exec_backend::cuda();

void test_reduce() {
    std::vector<std::int64_t> data(100);
    std::iota(data.begin(), data.end(), 1);
    CHECK(ak::reduce<std::int64_t>(ak::plus{}, data, {0, 256}, ex) == 5050);
    const std::int64_t sentinel = std::numeric_limits<std::int64_t>::lowest();
    CHECK(ak::reduce<std::int64_t>(ak::maximum{}, std::span<const std::int64_t>{}, {sentinel, 256}, ex) == sentinel);

    std::mt19937_64 rng(7);
    const auto big = random_ints<std::int64_t>(rng, 100000, -10000, 10000);
    const std::int64_t want = std::accumulate(big.begin(), big.end(), std::int64_t{0});
    CHECK(ak::reduce<std::int64_t>(ak::plus{}, big, {0, 256}, ex) == want);
    CHECK(ak::reduce<std::int64_t>(std::plus<>{}, big, {0, 256}, ex) == want);
    CHECK(ak::reduce<std::int64_t>(ak::minimum{}, big, {std::numeric_limits<std::int64_t>::max(), 256}, ex) ==
          *std::min_element(big.begin(), big.end()));

    std::vector<float> f(100000);
    std::uniform_real_distribution<float> u(0.f, 1.f);
    for (auto& x : f) x = u(rng);
    double fw = 0;
    for (float x : f) fw += x;
    CHECK(approx_rel(ak::reduce<float>(ak::plus{}, f, {0.0f, 256}, ex), fw, 1e-5));

    const std::vector<int> small = {-3, 1, 2};
    CHECK(ak::mapreduce<int>(ak::absolute{}, ak::maximum{}, std::span<const int>(small), {0, 256}, ex) == 3);
    CHECK(ak::mapreduce<int>(ak::square{}, ak::plus{}, std::span<const int>(small), {0, 256}, ex) == 14);
}

void test_accumulate() {
    const std::vector<int> ones = {1, 1, 1, 1};
    auto inc = ak::accumulate<int>(ak::plus{}, ones, {ak::scan_mode::inclusive, 0, 4096}, ex);
    CHECK(inc == (std::vector<int>{1, 2, 3, 4}));
    const std::vector<int> xs = {1, 2, 3};
    auto exc = ak::accumulate<int>(ak::plus{}, xs, {ak::scan_mode::exclusive, 0, 4096}, ex);
    CHECK(exc == (std::vector<int>{0, 1, 3}));

    std::mt19937_64 rng(11);
    auto data = random_ints<std::int64_t>(rng, 100000, -10000, 10000);
    std::vector<std::int64_t> want(data.size());
    std::inclusive_scan(data.begin(), data.end(), want.begin());
    for (std::size_t chunk : {std::size_t{1}, std::size_t{7}, std::size_t{1024}}) {
        CHECK(ak::accumulate<std::int64_t>(ak::plus{}, data, {ak::scan_mode::inclusive, 0, chunk}, ex) == want);
    }
    // in place (scan.hpp:72-76) and argument errors before mutation (scan.hpp:32-37)
    auto inplace = data;
    ak::accumulate<std::int64_t>(ak::plus{}, std::span<const std::int64_t>(inplace),
                                 {ak::scan_mode::inclusive, 0, 4096}, ex, std::span<std::int64_t>(inplace));
    CHECK(inplace == want);
    std::vector<std::int64_t> short_out(10);
    CHECK_THROWS_AS(ak::accumulate<std::int64_t>(ak::plus{}, std::span<const std::int64_t>(data),
                                                 {ak::scan_mode::inclusive, 0, 4096}, ex,
                                                 std::span<std::int64_t>(short_out)),
                    std::invalid_argument);
    CHECK_THROWS_AS(ak::accumulate<std::int64_t>(ak::plus{}, data, {ak::scan_mode::inclusive, 0, 0}, ex),
                    std::invalid_argument);
    // non-neutral init seeds position 0 (scan.hpp:12-16)
    auto seeded = ak::accumulate<std::int64_t>(ak::plus{}, std::vector<std::int64_t>{1, 2, 3},
                                               {ak::scan_mode::inclusive, 100, 4096}, ex);
    CHECK(seeded == (std::vector<std::int64_t>{101, 103, 106}));
}

void test_search() {
    const std::vector<int> hay = {1, 2, 4, 4, 7};
    const std::vector<int> needles = {4, 0, 9};
    CHECK(ak::searchsorted<int>(hay, needles, ak::search_side::first, ex) == (std::vector<std::size_t>{2, 0, 5}));
    CHECK(ak::searchsorted<int>(hay, needles, ak::search_side::last, ex) == (std::vector<std::size_t>{4, 0, 5}));
    CHECK(ak::search_first<int>(hay, 4) == 2);
    CHECK(ak::search_last<int>(hay, 4) == 4);
    const std::vector<int> unsorted = {3, 1, 2};
    CHECK_THROWS_AS(ak::searchsorted<int>(unsorted, needles, ak::search_side::first, ex, std::less<int>{}, true),
                    std::invalid_argument);
}

void test_sort() {
    std::vector<int> a = {3, 2, 1};
    auto bufs = ak::sort_buffers<int>::with_capacity(3);
    ak::merge_sort(std::span<int>(a), bufs, ex);
    CHECK(a == (std::vector<int>{1, 2, 3}));

    std::mt19937_64 rng(42);
    std::vector<std::int64_t> k(1000000);
    for (auto& x : k) x = static_cast<std::int64_t>(rng());
    auto want = k;
    std::stable_sort(want.begin(), want.end());
    CHECK(ak::merge_sort_copy<std::int64_t>(k, ex) == want);
    auto desc = k;
    auto want_desc = k;
    std::stable_sort(want_desc.begin(), want_desc.end(), std::greater<std::int64_t>{});
    auto b2 = ak::sort_buffers<std::int64_t>::with_capacity(k.size());
    ak::merge_sort(std::span<std::int64_t>(desc), b2, ex, std::greater<std::int64_t>{});
    CHECK(desc == want_desc);

    // undersized scratch throws before mutation (sort.hpp:182-184)
    std::vector<int> keep = {5, 4, 3};
    std::vector<int> tiny(2);
    CHECK_THROWS_AS(ak::merge_sort(std::span<int>(keep), std::span<int>(tiny), ex), std::invalid_argument);
    CHECK(keep == (std::vector<int>{5, 4, 3}));

    // device-resident spans sort in place
    {
        const std::size_t n = 1 << 19;  // <= k.size()
        void *d = nullptr, *s = nullptr;
        ak::detail::check(ak_malloc(ex.ctx(), n * 8, &d));
        ak::detail::check(ak_malloc(ex.ctx(), n * 8, &s));
        ak::detail::check(ak_memcpy(ex.ctx(), d, k.data(), n * 8));
        ak::merge_sort(std::span<std::int64_t>(static_cast<std::int64_t*>(d), n),
                       std::span<std::int64_t>(static_cast<std::int64_t*>(s), n), ex);
        std::vector<std::int64_t> got(n), w(k.begin(), k.begin() + n);
        std::stable_sort(w.begin(), w.end());
        ak::detail::check(ak_memcpy(ex.ctx(), got.data(), d, n * 8));
        CHECK(got == w);
        ak_free(ex.ctx(), d);
        ak_free(ex.ctx(), s);
    }
}

void test_sortperm() {
    const std::vector<int> d = {30, 10, 20};
    CHECK(ak::sortperm<int>(d, ex) == (std::vector<std::size_t>{1, 2, 0}));
    CHECK(ak::sortperm_lowmem<int>(d, ex) == (std::vector<std::size_t>{1, 2, 0}));
    const std::vector<int> eq(5, 7);
    CHECK(ak::sortperm<int>(eq, ex) == (std::vector<std::size_t>{0, 1, 2, 3, 4}));
    // -0.0 == +0.0 keeps input order
    const std::vector<float> z = {+0.0f, -0.0f, 1.0f, -0.0f, +0.0f, -1.0f};
    CHECK((ak::sortperm<float, std::uint32_t>(z, ex)) == (std::vector<std::uint32_t>{5, 0, 1, 3, 4, 2}));
    CHECK((ak::sortperm_lowmem<float, std::int64_t>(z, ex)) == (std::vector<std::int64_t>{5, 0, 1, 3, 4, 2}));

    std::mt19937_64 rng(3);
    std::uniform_real_distribution<float> u(-1e6f, 1e6f);
    std::vector<float> f(300000);
    for (auto& x : f) x = u(rng);
    for (std::size_t i = 0; i < f.size(); i += 5) f[i] = f[1];  // ties
    std::vector<std::int32_t> want(f.size());
    std::iota(want.begin(), want.end(), 0);
    std::stable_sort(want.begin(), want.end(), [&](std::int32_t a, std::int32_t b) { return f[a] < f[b]; });
    CHECK((ak::sortperm<float, std::int32_t>(f, ex)) == want);
    CHECK((ak::sortperm_lowmem<float, std::int32_t>(f, ex)) == want);

    // by_key: ties keep payload order
    std::vector<int> keys = {2, 1, 2, 1};
    std::vector<std::int32_t> pay = {10, 30, 20, 40};
    auto kb = ak::sort_by_key_buffers<int, std::int32_t>::with_capacity(4);
    ak::merge_sort_by_key(std::span<int>(keys), std::span<std::int32_t>(pay), kb, ex);
    CHECK(keys == (std::vector<int>{1, 1, 2, 2}));
    CHECK(pay == (std::vector<std::int32_t>{30, 40, 10, 20}));
    std::vector<std::int32_t> bad(3);
    CHECK_THROWS_AS(ak::merge_sort_by_key(std::span<int>(keys), std::span<std::int32_t>(bad), kb, ex),
                    std::invalid_argument);
    // scratch contract: lowmem <= 2/3 of sortperm
    CHECK(3 * ak::sortperm_lowmem_buffers<std::size_t>::required_bytes(1000000) <=
          2 * ak::sortperm_buffers<std::int64_t, std::size_t>::required_bytes(1000000));
}

void test_sihsort() {
    // P=2, [1,2,9] and [3,8,10], splitter 5 -> rank0 {1,2,3}, rank1 {8,9,10}
    {
        ak::sim::world w(2);
        std::vector<std::vector<std::int64_t>> out(2);
        ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
            const auto r = comm.rank();
            const auto e = ak::exec_backend::cuda();
            std::vector<std::int64_t> mine = r == 0 ? std::vector<std::int64_t>{1, 2, 9}
                                                    : std::vector<std::int64_t>{3, 8, 10};
            out[r] = ak::sihsort<std::int64_t>(mine, comm, ak::sih_config{}, e).first;
        });
        CHECK(out[0] == (std::vector<std::int64_t>{1, 2, 3}));
        CHECK(out[1] == (std::vector<std::int64_t>{8, 9, 10}));
    }
    // all-equal 1000/rank at P=4 -> 4000/0/0/0, 4 rounds, not converged
    {
        ak::sim::world w(4);
        std::vector<std::size_t> sizes(4);
        std::vector<ak::sih_stats> stats(4);
        ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
            const auto e = ak::exec_backend::cuda();
            auto res = ak::sihsort<std::int64_t>(std::vector<std::int64_t>(1000, 7), comm, ak::sih_config{}, e,
                                                 ak::cuda_sorter{});
            sizes[comm.rank()] = res.first.size();
            stats[comm.rank()] = res.second;
        });
        CHECK(sizes == (std::vector<std::size_t>{4000, 0, 0, 0}));
        CHECK(stats[0].rounds_used == 4);
        CHECK(!stats[0].converged);
    }
    // uniform keys at P=4: globally sorted concatenation, multiset preserved
    {
        const std::size_t P = 4, n = 200000;
        ak::sim::world w(P);
        std::vector<std::vector<std::uint64_t>> in(P), out(P);
        std::vector<std::uint64_t> all;
        for (std::size_t r = 0; r < P; ++r) {
            std::mt19937_64 rng(42 + 0x9e3779b97f4a7c15ULL * (r + 1));  // bench.cpp:164-173
            in[r].resize(n);
            for (auto& x : in[r]) x = rng();
            all.insert(all.end(), in[r].begin(), in[r].end());
        }
        ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
            const auto e = ak::exec_backend::cuda();
            out[comm.rank()] = ak::sihsort<std::uint64_t>(in[comm.rank()], comm, ak::sih_config{}, e).first;
        });
        std::vector<std::uint64_t> cat;
        for (auto& o : out) cat.insert(cat.end(), o.begin(), o.end());
        std::sort(all.begin(), all.end());
        CHECK(cat == all);
    }
    // a rank failure aborts the world and is rethrown (sim_comm.hpp:203-208)
    {
        ak::sim::world w(2);
        bool threw = false;
        try {
            ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
                if (comm.rank() == 1) throw std::runtime_error("injected");
                const auto e = ak::exec_backend::cuda();
                (void)ak::sihsort<std::int64_t>(std::vector<std::int64_t>{1, 2, 3}, comm, ak::sih_config{}, e);
            });
        } catch (const std::runtime_error&) {
            threw = true;
        }
        CHECK(threw);
    }
}

void test_sihsort_perm() {  // the distributed sortperm extension: stable global order + permutation
    // P=2, [5,1,5] and [1,5,0] -> global keys [5,1,5,1,5,0]; stable order: 0@5, 1@1, 1@3, 5@0, 5@2, 5@4
    ak::sim::world w(2);
    std::vector<std::vector<float>> keys(2);
    std::vector<std::vector<std::uint64_t>> idx(2);
    ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
        const auto r = comm.rank();
        const auto e = ak::exec_backend::cuda();
        std::vector<float> mine = r == 0 ? std::vector<float>{5, 1, 5} : std::vector<float>{1, 5, 0};
        auto [k, i, st] = ak::sihsort_perm<float>(std::span<const float>(mine), comm, ak::sih_config{}, e);
        keys[r] = k;
        idx[r] = i;
    });
    std::vector<float> ck;
    std::vector<std::uint64_t> ci;
    for (int r = 0; r < 2; ++r) {
        ck.insert(ck.end(), keys[r].begin(), keys[r].end());
        ci.insert(ci.end(), idx[r].begin(), idx[r].end());
    }
    CHECK(ck == (std::vector<float>{0, 1, 1, 5, 5, 5}));
    CHECK(ci == (std::vector<std::uint64_t>{5, 1, 3, 0, 2, 4}));
}

void test_sihsort_stages() {  // SPEC.md:282-325 known answers for the stage functions
    const std::vector<std::int64_t> ten{1, 2, 3, 4, 5, 6, 7, 8, 9, 10};
    CHECK(ak::sample_local<std::int64_t>(ten, 3) == (std::vector<std::int64_t>{1, 6, 10}));
    CHECK(ak::sample_local<std::int64_t>(ten, 1) == (std::vector<std::int64_t>{6}));
    CHECK(ak::sample_local<std::int64_t>(ten, 99).size() == 10);                              // k clamps to n
    CHECK(ak::sample_local<std::int64_t>(std::span<const std::int64_t>{}, 4).empty());
    const std::vector<std::int64_t> two{0, 10};
    const auto h = ak::build_interpolated_histogram<std::int64_t>(two, 2);
    CHECK(h.bin_edges == (std::vector<long double>{0.0L, 5.0L, 10.0L}));
    CHECK(h.counts == (std::vector<std::uint64_t>{1, 1}));
    CHECK(h.total == 2);
    const auto deg = ak::build_interpolated_histogram<std::int64_t>(std::vector<std::int64_t>(5, 7), 4);
    CHECK(deg.counts == (std::vector<std::uint64_t>{5}));  // degenerate range -> one bin
    CHECK(ak::select_splitters<std::int64_t>(h, 2).values == (std::vector<std::int64_t>{5}));
    CHECK(ak::select_splitters<std::int64_t>(h, 1).values.empty());
    // redistribute: P=2, [1,2,9] / [3,8,10], splitter 5 -> rank0 [1,2,3], rank1 [9,8,10]
    // (source-rank concatenation, not merged); a key equal to the splitter goes to
    // the lower rank
    {
        ak::sim::world w(2);
        std::vector<std::vector<std::int64_t>> out(2), tie(2);
        ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
            const auto e = ak::exec_backend::cuda();
            const auto r = comm.rank();
            const std::vector<std::int64_t> mine = r == 0 ? std::vector<std::int64_t>{1, 2, 9}
                                                          : std::vector<std::int64_t>{3, 8, 10};
            out[r] = ak::redistribute<std::int64_t>(mine, ak::splitter_set<std::int64_t>{{5}}, comm, 6, e);
            const std::vector<std::int64_t> t = r == 0 ? std::vector<std::int64_t>{5, 6} : std::vector<std::int64_t>{4, 5};
            tie[r] = ak::redistribute<std::int64_t>(t, ak::splitter_set<std::int64_t>{{5}}, comm, 4, e);
        });
        CHECK(out[0] == (std::vector<std::int64_t>{1, 2, 3}));
        CHECK(out[1] == (std::vector<std::int64_t>{9, 8, 10}));
        CHECK(tie[0] == (std::vector<std::int64_t>{5, 4, 5}));
        CHECK(tie[1] == (std::vector<std::int64_t>{6}));
    }
    // refine_splitters: a bad splitter on uniform data is corrected to a balanced one
    {
        const std::size_t P = 2, n = 100000;
        ak::sim::world w(P);
        std::vector<ak::refine_result<std::int64_t>> res(P);
        ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
            const auto e = ak::exec_backend::cuda();
            std::vector<std::int64_t> mine(n);
            for (std::size_t i = 0; i < n; ++i) mine[i] = static_cast<std::int64_t>(i * P + comm.rank());
            res[comm.rank()] = ak::refine_splitters<std::int64_t>(mine, ak::splitter_set<std::int64_t>{{10}}, comm,
                                                                  ak::sih_config{}, e);
        });
        CHECK(res[0].converged && res[1].converged);
        CHECK(res[0].splitters.values == res[1].splitters.values);
        CHECK(res[0].rounds_used >= 2);
        const auto s = res[0].splitters.values[0];
        CHECK(s > 75000 && s < 125000);  // within imbalance_tol 0.25 of n_total / 2
    }
}

void test_rank_comm() {  // sim_comm.hpp:84-181: messaging, values, all_reduce(merge), counters
    const std::size_t P = 4;
    ak::sim::world w(P);
    std::vector<std::vector<std::int64_t>> got(P), red(P);
    std::vector<ak::sim::rank_counters> ctr(P);
    std::vector<std::string> err(P);
    ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
        const auto e = ak::exec_backend::cuda();
        const std::size_t r = comm.rank();
        // ring of payload messages, then a control message back
        const std::vector<std::int64_t> mine{static_cast<std::int64_t>(r), 10, 20};
        comm.send_values<std::int64_t>((r + 1) % P, mine, ak::sim::traffic_class::payload, e);
        got[r] = comm.recv_values<std::int64_t>((r + P - 1) % P, e);
        const std::byte b[3] = {std::byte{1}, std::byte{2}, std::byte{3}};
        comm.send((r + P - 1) % P, std::span<const std::byte>(b, 3), ak::sim::traffic_class::control, e);
        const auto back = comm.recv((r + 1) % P, e);
        if (back.size() != 3 || back[2] != std::byte{3}) err[r] = "control message";
        // a 3-byte message cannot be read as int64 values (sim_comm.hpp:108-112)
        comm.send((r + 1) % P, std::span<const std::byte>(b, 3), ak::sim::traffic_class::payload, e);
        try {
            (void)comm.recv_values<std::int64_t>((r + P - 1) % P, e);
            err[r] = "no transport_error";
        } catch (const ak::sim::transport_error&) {
        }
        // non-commutative merge: the reference's binomial tree order, identical on every rank
        red[r] = comm.all_reduce(std::vector<std::int64_t>{static_cast<std::int64_t>(r + 1)},
                                 [](std::vector<std::int64_t>& a, const std::vector<std::int64_t>& in) {
                                     a[0] = a[0] * 10 + in[0];
                                 },
                                 e);
        ctr[r] = comm.counters();
    });
    for (std::size_t r = 0; r < P; ++r) {
        CHECK(err[r].empty());
        CHECK(got[r] == (std::vector<std::int64_t>{static_cast<std::int64_t>((r + P - 1) % P), 10, 20}));
        CHECK(red[r] == (std::vector<std::int64_t>{154}));  // ((1*10+3)*10 + (2*10+4))
        CHECK(ctr[r].p2p_sends == 3);
        CHECK(ctr[r].p2p_bytes == 24 + 3 + 3);
        CHECK(ctr[r].collective_ops == 1);
        CHECK(ctr[r].control_bytes_peak == 3);
    }
    CHECK(ctr[0].collective_sends == 2 && ctr[1].collective_sends == 2);  // binomial tree, P = 4
    CHECK(ctr[2].collective_sends == 1 && ctr[3].collective_sends == 1);
    CHECK_THROWS_AS(ak::sim::world(0), std::invalid_argument);
    CHECK_THROWS_AS(ak::sim::world(2, 0), std::invalid_argument);
}

void test_predicates() {  // test_primitives.cpp:206-263 with comparison functors for the lambdas
    const std::vector<int> zeros(100, 0), ones(100, 1);
    for (auto algo : {ak::predicate_algo::early_exit, ak::predicate_algo::via_mapreduce}) {
        CHECK(!ak::any_pred<int>(zeros, ak::pred::gt<int>{0}, ex, algo));
        CHECK(ak::all_pred<int>(ones, ak::pred::eq<int>{1}, ex, algo));
        CHECK(!ak::any_pred<int>(std::span<const int>{}, ak::pred::gt<int>{0}, ex, algo));
        CHECK(ak::all_pred<int>(std::span<const int>{}, ak::pred::gt<int>{0}, ex, algo));
    }
    std::mt19937_64 rng(14);
    std::vector<std::uint8_t> bytes(100000);
    for (auto& b : bytes) b = (rng() & 0xfff) == 0 ? 1 : 0;  // sparse trues
    bool want = false;
    for (auto b : bytes) want = want || b != 0;
    CHECK(ak::any_pred<std::uint8_t>(bytes, ak::pred::ne<std::uint8_t>{0}, ex) == want);
    std::mt19937_64 r2(15);
    for (int inst = 0; inst < 300; ++inst) {
        const std::size_t n = r2() % 200;
        const auto data = random_ints<std::int32_t>(r2, n, -10000, 10000);
        const auto cut = static_cast<std::int32_t>(r2() % 20001) - 10000;
        bool any = false, all = true;
        for (auto v : data) {
            any = any || v < cut;
            all = all && v < cut;
        }
        CHECK(ak::any_pred<std::int32_t>(data, ak::pred::lt<std::int32_t>{cut}, ex) == any);
        CHECK(ak::all_pred<std::int32_t>(data, ak::pred::lt<std::int32_t>{cut}, ex,
                                         ak::predicate_algo::via_mapreduce) == all);
        CHECK(ak::all_pred<std::int32_t>(data, ak::pred::lt<std::int32_t>{cut}, ex) ==
              !ak::any_pred<std::int32_t>(data, ak::pred::ge<std::int32_t>{cut}, ex));  // duality
    }
}

void test_distributed_reduce_scan() {  // 4 ranks on one GPU: slices of the global reduce / scan
    const std::size_t P = 4;
    std::mt19937_64 rng(21);
    std::vector<std::vector<std::int64_t>> parts(P);
    std::vector<std::int64_t> all;
    for (std::size_t r = 0; r < P; ++r) {
        parts[r] = random_ints<std::int64_t>(rng, 10000 + 977 * r, -10000, 10000);
        all.insert(all.end(), parts[r].begin(), parts[r].end());
    }
    std::vector<std::int64_t> scan_all(all.size());
    std::inclusive_scan(all.begin(), all.end(), scan_all.begin());
    const std::int64_t total = scan_all.back();
    std::vector<std::int64_t> sums(P), mins(P);
    std::vector<std::vector<std::int64_t>> scans(P);
    ak::sim::world w(P);
    ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) {
        const auto e = ak::exec_backend::cuda();
        const auto r = comm.rank();
        sums[r] = ak::reduce_all<std::int64_t>(ak::plus{}, parts[r], {0, 256}, comm, e);
        mins[r] = ak::reduce_all<std::int64_t>(ak::minimum{}, parts[r], {std::numeric_limits<std::int64_t>::max(), 256},
                                               comm, e);
        scans[r] = ak::accumulate_all<std::int64_t>(ak::plus{}, parts[r], {ak::scan_mode::inclusive, 0, 4096}, comm, e);
    });
    std::vector<std::int64_t> cat;
    for (std::size_t r = 0; r < P; ++r) {
        CHECK(sums[r] == total);
        CHECK(mins[r] == *std::min_element(all.begin(), all.end()));
        cat.insert(cat.end(), scans[r].begin(), scans[r].end());
    }
    CHECK(cat == scan_all);
}

void test_partition() {  // test_exec.cpp:18-22
    CHECK(ak::partition(10, 3) == (std::vector<ak::index_range>{{0, 4}, {4, 7}, {7, 10}}));
    CHECK(ak::partition(2, 5).size() == 2);
    CHECK(ak::partition(0, 4).empty());
    CHECK_THROWS_AS(ak::partition(5, 0), std::invalid_argument);
}

}  // namespace

int main() {
    const std::pair<const char*, void (*)()> tests[] = {
        {"partition", test_partition}, {"reduce", test_reduce},     {"accumulate", test_accumulate},
        {"search", test_search},       {"sort", test_sort},         {"sortperm", test_sortperm},
        {"sihsort", test_sihsort},     {"sihsort_perm", test_sihsort_perm},     {"sihsort_stages", test_sihsort_stages},
        {"rank_comm", test_rank_comm}, {"predicates", test_predicates},
        {"distributed", test_distributed_reduce_scan}};
    for (const auto& [name, fn] : tests) {
        std::fprintf(stderr, "[ run ] %s\n", name);
        fn();
    }
    std::printf("test_dropin: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
