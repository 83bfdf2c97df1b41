// ak_bench -- the reference benchmark CLI's sorting subcommands (proj/tools/bench_main.cpp:67-93,
// src/bench.cpp:146-351) on the B200 build, written against the drop-in headers.
//
//   ak_bench sort-weak   [--per-rank N] [--ranks 1,2,4] [common]
//   ak_bench sort-strong [--n N]        [--ranks 1,2,4] [common]
//   ak_bench sihsort-sim [--per-rank N] [--ranks 4] [--load-fixtures DIR] [--save-fixtures DIR] [common]
//   common: --dtype i32|u32|i64|u64|f32|f64  --reps N(>=3)  --warmup N(>=1)  --seed S  --csv PATH
//           --cost-ratio R  --threads LIST (accepted, unused: the work runs on the GPU)
//           --transport loopback|nccl   --device-resident
//
// Same inputs (mt19937_64(seed + 0x9e3779b97f4a7c15*(r+1)), bench.cpp:164-173), same weak/strong
// per-rank counts (bench.cpp:175-190), same record table, CSV header and sihsort-sim stats block,
// same exit codes (0 ok, 2 usage error, 1 runtime failure). Ranks: `loopback` runs P logical
// ranks on GPU 0 (the reference's in-process world); `nccl` runs rank r on GPU r over NCCL (one
// host thread per GPU). By default, like the reference, each timed run sorts host vectors
// (H2D + device sort + D2H per rank); --device-resident keeps inputs and outputs in HBM.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "ak/csv.hpp"
#include "ak/fixture.hpp"
#include "ak/sihsort.hpp"

namespace {

struct usage_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

struct request {
    std::string which;
    std::string dtype = "f32";
    std::uint64_t n = 1'000'000, per_rank = 100'000;
    std::vector<std::uint64_t> ranks;
    std::uint64_t reps = 5, warmup = 1, seed = 42;
    double cost_ratio = 1.0;
    std::string csv, load_dir, save_dir, transport = "loopback";
    bool device_resident = false;
};

std::vector<std::uint64_t> parse_list(const std::string& s) {
    std::vector<std::uint64_t> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
        if (tok.empty()) throw usage_error("empty list element");
        out.push_back(std::stoull(tok));
    }
    return out;
}

template <typename T>
std::vector<T> random_keys(std::mt19937_64& rng, std::size_t count) {  // bench.cpp:44-62
    std::vector<T> out(count);
    if constexpr (std::is_integral_v<T>) {
        for (auto& v : out) v = static_cast<T>(rng());
    } else {
        std::uniform_real_distribution<T> dist(T(-1e6), T(1e6));
        for (auto& v : out) v = dist(rng);
    }
    return out;
}

std::vector<std::uint64_t> per_rank_counts(const request& req, std::uint64_t ranks) {  // bench.cpp:175-190
    std::vector<std::uint64_t> c(ranks, req.per_rank);
    if (req.which == "sort-strong")
        for (std::uint64_t r = 0; r < ranks; ++r) c[r] = req.n / ranks + (r < req.n % ranks ? 1 : 0);
    return c;
}

struct timing {
    double mean_ms = 0, stddev_ms = 0;
};

template <typename Body>
timing time_reps(std::uint64_t reps, std::uint64_t warmup, Body&& body) {  // bench.hpp:128-150
    for (std::uint64_t i = 0; i < warmup; ++i) body();
    std::vector<double> ms(reps);
    for (std::uint64_t i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        body();
        ms[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    timing t;
    for (double v : ms) t.mean_ms += v;
    t.mean_ms /= static_cast<double>(reps);
    if (reps > 1) {
        double ss = 0;
        for (double v : ms) ss += (v - t.mean_ms) * (v - t.mean_ms);
        t.stddev_ms = std::sqrt(ss / static_cast<double>(reps - 1));
    }
    return t;
}

struct world_result {
    std::vector<ak::sih_stats> stats;
    std::vector<std::uint64_t> out_counts;
};

// Per-rank state created once, outside the timed region: an exec handle (device context
// and scratch) per rank, NCCL communicators, and device-resident buffers when requested.
template <typename T>
struct world_state {
    std::vector<ak::exec_backend> ex;
    std::vector<std::unique_ptr<ak::nccl::rank_comm>> nccl;
    std::vector<void*> din, dout;
    std::vector<std::uint64_t> cap;
    ~world_state() {
        for (std::size_t r = 0; r < din.size(); ++r) {
            if (din[r]) ak_free(ex[r].ctx(), din[r]);
            if (dout[r]) ak_free(ex[r].ctx(), dout[r]);
        }
    }
};

template <typename T>
void setup(const request& req, const std::vector<std::vector<T>>& in, world_state<T>& ws) {
    const std::size_t P = in.size();
    const bool nccl = req.transport == "nccl";
    for (std::size_t r = 0; r < P; ++r) ws.ex.push_back(ak::exec_backend::cuda(nccl ? static_cast<int>(r) : 0));
    if (nccl) {
        const auto id = ak::nccl::make_unique_id();
        ws.nccl.resize(P);
        std::vector<std::thread> th;  // ncclCommInitRank blocks until every rank joins
        std::vector<std::exception_ptr> err(P);
        for (std::size_t r = 0; r < P; ++r)
            th.emplace_back([&, r] {
                try {
                    ws.nccl[r] = std::make_unique<ak::nccl::rank_comm>(id, P, r, static_cast<int>(r));
                } catch (...) {
                    err[r] = std::current_exception();
                }
            });
        for (auto& t : th) t.join();
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
    }
    if (req.device_resident) {
        std::uint64_t total = 0;
        for (auto& v : in) total += v.size();
        ws.din.assign(P, nullptr);
        ws.dout.assign(P, nullptr);
        ws.cap.assign(P, total + 65536);  // any rank may receive everything (skewed keys)
        for (std::size_t r = 0; r < P; ++r) {
            ak::detail::check(ak_malloc(ws.ex[r].ctx(), std::max<std::size_t>(1, in[r].size()) * sizeof(T), &ws.din[r]));
            ak::detail::check(ak_malloc(ws.ex[r].ctx(), ws.cap[r] * sizeof(T), &ws.dout[r]));
            ak::detail::check(ak_memcpy(ws.ex[r].ctx(), ws.din[r], in[r].data(), in[r].size() * sizeof(T)));
        }
    }
}

// One rank's sort: host vectors (reference semantics) or device-resident buffers.
template <typename T, typename Comm>
void rank_sort(const request& req, const std::vector<T>& in, Comm& comm, world_state<T>& ws, world_result& res,
               std::size_t r) {
    if (!req.device_resident) {
        auto [out, st] = ak::sihsort<T>(in, comm, ak::sih_config{}, ws.ex[r]);
        res.stats[r] = st;
        res.out_counts[r] = out.size();
        return;
    }
    ak::sih_stats st;
    res.out_counts[r] = ak::sihsort_device<T>(std::span<const T>(static_cast<const T*>(ws.din[r]), in.size()),
                                              std::span<T>(static_cast<T*>(ws.dout[r]), ws.cap[r]), comm,
                                              ak::sih_config{}, ws.ex[r], &st);
    res.stats[r] = st;
}

template <typename T>
world_result run_world_sort(const request& req, const std::vector<std::vector<T>>& inputs, world_state<T>& ws) {
    const std::size_t P = inputs.size();
    world_result res;
    res.stats.resize(P);
    res.out_counts.resize(P);
    if (req.transport == "nccl") {  // one host thread per GPU, one NCCL rank each
        std::vector<std::thread> th;
        std::vector<std::exception_ptr> err(P);
        for (std::size_t r = 0; r < P; ++r)
            th.emplace_back([&, r] {
                try {
                    rank_sort<T>(req, inputs[r], *ws.nccl[r], ws, res, r);
                } catch (...) {
                    err[r] = std::current_exception();
                }
            });
        for (auto& t : th) t.join();
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
        return res;
    }
    ak::sim::world w(P);  // P logical ranks on GPU 0 (sim_comm.hpp:41-218)
    ak::sim::run_ranks(w, [&](ak::sim::rank_comm& comm) { rank_sort<T>(req, inputs[comm.rank()], comm, ws, res, comm.rank()); });
    return res;
}

template <typename T>
std::vector<std::vector<T>> rank_inputs(const request& req, std::uint64_t ranks) {
    std::vector<std::vector<T>> in(ranks);
    if (!req.load_dir.empty()) {
        for (std::uint64_t r = 0; r < ranks; ++r) {
            const auto path = std::filesystem::path(req.load_dir) / ("rank_" + std::to_string(r) + ".sihs");
            std::uint32_t fr = 0;
            in[r] = ak::read_fixture<T>(path, &fr);
            if (fr != r)
                throw std::runtime_error("fixture " + path.string() + " carries rank " + std::to_string(fr) +
                                         ", expected " + std::to_string(r));
        }
    } else {
        const auto counts = per_rank_counts(req, ranks);
        for (std::uint64_t r = 0; r < ranks; ++r) {
            std::mt19937_64 rng(req.seed + 0x9e3779b97f4a7c15ULL * (r + 1));
            in[r] = random_keys<T>(rng, counts[r]);
        }
    }
    if (!req.save_dir.empty()) {
        std::filesystem::create_directories(req.save_dir);
        for (std::uint64_t r = 0; r < ranks; ++r)
            ak::write_fixture<T>(std::filesystem::path(req.save_dir) / ("rank_" + std::to_string(r) + ".sihs"),
                                 static_cast<std::uint32_t>(r), std::span<const T>(in[r]));
    }
    return in;
}

template <typename T>
std::vector<ak::bench::bench_record> run_typed(const request& req, std::string* stats_text) {
    std::vector<ak::bench::bench_record> records;
    for (std::uint64_t ranks : req.ranks) {
        if (ranks == 0) throw usage_error("ranks must be >= 1");
        const auto inputs = rank_inputs<T>(req, ranks);
        std::uint64_t total = 0;
        for (auto& v : inputs) total += v.size();
        world_state<T> ws;
        setup<T>(req, inputs, ws);
        world_result last;
        const timing t = time_reps(req.reps, req.warmup, [&] { last = run_world_sort<T>(req, inputs, ws); });
        ak::bench::bench_record rec;
        rec.case_name = req.which;
        rec.dtype = ak::dtype_name(ak::dtype_of<T>());
        rec.n = total / ranks;
        rec.workers = ranks;
        rec.reps = req.reps;
        rec.mean_ms = t.mean_ms;
        rec.stddev_ms = t.stddev_ms;
        rec.throughput_gbps = static_cast<double>(total * sizeof(T)) / 1e9 / (t.mean_ms / 1e3);  // bench.cpp:74-76
        rec.normalized_ms = t.mean_ms * req.cost_ratio;
        records.push_back(rec);
        if (req.which == "sihsort-sim" && stats_text) {  // bench.cpp:336-349
            double max_imb = 0;
            const double mean_out = static_cast<double>(total) / static_cast<double>(ranks);
            for (auto c : last.out_counts)
                if (mean_out > 0) max_imb = std::max(max_imb, static_cast<double>(c) / mean_out);
            std::ostringstream os;
            os << "case=sihsort-sim\n"
               << "dtype=" << rec.dtype << "\n"
               << "ranks=" << ranks << "\n"
               << "total_elements=" << total << "\n"
               << "rounds=" << last.stats[0].rounds_used << "\n"
               << "converged=" << (last.stats[0].converged ? 1 : 0) << "\n"
               << "max_imbalance=" << max_imb << "\n";
            for (std::uint64_t r = 0; r < ranks; ++r)
                os << "msg_count_rank_" << r << "=" << last.stats[r].redistribution_sends << "\n"
                   << "collectives_rank_" << r << "=" << last.stats[r].collective_ops << "\n"
                   << "out_count_rank_" << r << "=" << last.stats[r].output_count << "\n";
            *stats_text = os.str();
            break;  // sihsort-sim runs one rank count
        }
    }
    return records;
}

void print_records(const std::vector<ak::bench::bench_record>& records) {  // bench_main.cpp:16-28
    std::printf("%-12s %-6s %12s %8s %6s %12s %12s %14s %14s\n", "case", "dtype", "n", "workers", "reps", "mean_ms",
                "stddev_ms", "gbps", "normalized_ms");
    for (const auto& r : records)
        std::printf("%-12s %-6s %12llu %8llu %6llu %12.4f %12.4f %14.4f %14.4f\n", r.case_name.c_str(),
                    r.dtype.c_str(), static_cast<unsigned long long>(r.n), static_cast<unsigned long long>(r.workers),
                    static_cast<unsigned long long>(r.reps), r.mean_ms, r.stddev_ms, r.throughput_gbps,
                    r.normalized_ms);
}

request parse(int argc, char** argv) {
    if (argc < 2) throw usage_error("a subcommand is required: sort-weak | sort-strong | sihsort-sim");
    request req;
    req.which = argv[1];
    if (req.which == "rbf" || req.which == "ljg")
        throw usage_error(req.which + " is an arithmetic benchmark outside the B200 build's sorting path");
    if (req.which != "sort-weak" && req.which != "sort-strong" && req.which != "sihsort-sim")
        throw usage_error("unknown subcommand " + req.which);
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw usage_error("option " + a + " needs a value");
            return argv[++i];
        };
        if (a == "--dtype") req.dtype = val();
        else if (a == "--reps") req.reps = std::stoull(val());
        else if (a == "--warmup") req.warmup = std::stoull(val());
        else if (a == "--seed") req.seed = std::stoull(val());
        else if (a == "--cost-ratio") req.cost_ratio = std::stod(val());
        else if (a == "--csv") req.csv = val();
        else if (a == "--threads") (void)parse_list(val());
        else if (a == "--ranks") req.ranks = parse_list(val());
        else if (a == "--n" && req.which == "sort-strong") req.n = std::stoull(val());
        else if (a == "--per-rank" && req.which != "sort-strong") req.per_rank = std::stoull(val());
        else if (a == "--load-fixtures" && req.which == "sihsort-sim") req.load_dir = val();
        else if (a == "--save-fixtures" && req.which == "sihsort-sim") req.save_dir = val();
        else if (a == "--transport") req.transport = val();
        else if (a == "--device-resident") req.device_resident = true;
        else throw usage_error("unknown option " + a + " for " + req.which);
    }
    if (req.ranks.empty()) req.ranks = {req.which == "sihsort-sim" ? 4ull : 1ull};
    if (req.reps < 3) throw usage_error("--reps must be >= 3");  // bench.cpp:82-89
    if (req.warmup < 1) throw usage_error("--warmup must be >= 1");
    if (req.transport != "loopback" && req.transport != "nccl") throw usage_error("--transport loopback|nccl");
    return req;
}

}  // namespace

int main(int argc, char** argv) {
    request req;
    try {
        req = parse(argc, argv);
    } catch (const std::exception& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return 2;
    }
    try {
        const auto code = ak::dtype_from_name(req.dtype);
        if (!code) {
            std::cerr << "unknown dtype: " << req.dtype << "\n";
            return 2;
        }
        std::string stats;
        std::vector<ak::bench::bench_record> records;
        switch (*code) {
            case ak::dtype_code::i32: records = run_typed<std::int32_t>(req, &stats); break;
            case ak::dtype_code::u32: records = run_typed<std::uint32_t>(req, &stats); break;
            case ak::dtype_code::i64: records = run_typed<std::int64_t>(req, &stats); break;
            case ak::dtype_code::u64: records = run_typed<std::uint64_t>(req, &stats); break;
            case ak::dtype_code::f32: records = run_typed<float>(req, &stats); break;
            case ak::dtype_code::f64: records = run_typed<double>(req, &stats); break;
            default:
                std::cerr << "usage error: dtype " << req.dtype << " has no device sort in the B200 build\n";
                return 2;
        }
        std::cout << stats;
        print_records(records);
        if (!req.csv.empty()) ak::bench::emit_csv(std::filesystem::path(req.csv), records);
    } catch (const usage_error& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
