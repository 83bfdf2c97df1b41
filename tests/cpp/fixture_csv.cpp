// fixture_csv.cpp -- driver for tests/test_fixture_csv.py: the B200 build's SIHS fixture and
// CSV headers (include/ak/{fixture,csv,dtype}.hpp), exercised against the reference's own
// implementation (oracle/_ref). No GPU needed.
//   fixture_csv write <path> <rank> <dtype> <n> <seed>   keys: mt19937_64(seed) as in bench.cpp
//   fixture_csv read  <path> <dtype>                      prints "rank count sum_u64"
//   fixture_csv csv   <path>                              emits the records test_fixture_csv.py expects
//   fixture_csv parse <path>                              parses and re-emits to stdout
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <random>
#include <string>
#include <vector>

#include "ak/csv.hpp"
#include "ak/fixture.hpp"

template <typename T>
int do_write(const char* path, std::uint32_t rank, std::uint64_t n, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<T> v(n);
    for (auto& x : v) {
        if constexpr (std::is_integral_v<T>) x = static_cast<T>(rng());
        else x = std::uniform_real_distribution<T>(T(-1e6), T(1e6))(rng);
    }
    ak::write_fixture<T>(path, rank, std::span<const T>(v));
    return 0;
}

template <typename T>
int do_read(const char* path) {
    std::uint32_t rank = 0;
    const auto v = ak::read_fixture<T>(path, &rank);
    std::uint64_t sum = 0;
    for (const T& x : v) {
        std::uint64_t b = 0;
        std::memcpy(&b, &x, sizeof(T));
        sum = sum * 1099511628211ull + b;
    }
    std::printf("%u %llu %llu\n", rank, static_cast<unsigned long long>(v.size()), static_cast<unsigned long long>(sum));
    return 0;
}

std::vector<ak::bench::bench_record> sample_records() {
    std::vector<ak::bench::bench_record> r(3);
    r[0] = {"sort-weak", "i64", 100000, 1, 5, 1.25, 0.015625, 0.64, 1.25};
    r[1] = {"sihsort-sim", "f32", 268435456, 8, 3, 12.345678901234, 0.1, 1234.5678901, 271.6};
    r[2] = {"odd,\"name\"", "u64", 7, 2, 3, 1e-9, 0, 3.14159265358979, 2.0};
    return r;
}

int main(int argc, char** argv) {
    try {
        const std::string mode = argc > 1 ? argv[1] : "";
        if (mode == "write" && argc == 7) {
            const std::string dt = argv[4];
            const auto rank = static_cast<std::uint32_t>(std::stoul(argv[3]));
            const auto n = std::stoull(argv[5]);
            const auto seed = std::stoull(argv[6]);
            if (dt == "i32") return do_write<std::int32_t>(argv[2], rank, n, seed);
            if (dt == "i64") return do_write<std::int64_t>(argv[2], rank, n, seed);
            if (dt == "f32") return do_write<float>(argv[2], rank, n, seed);
            if (dt == "f64") return do_write<double>(argv[2], rank, n, seed);
            if (dt == "u64") return do_write<std::uint64_t>(argv[2], rank, n, seed);
        } else if (mode == "read" && argc == 4) {
            const std::string dt = argv[3];
            if (dt == "i32") return do_read<std::int32_t>(argv[2]);
            if (dt == "i64") return do_read<std::int64_t>(argv[2]);
            if (dt == "f32") return do_read<float>(argv[2]);
            if (dt == "f64") return do_read<double>(argv[2]);
            if (dt == "u64") return do_read<std::uint64_t>(argv[2]);
        } else if (mode == "csv" && argc == 3) {
            ak::bench::emit_csv(std::filesystem::path(argv[2]), sample_records());
            return 0;
        } else if (mode == "parse" && argc == 3) {
            ak::bench::emit_csv(std::cout, ak::bench::parse_csv(argv[2]));
            return 0;
        }
        std::cerr << "bad arguments\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
