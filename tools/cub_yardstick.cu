// cub_yardstick.cu -- ADVISORY yardstick only (CUB must not be used
// inside the product). Times CUB's radix sort / scan / reduce on the same shapes
// the product kernels are measured on, so the roofline fractions in profiles/
// have a library reference point on the same B200.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/cub_yardstick.cu -o build/cub_yardstick
//   build/cub_yardstick [log2n=28]
// Every CUB call's status is checked (r01's run printed 0.003 ms for SortKeys: the call had
// failed on a 64-bit item count and nothing noticed). Item counts are passed as int (n < 2^31).
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <random>
#include <vector>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)

template <typename F>
float time_ms(F&& f, int reps = 5) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    f();
    CK(cudaDeviceSynchronize());
    float best = 1e30f, sum = 0;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a));
        f();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
        sum += ms;
    }
    return sum / reps;
}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? std::atoi(argv[1]) : 28;
    const size_t n = size_t(1) << lg;
    if (lg > 30) {
        std::fprintf(stderr, "log2n <= 30\n");
        return 2;
    }
    const int ni = static_cast<int>(n);
    std::vector<int64_t> h(n);
    std::mt19937_64 rng(42);
    for (auto& v : h) v = static_cast<int64_t>(rng());
    int64_t *k0, *k1;
    CK(cudaMalloc(&k0, n * 8));
    CK(cudaMalloc(&k1, n * 8));
    CK(cudaMemcpy(k0, h.data(), n * 8, cudaMemcpyHostToDevice));
    void* tmp = nullptr;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, ni));
    size_t tb2 = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb2, k0, k1, ni));
    tb = std::max(tb, tb2) + (size_t(1) << 20);
    CK(cudaMalloc(&tmp, tb));
    float ms = time_ms([&] {
        size_t t = tb;
        CK(cub::DeviceRadixSort::SortKeys(tmp, t, k0, k1, ni));
    });
    {
        std::vector<int64_t> o(n);
        CK(cudaMemcpy(o.data(), k1, n * 8, cudaMemcpyDeviceToHost));
        for (size_t i = 1; i < n; ++i)
            if (o[i - 1] > o[i]) {
                std::fprintf(stderr, "cub SortKeys output not sorted at %zu\n", i);
                return 1;
            }
    }
    std::printf("cub SortKeys int64 n=2^%d: %.3f ms  (%.1f GB/s keys, output checked sorted)\n", lg, ms,
                n * 8 / 1e6 / ms);
    ms = time_ms([&] {
        size_t t = tb;
        CK(cub::DeviceScan::InclusiveSum(tmp, t, k0, k1, ni));
    });
    std::printf("cub InclusiveSum int64 n=2^%d: %.3f ms  (%.1f GB/s r+w)\n", lg, ms, n * 16 / 1e6 / ms);
    ms = time_ms([&] {
        size_t t = tb;
        CK(cub::DeviceReduce::Sum(tmp, t, k0, k1, ni));
    });
    std::printf("cub Reduce int64 n=2^%d: %.3f ms  (%.1f GB/s)\n", lg, ms, n * 8 / 1e6 / ms);
    // f32 keys + i32 payload (config 2 shape at n)
    float* f0 = reinterpret_cast<float*>(k0);
    float* f1 = reinterpret_cast<float*>(k1);
    int32_t* v0 = reinterpret_cast<int32_t*>(k0) + n;
    int32_t* v1 = reinterpret_cast<int32_t*>(k1) + n;
    std::uniform_real_distribution<float> U(-1e6f, 1e6f);
    std::vector<float> hf(n);
    for (auto& v : hf) v = U(rng);
    CK(cudaMemcpy(f0, hf.data(), n * 4, cudaMemcpyHostToDevice));
    size_t tb3 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb3, f0, f1, v0, v1, ni));
    if (tb3 > tb) {
        CK(cudaFree(tmp));
        tb = tb3;
        CK(cudaMalloc(&tmp, tb));
    }
    ms = time_ms([&] {
        size_t t = tb;
        CK(cub::DeviceRadixSort::SortPairs(tmp, t, f0, f1, v0, v1, ni));
    });
    std::printf("cub SortPairs f32/i32 n=2^%d: %.3f ms\n", lg, ms);
    float* g = reinterpret_cast<float*>(k1);
    ms = time_ms([&] {
        size_t t = tb;
        CK(cub::DeviceScan::InclusiveSum(tmp, t, f0, g, ni));
    });
    std::printf("cub InclusiveSum f32 n=2^%d: %.3f ms  (%.1f GB/s r+w)\n", lg, ms, n * 8 / 1e6 / ms);
    return 0;
}
