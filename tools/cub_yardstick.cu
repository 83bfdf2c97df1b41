// cub_yardstick.cu -- ADVISORY yardstick only (CUB must not be used
// inside the product). Times CUB's radix sort / scan / reduce on the same shapes
// the product kernels are measured on, so the roofline fractions in profiles/
// have a library reference point on the same B200.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/cub_yardstick.cu -o build/cub_yardstick
//   build/cub_yardstick [log2n=28]
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
    std::vector<int64_t> h(n);
    std::mt19937_64 rng(42);
    for (auto& v : h) v = static_cast<int64_t>(rng());
    int64_t *k0, *k1;
    CK(cudaMalloc(&k0, n * 8));
    CK(cudaMalloc(&k1, n * 8));
    CK(cudaMemcpy(k0, h.data(), n * 8, cudaMemcpyHostToDevice));
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, n);
    size_t tb2 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb2, k0, k1, n);
    tb = std::max(tb, tb2) + (size_t(1) << 20);
    CK(cudaMalloc(&tmp, tb));
    float ms = time_ms([&] {
        size_t t = tb;
        cub::DeviceRadixSort::SortKeys(tmp, t, k0, k1, n);
    });
    std::printf("cub SortKeys int64 n=2^%d: %.3f ms  (%.1f GB/s keys)\n", lg, ms, n * 8 / 1e6 / ms);
    ms = time_ms([&] {
        size_t t = tb;
        cub::DeviceScan::InclusiveSum(tmp, t, k0, k1, n);
    });
    std::printf("cub InclusiveSum int64 n=2^%d: %.3f ms  (%.1f GB/s r+w)\n", lg, ms, n * 16 / 1e6 / ms);
    ms = time_ms([&] {
        size_t t = tb;
        cub::DeviceReduce::Sum(tmp, t, k0, k1, n);
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
    cub::DeviceRadixSort::SortPairs(nullptr, tb3, f0, f1, v0, v1, n);
    if (tb3 > tb) {
        CK(cudaFree(tmp));
        tb = tb3;
        CK(cudaMalloc(&tmp, tb));
    }
    ms = time_ms([&] {
        size_t t = tb;
        cub::DeviceRadixSort::SortPairs(tmp, t, f0, f1, v0, v1, n);
    });
    std::printf("cub SortPairs f32/i32 n=2^%d: %.3f ms\n", lg, ms);
    float* g = reinterpret_cast<float*>(k1);
    ms = time_ms([&] {
        size_t t = tb;
        cub::DeviceScan::InclusiveSum(tmp, t, f0, g, n);
    });
    std::printf("cub InclusiveSum f32 n=2^%d: %.3f ms  (%.1f GB/s r+w)\n", lg, ms, n * 8 / 1e6 / ms);
    return 0;
}
