// ak_common.cuh -- shared device/host helpers for libak_cuda.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libak_cuda is built for sm_100a (B200) only"
#endif

namespace akb {

// ---------------------------------------------------------------------------
// Errors. The C ABI maps these to status codes; the C++ drop-in headers map the
// codes back to the reference's exception types (sort.hpp:182-184 etc.).
// ---------------------------------------------------------------------------
struct invalid_argument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct protocol_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct transport_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct capacity_error : std::runtime_error {
    std::uint64_t required;
    capacity_error(const std::string& m, std::uint64_t req) : std::runtime_error(m), required(req) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define AKB_CUDA(x) ::akb::cuda_check((x), #x)

// ---------------------------------------------------------------------------
// Key traits: map a key to unsigned bits whose unsigned order equals the
// reference comparator order (std::less, sort.hpp:180). Floats: -0.0 is
// canonicalised to +0.0 first so that -0.0 == +0.0 as under operator< and a
// stable radix pass keeps their input order. NaN is
// unsupported, as in the reference.
// ---------------------------------------------------------------------------
template <typename T>
struct key_traits;

template <>
struct key_traits<std::uint32_t> {
    using bits = std::uint32_t;
    static constexpr int nbits = 32;
    __host__ __device__ static bits to_ordered(std::uint32_t v) { return v; }
};
template <>
struct key_traits<std::int32_t> {
    using bits = std::uint32_t;
    static constexpr int nbits = 32;
    __host__ __device__ static bits to_ordered(std::int32_t v) {
        return static_cast<bits>(v) ^ 0x80000000u;
    }
};
template <>
struct key_traits<std::uint64_t> {
    using bits = std::uint64_t;
    static constexpr int nbits = 64;
    __host__ __device__ static bits to_ordered(std::uint64_t v) { return v; }
};
template <>
struct key_traits<std::int64_t> {
    using bits = std::uint64_t;
    static constexpr int nbits = 64;
    __host__ __device__ static bits to_ordered(std::int64_t v) {
        return static_cast<bits>(v) ^ 0x8000000000000000ull;
    }
};
template <>
struct key_traits<float> {
    using bits = std::uint32_t;
    static constexpr int nbits = 32;
    __host__ __device__ static bits to_ordered(float v) {
        bits b;
        memcpy(&b, &v, 4);
        if (b == 0x80000000u) b = 0;  // -0.0 -> +0.0
        const bits mask = (b & 0x80000000u) ? 0xffffffffu : 0x80000000u;
        return b ^ mask;
    }
};
template <>
struct key_traits<double> {
    using bits = std::uint64_t;
    static constexpr int nbits = 64;
    __host__ __device__ static bits to_ordered(double v) {
        bits b;
        memcpy(&b, &v, 8);
        if (b == 0x8000000000000000ull) b = 0;
        const bits mask = (b & 0x8000000000000000ull) ? ~0ull : 0x8000000000000000ull;
        return b ^ mask;
    }
};

template <typename T>
__host__ __device__ inline typename key_traits<T>::bits ordered(T v, bool desc) {
    auto o = key_traits<T>::to_ordered(v);
    return desc ? static_cast<typename key_traits<T>::bits>(~o) : o;
}

// Strict "less" on keys with the reference semantics (operator< / std::greater).
template <typename T>
__host__ __device__ inline bool key_less(T a, T b, bool desc) {
    return desc ? (b < a) : (a < b);
}

__device__ __forceinline__ std::uint32_t lanemask_lt() {
    std::uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ std::uint64_t ld_relaxed_u64(const std::uint64_t* p) {
    std::uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(std::uint64_t* p, std::uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ std::uint32_t ld_acquire_u32(const std::uint32_t* p) {
    std::uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(std::uint32_t* p, std::uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16-byte look-back descriptors {value bits, status word}: one aligned 128-bit
// access, so a reader sees value and status from the same publication without a
// release/acquire pair (which compile to MEMBAR.ALL.GPU / CCTL.IVALL on sm_100a).
__device__ __forceinline__ void st_relaxed_desc(std::uint64_t* p, std::uint64_t value, std::uint64_t status) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(value), "l"(status) : "memory");
}
__device__ __forceinline__ void ld_relaxed_desc(const std::uint64_t* p, std::uint64_t& value, std::uint64_t& status) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(value), "=l"(status) : "l"(p) : "memory");
}

inline std::uint64_t ceil_div(std::uint64_t a, std::uint64_t b) { return (a + b - 1) / b; }

}  // namespace akb
