// predicates.cu -- any_pred / all_pred (reference include/ak/predicates.hpp:16-78).
//
// One grid-stride pass with 16-byte vector loads; `want` = true looks for an element
// satisfying the predicate (any), false for one violating it (all). The early-exit variant
// polls a device flag once per loop trip and stops every block once the outcome is decided
// (the reference's pred_poll_stride flag, predicates.hpp:24-52); the full-pass variant is
// the reference's via_mapreduce path. Both return identical results.
#include "predicates.cuh"

namespace akb {

namespace {

template <typename T>
__device__ __forceinline__ bool pred_eval(T x, int op, T v) {
    switch (op) {
        case PRED_LT: return x < v;
        case PRED_LE: return x <= v;
        case PRED_GT: return x > v;
        case PRED_GE: return x >= v;
        case PRED_EQ: return x == v;
        default: return x != v;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) pred_kernel(const T* __restrict__ x, std::uint64_t n, int op, T v, int want,
                                                   int early, unsigned* found) {
    constexpr int VEC = 16 / sizeof(T);
    const std::uint64_t S = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    const std::uint64_t g = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool w = want != 0;
    bool hit = false;
    const bool aligned = (reinterpret_cast<std::uintptr_t>(x) & 15) == 0;
    std::uint64_t done = 0;
    if (aligned) {
        const uint4* xv = reinterpret_cast<const uint4*>(x);
        const std::uint64_t nv = n / VEC;
        // block-uniform trip count, so the per-trip poll can be a block-wide vote
        for (std::uint64_t base = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x; base < nv; base += S) {
            if (early && __syncthreads_or(hit || *reinterpret_cast<volatile unsigned*>(found))) break;
            const std::uint64_t i = base + threadIdx.x;
            if (i < nv) {
                const uint4 q = __ldg(xv + i);
                const T* e = reinterpret_cast<const T*>(&q);
#pragma unroll
                for (int k = 0; k < VEC; ++k) hit |= pred_eval(e[k], op, v) == w;
            }
            if (early && hit) *reinterpret_cast<volatile unsigned*>(found) = 1u;
        }
        done = nv * VEC;
    }
    for (std::uint64_t i = done + g; i < n; i += S) hit |= pred_eval(x[i], op, v) == w;  // tail
    if (__any_sync(0xffffffffu, hit) && (threadIdx.x & 31) == 0) atomicOr(found, 1u);
}

}  // namespace

template <typename T>
bool find_decider(ak_ctx* c, const T* x, std::uint64_t n, int op, T v, bool want, bool early) {
    if (n == 0) return false;
    unsigned* flag = reinterpret_cast<unsigned*>(static_cast<char*>(c->small) + 196608 + 64);
    AKB_CUDA(cudaMemsetAsync(flag, 0, 4, c->stream));
    std::uint64_t blocks = ceil_div(n, 256 * (16 / sizeof(T)) * 4);
    if (blocks > static_cast<std::uint64_t>(c->sm_count) * 8) blocks = static_cast<std::uint64_t>(c->sm_count) * 8;
    if (blocks < 1) blocks = 1;
    const int tok = ctx_prof_begin(c, KF_OTHER);
    pred_kernel<T><<<static_cast<unsigned>(blocks), 256, 0, c->stream>>>(x, n, op, v, want ? 1 : 0, early ? 1 : 0,
                                                                          flag);
    AKB_CUDA(cudaGetLastError());
    ctx_prof_end(c, tok);
    c->kernel_launches += 1;
    unsigned* h = static_cast<unsigned*>(ctx_pinned(c, 4));
    AKB_CUDA(cudaMemcpyAsync(h, flag, 4, cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    return *h != 0;
}

#define AKB_INST(T) template bool find_decider<T>(ak_ctx*, const T*, std::uint64_t, int, T, bool, bool);
AKB_INST(std::uint8_t)
AKB_INST(std::int8_t)
AKB_INST(std::int16_t)
AKB_INST(std::int32_t)
AKB_INST(std::uint32_t)
AKB_INST(std::int64_t)
AKB_INST(std::uint64_t)
AKB_INST(float)
AKB_INST(double)

}  // namespace akb
