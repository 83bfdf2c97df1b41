// ak/exec.hpp -- drop-in for the reference's proj/include/ak/exec.hpp (exec.hpp:13-98)
// on the B200 build. The dispatch handle gains exec_kind::cuda: an exec_backend owns one
// ak_ctx (device + CUDA stream + device scratch arena) of libak_cuda.so, shared by copies
// (exec.hpp:31-35). Every primitive taking the handle runs on the GPU and blocks until
// done. sequential()/threaded() are kept so reference call sites compile
// unchanged; in this build they also return a CUDA handle (there is no CPU path).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ak_cuda.h"

namespace ak {

namespace sim {
/// Transport-level failure (sim_comm.hpp:19-21): aborted world, NCCL failure.
struct transport_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// Collective-protocol failure (sim_comm.hpp:24-26): ranks disagree on configuration.
struct protocol_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
}  // namespace sim

enum class exec_kind { sequential, threaded, cuda };

/// Half-open index interval [begin, end) (exec.hpp:17-24).
struct index_range {
    std::size_t begin = 0;
    std::size_t end = 0;

    std::size_t size() const noexcept { return end - begin; }
    bool operator==(const index_range&) const = default;
};

/// Splits [0, n) into min(p, n) contiguous chunks, sizes differing by at most one, the
/// remainder spread one per chunk from the front (exec.cpp:11-30). p == 0 throws.
inline std::vector<index_range> partition(std::size_t n, std::size_t p) {
    if (p == 0) throw std::invalid_argument("partition: p must be >= 1");
    const std::size_t chunks = n < p ? n : p;
    std::vector<index_range> out;
    out.reserve(chunks);
    if (chunks == 0) return out;
    const std::size_t base = n / chunks, extra = n % chunks;
    std::size_t b = 0;
    for (std::size_t i = 0; i < chunks; ++i) {
        const std::size_t len = base + (i < extra ? 1 : 0);
        out.push_back({b, b + len});
        b += len;
    }
    return out;
}

/// Raised when a sihsort output capacity is too small (device-buffer overloads only).
struct capacity_error : std::runtime_error {
    std::uint64_t required;
    capacity_error(const std::string& m, std::uint64_t r) : std::runtime_error(m), required(r) {}
};

namespace detail {

/// Maps an ak_status to the reference's exception types (SURVEY.md §8(b) "Errors").
inline void check(int status, std::uint64_t required = 0) {
    if (status == AK_OK) return;
    const std::string msg = ak_last_error();
    switch (status) {
        case AK_EINVAL: throw std::invalid_argument(msg);
        case AK_EPROTOCOL: throw sim::protocol_error(msg);
        case AK_ETRANSPORT: throw sim::transport_error(msg);
        case AK_ECAPACITY: throw capacity_error(msg, required);
        default: throw std::runtime_error(msg);
    }
}

struct ctx_holder {
    ak_ctx* ctx = nullptr;
    int device = 0;
    explicit ctx_holder(int dev) : device(dev) { check(ak_ctx_create(dev, nullptr, &ctx)); }
    ctx_holder(const ctx_holder&) = delete;
    ctx_holder& operator=(const ctx_holder&) = delete;
    ~ctx_holder() {
        if (ctx) ak_ctx_destroy(ctx);
    }
};

inline int default_device() {
    const char* e = std::getenv("AK_DEVICE");
    return e ? std::atoi(e) : 0;
}

inline bool on_device(const void* p) { return p != nullptr && ak_pointer_is_device(p) == 1; }

}  // namespace detail

/// Execution handle: one GPU, one stream, one scratch arena. Copies share the context;
/// calls on one context are serialised and block the caller until complete.
class exec_backend {
public:
    static exec_backend cuda(int device = detail::default_device()) {
        return exec_backend(std::make_shared<detail::ctx_holder>(device));
    }
    /// Kept for source compatibility (exec.hpp:38): runs on the GPU in this build.
    static exec_backend sequential() { return cuda(); }
    /// Kept for source compatibility (exec.hpp:41): the worker count must be >= 1
    /// (exec.cpp:33-35) and is otherwise ignored: the work runs on the GPU.
    static exec_backend threaded(std::size_t thread_count) {
        if (thread_count == 0) throw std::invalid_argument("exec_backend::threaded: thread_count must be >= 1");
        return cuda();
    }
    static exec_backend threaded() { return cuda(); }

    exec_kind kind() const noexcept { return exec_kind::cuda; }
    std::size_t thread_count() const noexcept { return 1; }
    int device() const noexcept { return h_->device; }
    ak_ctx* ctx() const noexcept { return h_->ctx; }
    /// Device time per kernel family (AK_KF_*), for measurement tools.
    void set_profiling(bool on) const { detail::check(ak_ctx_set_profiling(h_->ctx, on ? 1 : 0)); }
    std::uint64_t kernel_launches() const noexcept { return ak_ctx_kernel_launches(h_->ctx); }

private:
    explicit exec_backend(std::shared_ptr<detail::ctx_holder> h) : h_(std::move(h)) {}
    std::shared_ptr<detail::ctx_holder> h_;
};

namespace detail {

/// Process-wide handle for the reference entry points that take no exec_backend
/// (search_first/search_last, rank_comm::all_reduce_sum).
inline const exec_backend& default_backend() {
    static const exec_backend ex = exec_backend::cuda();
    return ex;
}

/// Device buffer owned by one call (host-span overloads stage through HBM).
template <typename T>
struct device_buffer {
    ak_ctx* c = nullptr;
    T* p = nullptr;
    std::size_t n = 0;
    device_buffer(ak_ctx* ctx, std::size_t count) : c(ctx), n(count) {
        if (n) {
            void* v = nullptr;
            check(ak_malloc(c, n * sizeof(T), &v));
            p = static_cast<T*>(v);
        }
    }
    device_buffer(const device_buffer&) = delete;
    device_buffer& operator=(const device_buffer&) = delete;
    ~device_buffer() {
        if (p) ak_free(c, p);
    }
    void upload(const T* host, std::size_t count) {
        if (count) check(ak_memcpy(c, p, host, count * sizeof(T)));
    }
    void download(T* host, std::size_t count) const {
        if (count) check(ak_memcpy(c, host, p, count * sizeof(T)));
    }
};

}  // namespace detail

}  // namespace ak
