// ak/sim_comm.hpp -- drop-in for proj/include/ak/sim_comm.hpp (sim_comm.hpp:16-218), B200 build.
//
// Two communicators with the reference's method shape:
//   * ak::sim::world / rank_comm / run_ranks: P logical ranks in ONE process on ONE GPU,
//     one host thread per rank (the reference's in-process world, sim_comm.hpp:41-218).
//     Collectives are host-level; sihsort slices move device to device.
//   * ak::nccl::rank_comm: one rank per GPU (one process or thread each) over NCCL,
//     NVLink 5 / NVSwitch -- the production transport for the 8xB200 sample sort.
// Both abort on failure so blocked peers wake with sim::transport_error.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "ak/exec.hpp"

namespace ak {

namespace sim {

/// P logical ranks on one device (sim_comm.hpp:45-80). queue_capacity is accepted for
/// source compatibility; the device exchange needs no bounded FIFO.
class world {
public:
    explicit world(std::size_t ranks, std::size_t queue_capacity = 64) {
        (void)queue_capacity;
        if (ranks == 0) throw std::invalid_argument("world: rank count must be >= 1");
        detail::check(ak_world_create(static_cast<int>(ranks), &w_));
    }
    world(const world&) = delete;
    world& operator=(const world&) = delete;
    ~world() {
        if (w_) ak_world_destroy(w_);
    }
    std::size_t size() const noexcept { return static_cast<std::size_t>(ak_world_size(w_)); }
    void abort() noexcept { ak_world_abort(w_); }
    ak_world* handle() const noexcept { return w_; }

private:
    ak_world* w_ = nullptr;
};

/// Per-rank handle (sim_comm.hpp:84-181); used by one thread.
class rank_comm {
public:
    rank_comm(world& w, std::size_t rank) { detail::check(ak_comm_loopback_create(w.handle(), static_cast<int>(rank), &c_)); }
    rank_comm(const rank_comm&) = delete;
    rank_comm& operator=(const rank_comm&) = delete;
    ~rank_comm() {
        if (c_) ak_comm_destroy(c_);
    }
    std::size_t rank() const noexcept { return static_cast<std::size_t>(ak_comm_rank(c_)); }
    std::size_t world_size() const noexcept { return static_cast<std::size_t>(ak_comm_size(c_)); }
    /// all_reduce_sum of a u64 vector (sim_comm.hpp:151-156).
    std::vector<std::uint64_t> all_reduce_sum(std::vector<std::uint64_t> v,
                                              const exec_backend& ex = detail::default_backend()) {
        detail::check(ak_comm_allreduce_sum_u64(c_, ex.ctx(), v.data(), v.size()));
        return v;
    }
    ak_comm* handle() const noexcept { return c_; }

private:
    ak_comm* c_ = nullptr;
};

/// Runs fn(rank_comm&) on one thread per rank; the first exception aborts the world and
/// is rethrown after every thread has joined (sim_comm.hpp:187-218).
template <typename Fn>
void run_ranks(world& w, Fn&& fn) {
    const std::size_t P = w.size();
    std::vector<std::thread> threads;
    std::mutex mu;
    std::exception_ptr first;
    for (std::size_t r = 0; r < P; ++r) {
        threads.emplace_back([&, r] {
            try {
                rank_comm comm(w, r);
                fn(comm);
            } catch (...) {
                {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!first) first = std::current_exception();
                }
                w.abort();
            }
        });
    }
    for (auto& t : threads) t.join();
    if (first) std::rethrow_exception(first);
}

}  // namespace sim

namespace nccl {

using unique_id = std::array<unsigned char, 128>;

/// ncclGetUniqueId on one rank, then shared with the others (e.g. over torch.distributed).
inline unique_id make_unique_id() {
    unique_id id{};
    detail::check(ak_nccl_unique_id(id.data(), id.size()));
    return id;
}

/// One GPU's rank of an NCCL world (replaces sim::rank_comm across GPUs).
class rank_comm {
public:
    rank_comm(const unique_id& id, std::size_t nranks, std::size_t rank, int device) {
        detail::check(ak_comm_nccl_create(id.data(), static_cast<int>(nranks), static_cast<int>(rank), device, &c_));
    }
    rank_comm(const rank_comm&) = delete;
    rank_comm& operator=(const rank_comm&) = delete;
    ~rank_comm() {
        if (c_) ak_comm_destroy(c_);
    }
    std::size_t rank() const noexcept { return static_cast<std::size_t>(ak_comm_rank(c_)); }
    std::size_t world_size() const noexcept { return static_cast<std::size_t>(ak_comm_size(c_)); }
    std::vector<std::uint64_t> all_reduce_sum(std::vector<std::uint64_t> v,
                                              const exec_backend& ex = detail::default_backend()) {
        detail::check(ak_comm_allreduce_sum_u64(c_, ex.ctx(), v.data(), v.size()));
        return v;
    }
    ak_comm* handle() const noexcept { return c_; }

private:
    ak_comm* c_ = nullptr;
};

}  // namespace nccl

}  // namespace ak
