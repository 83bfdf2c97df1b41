// ak/sim_comm.hpp -- drop-in for proj/include/ak/sim_comm.hpp (sim_comm.hpp:16-218), B200 build.
//
// Two communicators with the reference's method shape:
//   * ak::sim::world / rank_comm / run_ranks: P logical ranks in ONE process on ONE GPU,
//     one host thread per rank (the reference's in-process world, sim_comm.hpp:41-218).
//     Collectives are host-level; sihsort slices move device to device.
//   * ak::nccl::rank_comm: one rank per GPU (one process or thread each) over NCCL,
//     NVLink 5 / NVSwitch -- the production transport for the 8xB200 sample sort;
//   * ak::ipc::rank_comm: one process per GPU, peer memory through CUDA IPC (the exchange is
//     fused into the merge), control collectives from caller callbacks.
// Both abort on failure so blocked peers wake with sim::transport_error.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "ak/exec.hpp"

namespace ak {

namespace sim {

/// payload: bulk redistribution traffic; control: everything else (sim_comm.hpp:28-31).
enum class traffic_class { control, payload };

/// sim_comm.hpp:33-39. On the B200 build collective_sends counts the messages this rank
/// would send in the reference's binomial reduce + broadcast tree (the device transports
/// gather instead), and control_bytes_peak covers user control-class messages (loopback world).
struct rank_counters {
    std::uint64_t p2p_sends = 0;
    std::uint64_t p2p_bytes = 0;
    std::uint64_t collective_ops = 0;
    std::uint64_t collective_sends = 0;
    std::uint64_t control_bytes_peak = 0;
};

}  // namespace sim

namespace detail {

/// rank_comm's messaging / collective methods (sim_comm.hpp:84-181) over any ak_comm.
template <typename Derived>
class comm_ops {
public:
    /// point-to-point message (sim_comm.hpp:92-94)
    void send(std::size_t dest, std::span<const std::byte> bytes, sim::traffic_class cls = sim::traffic_class::payload,
              const exec_backend& ex = default_backend()) {
        check(ak_comm_send(h(), ex.ctx(), static_cast<int>(dest), bytes.data(), bytes.size(),
                           cls == sim::traffic_class::control ? 1 : 0));
    }
    /// next message from src, FIFO per pair (sim_comm.hpp:95-96)
    std::vector<std::byte> recv(std::size_t src, const exec_backend& ex = default_backend()) {
        std::vector<std::byte> out(256);
        for (;;) {
            std::uint64_t n = 0;
            const int rc = ak_comm_recv(h(), ex.ctx(), static_cast<int>(src), out.data(), out.size(), &n);
            if (rc == AK_ECAPACITY) {  // the message stays pending: retry with room
                out.resize(n);
                continue;
            }
            check(rc, n);
            out.resize(n);
            return out;
        }
    }
    template <typename T>
    void send_values(std::size_t dest, std::span<const T> values, sim::traffic_class cls = sim::traffic_class::payload,
                     const exec_backend& ex = default_backend()) {
        static_assert(std::is_trivially_copyable_v<T>);
        send(dest, std::as_bytes(values), cls, ex);
    }
    template <typename T>
    std::vector<T> recv_values(std::size_t src, const exec_backend& ex = default_backend()) {
        static_assert(std::is_trivially_copyable_v<T>);
        const auto bytes = recv(src, ex);
        if (bytes.size() % sizeof(T) != 0)  // sim_comm.hpp:108-112
            throw sim::transport_error("recv_values: message size " + std::to_string(bytes.size()) +
                                       " is not a multiple of the element size (pair " + std::to_string(src) +
                                       " -> " + std::to_string(static_cast<const Derived*>(this)->rank()) + ")");
        std::vector<T> out(bytes.size() / sizeof(T));
        if (!bytes.empty()) std::memcpy(out.data(), bytes.data(), bytes.size());
        return out;
    }
    /// all_reduce of equal-length vectors (sim_comm.hpp:124-149): the vectors are gathered and
    /// folded in the reference's binomial-tree order (reduce to rank 0 by halving distances),
    /// so any merge -- commutative or not -- gives the reference's result on every rank.
    template <typename T, typename Merge>
    std::vector<T> all_reduce(std::vector<T> local, Merge merge, const exec_backend& ex = default_backend()) {
        static_assert(std::is_trivially_copyable_v<T>);
        const std::size_t p = static_cast<const Derived*>(this)->world_size();
        const std::size_t len = local.size();
        std::vector<T> all(len * p);
        // one gather; the loopback world rejects unequal lengths with sim::protocol_error
        // (sim_comm.hpp:171-176), NCCL ranks must agree on the length as the reference requires
        check(ak_comm_allgather(h(), ex.ctx(), local.data(), len * sizeof(T), all.data()));
        std::vector<std::vector<T>> acc(p);
        for (std::size_t q = 0; q < p; ++q) acc[q].assign(all.begin() + q * len, all.begin() + (q + 1) * len);
        std::size_t m = 1;
        while (m * 2 < p) m *= 2;
        for (; m >= 1; m >>= 1)
            for (std::size_t r = 0; r < m && r + m < p; ++r) merge(acc[r], acc[r + m]);
        return acc[0];
    }
    template <typename T>
    std::vector<T> all_reduce_sum(std::vector<T> local, const exec_backend& ex = default_backend()) {
        return all_reduce(std::move(local),
                          [](std::vector<T>& a, const std::vector<T>& b) {
                              for (std::size_t i = 0; i < a.size(); ++i) a[i] += b[i];
                          },
                          ex);
    }
    sim::rank_counters counters() const {
        ak_rank_counters c{};
        check(ak_comm_counters(h(), &c));
        return {c.p2p_sends, c.p2p_bytes, c.collective_ops, c.collective_sends, c.control_bytes_peak};
    }

private:
    ak_comm* h() const { return static_cast<const Derived*>(this)->handle(); }
};

}  // namespace detail

namespace sim {

/// P logical ranks on one device (sim_comm.hpp:45-80); queue_capacity bounds each ordered
/// pair's FIFO of user messages (send blocks while it is full). The sihsort exchange moves
/// device slices directly and needs no FIFO.
class world {
public:
    explicit world(std::size_t ranks, std::size_t queue_capacity = 64) {
        detail::check(ak_world_create_ex(static_cast<int>(ranks), queue_capacity, &w_));
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
class rank_comm : public detail::comm_ops<rank_comm> {
public:
    rank_comm(world& w, std::size_t rank) { detail::check(ak_comm_loopback_create(w.handle(), static_cast<int>(rank), &c_)); }
    rank_comm(const rank_comm&) = delete;
    rank_comm& operator=(const rank_comm&) = delete;
    ~rank_comm() {
        if (c_) ak_comm_destroy(c_);
    }
    std::size_t rank() const noexcept { return static_cast<std::size_t>(ak_comm_rank(c_)); }
    std::size_t world_size() const noexcept { return static_cast<std::size_t>(ak_comm_size(c_)); }
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

/// One GPU's rank of an NCCL world (replaces sim::rank_comm across GPUs). send / recv are
/// rendezvous (a send returns once the peer has received).
class rank_comm : public detail::comm_ops<rank_comm> {
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
    ak_comm* handle() const noexcept { return c_; }

private:
    ak_comm* c_ = nullptr;
};

}  // namespace nccl

namespace ipc {

/// One process per GPU without NCCL: the SIHSort exchange reads the peers' sorted arrays
/// through CUDA IPC mappings (fused into the P-way merge; NVLink P2P between GPUs, or
/// processes sharing one GPU), and the caller supplies the tiny control collectives -- e.g.
/// an MPI / gloo allgather of `bytes` per rank (rank order) and a u64 sum allreduce.
class rank_comm : public detail::comm_ops<rank_comm> {
public:
    using allgather_fn = ak_allgather_fn;       // int (void* user, const void* in, uint64_t bytes, void* out)
    using allreduce_fn = ak_allreduce_u64_fn;  // int (void* user, uint64_t* inout, uint64_t n)
    rank_comm(std::size_t nranks, std::size_t rank, int device, void* user, allgather_fn ag, allreduce_fn ar) {
        detail::check(ak_comm_ipc_create(static_cast<int>(nranks), static_cast<int>(rank), device, user, ag, ar, &c_));
    }
    rank_comm(const rank_comm&) = delete;
    rank_comm& operator=(const rank_comm&) = delete;
    ~rank_comm() {
        if (c_) ak_comm_destroy(c_);
    }
    std::size_t rank() const noexcept { return static_cast<std::size_t>(ak_comm_rank(c_)); }
    std::size_t world_size() const noexcept { return static_cast<std::size_t>(ak_comm_size(c_)); }
    ak_comm* handle() const noexcept { return c_; }

private:
    ak_comm* c_ = nullptr;
};

}  // namespace ipc

}  // namespace ak
