// sihsort.cuh -- device rank policy, NCCL transport and the loopback world.
#pragma once

#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

#include "ctx.cuh"
#include "sih_protocol.hpp"

namespace akb {

// NCCL transport (one communicator per GPU/process); replaces the reference's
// in-process sim::rank_comm (sim_comm.hpp:84-156) over NVLink/NVSwitch.
struct nccl_comm final : comm_iface {
    ncclComm_t comm = nullptr;
    int r = 0, p = 1, device = 0;
    cudaStream_t stream = nullptr;  // set per call by the caller's ctx
    void* d_stage = nullptr;
    std::size_t d_stage_bytes = 0;
    void* h_stage = nullptr;
    std::size_t h_stage_bytes = 0;
    std::uint64_t bytes_sent = 0;

    ~nccl_comm() override;
    int rank() const override { return r; }
    int size() const override { return p; }
    void allgather(const void* in, std::size_t bytes, void* out) override;
    void allreduce_sum_u64(std::uint64_t* inout, std::size_t n) override;
    void exchange(const void* send_base, const std::uint64_t* send_off, const std::uint64_t* send_cnt,
                  void* recv_base, const std::uint64_t* recv_off, const std::uint64_t* recv_cnt,
                  std::size_t elem_bytes) override;
    void abort() noexcept override;
    void stage(std::size_t bytes);
};

// P logical ranks in one process on one GPU (device analogue of sim::world,
// sim_comm.hpp:41-80): host-level collectives, device-to-device slice copies.
struct loopback_world {
    explicit loopback_world(int ranks);
    int P;
    std::mutex mu;
    std::condition_variable cv;
    std::uint64_t generation = 0;
    int arrived = 0;
    bool aborted = false;
    std::vector<std::vector<char>> slots;
    void barrier();
    void abort() noexcept;
};

struct loopback_comm final : comm_iface {
    loopback_world* w;
    int r;
    cudaStream_t stream;
    loopback_comm(loopback_world* world, int rank_, cudaStream_t s) : w(world), r(rank_), stream(s) {}
    int rank() const override { return r; }
    int size() const override { return w->P; }
    void allgather(const void* in, std::size_t bytes, void* out) override;
    void allreduce_sum_u64(std::uint64_t* inout, std::size_t n) override;
    void exchange(const void* send_base, const std::uint64_t* send_off, const std::uint64_t* send_cnt,
                  void* recv_base, const std::uint64_t* recv_off, const std::uint64_t* recv_cnt,
                  std::size_t elem_bytes) override;
    void abort() noexcept override { w->abort(); }
};

// Device sihsort on one rank: d_in (n keys, not modified) -> d_out (capacity cap).
template <typename T>
std::uint64_t sihsort_device(ak_ctx* c, comm_iface& comm, const T* d_in, std::uint64_t n, T* d_out,
                             std::uint64_t cap, const sih_config_c& cfg, sih_stats_c& st,
                             std::vector<T>* splitters = nullptr);

}  // namespace akb
