// sihsort.cuh -- device rank policy, NCCL transport and the loopback world.
#pragma once

#include <nccl.h>

#include <condition_variable>
#include <deque>
#include <cstdint>
#include <mutex>
#include <vector>

#include "ctx.cuh"
#include "sih_protocol.hpp"

namespace akb {

// Peer-store exchange (K7 without a library): ONE launch copies every outgoing slice straight
// into its destination rank's receive buffer -- on this device (loopback ranks) or in a peer
// GPU's HBM mapped by CUDA IPC (P2P stores over NVLink/NVSwitch). SM-driven 16-byte
// (8/4-byte when the two ends are not co-aligned) vector copies, no staging.
struct copy_seg {
    const void* src;
    void* dst;
    std::uint64_t bytes;
};
void peer_store(cudaStream_t s, int sm_count, const std::vector<copy_seg>& segs);

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
    void bind(void* s, int) override { stream = static_cast<cudaStream_t>(s); }
    std::uint64_t payload_bytes_sent() const override { return bytes_sent; }
    void send_bytes(int dest, const void* p, std::size_t n, bool control) override;
    std::vector<char> recv_bytes(int src) override;
    void stage(std::size_t bytes);
};

// One process per GPU, bulk slices moved by peer_store into the peers' receive buffers
// (CUDA IPC handles exchanged over the control plane, mappings cached); control messages
// (allgather / allreduce, tiny) go through caller callbacks -- e.g. torch.distributed gloo.
// Works between processes on different GPUs (NVLink P2P) and on the same GPU.
struct ipc_comm final : comm_iface {
    int r, p, device;
    void* user;
    akb_allgather_fn ag;
    akb_allreduce_fn ar;
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    std::uint64_t bytes_sent = 0;
    struct mapping {
        std::vector<char> handle;  // cudaIpcMemHandle_t bytes of the peer allocation
        char* base = nullptr;      // its base, opened in this process
    };
    std::vector<mapping> peers;    // current mapping per peer rank
    ipc_comm(int rank_, int size_, int dev, void* u, akb_allgather_fn a, akb_allreduce_fn b)
        : r(rank_), p(size_), device(dev), user(u), ag(a), ar(b), peers(size_), pulled(size_) {}
    ~ipc_comm() override;
    int rank() const override { return r; }
    int size() const override { return p; }
    void allgather(const void* in, std::size_t bytes, void* out) override;
    void allreduce_sum_u64(std::uint64_t* inout, std::size_t n) override;
    void exchange(const void* send_base, const std::uint64_t* send_off, const std::uint64_t* send_cnt,
                  void* recv_base, const std::uint64_t* recv_off, const std::uint64_t* recv_cnt,
                  std::size_t elem_bytes) override;
    void bind(void* s, int sms) override {
        stream = static_cast<cudaStream_t>(s);
        sm_count = sms;
    }
    std::uint64_t payload_bytes_sent() const override { return bytes_sent; }
    bool map_peers(const void* local, std::vector<const void*>& out) override;
    void peers_released() override;
    void add_pulled(std::uint64_t b) { bytes_sent += b; }
    // mappings of peer buffers for map_peers (separate from the receive-buffer ones)
    std::vector<mapping> pulled;
    char* open_peer(mapping& m, const cudaIpcMemHandle_t& h);
};

// P logical ranks in one process on one GPU (device analogue of sim::world,
// sim_comm.hpp:41-80): host-level collectives, device-to-device slice copies.
struct loopback_world {
    explicit loopback_world(int ranks, std::size_t queue_capacity = 64);
    int P;
    std::size_t capacity;  // messages queued per ordered pair before send blocks (sim_comm.hpp:47)
    std::mutex mu;
    std::condition_variable cv;
    std::uint64_t generation = 0;
    int arrived = 0;
    bool aborted = false;
    std::vector<std::vector<char>> slots;
    struct message {
        std::vector<char> bytes;
        bool control;
    };
    std::vector<std::deque<message>> chan;  // src * P + dst
    std::vector<std::uint64_t> queued_control, peak_control;
    void barrier();
    void abort() noexcept;
    void send(int src, int dst, const void* p, std::size_t n, bool control);
    std::vector<char> recv(int src, int dst);
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
    void bind(void* s, int sms) override {
        stream = static_cast<cudaStream_t>(s);
        sm_count = sms;
    }
    void send_bytes(int dest, const void* p, std::size_t n, bool control) override;
    std::vector<char> recv_bytes(int src) override;
    counters_c counters() const override;
    bool map_peers(const void* local, std::vector<const void*>& out) override;  // same process and GPU
    void peers_released() override { w->barrier(); }
    int sm_count = 148;
};

// Device sihsort on one rank: d_in (n keys, not modified) -> d_out (capacity cap).
template <typename T>
std::uint64_t sihsort_device(ak_ctx* c, comm_iface& comm, const T* d_in, std::uint64_t n, T* d_out,
                             std::uint64_t cap, const sih_config_c& cfg, sih_stats_c& st,
                             std::vector<T>* splitters = nullptr);

// Distributed sortperm (new; the reference sihsort is keys-only): d_out / d_idx (capacity cap)
// = this rank's slice of the globally stable order of all ranks' keys, as keys and their
// global indices (rank r's key i has global index sum_{q<r} n_q + i).
template <typename T>
std::uint64_t sihsort_perm_device(ak_ctx* c, comm_iface& comm, const T* d_in, std::uint64_t n, T* d_out,
                                  std::uint64_t* d_idx, std::uint64_t cap, const sih_config_c& cfg,
                                  sih_stats_c& st);

// Public stage functions (sihsort.hpp:264-501) over a caller's sorted device keys.
template <typename T>
std::uint64_t sample_local_device(ak_ctx* c, const T* sorted, std::uint64_t n, std::uint64_t k, T* host_out);
template <typename T>
refine_out refine_device(ak_ctx* c, comm_iface& comm, const T* sorted, std::uint64_t n, std::vector<T>& spl,
                         const sih_config_c& cfg);
// returns the received element count; *sends / *bytes accumulate the reference's accounting
template <typename T>
std::uint64_t redistribute_device(ak_ctx* c, comm_iface& comm, const T* sorted, std::uint64_t n,
                                  const std::vector<T>& spl, T* out, std::uint64_t cap, std::uint64_t* sends,
                                  std::uint64_t* bytes, std::uint64_t n_total);

}  // namespace akb
