// sihsort.cu -- device policy of the SIHSort protocol, NCCL and loopback transports.
#include <cstdlib>
#include <cstring>
#include <string>

#include "radix_sort.cuh"
#include "search_merge.cuh"
#include "sihsort.cuh"

namespace akb {

// ---------------------------------------------------------------------------
// NCCL transport
// ---------------------------------------------------------------------------
namespace {
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw transport_error(std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace
#define AKB_NCCL(x) nccl_check((x), #x)

nccl_comm::~nccl_comm() {
    if (comm) ncclCommDestroy(comm);
    if (d_stage) cudaFree(d_stage);
    if (h_stage) cudaFreeHost(h_stage);
}

void nccl_comm::abort() noexcept {
    if (comm) {
        ncclCommAbort(comm);
        comm = nullptr;
    }
}

void nccl_comm::stage(std::size_t bytes) {
    if (bytes > d_stage_bytes) {
        if (d_stage) {
            AKB_CUDA(cudaStreamSynchronize(stream));
            AKB_CUDA(cudaFree(d_stage));
        }
        AKB_CUDA(cudaMalloc(&d_stage, bytes));
        d_stage_bytes = bytes;
    }
    if (bytes > h_stage_bytes) {
        if (h_stage) AKB_CUDA(cudaFreeHost(h_stage));
        AKB_CUDA(cudaMallocHost(&h_stage, bytes));
        h_stage_bytes = bytes;
    }
}

void nccl_comm::allgather(const void* in, std::size_t bytes, void* out) {
    stage(bytes * (p + 1));
    char* h = static_cast<char*>(h_stage);
    std::memcpy(h, in, bytes);
    char* d = static_cast<char*>(d_stage);
    AKB_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream));
    AKB_NCCL(ncclAllGather(d, d + bytes, bytes, ncclChar, comm, stream));
    AKB_CUDA(cudaMemcpyAsync(h + bytes, d + bytes, bytes * p, cudaMemcpyDeviceToHost, stream));
    AKB_CUDA(cudaStreamSynchronize(stream));
    std::memcpy(out, h + bytes, bytes * p);
}

void nccl_comm::allreduce_sum_u64(std::uint64_t* inout, std::size_t n) {
    if (n == 0) return;
    const std::size_t bytes = n * sizeof(std::uint64_t);
    stage(bytes);
    std::memcpy(h_stage, inout, bytes);
    AKB_CUDA(cudaMemcpyAsync(d_stage, h_stage, bytes, cudaMemcpyHostToDevice, stream));
    AKB_NCCL(ncclAllReduce(d_stage, d_stage, n, ncclUint64, ncclSum, comm, stream));
    AKB_CUDA(cudaMemcpyAsync(h_stage, d_stage, bytes, cudaMemcpyDeviceToHost, stream));
    AKB_CUDA(cudaStreamSynchronize(stream));
    std::memcpy(inout, h_stage, bytes);
}

void nccl_comm::exchange(const void* send_base, const std::uint64_t* send_off,
                         const std::uint64_t* send_cnt, void* recv_base, const std::uint64_t* recv_off,
                         const std::uint64_t* recv_cnt, std::size_t eb) {
    // one grouped all-to-all-v: P-1 sends + P-1 receives (NCCL 2.27 has no alltoallv)
    AKB_NCCL(ncclGroupStart());
    for (int q = 0; q < p; ++q) {
        if (q == r) continue;
        if (send_cnt[q])
            AKB_NCCL(ncclSend(static_cast<const char*>(send_base) + send_off[q] * eb, send_cnt[q] * eb,
                              ncclChar, q, comm, stream));
        if (recv_cnt[q])
            AKB_NCCL(ncclRecv(static_cast<char*>(recv_base) + recv_off[q] * eb, recv_cnt[q] * eb, ncclChar,
                              q, comm, stream));
        bytes_sent += send_cnt[q] * eb;
    }
    AKB_NCCL(ncclGroupEnd());
}

// ---------------------------------------------------------------------------
// Loopback world
// ---------------------------------------------------------------------------
loopback_world::loopback_world(int ranks) : P(ranks), slots(ranks) {}

void loopback_world::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw transport_error("loopback: world aborted");
    const std::uint64_t gen = generation;
    if (++arrived == P) {
        arrived = 0;
        ++generation;
        cv.notify_all();
        return;
    }
    cv.wait(lk, [&] { return generation != gen || aborted; });
    if (aborted) throw transport_error("loopback: world aborted");
}

void loopback_world::abort() noexcept {
    {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
    }
    cv.notify_all();
}

void loopback_comm::allgather(const void* in, std::size_t bytes, void* out) {
    {
        std::lock_guard<std::mutex> lk(w->mu);
        w->slots[r].assign(static_cast<const char*>(in), static_cast<const char*>(in) + bytes);
    }
    w->barrier();
    {
        std::lock_guard<std::mutex> lk(w->mu);
        for (int q = 0; q < w->P; ++q) {
            if (w->slots[q].size() != bytes) throw protocol_error("loopback: collective size mismatch");
            std::memcpy(static_cast<char*>(out) + q * bytes, w->slots[q].data(), bytes);
        }
    }
    w->barrier();
}

void loopback_comm::allreduce_sum_u64(std::uint64_t* inout, std::size_t n) {
    std::vector<std::uint64_t> all(n * w->P);
    allgather(inout, n * sizeof(std::uint64_t), all.data());
    for (std::size_t i = 0; i < n; ++i) {
        std::uint64_t s = 0;
        for (int q = 0; q < w->P; ++q) s += all[q * n + i];
        inout[i] = s;
    }
}

void loopback_comm::exchange(const void* send_base, const std::uint64_t* send_off,
                             const std::uint64_t* send_cnt, void* recv_base, const std::uint64_t* recv_off,
                             const std::uint64_t*, std::size_t eb) {
    // publish (recv_base, recv_off[src] for every src) so senders can push
    const int P = w->P;
    std::vector<std::uint64_t> mine(P + 1), all((P + 1) * P);
    mine[0] = reinterpret_cast<std::uint64_t>(recv_base);
    for (int q = 0; q < P; ++q) mine[q + 1] = recv_off[q];
    allgather(mine.data(), mine.size() * sizeof(std::uint64_t), all.data());
    for (int q = 0; q < P; ++q) {
        if (q == r || send_cnt[q] == 0) continue;
        char* dst = reinterpret_cast<char*>(all[q * (P + 1)]) + all[q * (P + 1) + 1 + r] * eb;
        AKB_CUDA(cudaMemcpyAsync(dst, static_cast<const char*>(send_base) + send_off[q] * eb,
                                 send_cnt[q] * eb, cudaMemcpyDeviceToDevice, stream));
    }
    AKB_CUDA(cudaStreamSynchronize(stream));
    w->barrier();
}

// ---------------------------------------------------------------------------
// Device rank policy
// ---------------------------------------------------------------------------
namespace {

template <typename T>
struct device_local {
    ak_ctx* c;
    const T* d_in;
    std::uint64_t n;
    T* d_out;
    std::uint64_t cap;
    std::size_t P, me;
    T* sorted = nullptr;  // local sort #1 result
    T* X = nullptr;       // radix scratch, then merge ping-pong
    T* R = nullptr;       // receive buffer
    bool direct = false;  // P == 1: sorted straight into d_out
    std::vector<std::uint64_t> roff;

    std::uint64_t size() const { return n; }
    std::uint64_t capacity() const { return cap; }

    void sort_local() {
        direct = (P == 1 && cap >= n);
        const std::uint64_t xn = std::max<std::uint64_t>(n, cap);
        std::size_t need = arena::need(xn * sizeof(T)) + 256;
        if (!direct) need += arena::need(n * sizeof(T)) + arena::need(cap * sizeof(T)) + 512;
        ctx_reserve_aux(c, need);
        arena a{static_cast<char*>(c->aux), c->aux_bytes};
        X = a.take<T>(xn);
        if (!direct) {
            sorted = a.take<T>(n);
            R = a.take<T>(cap);
        } else {
            sorted = d_out;
        }
        radix_sort<T, std::uint32_t>(c, SORT_KEYS, d_in, sorted, X, nullptr, nullptr, nullptr, n, false,
                                     true);
    }

    void samples(std::uint64_t k, std::vector<T>& s, T& front, T& back) {
        T* dev = reinterpret_cast<T*>(ctx_split(c, k + 2));
        k = gather_samples<T>(c, sorted, n, k, dev);
        T* h = static_cast<T*>(ctx_pinned(c, (k + 2) * sizeof(T)));
        AKB_CUDA(cudaMemcpyAsync(h, dev, (k + 2) * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        front = h[0];
        back = h[1];
        s.assign(h + 2, h + 2 + k);
    }

    void upper_bounds(const std::vector<T>& v, std::vector<std::uint64_t>& out) {
        out.assign(v.size(), 0);
        if (v.empty()) return;
        const std::size_t m = v.size();
        char* small = static_cast<char*>(c->small) + 262144;  // needles | results
        T* d_needles = reinterpret_cast<T*>(small);
        std::uint64_t* d_res = reinterpret_cast<std::uint64_t*>(small + 131072);
        if (m * sizeof(T) > 131072) throw invalid_argument("sihsort: too many ranks for staging");
        char* h = static_cast<char*>(ctx_pinned(c, m * (sizeof(T) + 8)));
        std::memcpy(h, v.data(), m * sizeof(T));
        AKB_CUDA(cudaMemcpyAsync(d_needles, h, m * sizeof(T), cudaMemcpyHostToDevice, c->stream));
        searchsorted<T>(c, sorted, n, d_needles, m, 1, 0, d_res);
        AKB_CUDA(cudaMemcpyAsync(h + m * sizeof(T), d_res, m * 8, cudaMemcpyDeviceToHost, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        std::memcpy(out.data(), h + m * sizeof(T), m * 8);
    }

    void exchange(comm_iface& comm, const std::vector<std::uint64_t>& bounds,
                  const std::vector<std::uint64_t>& recv_counts) {
        roff.assign(P, 0);
        std::uint64_t o = 0;
        for (std::size_t s = 0; s < P; ++s) {
            roff[s] = o;
            if (s != me) o += recv_counts[s];
        }
        if (P == 1) return;
        std::vector<std::uint64_t> soff(P), scnt(P);
        for (std::size_t d = 0; d < P; ++d) {
            soff[d] = bounds[d];
            scnt[d] = bounds[d + 1] - bounds[d];
        }
        const int tok = ctx_prof_begin(c, KF_EXCHANGE);
        comm.exchange(sorted, soff.data(), scnt.data(), R, roff.data(), recv_counts.data(), sizeof(T));
        ctx_prof_end(c, tok);
    }

    // P-way merge of the runs in source-rank order (replaces local sort #2,
    // sihsort.hpp:555): merge_runs (K8), last level lands in d_out.
    std::uint64_t merge_runs(const std::vector<std::uint64_t>& bounds,
                             const std::vector<std::uint64_t>& recv_counts) {
        std::uint64_t total = 0;
        for (std::size_t s = 0; s < P; ++s) total += recv_counts[s];
        if (direct) return n;
        struct run {
            const T* p;
            std::uint64_t len, off;
        };
        std::vector<run> runs;
        std::uint64_t off = 0;
        for (std::size_t s = 0; s < P; ++s) {
            const T* p = s == me ? sorted + bounds[me] : R + roff[s];
            runs.push_back({p, recv_counts[s], off});
            off += recv_counts[s];
        }
        // drop empty runs (they contribute nothing); keep order
        std::vector<run> live;
        for (auto& rr : runs)
            if (rr.len) live.push_back(rr);
        if (live.empty()) return 0;
        if (live.size() == 1) {
            AKB_CUDA(cudaMemcpyAsync(d_out, live[0].p, live[0].len * sizeof(T), cudaMemcpyDeviceToDevice,
                                     c->stream));
            return total;
        }
        {
            // P-way merge tree (K8, search_merge.cu); X is free scratch at this point
            std::vector<const T*> ptrs;
            std::vector<std::uint64_t> lens;
            for (auto& rr : live) {
                ptrs.push_back(rr.p);
                lens.push_back(rr.len);
            }
            akb::merge_runs<T>(c, static_cast<int>(live.size()), ptrs.data(), lens.data(), d_out, X, false);
            return total;
        }
    }
};

}  // namespace

template <typename T>
std::uint64_t sihsort_device(ak_ctx* c, comm_iface& comm, const T* d_in, std::uint64_t n, T* d_out,
                             std::uint64_t cap, const sih_config_c& cfg, sih_stats_c& st,
                             std::vector<T>* splitters) {
    device_local<T> L{c, d_in, n, d_out, cap, static_cast<std::size_t>(comm.size()),
                      static_cast<std::size_t>(comm.rank())};
    sihsort_run<T>(comm, L, cfg, st, splitters);
    return st.output_count;
}

#define AKB_INST(T)                                                                                  \
    template std::uint64_t sihsort_device<T>(ak_ctx*, comm_iface&, const T*, std::uint64_t, T*,      \
                                             std::uint64_t, const sih_config_c&, sih_stats_c&,      \
                                             std::vector<T>*);
AKB_INST(std::int32_t)
AKB_INST(std::uint32_t)
AKB_INST(std::int64_t)
AKB_INST(std::uint64_t)
AKB_INST(float)
AKB_INST(double)

}  // namespace akb
