// sihsort.cu -- device policy of the SIHSort protocol, NCCL and loopback transports.
#include <algorithm>
#include <cstring>
#include <string>

#include "radix_sort.cuh"
#include "search_merge.cuh"
#include "sihsort.cuh"

namespace akb {

// ---------------------------------------------------------------------------
// Peer-store exchange kernel
// ---------------------------------------------------------------------------
namespace {

constexpr int PS_MAX_SEGS = 32;  // segments per launch (P - 1 <= 31 peers)
constexpr int PS_BLOCK = 512;
constexpr int PS_UNROLL = 4;

struct ps_args {
    copy_seg seg[PS_MAX_SEGS];
};

// Copies `bytes` (a multiple of 4) from src to dst with vectors of W bytes; src and dst are
// co-aligned modulo W after the head.
template <typename V>
__device__ __forceinline__ void copy_vec(const char* __restrict__ src, char* __restrict__ dst, std::uint64_t bytes,
                                         std::uint64_t t, std::uint64_t nt) {
    constexpr std::uint64_t W = sizeof(V);
    const std::uint64_t head = ((W - (reinterpret_cast<std::uintptr_t>(dst) & (W - 1))) & (W - 1)) < bytes
                                   ? ((W - (reinterpret_cast<std::uintptr_t>(dst) & (W - 1))) & (W - 1))
                                   : bytes;
    for (std::uint64_t i = 4 * t; i < head; i += 4 * nt)
        *reinterpret_cast<std::uint32_t*>(dst + i) = *reinterpret_cast<const std::uint32_t*>(src + i);
    const std::uint64_t nv = (bytes - head) / W;
    const V* s = reinterpret_cast<const V*>(src + head);
    V* d = reinterpret_cast<V*>(dst + head);
    std::uint64_t i = t;
    for (; i + (PS_UNROLL - 1) * nt < nv; i += PS_UNROLL * nt) {
        V v[PS_UNROLL];
#pragma unroll
        for (int u = 0; u < PS_UNROLL; ++u) v[u] = __ldcs(s + i + u * nt);  // streamed: read once
#pragma unroll
        for (int u = 0; u < PS_UNROLL; ++u) d[i + u * nt] = v[u];
    }
    for (; i < nv; i += nt) d[i] = __ldcs(s + i);
    for (std::uint64_t j = head + nv * W + 4 * t; j < bytes; j += 4 * nt)
        *reinterpret_cast<std::uint32_t*>(dst + j) = *reinterpret_cast<const std::uint32_t*>(src + j);
}

// blockIdx.y = segment; the x-blocks of a segment stride over its bytes.
__global__ void __launch_bounds__(PS_BLOCK) peer_store_kernel(ps_args a) {
    const copy_seg g = a.seg[blockIdx.y];
    if (g.bytes == 0) return;
    const char* src = static_cast<const char*>(g.src);
    char* dst = static_cast<char*>(g.dst);
    const std::uint64_t t = static_cast<std::uint64_t>(blockIdx.x) * PS_BLOCK + threadIdx.x;
    const std::uint64_t nt = static_cast<std::uint64_t>(gridDim.x) * PS_BLOCK;
    const std::uintptr_t mis = reinterpret_cast<std::uintptr_t>(src) ^ reinterpret_cast<std::uintptr_t>(dst);
    if ((mis & 15) == 0) copy_vec<uint4>(src, dst, g.bytes, t, nt);
    else if ((mis & 7) == 0) copy_vec<uint2>(src, dst, g.bytes, t, nt);
    else copy_vec<std::uint32_t>(src, dst, g.bytes, t, nt);
}

}  // namespace

void peer_store(cudaStream_t s, int sm_count, const std::vector<copy_seg>& segs) {
    for (std::size_t b = 0; b < segs.size(); b += PS_MAX_SEGS) {
        ps_args a{};
        int k = 0;
        std::uint64_t biggest = 0;
        for (std::size_t i = b; i < segs.size() && k < PS_MAX_SEGS; ++i) {
            if (segs[i].bytes % 4) throw invalid_argument("peer_store: slice bytes must be a multiple of 4");
            a.seg[k++] = segs[i];
            biggest = std::max<std::uint64_t>(biggest, segs[i].bytes);
        }
        if (biggest == 0) continue;
        // ~4 resident CTAs per SM shared by the segments, enough bytes in flight per segment
        const std::uint64_t want = ceil_div(biggest, static_cast<std::uint64_t>(PS_BLOCK) * 16 * PS_UNROLL);
        const unsigned gx = static_cast<unsigned>(
            std::max<std::uint64_t>(1, std::min<std::uint64_t>(want, std::max(1, 4 * sm_count / k))));
        peer_store_kernel<<<dim3(gx, k), PS_BLOCK, 0, s>>>(a);
        AKB_CUDA(cudaGetLastError());
    }
}

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

// rank_comm::send / recv over NCCL: an 8-byte length, then the bytes, staged through HBM.
// Rendezvous semantics: the call returns when the peer has received (NCCL point-to-point),
// unlike the reference's buffered FIFO -- callers must order matching pairs.
void nccl_comm::send_bytes(int dest, const void* p, std::size_t n, bool) {
    if (dest == r || dest < 0 || dest >= this->p) throw transport_error("send: invalid destination rank");
    stage(n + 8);
    char* h = static_cast<char*>(h_stage);
    const std::uint64_t len = n;
    std::memcpy(h, &len, 8);
    if (n) std::memcpy(h + 8, p, n);
    AKB_CUDA(cudaMemcpyAsync(d_stage, h, n + 8, cudaMemcpyHostToDevice, stream));
    AKB_NCCL(ncclSend(d_stage, 8, ncclChar, dest, comm, stream));
    if (n) AKB_NCCL(ncclSend(static_cast<char*>(d_stage) + 8, n, ncclChar, dest, comm, stream));
    AKB_CUDA(cudaStreamSynchronize(stream));
    ctr.p2p_sends += 1;
    ctr.p2p_bytes += n;
}

std::vector<char> nccl_comm::recv_bytes(int src) {
    if (src == r || src < 0 || src >= p) throw transport_error("recv: invalid source rank");
    stage(8);
    AKB_NCCL(ncclRecv(d_stage, 8, ncclChar, src, comm, stream));
    AKB_CUDA(cudaMemcpyAsync(h_stage, d_stage, 8, cudaMemcpyDeviceToHost, stream));
    AKB_CUDA(cudaStreamSynchronize(stream));
    std::uint64_t len = 0;
    std::memcpy(&len, h_stage, 8);
    std::vector<char> out(len);
    if (len) {
        stage(len);
        AKB_NCCL(ncclRecv(d_stage, len, ncclChar, src, comm, stream));
        AKB_CUDA(cudaMemcpyAsync(h_stage, d_stage, len, cudaMemcpyDeviceToHost, stream));
        AKB_CUDA(cudaStreamSynchronize(stream));
        std::memcpy(out.data(), h_stage, len);
    }
    return out;
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
loopback_world::loopback_world(int ranks, std::size_t queue_capacity)
    : P(ranks), capacity(queue_capacity), slots(ranks), chan(static_cast<std::size_t>(ranks) * ranks),
      queued_control(ranks, 0), peak_control(ranks, 0) {}

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

void loopback_world::send(int src, int dst, const void* p, std::size_t n, bool control) {
    std::unique_lock<std::mutex> lk(mu);
    if (src == dst || dst < 0 || dst >= P)
        throw transport_error("send: invalid pair " + std::to_string(src) + " -> " + std::to_string(dst));
    auto& q = chan[static_cast<std::size_t>(src) * P + dst];
    cv.wait(lk, [&] { return aborted || q.size() < capacity; });  // bounded FIFO (sim_comm.cpp:50)
    if (aborted)
        throw transport_error("send: world aborted (pair " + std::to_string(src) + " -> " + std::to_string(dst) + ")");
    q.push_back({std::vector<char>(static_cast<const char*>(p), static_cast<const char*>(p) + n), control});
    if (control) {
        queued_control[dst] += n;
        peak_control[dst] = std::max(peak_control[dst], queued_control[dst]);
    }
    cv.notify_all();
}

std::vector<char> loopback_world::recv(int src, int dst) {
    std::unique_lock<std::mutex> lk(mu);
    if (src == dst || src < 0 || src >= P)
        throw transport_error("recv: invalid pair " + std::to_string(src) + " -> " + std::to_string(dst));
    auto& q = chan[static_cast<std::size_t>(src) * P + dst];
    cv.wait(lk, [&] { return aborted || !q.empty(); });
    if (aborted)
        throw transport_error("recv: world aborted (pair " + std::to_string(src) + " -> " + std::to_string(dst) + ")");
    message m = std::move(q.front());
    q.pop_front();
    if (m.control) queued_control[dst] -= m.bytes.size();
    cv.notify_all();
    return std::move(m.bytes);
}

void loopback_comm::send_bytes(int dest, const void* p, std::size_t n, bool control) {
    w->send(r, dest, p, n, control);
    ctr.p2p_sends += 1;
    ctr.p2p_bytes += n;
}

std::vector<char> loopback_comm::recv_bytes(int src) { return w->recv(src, r); }

comm_iface::counters_c loopback_comm::counters() const {
    counters_c c = ctr;
    std::lock_guard<std::mutex> lk(w->mu);
    c.control_bytes_peak = w->peak_control[r];
    return c;
}

bool loopback_comm::map_peers(const void* local, std::vector<const void*>& out) {
    // every rank is a thread of this process on this GPU: its pointer is valid here as is
    const std::uint64_t mine = reinterpret_cast<std::uint64_t>(local);
    std::vector<std::uint64_t> all(w->P);
    allgather(&mine, sizeof(mine), all.data());
    out.resize(w->P);
    for (int q = 0; q < w->P; ++q) out[q] = reinterpret_cast<const void*>(all[q]);
    return true;
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
    std::vector<copy_seg> segs;
    for (int q = 0; q < P; ++q) {
        if (q == r || send_cnt[q] == 0) continue;
        char* dst = reinterpret_cast<char*>(all[q * (P + 1)]) + all[q * (P + 1) + 1 + r] * eb;
        segs.push_back({static_cast<const char*>(send_base) + send_off[q] * eb, dst, send_cnt[q] * eb});
    }
    peer_store(stream, sm_count, segs);
    AKB_CUDA(cudaStreamSynchronize(stream));
    w->barrier();
}

// ---------------------------------------------------------------------------
// CUDA IPC transport (one process per GPU)
// ---------------------------------------------------------------------------
namespace {

// base of the cudaMalloc allocation holding p (driver cuMemGetAddressRange, resolved at run
// time so the library needs no -lcuda)
char* allocation_base(const void* p) {
    using fn_t = int (*)(unsigned long long*, std::size_t*, unsigned long long);
    static fn_t fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<fn_t>(f);
    }();
    if (!fn) throw transport_error("ipc: cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    std::size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<unsigned long long>(p)) != 0)
        throw transport_error("ipc: receive buffer is not device memory of this process");
    return reinterpret_cast<char*>(base);
}

}  // namespace

ipc_comm::~ipc_comm() {
    for (auto& m : peers)
        if (m.base) cudaIpcCloseMemHandle(m.base);
    for (auto& m : pulled)
        if (m.base) cudaIpcCloseMemHandle(m.base);
}

char* ipc_comm::open_peer(mapping& m, const cudaIpcMemHandle_t& h) {
    const char* hb = reinterpret_cast<const char*>(&h);
    if (!m.base || m.handle.size() != sizeof(h) || std::memcmp(m.handle.data(), hb, sizeof(h)) != 0) {
        if (m.base) AKB_CUDA(cudaIpcCloseMemHandle(m.base));
        m.base = nullptr;
        void* ptr = nullptr;
        AKB_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        m.base = static_cast<char*>(ptr);
        m.handle.assign(hb, hb + sizeof(h));
    }
    return m.base;
}

bool ipc_comm::map_peers(const void* local, std::vector<const void*>& out) {
    struct rec {
        cudaIpcMemHandle_t h;
        std::uint64_t off;
        std::uint64_t has;
    };
    rec mine{};
    if (local) {
        char* base = allocation_base(local);
        AKB_CUDA(cudaIpcGetMemHandle(&mine.h, base));
        mine.off = static_cast<std::uint64_t>(static_cast<const char*>(local) - base);
        mine.has = 1;
    }
    std::vector<rec> all(p);
    allgather(&mine, sizeof(rec), all.data());
    out.assign(p, nullptr);
    for (int q = 0; q < p; ++q) {
        if (q == r) {
            out[q] = local;
            continue;
        }
        if (!all[q].has) continue;
        out[q] = open_peer(pulled[q], all[q].h) + all[q].off;
    }
    return true;
}

void ipc_comm::peers_released() {
    std::uint8_t one = 1;
    std::vector<std::uint8_t> ack(p);
    allgather(&one, 1, ack.data());
}

void ipc_comm::allgather(const void* in, std::size_t bytes, void* out) {
    if (ag(user, in, bytes, out) != 0) throw transport_error("ipc: control allgather failed");
}

void ipc_comm::allreduce_sum_u64(std::uint64_t* inout, std::size_t n) {
    if (n && ar(user, inout, n) != 0) throw transport_error("ipc: control allreduce failed");
}

void ipc_comm::exchange(const void* send_base, const std::uint64_t* send_off, const std::uint64_t* send_cnt,
                        void* recv_base, const std::uint64_t* recv_off, const std::uint64_t*, std::size_t eb) {
    // 1. publish {IPC handle of my receive allocation, offset of recv_base in it, my recv_off[]};
    //    the allgather is also the barrier: every receive buffer is allocated and idle after it
    struct rec_head {
        cudaIpcMemHandle_t h;
        std::uint64_t off;
        std::uint64_t has;
    };
    const std::size_t rec = sizeof(rec_head) + static_cast<std::size_t>(p) * sizeof(std::uint64_t);
    std::vector<char> mine(rec), all(rec * p);
    rec_head hd{};
    if (recv_base) {
        char* base = allocation_base(recv_base);
        AKB_CUDA(cudaIpcGetMemHandle(&hd.h, base));
        hd.off = static_cast<std::uint64_t>(static_cast<char*>(recv_base) - base);
        hd.has = 1;
    }
    std::memcpy(mine.data(), &hd, sizeof(hd));
    std::memcpy(mine.data() + sizeof(hd), recv_off, p * sizeof(std::uint64_t));
    allgather(mine.data(), rec, all.data());
    // 2. map every destination (cached while the peer keeps its allocation), one launch for all
    std::vector<copy_seg> segs;
    for (int q = 0; q < p; ++q) {
        if (q == r || send_cnt[q] == 0) continue;
        rec_head h;
        std::memcpy(&h, all.data() + q * rec, sizeof(h));
        if (!h.has) throw protocol_error("ipc: peer posted no receive buffer for a non-empty slice");
        std::uint64_t roff_q_me;
        std::memcpy(&roff_q_me, all.data() + q * rec + sizeof(h) + r * sizeof(std::uint64_t), sizeof(roff_q_me));
        mapping& m = peers[q];
        const char* hb = reinterpret_cast<const char*>(&h.h);
        if (!m.base || m.handle.size() != sizeof(h.h) || std::memcmp(m.handle.data(), hb, sizeof(h.h)) != 0) {
            if (m.base) AKB_CUDA(cudaIpcCloseMemHandle(m.base));
            m.base = nullptr;
            void* ptr = nullptr;
            AKB_CUDA(cudaIpcOpenMemHandle(&ptr, h.h, cudaIpcMemLazyEnablePeerAccess));
            m.base = static_cast<char*>(ptr);
            m.handle.assign(hb, hb + sizeof(h.h));
        }
        segs.push_back({static_cast<const char*>(send_base) + send_off[q] * eb, m.base + h.off + roff_q_me * eb,
                        send_cnt[q] * eb});
        bytes_sent += send_cnt[q] * eb;
    }
    peer_store(stream, sm_count, segs);
    AKB_CUDA(cudaStreamSynchronize(stream));
    // 3. every rank's stores have landed before anyone reads its receive buffer
    std::uint8_t one = 1;
    std::vector<std::uint8_t> ack(p);
    allgather(&one, 1, ack.data());
}

// ---------------------------------------------------------------------------
// Device rank policy
// ---------------------------------------------------------------------------
namespace {

// #elements <= v[j] in the sorted device array (search_last), for each host needle v[j]
template <typename T>
void device_upper_bounds(ak_ctx* c, const T* sorted, std::uint64_t n, const std::vector<T>& v,
                         std::vector<std::uint64_t>& out) {
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

// Stage policy over a caller's already-sorted device keys (the public stage functions).
template <typename T>
struct sorted_view {
    ak_ctx* c;
    const T* sorted;
    std::uint64_t n;
    void upper_bounds(const std::vector<T>& v, std::vector<std::uint64_t>& out) {
        device_upper_bounds<T>(c, sorted, n, v, out);
    }
};

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
        device_upper_bounds<T>(c, sorted, n, v, out);
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

    const void* sorted_buffer() const { return sorted; }

    // The exchange fused into the P-way merge: run s is read straight from source rank s's
    // sorted array (peers[s]: this GPU, or its HBM over NVLink through a CUDA IPC mapping),
    // at the offset of this rank's slice there (row s of the count matrix), and merged in
    // source-rank order into d_out -- no receive buffer, no separate copy pass.
    std::uint64_t merge_from_peers(const std::vector<const void*>& peers, const std::vector<std::uint64_t>& mat) {
        std::vector<const T*> ptrs;
        std::vector<std::uint64_t> lens;
        std::uint64_t total = 0, remote = 0;
        for (std::size_t s = 0; s < P; ++s) {
            const std::uint64_t len = mat[s * (P + 1) + me];
            if (!len) continue;
            std::uint64_t off = 0;
            for (std::size_t d = 0; d < me; ++d) off += mat[s * (P + 1) + d];
            if (!peers[s]) throw protocol_error("sihsort: a source rank with data mapped no buffer");
            ptrs.push_back(static_cast<const T*>(peers[s]) + off);
            lens.push_back(len);
            total += len;
            if (s != me) remote += len * sizeof(T);
        }
        if (total > cap) throw invalid_argument("sihsort: internal capacity");
        const int tok = ctx_prof_begin(c, KF_EXCHANGE);  // transfer and merge are one step here
        if (ptrs.size() == 1) {
            AKB_CUDA(cudaMemcpyAsync(d_out, ptrs[0], total * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
        } else if (!ptrs.empty()) {
            akb::merge_runs<T>(c, static_cast<int>(ptrs.size()), ptrs.data(), lens.data(), d_out, X, false);
        }
        ctx_prof_end(c, tok);
        AKB_CUDA(cudaStreamSynchronize(c->stream));  // every read of peer memory has finished
        pulled_bytes += remote;
        return total;
    }
    std::uint64_t pulled_bytes = 0;

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

__global__ void iota_u64_kernel(std::uint64_t* __restrict__ out, std::uint64_t n, std::uint64_t base) {
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = base + i;
}

// Distributed sortperm (new work: the reference sihsort is keys-only,
// sihsort.hpp:472-501): the SIHSort protocol over (key, global index) pairs. Local sort #1
// is the stable by-key radix sort of (key, offset + i); splitters, refinement and the count
// exchange run on the keys exactly as for sihsort; the exchange moves keys and indices; the
// second local sort is the stable by-key sort of the received runs concatenated in
// source-rank order (sihsort.hpp:555 sorts again too), so ties keep ascending global index:
// the ranks' outputs concatenated are the globally STABLE sort order and its permutation.
template <typename T>
struct device_local_perm {
    ak_ctx* c;
    const T* d_in;
    std::uint64_t n;
    T* d_out;
    std::uint64_t* d_idx;
    std::uint64_t cap;
    std::size_t P, me;
    std::uint64_t offset;  // global index of this rank's first key
    T* sorted = nullptr;
    std::uint64_t* sidx = nullptr;
    T* X = nullptr;
    std::uint64_t* XV = nullptr;
    T* R = nullptr;
    std::uint64_t* RV = nullptr;
    bool direct = false;
    std::vector<std::uint64_t> roff;
    std::uint64_t payload_bytes = 0;  // index bytes sent to other ranks

    bool peer_merge() const { return false; }
    std::uint64_t size() const { return n; }
    std::uint64_t capacity() const { return cap; }

    void sort_local() {
        direct = (P == 1 && cap >= n);
        const std::uint64_t xn = std::max<std::uint64_t>(n, cap);
        std::size_t need = arena::need(xn * sizeof(T)) + arena::need(xn * 8) + 512;
        if (!direct)
            need += arena::need(n * sizeof(T)) + arena::need(n * 8) + arena::need(cap * sizeof(T)) +
                    arena::need(cap * 8) + 1024;
        ctx_reserve_aux(c, need);
        arena a{static_cast<char*>(c->aux), c->aux_bytes};
        X = a.take<T>(xn);
        XV = a.take<std::uint64_t>(xn);
        if (!direct) {
            sorted = a.take<T>(n);
            sidx = a.take<std::uint64_t>(n);
            R = a.take<T>(cap);
            RV = a.take<std::uint64_t>(cap);
        } else {
            sorted = d_out;
            sidx = d_idx;
        }
        if (n == 0) return;
        iota_u64_kernel<<<static_cast<unsigned>(std::min<std::uint64_t>(ceil_div(n, 256), 4096)), 256, 0, c->stream>>>(
            sidx, n, offset);
        AKB_CUDA(cudaGetLastError());
        c->kernel_launches += 1;
        radix_sort<T, std::uint64_t>(c, SORT_PAIRS, d_in, sorted, X, sidx, sidx, XV, n, false, true);
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
        device_upper_bounds<T>(c, sorted, n, v, out);
    }

    const void* sorted_buffer() const { return sorted; }

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
            if (d != me) payload_bytes += scnt[d] * sizeof(std::uint64_t);
        }
        const int tok = ctx_prof_begin(c, KF_EXCHANGE);
        comm.exchange(sorted, soff.data(), scnt.data(), R, roff.data(), recv_counts.data(), sizeof(T));
        comm.exchange(sidx, soff.data(), scnt.data(), RV, roff.data(), recv_counts.data(), sizeof(std::uint64_t));
        ctx_prof_end(c, tok);
    }

    std::uint64_t merge_from_peers(const std::vector<const void*>&, const std::vector<std::uint64_t>&) {
        throw invalid_argument("sihsort_perm: no pull-merge for payload sorts");
    }

    // local sort #2: the runs concatenated in source-rank order, then the stable by-key sort
    std::uint64_t merge_runs(const std::vector<std::uint64_t>& bounds,
                             const std::vector<std::uint64_t>& recv_counts) {
        if (direct) return n;
        std::uint64_t total = 0;
        for (std::size_t s = 0; s < P; ++s) {
            const std::uint64_t len = recv_counts[s];
            if (len) {
                const T* pk = s == me ? sorted + bounds[me] : R + roff[s];
                const std::uint64_t* pv = s == me ? sidx + bounds[me] : RV + roff[s];
                AKB_CUDA(cudaMemcpyAsync(d_out + total, pk, len * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
                AKB_CUDA(cudaMemcpyAsync(d_idx + total, pv, len * 8, cudaMemcpyDeviceToDevice, c->stream));
            }
            total += len;
        }
        if (total > 1)
            radix_sort<T, std::uint64_t>(c, SORT_PAIRS, d_out, d_out, X, d_idx, d_idx, XV, total, false, true);
        return total;
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
    if (L.pulled_bytes)
        if (auto* ic = dynamic_cast<ipc_comm*>(&comm)) ic->add_pulled(L.pulled_bytes);
    return st.output_count;
}

template <typename T>
std::uint64_t sihsort_perm_device(ak_ctx* c, comm_iface& comm, const T* d_in, std::uint64_t n, T* d_out,
                                  std::uint64_t* d_idx, std::uint64_t cap, const sih_config_c& cfg,
                                  sih_stats_c& st) {
    const std::size_t P = static_cast<std::size_t>(comm.size());
    const std::size_t me = static_cast<std::size_t>(comm.rank());
    // global index offsets: one control allgather of the per-rank counts (not a collective of
    // the reference's accounting, like the count exchange)
    std::vector<std::uint64_t> all(P);
    comm.allgather(&n, sizeof(n), all.data());
    std::uint64_t offset = 0;
    for (std::size_t r = 0; r < me; ++r) offset += all[r];
    device_local_perm<T> L{c, d_in, n, d_out, d_idx, cap, P, me, offset};
    sihsort_run<T>(comm, L, cfg, st);
    st.redistribution_bytes += L.payload_bytes;
    comm.ctr.p2p_bytes += L.payload_bytes;
    return st.output_count;
}

// ---- public stage functions (sihsort.hpp:264-501) ----

template <typename T>
std::uint64_t sample_local_device(ak_ctx* c, const T* sorted, std::uint64_t n, std::uint64_t k, T* host_out) {
    if (n == 0 || k == 0) return 0;
    k = std::min(k, n);
    T* dev = reinterpret_cast<T*>(ctx_split(c, k + 2));
    k = gather_samples<T>(c, sorted, n, k, dev);
    AKB_CUDA(cudaMemcpyAsync(host_out, dev + 2, k * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    return k;
}

template <typename T>
refine_out refine_device(ak_ctx* c, comm_iface& comm, const T* sorted, std::uint64_t n, std::vector<T>& spl,
                         const sih_config_c& cfg) {
    if (spl.size() + 1 != static_cast<std::size_t>(comm.size()) && !spl.empty())
        throw invalid_argument("refine_splitters: need world_size - 1 splitters");
    sorted_view<T> L{c, sorted, n};
    T lo{}, hi{};
    if (n > 0) {
        T* h = static_cast<T*>(ctx_pinned(c, 2 * sizeof(T)));
        AKB_CUDA(cudaMemcpyAsync(h, sorted, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
        AKB_CUDA(cudaMemcpyAsync(h + 1, sorted + n - 1, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        lo = h[0];
        hi = h[1];
    }
    const refine_out r = refine_run<T>(comm, L, spl, n, lo, hi, cfg);
    for (std::uint64_t i = 0; i < r.collectives; ++i) comm.count_collective();
    return r;
}

template <typename T>
std::uint64_t redistribute_device(ak_ctx* c, comm_iface& comm, const T* sorted, std::uint64_t n,
                                  const std::vector<T>& spl, T* out, std::uint64_t cap, std::uint64_t* sends,
                                  std::uint64_t* bytes, std::uint64_t n_total) {
    const std::size_t P = static_cast<std::size_t>(comm.size());
    const std::size_t me = static_cast<std::size_t>(comm.rank());
    if (spl.size() + 1 != P) throw invalid_argument("redistribute: need world_size - 1 splitters");
    sorted_view<T> L{c, sorted, n};
    std::vector<std::uint64_t> bounds, rc;
    count_exchange<T>(comm, L, spl, n, cap, bounds, rc);
    // output = the P received runs concatenated in SOURCE-RANK order, own slice included
    // (sihsort.hpp:490-499): offsets are the exclusive scan of the receive counts
    std::vector<std::uint64_t> roff(P, 0), soff(P), scnt(P);
    std::uint64_t o = 0;
    for (std::size_t s = 0; s < P; ++s) {
        roff[s] = o;
        o += rc[s];
        soff[s] = bounds[s];
        scnt[s] = bounds[s + 1] - bounds[s];
    }
    if (scnt[me])
        AKB_CUDA(cudaMemcpyAsync(out + roff[me], sorted + bounds[me], scnt[me] * sizeof(T), cudaMemcpyDeviceToDevice,
                                 c->stream));
    const bool tail = proto::tail_mode<T>(n_total);
    for (std::size_t d = 0; d < P; ++d) {
        if (d == me) continue;
        const std::uint64_t b = tail ? (scnt[d] + 1) * sizeof(T) : 8 + scnt[d] * sizeof(T);
        *sends += 1;
        *bytes += b;
        comm.ctr.p2p_sends += 1;
        comm.ctr.p2p_bytes += b;
    }
    if (P > 1) {
        const int tok = ctx_prof_begin(c, KF_EXCHANGE);
        comm.exchange(sorted, soff.data(), scnt.data(), out, roff.data(), rc.data(), sizeof(T));
        ctx_prof_end(c, tok);
    }
    AKB_CUDA(cudaStreamSynchronize(c->stream));
    return o;
}

#define AKB_INST(T)                                                                                  \
    template std::uint64_t sihsort_device<T>(ak_ctx*, comm_iface&, const T*, std::uint64_t, T*,      \
                                             std::uint64_t, const sih_config_c&, sih_stats_c&,      \
                                             std::vector<T>*);                                      \
    template std::uint64_t sihsort_perm_device<T>(ak_ctx*, comm_iface&, const T*, std::uint64_t, T*,  \
                                                  std::uint64_t*, std::uint64_t, const sih_config_c&,   \
                                                  sih_stats_c&);                                        \
    template std::uint64_t sample_local_device<T>(ak_ctx*, const T*, std::uint64_t, std::uint64_t, T*); \
    template refine_out refine_device<T>(ak_ctx*, comm_iface&, const T*, std::uint64_t, std::vector<T>&,  \
                                         const sih_config_c&);                                          \
    template std::uint64_t redistribute_device<T>(ak_ctx*, comm_iface&, const T*, std::uint64_t,          \
                                                  const std::vector<T>&, T*, std::uint64_t, std::uint64_t*, \
                                                  std::uint64_t*, std::uint64_t);
AKB_INST(std::int32_t)
AKB_INST(std::uint32_t)
AKB_INST(std::int64_t)
AKB_INST(std::uint64_t)
AKB_INST(float)
AKB_INST(double)

}  // namespace akb
