// sih_protocol.hpp -- host-side SIHSort protocol (no CUDA in this header).
//
// The rank-local protocol of the reference's sihsort (sihsort.hpp:21-569),
// written once and instantiated with
//   * a communicator (comm_iface): NCCL across GPUs, an in-process loopback
//     world of P ranks on one GPU (the reference sim::world, sim_comm.hpp),
//     or caller-supplied callbacks;
//   * a rank-local data policy (Local): libak_cuda.so's device policy keeps
//     the keys in HBM (radix sort, device gather/searchsorted, P-way merge).
// Splitter math is host long double, identical to the reference expression by
// expression, so per-rank outputs and stats match the reference exactly.
//
// Local policy contract:
//   std::uint64_t size() const;                         local element count n
//   std::uint64_t capacity() const;                     output capacity
//   void sort_local();                                  local sort 1 of 2 (sihsort.hpp:520)
//   void samples(std::uint64_t k, std::vector<T>& s, T& front, T& back);
//   void upper_bounds(const std::vector<T>& v, std::vector<std::uint64_t>& out);
//   void exchange(comm_iface&, const std::vector<std::uint64_t>& bounds,
//                 const std::vector<std::uint64_t>& recv_counts);
//   std::uint64_t merge_runs(const std::vector<std::uint64_t>& bounds,
//                            const std::vector<std::uint64_t>& recv_counts);  // sort 2 of 2
//   const void* sorted_buffer() const;   // the sorted local keys (peers read their slices)
//   std::uint64_t merge_from_peers(const std::vector<const void*>& peers,
//                                  const std::vector<std::uint64_t>& count_matrix);
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace akb {

// C-layout mirrors of sih_config / sih_stats (sihsort.hpp:21-53).
struct sih_config_c {
    std::uint64_t sample_per_rank;
    std::uint64_t bins;
    std::uint64_t max_refine_rounds;
    double imbalance_tol;
};
struct sih_stats_c {
    std::uint64_t rounds_used;
    std::uint64_t converged;
    double max_deviation;
    std::uint64_t redistribution_sends;
    std::uint64_t redistribution_bytes;
    std::uint64_t collective_ops;
    std::uint64_t output_count;
};

struct proto_protocol_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct proto_capacity_error : std::runtime_error {
    std::uint64_t required;
    proto_capacity_error(const std::string& m, std::uint64_t r) : std::runtime_error(m), required(r) {}
};

// Transport. allgather/allreduce are host-level (tiny control messages);
// exchange moves the bulk slices (pointers are device pointers for the
// device policy). Self slices never go through exchange.
struct comm_iface {
    virtual ~comm_iface() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    virtual void allgather(const void* in, std::size_t bytes, void* out) = 0;
    virtual void allreduce_sum_u64(std::uint64_t* inout, std::size_t n) = 0;
    // for every peer p != rank(): send send_cnt[p] elements at send_base + send_off[p],
    // receive recv_cnt[p] elements into recv_base + recv_off[p]
    virtual void exchange(const void* send_base, const std::uint64_t* send_off,
                          const std::uint64_t* send_cnt, void* recv_base,
                          const std::uint64_t* recv_off, const std::uint64_t* recv_cnt,
                          std::size_t elem_bytes) = 0;
    virtual void abort() noexcept {}
    // the caller's ctx stream (cudaStream_t) and SM count, set before every call that
    // may use the transport (device transports enqueue their copies there)
    virtual void bind(void* /*stream*/, int /*sm_count*/) {}
    // bulk payload bytes this rank has pushed to peers through exchange() (counters)
    virtual std::uint64_t payload_bytes_sent() const { return 0; }
    // user point-to-point messages of rank_comm::send / recv (sim_comm.hpp:92-121): host
    // bytes, FIFO per ordered pair; control = traffic_class::control
    virtual void send_bytes(int /*dest*/, const void* /*p*/, std::size_t /*n*/, bool /*control*/) {
        throw std::runtime_error("transport: point-to-point messages are not supported by this communicator");
    }
    virtual std::vector<char> recv_bytes(int /*src*/) {
        throw std::runtime_error("transport: point-to-point messages are not supported by this communicator");
    }
    // Peer memory: every rank passes one device buffer; on success out[q] is rank q's buffer
    // as addressable from this rank (the same process / GPU, or a CUDA IPC mapping over
    // NVLink). Collective. false (nothing done) when the transport cannot map peers (NCCL).
    virtual bool map_peers(const void* /*local*/, std::vector<const void*>& /*out*/) { return false; }
    // after the ranks' reads of mapped peer buffers: every read has finished (collective)
    virtual void peers_released() {}
    // rank_counters (sim_comm.hpp:33-39)
    struct counters_c {
        std::uint64_t p2p_sends = 0, p2p_bytes = 0, collective_ops = 0, collective_sends = 0,
                      control_bytes_peak = 0;
    };
    virtual counters_c counters() const { return ctr; }
    // one collective of the reference's accounting: 1 op, and the messages this rank would
    // send in its binomial reduce-to-0 + broadcast tree (sim_comm.hpp:124-149)
    void count_collective() {
        ctr.collective_ops += 1;
        ctr.collective_sends += tree_sends(rank(), size());
    }
    static std::uint64_t tree_sends(int r, int p) {
        std::uint64_t s = 0;
        int m = 1;
        while (m * 2 < p) m *= 2;
        for (; m >= 1; m >>= 1)
            if (r >= m && r < 2 * m) {
                ++s;
                break;
            }
        for (m = 1; m < p; m <<= 1)
            if (r < m && r + m < p) ++s;
        return s;
    }
    counters_c ctr;
};

// Callback-backed transport: lets any runtime (torch.distributed, MPI, ...)
// provide the collectives through a C ABI.
extern "C" {
typedef int (*akb_allgather_fn)(void* user, const void* in, std::uint64_t bytes, void* out);
typedef int (*akb_allreduce_fn)(void* user, std::uint64_t* inout, std::uint64_t n);
typedef int (*akb_exchange_fn)(void* user, const void* send_base, const std::uint64_t* send_off,
                               const std::uint64_t* send_cnt, void* recv_base,
                               const std::uint64_t* recv_off, const std::uint64_t* recv_cnt,
                               std::uint64_t elem_bytes);
}

struct callback_comm final : comm_iface {
    int r, p;
    void* user;
    akb_allgather_fn ag;
    akb_allreduce_fn ar;
    akb_exchange_fn ex;
    callback_comm(int rank_, int size_, void* u, akb_allgather_fn a, akb_allreduce_fn b,
                  akb_exchange_fn e)
        : r(rank_), p(size_), user(u), ag(a), ar(b), ex(e) {}
    int rank() const override { return r; }
    int size() const override { return p; }
    void allgather(const void* in, std::size_t bytes, void* out) override {
        if (ag(user, in, bytes, out) != 0) throw std::runtime_error("callback allgather failed");
    }
    void allreduce_sum_u64(std::uint64_t* inout, std::size_t n) override {
        if (ar(user, inout, n) != 0) throw std::runtime_error("callback allreduce failed");
    }
    void exchange(const void* sb, const std::uint64_t* so, const std::uint64_t* sc, void* rb,
                  const std::uint64_t* ro, const std::uint64_t* rc, std::size_t eb) override {
        if (ex(user, sb, so, sc, rb, ro, rc, eb) != 0) throw std::runtime_error("callback exchange failed");
    }
};

namespace proto {

template <typename T>
inline long double to_ld(T v) {
    return static_cast<long double>(v);
}

// ld_to_key (sihsort.hpp:63-74)
template <typename T>
T ld_to_key(long double x) {
    if constexpr (std::is_integral_v<T>) {
        x = std::floor(x + 0.5L);
        if (x <= to_ld(std::numeric_limits<T>::min())) return std::numeric_limits<T>::min();
        if (x >= to_ld(std::numeric_limits<T>::max())) return std::numeric_limits<T>::max();
        return static_cast<T>(x);
    } else {
        return static_cast<T>(x);
    }
}

// equal_width_edges (sihsort.hpp:76-88)
inline std::vector<long double> edges(long double lo, long double hi, std::size_t bins) {
    if (!(lo < hi)) return {lo, lo};
    std::vector<long double> e(bins + 1);
    for (std::size_t i = 0; i <= bins; ++i)
        e[i] = lo + (hi - lo) * static_cast<long double>(i) / static_cast<long double>(bins);
    e.front() = lo;
    e.back() = hi;
    return e;
}

// count_into_bins (sihsort.hpp:91-106)
template <typename T>
void count_bins(const std::vector<T>& samples, const std::vector<long double>& e,
                std::vector<std::uint64_t>& counts) {
    const long double lo = e.front(), hi = e.back();
    const std::size_t k = counts.size();
    for (const T& s : samples) {
        std::size_t bin = 0;
        if (lo < hi) {
            const long double frac = (to_ld(s) - lo) / (hi - lo);
            const auto raw = static_cast<long long>(std::floor(frac * static_cast<long double>(k)));
            bin = raw <= 0 ? 0 : std::min<std::size_t>(static_cast<std::size_t>(raw), k - 1);
        }
        ++counts[bin];
    }
}

// build_interpolated_histogram (sihsort.hpp:286-305) over a rank's gathered samples
struct histogram {
    std::vector<long double> edges;
    std::vector<std::uint64_t> counts;
    std::uint64_t total = 0;
};
template <typename T>
histogram build_histogram(const std::vector<T>& samples, std::size_t bins) {
    histogram h;
    if (samples.empty() || bins == 0) {
        h.edges = {0.0L, 0.0L};
        h.counts = {0};
        return h;
    }
    T lo = samples[0], hi = samples[0];
    for (const T& v : samples) {
        if (v < lo) lo = v;
        if (hi < v) hi = v;
    }
    h.edges = edges(to_ld(lo), to_ld(hi), bins);
    h.counts.assign(h.edges.size() - 1, 0);
    count_bins(samples, h.edges, h.counts);
    h.total = samples.size();
    return h;
}

// select_splitters (sihsort.hpp:310-349)
template <typename T>
std::vector<T> select(const std::vector<long double>& e, const std::vector<std::uint64_t>& counts,
                      std::uint64_t total, std::size_t world) {
    std::vector<T> out;
    if (world <= 1) return out;
    out.reserve(world - 1);
    if (total == 0) {
        out.assign(world - 1, ld_to_key<T>(e.front()));
        return out;
    }
    const std::size_t k = counts.size();
    std::uint64_t cum = 0;
    std::size_t bin = 0;
    for (std::size_t j = 1; j < world; ++j) {
        const long double target =
            static_cast<long double>(total) * static_cast<long double>(j) / static_cast<long double>(world);
        while (bin < k && static_cast<long double>(cum + counts[bin]) < target) {
            cum += counts[bin];
            ++bin;
        }
        long double value;
        if (bin >= k) {
            value = e.back();
        } else {
            const long double frac = counts[bin] == 0
                                         ? 0.0L
                                         : (target - static_cast<long double>(cum)) /
                                               static_cast<long double>(counts[bin]);
            value = e[bin] + frac * (e[bin + 1] - e[bin]);
        }
        T key = ld_to_key<T>(value);
        if (!out.empty() && key < out.back()) key = out.back();
        out.push_back(key);
    }
    return out;
}

template <typename T>
struct summary {
    std::uint64_t n = 0;
    std::uint64_t samples = 0;
    T data_min{}, data_max{}, sample_min{}, sample_max{};
};

// global_summary (sihsort.hpp:221-238): allgather + order-independent fold.
template <typename T>
summary<T> global_summary(comm_iface& comm, const summary<T>& mine) {
    const int P = comm.size();
    std::vector<summary<T>> all(P);
    comm.allgather(&mine, sizeof(summary<T>), all.data());
    summary<T> a = all[0];
    for (int r = 1; r < P; ++r) {
        const summary<T>& b = all[r];
        if (b.n > 0) {
            if (a.n == 0 || b.data_min < a.data_min) a.data_min = b.data_min;
            if (a.n == 0 || a.data_max < b.data_max) a.data_max = b.data_max;
        }
        if (b.samples > 0) {
            if (a.samples == 0 || b.sample_min < a.sample_min) a.sample_min = b.sample_min;
            if (a.samples == 0 || a.sample_max < b.sample_max) a.sample_max = b.sample_max;
        }
        a.n += b.n;
        a.samples += b.samples;
    }
    return a;
}

// piggyback_tail_mode (sihsort.hpp:129-141): only used to report the
// reference-equivalent redistribution_bytes.
template <typename T>
bool tail_mode(std::uint64_t n_total) {
    if constexpr (std::is_integral_v<T>) {
        using U = std::make_unsigned_t<T>;
        return static_cast<unsigned long long>(n_total) <=
               static_cast<unsigned long long>(std::min<U>(static_cast<U>(std::numeric_limits<T>::max()),
                                                           static_cast<U>(~0ULL)));
    } else {
        (void)n_total;
        return false;
    }
}

}  // namespace proto

struct refine_out {
    std::uint64_t rounds_used = 0;
    std::uint64_t converged = 0;
    double max_deviation = 0.0;
    std::uint64_t collectives = 0;
};

// refine_splitters (sihsort.hpp:364-464) on a rank whose sorted keys the policy holds (n keys,
// local min / max data_min / data_max when n > 0); spl is refined in place. Collective.
template <typename T, typename Local>
refine_out refine_run(comm_iface& comm, Local& L, std::vector<T>& spl, std::uint64_t n, T data_min, T data_max,
                      const sih_config_c& cfg) {
    refine_out st;
    const std::size_t P = static_cast<std::size_t>(comm.size());
    if (cfg.max_refine_rounds == 0) return st;
    proto::summary<T> rs;
    rs.n = n;
    if (n > 0) {
        rs.data_min = data_min;
        rs.data_max = data_max;
    }
    const proto::summary<T> s2 = proto::global_summary(comm, rs);
    ++st.collectives;
    const std::uint64_t n_total = s2.n;
    if (P <= 1 || spl.empty() || n_total == 0) {
        st.converged = 1;
        return st;
    }
    const long double ideal = static_cast<long double>(n_total) / static_cast<long double>(P);
    std::vector<T> lo(P - 1, s2.data_min), hi(P - 1, s2.data_max);
    std::vector<std::uint64_t> flo(P - 1, 0), fhi(P - 1, n_total);
    std::vector<bool> frozen(P - 1, false);
    std::vector<std::uint64_t> le;
    for (std::size_t round = 1; round <= cfg.max_refine_rounds; ++round) {
        L.upper_bounds(spl, le);
        comm.allreduce_sum_u64(le.data(), le.size());
        ++st.collectives;
        long double max_dev = 0.0L;
        for (std::size_t r = 0; r < P; ++r) {
            const std::uint64_t upper = r + 1 < P ? le[r] : n_total;
            const std::uint64_t lower = r > 0 ? le[r - 1] : 0;
            const long double bucket = static_cast<long double>(upper - lower);
            max_dev = std::max(max_dev, std::abs(bucket - ideal) / ideal);
        }
        st.rounds_used = round;
        st.max_deviation = static_cast<double>(max_dev);
        if (max_dev <= static_cast<long double>(cfg.imbalance_tol)) {
            st.converged = 1;
            break;
        }
        if (round == cfg.max_refine_rounds) break;
        for (std::size_t j = 0; j + 1 < P; ++j) {
            if (frozen[j]) continue;
            const long double target = ideal * static_cast<long double>(j + 1);
            const std::uint64_t measured = le[j];
            if (static_cast<long double>(measured) < target) {
                lo[j] = spl[j];
                flo[j] = measured;
            } else if (static_cast<long double>(measured) > target) {
                hi[j] = spl[j];
                fhi[j] = measured;
            } else {
                frozen[j] = true;
                continue;
            }
            if (!(lo[j] < hi[j]) || fhi[j] <= flo[j]) {
                frozen[j] = true;
                continue;
            }
            const long double frac = (target - static_cast<long double>(flo[j])) /
                                     static_cast<long double>(fhi[j] - flo[j]);
            const long double cand = proto::to_ld(lo[j]) + (proto::to_ld(hi[j]) - proto::to_ld(lo[j])) * frac;
            T key = proto::ld_to_key<T>(cand);
            if constexpr (std::is_integral_v<T>) {
                if (key <= lo[j]) key = static_cast<T>(lo[j] + 1);
                if (hi[j] < key) key = hi[j];
            } else {
                if (!(key > lo[j]) || !(key < hi[j]))
                    key = proto::ld_to_key<T>((proto::to_ld(lo[j]) + proto::to_ld(hi[j])) / 2);
                if (!(key > lo[j]) || !(key < hi[j])) {
                    frozen[j] = true;
                    continue;
                }
            }
            spl[j] = key;
        }
        for (std::size_t j = 1; j + 1 < P; ++j)
            if (spl[j] < spl[j - 1]) spl[j] = spl[j - 1];
    }
    return st;
}

// slice_bounds + P x P count exchange (with every rank's capacity) of redistribute
// (sihsort.hpp:110-123, :472-501): bounds (P+1) of this rank's slices, recv_counts (P) it
// receives from each source. Throws proto_capacity_error (on every rank alike) when some rank's
// capacity is short. Collective.
template <typename T, typename Local>
void count_exchange(comm_iface& comm, Local& L, const std::vector<T>& spl, std::uint64_t n, std::uint64_t capacity,
                    std::vector<std::uint64_t>& bounds, std::vector<std::uint64_t>& recv_counts,
                    std::vector<std::uint64_t>* matrix = nullptr) {
    const std::size_t P = static_cast<std::size_t>(comm.size());
    const std::size_t me = static_cast<std::size_t>(comm.rank());
    bounds.assign(P + 1, 0);
    {
        std::vector<std::uint64_t> cuts;
        L.upper_bounds(spl, cuts);
        for (std::size_t j = 0; j + 1 < P; ++j) bounds[j + 1] = cuts[j];
        bounds[P] = n;
    }
    // P x (P+1) matrix: row r = send counts of rank r to each dest, then its capacity
    std::vector<std::uint64_t> row(P + 1), mat((P + 1) * P);
    for (std::size_t d = 0; d < P; ++d) row[d] = bounds[d + 1] - bounds[d];
    row[P] = capacity;
    comm.allgather(row.data(), row.size() * sizeof(std::uint64_t), mat.data());
    recv_counts.assign(P, 0);
    for (std::size_t s = 0; s < P; ++s) recv_counts[s] = mat[s * (P + 1) + me];
    if (matrix) *matrix = mat;
    for (std::size_t r = 0; r < P; ++r) {
        std::uint64_t need = 0;
        for (std::size_t s = 0; s < P; ++s) need += mat[s * (P + 1) + r];
        if (need > mat[r * (P + 1) + P]) {
            std::uint64_t mine_need = 0;
            for (std::size_t s = 0; s < P; ++s) mine_need += recv_counts[s];
            throw proto_capacity_error("sihsort: output capacity too small on rank " + std::to_string(r),
                                       mine_need);
        }
    }
}

// A rank policy may opt out of the fused pull-merge (bool peer_merge() const): the
// payload-carrying distributed sortperm exchanges first, then sorts its received runs.
template <typename Local>
bool peer_merge_ok(const Local& L) {
    if constexpr (requires { L.peer_merge(); }) return L.peer_merge();
    else return true;
}

// The whole per-rank protocol (sihsort.hpp:508-559).
template <typename T, typename Local>
void sihsort_run(comm_iface& comm, Local& L, const sih_config_c& cfg, sih_stats_c& st,
                 std::vector<T>* splitters_out = nullptr) {
    const std::size_t P = static_cast<std::size_t>(comm.size());
    const std::size_t me = static_cast<std::size_t>(comm.rank());
    const std::uint64_t spr = cfg.sample_per_rank > 0 ? cfg.sample_per_rank : 32 * P;
    const std::uint64_t bins = cfg.bins > 0 ? cfg.bins : 8 * P;
    std::memset(&st, 0, sizeof(st));
    std::uint64_t collectives = 0;

    // check_consistent_config (sihsort.hpp:240-256)
    {
        const std::uint64_t sig[4] = {cfg.sample_per_rank, cfg.bins, cfg.max_refine_rounds,
                                      std::bit_cast<std::uint64_t>(cfg.imbalance_tol)};
        std::vector<std::uint64_t> all(4 * P);
        comm.allgather(sig, sizeof(sig), all.data());
        ++collectives;
        for (std::size_t r = 0; r < P; ++r)
            for (int i = 0; i < 4; ++i)
                if (all[4 * r + i] != sig[i])
                    throw proto_protocol_error("sihsort: configuration differs across ranks");
    }

    L.sort_local();  // local sort 1 of 2
    const std::uint64_t n = L.size();

    // sample_local + global_summary (sihsort.hpp:522-523)
    std::vector<T> samples;
    proto::summary<T> mine;
    mine.n = n;
    if (n > 0) {
        const std::uint64_t k = std::min<std::uint64_t>(spr, n);
        if (P > 1) {
            L.samples(k, samples, mine.data_min, mine.data_max);
            mine.samples = samples.size();
            if (!samples.empty()) {
                mine.sample_min = samples.front();
                mine.sample_max = samples.back();
            }
        } else {
            // one rank: select_splitters returns P - 1 = 0 splitters and refine stops before
            // reading the bounds, so the sample VALUES are never used; only their count enters
            // the protocol (the histogram allreduce happens iff samples exist). The device
            // gather and its host round trip are skipped.
            mine.samples = k;
        }
    }
    const proto::summary<T> g = proto::global_summary(comm, mine);
    ++collectives;

    std::vector<T> spl;
    if (g.samples == 0) {
        spl.assign(P > 0 ? P - 1 : 0, T{});
    } else {
        // distributed histogram (sihsort.hpp:526-540)
        const auto e = proto::edges(proto::to_ld(g.sample_min), proto::to_ld(g.sample_max), bins);
        std::vector<std::uint64_t> counts(e.size() - 1, 0);
        proto::count_bins(samples, e, counts);
        comm.allreduce_sum_u64(counts.data(), counts.size());
        ++collectives;
        spl = proto::select<T>(e, counts, g.samples, P);
    }

    // refine_splitters (sihsort.hpp:364-464)
    {
        refine_out r = refine_run<T>(comm, L, spl, n, mine.data_min, mine.data_max, cfg);
        collectives += r.collectives;
        st.rounds_used = r.rounds_used;
        st.converged = r.converged;
        st.max_deviation = r.max_deviation;
    }

    // redistribute (sihsort.hpp:472-501): slice_bounds + count exchange + payload
    std::vector<std::uint64_t> bounds, recv_counts, mat;
    count_exchange<T>(comm, L, spl, n, L.capacity(), bounds, recv_counts, &mat);
    // (the count allgather replaces the reference's piggybacked counts: not a collective of the
    //  reference's accounting, so not counted in collective_ops)
    std::vector<std::uint64_t> row(P);
    for (std::size_t d = 0; d < P; ++d) row[d] = bounds[d + 1] - bounds[d];
    const bool tail = proto::tail_mode<T>(g.n);
    for (std::size_t d = 0; d < P; ++d) {
        if (d == me) continue;
        const std::uint64_t len = row[d];
        st.redistribution_sends += 1;
        st.redistribution_bytes += tail ? (len + 1) * sizeof(T) : 8 + len * sizeof(T);
    }
    // exchange + local sort 2 of 2: when the transport maps the peers' sorted arrays, the P-way
    // merge reads every incoming run straight from its source rank (the all-to-all fused into
    // the merge: no copy through a receive buffer); otherwise the runs are exchanged first
    std::vector<const void*> peers;
    if (P > 1 && peer_merge_ok(L) && comm.map_peers(L.sorted_buffer(), peers)) {
        st.output_count = L.merge_from_peers(peers, mat);
        comm.peers_released();
    } else {
        L.exchange(comm, bounds, recv_counts);
        st.output_count = L.merge_runs(bounds, recv_counts);
    }
    st.collective_ops = collectives;
    for (std::uint64_t i = 0; i < collectives; ++i) comm.count_collective();
    comm.ctr.p2p_sends += st.redistribution_sends;
    comm.ctr.p2p_bytes += st.redistribution_bytes;
    if (splitters_out) *splitters_out = spl;
}

}  // namespace akb
