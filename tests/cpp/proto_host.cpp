// proto_host.cpp -- TEST-ONLY instantiation of the product SIHSort protocol
// (paper_2507_16710_b200/csrc/sih_protocol.hpp) with a host-memory rank policy
// and the callback transport, so the multi-rank host logic (config check,
// summaries, histogram, splitter selection + refinement, count exchange,
// redistribution bookkeeping) runs across real processes over torch.distributed
// gloo on a CPU-only machine. The rank-local data ops here are plain std::
// algorithms standing in for the device policy (test infrastructure only).
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "sih_protocol.hpp"

namespace {

template <typename T>
struct host_local {
    const T* in;
    std::uint64_t n;
    T* out;
    std::uint64_t cap;
    std::size_t P, me;
    std::vector<T> sorted, recv;
    std::vector<std::uint64_t> roff;

    std::uint64_t size() const { return n; }
    std::uint64_t capacity() const { return cap; }
    void sort_local() {
        sorted.assign(in, in + n);
        std::stable_sort(sorted.begin(), sorted.end());
    }
    void samples(std::uint64_t k, std::vector<T>& s, T& front, T& back) {
        front = sorted.front();
        back = sorted.back();
        s.clear();
        if (k == 1) {
            s.push_back(sorted[n / 2]);
            return;
        }
        for (std::uint64_t j = 0; j < k; ++j) s.push_back(sorted[(2 * j * (n - 1) + (k - 1)) / (2 * (k - 1))]);
    }
    void upper_bounds(const std::vector<T>& v, std::vector<std::uint64_t>& o) {
        o.resize(v.size());
        for (std::size_t i = 0; i < v.size(); ++i)
            o[i] = std::upper_bound(sorted.begin(), sorted.end(), v[i]) - sorted.begin();
    }
    void exchange(akb::comm_iface& comm, const std::vector<std::uint64_t>& bounds,
                  const std::vector<std::uint64_t>& rc) {
        roff.assign(P, 0);
        std::uint64_t o = 0;
        for (std::size_t s = 0; s < P; ++s) {
            roff[s] = o;
            if (s != me) o += rc[s];
        }
        recv.resize(o + 1);
        std::vector<std::uint64_t> so(P), sc(P);
        for (std::size_t d = 0; d < P; ++d) {
            so[d] = bounds[d];
            sc[d] = bounds[d + 1] - bounds[d];
        }
        comm.exchange(sorted.data(), so.data(), sc.data(), recv.data(), roff.data(), rc.data(), sizeof(T));
    }
    std::uint64_t merge_runs(const std::vector<std::uint64_t>& bounds, const std::vector<std::uint64_t>& rc) {
        std::vector<T> all;
        for (std::size_t s = 0; s < P; ++s) {
            if (s == me) all.insert(all.end(), sorted.begin() + bounds[me], sorted.begin() + bounds[me + 1]);
            else all.insert(all.end(), recv.begin() + roff[s], recv.begin() + roff[s] + rc[s]);
        }
        std::stable_sort(all.begin(), all.end());  // local sort 2 of 2 (sihsort.hpp:555)
        std::copy(all.begin(), all.end(), out);
        return all.size();
    }
    // peer-mapped variant (only with a transport that maps peers; the callback one does not)
    const void* sorted_buffer() const { return sorted.data(); }
    std::uint64_t merge_from_peers(const std::vector<const void*>& peers, const std::vector<std::uint64_t>& mat) {
        std::vector<T> all;
        for (std::size_t s = 0; s < P; ++s) {
            std::uint64_t off = 0;
            for (std::size_t d = 0; d < me; ++d) off += mat[s * (P + 1) + d];
            const T* src = static_cast<const T*>(peers[s]) + off;
            all.insert(all.end(), src, src + mat[s * (P + 1) + me]);
        }
        std::stable_sort(all.begin(), all.end());
        std::copy(all.begin(), all.end(), out);
        return all.size();
    }
};

thread_local std::string g_err;

}  // namespace

extern "C" const char* proto_last_error() { return g_err.c_str(); }

extern "C" int proto_sihsort_i64(int rank, int size, void* user, akb::akb_allgather_fn ag,
                                 akb::akb_allreduce_fn ar, akb::akb_exchange_fn ex,const std::int64_t* in, std::uint64_t n, std::int64_t* out,
                                 std::uint64_t cap, std::uint64_t* out_count, const akb::sih_config_c* cfg,
                                 akb::sih_stats_c* st) {
    try {
        akb::callback_comm comm(rank, size, user, ag, ar, ex);
        host_local<std::int64_t> L{in, n, out, cap, static_cast<std::size_t>(size), static_cast<std::size_t>(rank)};
        akb::sihsort_run<std::int64_t>(comm, L, *cfg, *st);
        *out_count = st->output_count;
        return 0;
    } catch (const akb::proto_protocol_error&) {
        return 2;
    } catch (const akb::proto_capacity_error& e) {
        *out_count = e.required;
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    } catch (...) {
        return 9;
    }
}
