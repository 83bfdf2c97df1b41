// ctx.cuh -- the execution handle behind the C ABI.
//
// One ak_ctx is the device analogue of the reference's exec_backend handle
// (exec.hpp:31-60): a device, a stream, and the scratch the kernels need
// beyond the caller-owned buffers of sort.hpp:22-65 (look-back tile status,
// digit histograms, tile counters). Calls on one handle are serialised by a
// mutex (reference thread_pool.hpp:37) and, in blocking mode (the default,
// reference SPEC.md:64), synchronise the stream before returning.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <utility>
#include <vector>

#include "ak_common.cuh"

struct ak_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int blocking = 1;
    int sm_count = 148;
    std::mutex mu;

    // general scratch (carved per call; contents undefined between calls)
    void* aux = nullptr;
    std::size_t aux_bytes = 0;

    // radix look-back status: 64-bit self-contained words, epoch tagged so the
    // buffer is never cleared between passes (cleared on growth / tag wrap)
    std::uint64_t* lookback = nullptr;
    std::size_t lookback_words = 0;
    std::uint32_t lb_epoch = 0;

    // scan look-back: one 16-byte descriptor per tile {value bits, status | tag}
    std::uint32_t* scan_flags = nullptr;  // unused (kept for layout stability)
    std::uint64_t* scan_vals = nullptr;   // [2 * tiles]
    std::size_t scan_tiles = 0;
    std::uint32_t scan_epoch = 0;

    // small fixed region: tile counters, histograms, offsets, reduce partials
    void* small = nullptr;
    std::size_t small_bytes = 0;

    // merge-path split points
    std::uint64_t* split = nullptr;
    std::size_t split_cap = 0;

    // hybrid radix sort: range cut points + oversized-range list
    std::uint64_t* cuts = nullptr;
    std::size_t cuts_cap = 0;

    // hybrid radix sort, MSD passes: 16-bit joint histogram + 16-bit / 8-bit bucket cursors
    std::uint64_t* msd = nullptr;
    // third MSD level: [2^24 u64 cursors][2^24 u32 counts][4096 u64 chunk sums]
    std::uint64_t* msd3 = nullptr;

    // work arena of the composite-key sortperm path (two 8-byte words per element)
    void* work = nullptr;
    std::size_t work_bytes = 0;

    // device staging for the *_host entry points (end-to-end path)
    void* stage = nullptr;
    std::size_t stage_bytes = 0;

    // pinned host staging for small device->host reads
    // blocks returned by ak_free, kept for reuse by ak_malloc (the C++ headers stage host
    // spans through per-call device buffers): size -> pointer, at most free_cap bytes held
    std::vector<std::pair<std::size_t, void*>> free_blocks;
    std::size_t free_bytes = 0;
    std::vector<std::pair<void*, std::size_t>> live_blocks;  // ak_malloc'd and not yet freed
    void* pinned = nullptr;
    std::size_t pinned_bytes = 0;

    // counters (reported by ak_ctx_stats)
    std::uint64_t kernel_launches = 0;

    // small keys-only sorts replayed as CUDA graphs (one launch), keyed by their buffers
    struct small_graph {
        const void* kin = nullptr;
        void* kout = nullptr;
        void* kalt = nullptr;
        std::uint64_t n = 0;
        int desc = 0;
        int width = 0;
        const void* cuts = nullptr;
        const void* pinned = nullptr;
        cudaGraphExec_t exec = nullptr;
        std::uint64_t launches = 0;
    };
    std::vector<small_graph> graphs;  // most recent last, at most 4
    small_graph last_small;           // key of the last eager run (captured on a repeat)

    // optional per-kernel-family timing with CUDA events on the launch stream
    int profiling = 0;
    struct timed {
        cudaEvent_t a, b;
        int family;
    };
    std::vector<timed> pending;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> event_pool;
    double family_ms[16] = {};
    std::uint64_t family_count[16] = {};
};

namespace akb {

// Radix look-back word layout: [63:62] flag, [61:48] tag, [47:0] count.
constexpr std::uint64_t LB_AGG = 1ull << 62;
constexpr std::uint64_t LB_INC = 2ull << 62;
constexpr int LB_TAG_SHIFT = 48;
constexpr std::uint32_t LB_TAG_MASK = (1u << 14) - 1;
constexpr std::uint64_t LB_COUNT_MASK = (1ull << 48) - 1;

// Scan flag word layout: [31:30] flag, [29:0] tag.
constexpr std::uint32_t SC_AGG = 1u << 30;
constexpr std::uint32_t SC_INC = 2u << 30;
constexpr std::uint32_t SC_TAG_MASK = (1u << 30) - 1;

constexpr std::size_t SMALL_BYTES = 1u << 20;  // 1 MiB

void ctx_reserve_aux(ak_ctx* c, std::size_t bytes);
// returns the tag to use for one radix pass over `tiles` tiles
std::uint32_t ctx_lookback_pass(ak_ctx* c, std::size_t tiles);
std::uint32_t ctx_scan_pass(ak_ctx* c, std::size_t tiles);
void ctx_finish(ak_ctx* c);  // synchronise when blocking
void* ctx_pinned(ak_ctx* c, std::size_t bytes);
std::uint64_t* ctx_split(ak_ctx* c, std::size_t count);
std::uint64_t* ctx_cuts(ak_ctx* c, std::size_t count);
// MSD-pass tables: [65536 joint counts][65536 16-bit cursors][256 8-bit cursors][8 spare]
// [64 scan-chunk sums][64 x 256 column partials]
std::uint64_t* ctx_msd(ak_ctx* c);
std::uint64_t* ctx_msd3(ak_ctx* c);
void* ctx_stage(ak_ctx* c, std::size_t bytes);
// Kernel attributes live in each device's context: set `func`'s attribute once per device
// (a process may drive several GPUs, one ctx each, from several threads).
void func_attr_once(const ak_ctx* c, const void* func, cudaFuncAttribute attr, int value);
template <typename F>
inline void smem_attr(const ak_ctx* c, F* func, std::size_t bytes) {
    func_attr_once(c, reinterpret_cast<const void*>(func), cudaFuncAttributeMaxDynamicSharedMemorySize,
                   static_cast<int>(bytes));
}
// ctx-owned work arena (grown on demand, reused); nullptr when the allocation fails
void* ctx_work(ak_ctx* c, std::size_t bytes);

// Kernel families for ak_ctx_kernel_time (C ABI: AK_KF_*).
enum kernel_family : int { KF_ONESWEEP = 0, KF_HIST = 1, KF_MERGE = 2, KF_REDUCE = 3, KF_SCAN = 4,
                           KF_SEARCH = 5, KF_EXCHANGE = 6, KF_OTHER = 7, KF_LOCAL = 8, KF_MSD = 9 };
// Bracket one launch with events when profiling is on (returns -1 when off).
int ctx_prof_begin(ak_ctx* c, int family);
void ctx_prof_end(ak_ctx* c, int token);
void ctx_prof_resolve(ak_ctx* c);  // requires the stream to be idle

// Bump allocator over ctx->aux with 256-byte alignment.
struct arena {
    char* base;
    std::size_t cap;
    std::size_t off = 0;
    template <typename T>
    T* take(std::size_t count) {
        off = (off + 255) & ~std::size_t(255);
        T* p = reinterpret_cast<T*>(base + off);
        off += count * sizeof(T);
        if (off > cap) throw cuda_error("internal: aux arena overflow");
        return p;
    }
    static std::size_t need(std::size_t bytes) { return (bytes + 255) & ~std::size_t(255); }
};

}  // namespace akb
