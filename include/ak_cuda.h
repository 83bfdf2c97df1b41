/*
 * ak_cuda.h -- C ABI of libak_cuda.so, the B200 (sm_100a) implementation of the
 * sorting-centred primitive hot path of arXiv 2507.16710 (AcceleratedKernels.jl),
 * drop-in for the reference C++ API in /root/reference/proj/include/ak.
 *
 * Conventions
 *   - Every entry point returns an ak_status; on failure ak_last_error() gives a
 *     thread-local message. Argument validation happens BEFORE any mutation or
 *     kernel launch, exactly where the reference throws std::invalid_argument.
 *   - Data pointers are DEVICE pointers unless the symbol ends in _host.
 *   - Calls on one ak_ctx are serialised and, in blocking mode (default, the
 *     reference contract SPEC.md:64), complete before returning. With
 *     ak_ctx_set_blocking(ctx, 0) kernels stay queued on the ctx stream.
 *   - Type suffixes: i32 u32 i64 u64 f32 f64 (keys); payloads are moved as
 *     opaque 32/64-bit words (b32/b64); sortperm indices are i32 or i64.
 *   - Comparator: desc = 0 is std::less<T>, desc = 1 is std::greater<T>.
 *     Floats: -0.0 == +0.0 (stable order kept); NaN unsupported (as the reference).
 *
 * Each declaration cites the reference interface it replaces.
 */
#ifndef AK_CUDA_H
#define AK_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AK_OK = 0,
    AK_EINVAL = 1,     /* std::invalid_argument (sort.hpp:182-184, scan.hpp:32-37, search.hpp:40-43) */
    AK_EPROTOCOL = 2,  /* ak::sim::protocol_error (sim_comm.hpp:24-26, sihsort.hpp:253-255) */
    AK_ETRANSPORT = 3, /* ak::sim::transport_error (sim_comm.hpp:19-21) / NCCL failure */
    AK_ECUDA = 4,      /* CUDA runtime failure */
    AK_ECAPACITY = 6,  /* sihsort output capacity too small; *out_count = required */
    AK_EINTERNAL = 9
} ak_status;

typedef struct ak_ctx ak_ctx;   /* exec_backend (exec.hpp:31-60) with exec_kind::cuda */
typedef struct ak_comm ak_comm; /* sim::rank_comm (sim_comm.hpp:84-181) over NCCL */

/* sih_config (sihsort.hpp:21-26); zero sample_per_rank/bins -> 32P / 8P */
typedef struct {
    uint64_t sample_per_rank;
    uint64_t bins;
    uint64_t max_refine_rounds;
    double imbalance_tol;
} ak_sih_config;

/* sih_stats (sihsort.hpp:45-53). redistribution_bytes uses the reference's
 * piggyback accounting (sihsort.hpp:143-160) so the numbers compare 1:1. */
typedef struct {
    uint64_t rounds_used;
    uint64_t converged;
    double max_deviation;
    uint64_t redistribution_sends;
    uint64_t redistribution_bytes;
    uint64_t collective_ops;
    uint64_t output_count;
} ak_sih_stats;

const char* ak_last_error(void);
const char* ak_version(void);

/* ---- handle (exec.hpp:38-46: exec_backend::sequential/threaded -> cuda) ---- */
int ak_ctx_create(int device, void* cuda_stream /* NULL: own stream */, ak_ctx** out);
int ak_ctx_destroy(ak_ctx* ctx);
int ak_ctx_set_blocking(ak_ctx* ctx, int blocking);
int ak_ctx_synchronize(ak_ctx* ctx);
int ak_ctx_reserve(ak_ctx* ctx, uint64_t aux_bytes);
uint64_t ak_ctx_kernel_launches(const ak_ctx* ctx);
void* ak_ctx_stream(const ak_ctx* ctx);
/* Per-kernel-family device time, bracketed by CUDA events on the ctx stream
 * (bench.py's live roofline). Families: */
enum { AK_KF_ONESWEEP = 0, AK_KF_HIST = 1, AK_KF_MERGE = 2, AK_KF_REDUCE = 3, AK_KF_SCAN = 4,
       AK_KF_SEARCH = 5, AK_KF_EXCHANGE = 6, AK_KF_OTHER = 7,
       AK_KF_LOCAL = 8 /* hybrid sort: on-chip range sort */,
       AK_KF_MSD = 9 /* hybrid sort: unstable top-digit partition passes */ };
int ak_ctx_set_profiling(ak_ctx* ctx, int on);
/* synchronises the stream, then reports accumulated ms and launch count */
int ak_ctx_kernel_time(ak_ctx* ctx, int family, double* ms, uint64_t* launches);
int ak_ctx_reset_kernel_time(ak_ctx* ctx);

/* ---- device memory helpers for host-side callers (drop-in headers) ---- */
int ak_malloc(ak_ctx* ctx, uint64_t bytes, void** out);
int ak_free(ak_ctx* ctx, void* p);
int ak_memcpy(ak_ctx* ctx, void* dst, const void* src, uint64_t bytes); /* any direction, blocking */

/* ---- scratch queries: sort_buffers::required_bytes (sort.hpp:22-65) ---- */
uint64_t ak_sort_scratch_bytes(uint64_t n, int key_bytes);
uint64_t ak_sort_by_key_scratch_bytes(uint64_t n, int key_bytes, int payload_bytes);
uint64_t ak_sortperm_scratch_bytes(uint64_t n, int key_bytes, int index_bytes);
uint64_t ak_sortperm_lowmem_scratch_bytes(uint64_t n, int index_bytes);
/* device scratch the ctx keeps beyond the caller buffers (look-back, histograms) */
uint64_t ak_sort_ctx_bytes(uint64_t n, int key_bytes);

/* ---- merge_sort (sort.hpp:180-194): stable, in place, scratch >= n ---- */
#define AK_DECL_SORT(S, T)                                                                      \
    int ak_merge_sort_##S(ak_ctx* ctx, T* data, uint64_t n, T* scratch, uint64_t scratch_n,      \
                          int desc);                                                            \
    int ak_merge_sort_host_##S(ak_ctx* ctx, T* host_data, uint64_t n, int desc);                \
    /* merge_sort_by_key (sort.hpp:211-229) */                                                  \
    int ak_merge_sort_by_key_##S##_b32(ak_ctx* ctx, T* keys, uint64_t n_keys, void* payload,     \
                                       uint64_t n_payload, T* scratch_keys, uint64_t sk_n,      \
                                       void* scratch_payload, uint64_t sp_n, int desc);         \
    int ak_merge_sort_by_key_##S##_b64(ak_ctx* ctx, T* keys, uint64_t n_keys, void* payload,     \
                                       uint64_t n_payload, T* scratch_keys, uint64_t sk_n,      \
                                       void* scratch_payload, uint64_t sp_n, int desc);         \
    /* sortperm (sort.hpp:238-262): working_keys + scratch_keys + scratch_index */             \
    int ak_sortperm_##S##_i32(ak_ctx* ctx, const T* data, uint64_t n, int32_t* out,             \
                              uint64_t out_n, T* working_keys, uint64_t wk_n, T* scratch_keys,  \
                              uint64_t sk_n, int32_t* scratch_index, uint64_t si_n, int desc);  \
    int ak_sortperm_##S##_i64(ak_ctx* ctx, const T* data, uint64_t n, int64_t* out,             \
                              uint64_t out_n, T* working_keys, uint64_t wk_n, T* scratch_keys,  \
                              uint64_t sk_n, int64_t* scratch_index, uint64_t si_n, int desc);  \
    /* sortperm_lowmem (sort.hpp:267-290): index scratch only */                                \
    int ak_sortperm_lowmem_##S##_i32(ak_ctx* ctx, const T* data, uint64_t n, int32_t* out,      \
                                     uint64_t out_n, int32_t* scratch_index, uint64_t si_n,     \
                                     int desc);                                                 \
    int ak_sortperm_lowmem_##S##_i64(ak_ctx* ctx, const T* data, uint64_t n, int64_t* out,      \
                                     uint64_t out_n, int64_t* scratch_index, uint64_t si_n,     \
                                     int desc);                                                 \
    /* reduce / mapreduce (reduce.hpp:62-75): op 0 sum 1 min 2 max; map 0 id 1 abs 2 square */  \
    int ak_reduce_##S(ak_ctx* ctx, const T* x, uint64_t n, int op, int map, T init,             \
                      T* host_result);                                                          \
    int ak_reduce_device_##S(ak_ctx* ctx, const T* x, uint64_t n, int op, int map, T init,      \
                             T* device_result);                                                 \
    /* accumulate (scan.hpp:29-79): out may alias x; chunk_size >= 1 (association is exact */  \
    /* for integers; floats accumulate in double) */                                            \
    int ak_accumulate_##S(ak_ctx* ctx, const T* x, uint64_t n, T* out, uint64_t out_n, int op,   \
                          int inclusive, T init, uint64_t chunk_size);                          \
    /* stable P-way merge of sorted device runs, ties to the lower run (the second local sort  */ \
    /* of sihsort.hpp:555 as a merge); 1 <= P <= 4096; scratch >= sum(lens) elements */          \
    int ak_merge_runs_##S(ak_ctx* ctx, int P, const T* const* runs, const uint64_t* lens, T* dst,  \
                          T* scratch, int desc);                                                \
    /* searchsorted (search.hpp:36-50): side 0 first, 1 last; out: device uint64[m] */          \
    int ak_searchsorted_##S(ak_ctx* ctx, const T* hay, uint64_t n, const T* needles,            \
                            uint64_t m, int side_last, int desc, int validate, uint64_t* out);   \
    /* sihsort (sihsort.hpp:508-569) over an NCCL communicator; in is not modified; */         \
    /* out has capacity out_cap; *out_count = elements written (or required). */               \
    int ak_sihsort_##S(ak_ctx* ctx, ak_comm* comm, const T* in, uint64_t n, T* out,             \
                       uint64_t out_cap, uint64_t* out_count, const ak_sih_config* cfg,         \
                       ak_sih_stats* stats);                                                    \
    int ak_sihsort_host_##S(ak_ctx* ctx, ak_comm* comm, const T* host_in, uint64_t n,           \
                            T* host_out, uint64_t out_cap, uint64_t* out_count,                 \
                            const ak_sih_config* cfg, ak_sih_stats* stats);                     \
    /* P logical ranks on ONE device (sim::world + run_ranks, sim_comm.hpp:41-218) */           \
    int ak_sihsort_loopback_##S(int device, uint64_t P, const T* const* in, const uint64_t* n,  \
                                T* const* out, const uint64_t* out_cap, uint64_t* out_count,    \
                                const ak_sih_config* cfg, ak_sih_stats* stats);                 \
    /* distributed sortperm (new: the reference sihsort is keys-only, sihsort.hpp:472-501): */ \
    /* this rank's slice of the globally STABLE order of all ranks' keys -> out (keys) and */   \
    /* out_idx (global indices: rank r's key i is sum of the lower ranks' n + i); capacity */   \
    /* out_cap for both; stats as sihsort plus the index bytes in redistribution_bytes */       \
    int ak_sihsort_perm_##S(ak_ctx* ctx, ak_comm* comm, const T* in, uint64_t n, T* out,        \
                            uint64_t* out_idx, uint64_t out_cap, uint64_t* out_count,           \
                            const ak_sih_config* cfg, ak_sih_stats* stats);                     \
    int ak_sihsort_perm_loopback_##S(int device, uint64_t P, const T* const* in,               \
                                     const uint64_t* n, T* const* out, uint64_t* const* out_idx, \
                                     const uint64_t* out_cap, uint64_t* out_count,              \
                                     const ak_sih_config* cfg, ak_sih_stats* stats);            \
    /* sihsort stages. sample_local (sihsort.hpp:264-282): k order statistics of the sorted */  \
    /* device keys -> host_out[min(k, n)] */                                                    \
    int ak_sample_local_##S(ak_ctx* ctx, const T* sorted, uint64_t n, uint64_t k, T* host_out,   \
                            uint64_t* count);                                                   \
    /* build_interpolated_histogram (sihsort.hpp:286-305) of host samples: edges[nbins + 1], */ \
    /* counts[nbins], nbins <= max(bins, 1) <= cap_bins */                                       \
    int ak_build_interpolated_histogram_##S(const T* samples, uint64_t m, uint64_t bins,         \
                                            long double* edges, uint64_t* counts,               \
                                            uint64_t cap_bins, uint64_t* nbins, uint64_t* total); \
    /* select_splitters (sihsort.hpp:310-349) -> out[world - 1] */                              \
    int ak_select_splitters_##S(const long double* edges, const uint64_t* counts, uint64_t nbins, \
                                uint64_t total, uint64_t world, T* out);                        \
    /* refine_splitters (sihsort.hpp:364-464), collective: host splitters[m] refined in place */ \
    int ak_refine_splitters_##S(ak_ctx* ctx, ak_comm* comm, const T* sorted, uint64_t n,         \
                                T* splitters, uint64_t m, const ak_sih_config* cfg,             \
                                uint64_t* rounds_used, int* converged, double* max_deviation);  \
    /* redistribute (sihsort.hpp:472-501), collective: out (device, capacity cap) = the P */     \
    /* received slices concatenated in source-rank order (own slice included); sends/bytes */   \
    /* = the reference's message accounting (may be NULL) */                                    \
    int ak_redistribute_##S(ak_ctx* ctx, ak_comm* comm, const T* sorted, uint64_t n,             \
                            const T* splitters, uint64_t m, uint64_t n_total, T* out,           \
                            uint64_t cap, uint64_t* out_count, uint64_t* sends, uint64_t* bytes);

/* int16 and int128 keys (dtype.hpp:14-21): the sort family only (merge_sort, by_key,
 * sortperm, sortperm_lowmem); int16 sorts widened to int32, int128 as a stable LSD over its
 * two 64-bit halves. Uses a ctx-owned work arena. */
typedef __int128 ak_int128;
#define AK_DECL_SORT_ONLY(S, T)                                                                 \
    int ak_merge_sort_##S(ak_ctx* ctx, T* data, uint64_t n, T* scratch, uint64_t scratch_n,      \
                          int desc);                                                            \
    int ak_merge_sort_host_##S(ak_ctx* ctx, T* host_data, uint64_t n, int desc);                \
    int ak_merge_sort_by_key_##S##_b32(ak_ctx* ctx, T* keys, uint64_t n_keys, void* payload,     \
                                       uint64_t n_payload, T* scratch_keys, uint64_t sk_n,      \
                                       void* scratch_payload, uint64_t sp_n, int desc);         \
    int ak_merge_sort_by_key_##S##_b64(ak_ctx* ctx, T* keys, uint64_t n_keys, void* payload,     \
                                       uint64_t n_payload, T* scratch_keys, uint64_t sk_n,      \
                                       void* scratch_payload, uint64_t sp_n, int desc);         \
    int ak_sortperm_##S##_i32(ak_ctx* ctx, const T* data, uint64_t n, int32_t* out,             \
                              uint64_t out_n, T* working_keys, uint64_t wk_n, T* scratch_keys,  \
                              uint64_t sk_n, int32_t* scratch_index, uint64_t si_n, int desc);  \
    int ak_sortperm_##S##_i64(ak_ctx* ctx, const T* data, uint64_t n, int64_t* out,             \
                              uint64_t out_n, T* working_keys, uint64_t wk_n, T* scratch_keys,  \
                              uint64_t sk_n, int64_t* scratch_index, uint64_t si_n, int desc);  \
    int ak_sortperm_lowmem_##S##_i32(ak_ctx* ctx, const T* data, uint64_t n, int32_t* out,      \
                                     uint64_t out_n, int32_t* scratch_index, uint64_t si_n,     \
                                     int desc);                                                 \
    int ak_sortperm_lowmem_##S##_i64(ak_ctx* ctx, const T* data, uint64_t n, int64_t* out,      \
                                     uint64_t out_n, int64_t* scratch_index, uint64_t si_n,     \
                                     int desc);
AK_DECL_SORT_ONLY(i16, int16_t)
AK_DECL_SORT_ONLY(i128, ak_int128)

AK_DECL_SORT(i32, int32_t)
AK_DECL_SORT(u32, uint32_t)
AK_DECL_SORT(i64, int64_t)
AK_DECL_SORT(u64, uint64_t)
AK_DECL_SORT(f32, float)
AK_DECL_SORT(f64, double)

/* ---- multi-rank reduce / scan over a communicator (the reference has
 * only single-process reduce.hpp / scan.hpp): local device pass + one allgather of the P rank
 * partials, folded in rank order; init must be neutral for the op (reduce.hpp:12-14) ---- */
#define AK_DECL_DIST(S, T)                                                                        \
    int ak_reduce_all_##S(ak_ctx* ctx, ak_comm* comm, const T* x, uint64_t n, int op, int map,     \
                          T init, T* host_result);                                                \
    int ak_accumulate_all_##S(ak_ctx* ctx, ak_comm* comm, const T* x, uint64_t n, T* out,         \
                              uint64_t out_n, int op, int inclusive, T init);
AK_DECL_DIST(i32, int32_t)
AK_DECL_DIST(u32, uint32_t)
AK_DECL_DIST(i64, int64_t)
AK_DECL_DIST(u64, uint64_t)
AK_DECL_DIST(f32, float)
AK_DECL_DIST(f64, double)

/* ---- any_pred / all_pred (predicates.hpp:57-78): element predicate x OP value with
 * OP 0 <, 1 <=, 2 >, 3 >=, 4 ==, 5 !=; algo 0 early_exit, 1 via_mapreduce (same result);
 * *result = 0/1. Empty input: any -> 0, all -> 1 ---- */
#define AK_DECL_PRED(S, T)                                                                        \
    int ak_any_pred_##S(ak_ctx* ctx, const T* x, uint64_t n, int op, T value, int algo, int* result); \
    int ak_all_pred_##S(ak_ctx* ctx, const T* x, uint64_t n, int op, T value, int algo, int* result);
AK_DECL_PRED(u8, uint8_t)
AK_DECL_PRED(i8, int8_t)
AK_DECL_PRED(i16, int16_t)
AK_DECL_PRED(i32, int32_t)
AK_DECL_PRED(u32, uint32_t)
AK_DECL_PRED(i64, int64_t)
AK_DECL_PRED(u64, uint64_t)
AK_DECL_PRED(f32, float)
AK_DECL_PRED(f64, double)

/* ---- communicators (replace sim::world / rank_comm / run_ranks) ---- */
int ak_nccl_unique_id(void* out, uint64_t bytes /* >= 128 */);
int ak_comm_nccl_create(const void* unique_id, int nranks, int rank, int device, ak_comm** out);
/* caller-provided transport (e.g. torch.distributed); exchange pointers are device pointers */
typedef int (*ak_allgather_fn)(void* user, const void* in, uint64_t bytes, void* out);
typedef int (*ak_allreduce_u64_fn)(void* user, uint64_t* inout, uint64_t n);
typedef int (*ak_exchange_fn)(void* user, const void* send_base, const uint64_t* send_off,
                              const uint64_t* send_cnt, void* recv_base, const uint64_t* recv_off,
                              const uint64_t* recv_cnt, uint64_t elem_bytes);
int ak_comm_callbacks_create(int nranks, int rank, void* user, ak_allgather_fn ag,
                             ak_allreduce_u64_fn ar, ak_exchange_fn ex, ak_comm** out);
/* one process per GPU, bulk slices moved by a peer-store kernel straight into the peers'
 * receive buffers (CUDA IPC mappings, P2P over NVLink/NVSwitch; same-GPU processes work too);
 * tiny control messages through the caller's allgather / allreduce callbacks (e.g. gloo).
 * Replaces sim_comm's send/recv of redistribute (sihsort.hpp:481-499, sim_comm.cpp:42-90). */
int ak_comm_ipc_create(int nranks, int rank, int device, void* user, ak_allgather_fn ag,
                       ak_allreduce_u64_fn ar, ak_comm** out);
/* bulk payload bytes this rank pushed to peers so far (NCCL / IPC transports; else 0) */
int ak_comm_bytes_sent(const ak_comm* comm, uint64_t* out);
/* sim::world + rank_comm (sim_comm.hpp:41-181) on ONE device: P logical ranks, each driven
 * by its own host thread and ak_ctx; collectives are host-level, slices move device to
 * device. abort() wakes every blocked rank with AK_ETRANSPORT (sim_comm.cpp:19-25). */
typedef struct ak_world ak_world;
int ak_world_create(int ranks, ak_world** out);
int ak_world_create_ex(int ranks, uint64_t queue_capacity, ak_world** out); /* sim_comm.hpp:45-47 */
/* rank_comm::send / recv (sim_comm.hpp:92-96): host bytes, FIFO per ordered pair. Loopback:
 * bounded queue (send blocks while queue_capacity messages wait); NCCL: rendezvous (returns
 * once the peer received). recv: if *n (the message size) exceeds cap, AK_ECAPACITY and the
 * message stays pending for the next recv from src. control: traffic_class::control. */
int ak_comm_send(ak_comm* comm, ak_ctx* ctx, int dest, const void* bytes, uint64_t n, int control);
int ak_comm_recv(ak_comm* comm, ak_ctx* ctx, int src, void* buf, uint64_t cap, uint64_t* n);
/* every rank's `bytes` (same on all ranks), gathered in rank order into out[P * bytes]; counted
 * as one collective (the basis of rank_comm::all_reduce(local, merge), sim_comm.hpp:124-149) */
int ak_comm_allgather(ak_comm* comm, ak_ctx* ctx, const void* in, uint64_t bytes, void* out);
/* rank_counters (sim_comm.hpp:33-39) */
typedef struct ak_rank_counters {
    uint64_t p2p_sends, p2p_bytes, collective_ops, collective_sends, control_bytes_peak;
} ak_rank_counters;
int ak_comm_counters(const ak_comm* comm, ak_rank_counters* out);
int ak_world_size(const ak_world* w);
int ak_world_abort(ak_world* w);
int ak_world_destroy(ak_world* w);
int ak_comm_loopback_create(ak_world* w, int rank, ak_comm** out);
/* 1 when p is device (or managed) memory, else 0: the C++ headers run host spans through
 * HBM staging and device spans in place */
int ak_pointer_is_device(const void* p);
int ak_comm_rank(const ak_comm* comm);
int ak_comm_size(const ak_comm* comm);
int ak_comm_allreduce_sum_u64(ak_comm* comm, ak_ctx* ctx, uint64_t* host_inout, uint64_t n);
int ak_comm_allreduce_max_f64(ak_comm* comm, ak_ctx* ctx, double* host_inout, uint64_t n);
int ak_comm_barrier(ak_comm* comm, ak_ctx* ctx);
int ak_comm_destroy(ak_comm* comm);

/* ---- bench input generation (reference bench.cpp:44-58, :164-173) ---- */
/* keys of rank r: mt19937_64(seed + 0x9e3779b97f4a7c15*(r+1)); ints static_cast<T>(rng()), */
/* floats uniform_real_distribution<T>(-1e6, 1e6). Host buffer. */
int ak_bench_keys(uint64_t seed, uint64_t rank, uint64_t n, int dtype_code, void* host_out);

#ifdef __cplusplus
}
#endif

#endif /* AK_CUDA_H */
