/*
 * ak_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity checker for the B200 build. Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load it. The product path (paper_2507_16710_b200 + libak_cuda.so)
 * never links or calls it.
 *
 * Every function restates an algorithm of the reference C++ library
 * (/root/reference/proj, AcceleratedKernels.jl restatement) and cites the
 * file:line it follows. Parity of this restatement is PINNED against the
 * reference itself: oracle/ref_shim.cpp compiles the reference headers and
 * sources in place into oracle/_ref/libakref.so, and
 * tests/golden/make_golden.py records reference outputs into tests/golden/.
 * tests/test_oracle.py checks this file against both.
 *
 * Types: i32, i64, u64, f32, f64 keys; sort comparator is operator< (std::less),
 * optionally reversed (std::greater). Floating point: -0.0 == +0.0 under <,
 * NaN unsupported (the reference sort is undefined on NaN).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Stable bottom-up merge sort of an index permutation.                      */
/* Follows sort.hpp:75-170 (co-rank free sequential form: a wins ties).      */
/* sortperm semantics sort.hpp:238-262: equal keys keep ascending indices.   */
/* ------------------------------------------------------------------------ */

#define ORC_LESS(T, a, b, desc) ((desc) ? ((b) < (a)) : ((a) < (b)))

#define ORC_DEFINE_SORTPERM(SUF, T)                                                          \
    ORC_API int orc_sortperm_##SUF(const T* data, uint64_t n, uint64_t* out, int desc) {     \
        uint64_t* tmp;                                                                       \
        uint64_t i, width;                                                                   \
        uint64_t *src, *dst;                                                                 \
        for (i = 0; i < n; ++i) out[i] = i;                                                  \
        if (n < 2) return 0;                                                                 \
        tmp = (uint64_t*)malloc(n * sizeof(uint64_t));                                       \
        if (!tmp) return -1;                                                                 \
        src = out;                                                                           \
        dst = tmp;                                                                           \
        for (width = 1; width < n; width *= 2) {                                             \
            uint64_t lo;                                                                     \
            for (lo = 0; lo < n; lo += 2 * width) {                                          \
                uint64_t mid = lo + width < n ? lo + width : n;                              \
                uint64_t hi = lo + 2 * width < n ? lo + 2 * width : n;                       \
                uint64_t ia = lo, ib = mid, o = lo;                                          \
                while (ia < mid && ib < hi) {                                                \
                    /* take from the left run unless right < left (sort.hpp:98) */           \
                    if (!ORC_LESS(T, data[src[ib]], data[src[ia]], desc))                   \
                        dst[o++] = src[ia++];                                                \
                    else                                                                     \
                        dst[o++] = src[ib++];                                                \
                }                                                                            \
                while (ia < mid) dst[o++] = src[ia++];                                       \
                while (ib < hi) dst[o++] = src[ib++];                                        \
            }                                                                                \
            { uint64_t* t = src; src = dst; dst = t; }                                       \
        }                                                                                    \
        if (src != out) memcpy(out, src, n * sizeof(uint64_t));                              \
        free(tmp);                                                                           \
        return 0;                                                                            \
    }                                                                                        \
    /* merge_sort (sort.hpp:180-194): stable in-place sort of the keys. */                   \
    ORC_API int orc_merge_sort_##SUF(T* data, uint64_t n, int desc) {                        \
        uint64_t* perm = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));                  \
        T* copy = (T*)malloc((n ? n : 1) * sizeof(T));                                       \
        uint64_t i;                                                                          \
        if (!perm || !copy) { free(perm); free(copy); return -1; }                           \
        orc_sortperm_##SUF(data, n, perm, desc);                                             \
        memcpy(copy, data, n * sizeof(T));                                                   \
        for (i = 0; i < n; ++i) data[i] = copy[perm[i]];                                     \
        free(perm); free(copy);                                                              \
        return 0;                                                                            \
    }

ORC_DEFINE_SORTPERM(i32, int32_t)
ORC_DEFINE_SORTPERM(u32, uint32_t)
ORC_DEFINE_SORTPERM(i64, int64_t)
ORC_DEFINE_SORTPERM(u64, uint64_t)
ORC_DEFINE_SORTPERM(f32, float)
ORC_DEFINE_SORTPERM(f64, double)

/* ------------------------------------------------------------------------ */
/* reduce / mapreduce (reduce.hpp:24-75).                                    */
/* With a neutral init the reference result equals the sequential left fold  */
/* for integer sums (exact) and min/max (order independent). The f32 oracle  */
/* accumulates in double: the reference's own f32 fold stalls at 2^24 per    */
/* chunk at the 2^30 config, so it is not authoritative.    */
/* op: 0 sum, 1 min, 2 max. map: 0 identity, 1 abs, 2 square.                */
/* ------------------------------------------------------------------------ */

#define ORC_DEFINE_REDUCE(SUF, T, ACC)                                                       \
    ORC_API ACC orc_reduce_##SUF(const T* x, uint64_t n, int op, int map, ACC init) {        \
        ACC acc = init;                                                                      \
        uint64_t i;                                                                          \
        for (i = 0; i < n; ++i) {                                                            \
            ACC v = (ACC)x[i];                                                               \
            if (map == 1) v = v < 0 ? -v : v;                                                \
            else if (map == 2) v = v * v;                                                    \
            if (op == 0) acc = acc + v;                                                      \
            else if (op == 1) acc = v < acc ? v : acc;                                       \
            else acc = acc < v ? v : acc;                                                    \
        }                                                                                    \
        return acc;                                                                          \
    }

/* integer sums wrap exactly like two's complement (computed in uint64) */
ORC_API int64_t orc_reduce_i64(const int64_t* x, uint64_t n, int op, int map, int64_t init) {
    uint64_t acc = (uint64_t)init;
    int64_t m = init;
    uint64_t i;
    for (i = 0; i < n; ++i) {
        int64_t v = x[i];
        if (map == 1) v = v < 0 ? (int64_t)(0 - (uint64_t)v) : v;
        else if (map == 2) v = (int64_t)((uint64_t)v * (uint64_t)v);
        if (op == 0) acc += (uint64_t)v;
        else if (op == 1) m = v < m ? v : m;
        else m = m < v ? v : m;
    }
    return op == 0 ? (int64_t)acc : m;
}
ORC_API int32_t orc_reduce_i32(const int32_t* x, uint64_t n, int op, int map, int32_t init) {
    uint32_t acc = (uint32_t)init;
    int32_t m = init;
    uint64_t i;
    for (i = 0; i < n; ++i) {
        int32_t v = x[i];
        if (map == 1) v = v < 0 ? (int32_t)(0u - (uint32_t)v) : v;
        else if (map == 2) v = (int32_t)((uint32_t)v * (uint32_t)v);
        if (op == 0) acc += (uint32_t)v;
        else if (op == 1) m = v < m ? v : m;
        else m = m < v ? v : m;
    }
    return op == 0 ? (int32_t)acc : m;
}
ORC_DEFINE_REDUCE(f32_f64acc, float, double)
ORC_DEFINE_REDUCE(f64, double, double)
ORC_API uint64_t orc_reduce_u64(const uint64_t* x, uint64_t n, int op, int map, uint64_t init) {
    uint64_t acc = init;
    uint64_t i;
    for (i = 0; i < n; ++i) {
        uint64_t v = x[i];
        if (map == 2) v = v * v;
        if (op == 0) acc += v;
        else if (op == 1) acc = v < acc ? v : acc;
        else acc = acc < v ? v : acc;
    }
    return acc;
}

/* ------------------------------------------------------------------------ */
/* accumulate (scan.hpp:29-79). Integer scans are association independent,  */
/* so the sequential scan (tests/test_utils.hpp:74-88) is exact. Float scans */
/* are given as a double-precision prefix for the tolerance check.           */
/* ------------------------------------------------------------------------ */

ORC_API void orc_scan_i64(const int64_t* x, uint64_t n, int64_t* out, int inclusive, int64_t init) {
    uint64_t acc = (uint64_t)init;
    uint64_t i;
    for (i = 0; i < n; ++i) {
        uint64_t v = (uint64_t)x[i]; /* read before write: out may alias x (scan.hpp:72-76) */
        if (inclusive) { acc += v; out[i] = (int64_t)acc; }
        else { out[i] = (int64_t)acc; acc += v; }
    }
}
ORC_API void orc_scan_i32(const int32_t* x, uint64_t n, int32_t* out, int inclusive, int32_t init) {
    uint32_t acc = (uint32_t)init;
    uint64_t i;
    for (i = 0; i < n; ++i) {
        uint32_t v = (uint32_t)x[i];
        if (inclusive) { acc += v; out[i] = (int32_t)acc; }
        else { out[i] = (int32_t)acc; acc += v; }
    }
}
ORC_API void orc_scan_f32_f64acc(const float* x, uint64_t n, double* out, int inclusive, double init) {
    double acc = init;
    uint64_t i;
    for (i = 0; i < n; ++i) {
        double v = (double)x[i];
        if (inclusive) { acc += v; out[i] = acc; }
        else { out[i] = acc; acc += v; }
    }
}
ORC_API void orc_scan_f64(const double* x, uint64_t n, double* out, int inclusive, double init) {
    orc_scan_f32_f64acc((const float*)0, 0, out, inclusive, init); /* no-op, keeps one code path */
    {
        double acc = init;
        uint64_t i;
        for (i = 0; i < n; ++i) {
            double v = x[i];
            if (inclusive) { acc += v; out[i] = acc; }
            else { out[i] = acc; acc += v; }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* searchsorted (search.hpp:16-50): first = #elements < v, last = #<= v.     */
/* ------------------------------------------------------------------------ */

#define ORC_DEFINE_SEARCH(SUF, T)                                                            \
    static uint64_t orc_lower_##SUF(const T* h, uint64_t n, T v, int desc) {                 \
        uint64_t lo = 0, hi = n;                                                             \
        while (lo < hi) {                                                                    \
            uint64_t mid = lo + (hi - lo) / 2;                                               \
            if (ORC_LESS(T, h[mid], v, desc)) lo = mid + 1; else hi = mid;                   \
        }                                                                                    \
        return lo;                                                                           \
    }                                                                                        \
    static uint64_t orc_upper_##SUF(const T* h, uint64_t n, T v, int desc) {                 \
        uint64_t lo = 0, hi = n;                                                             \
        while (lo < hi) {                                                                    \
            uint64_t mid = lo + (hi - lo) / 2;                                               \
            if (!ORC_LESS(T, v, h[mid], desc)) lo = mid + 1; else hi = mid;                  \
        }                                                                                    \
        return lo;                                                                           \
    }                                                                                        \
    ORC_API void orc_searchsorted_##SUF(const T* h, uint64_t n, const T* needles, uint64_t m, \
                                        int side_last, int desc, uint64_t* out) {            \
        uint64_t i;                                                                          \
        for (i = 0; i < m; ++i)                                                              \
            out[i] = side_last ? orc_upper_##SUF(h, n, needles[i], desc)                     \
                               : orc_lower_##SUF(h, n, needles[i], desc);                    \
    }

ORC_DEFINE_SEARCH(i32, int32_t)
ORC_DEFINE_SEARCH(u32, uint32_t)
ORC_DEFINE_SEARCH(i64, int64_t)
ORC_DEFINE_SEARCH(u64, uint64_t)
ORC_DEFINE_SEARCH(f32, float)
ORC_DEFINE_SEARCH(f64, double)

/* ------------------------------------------------------------------------ */
/* SIHSort protocol (sihsort.hpp:57-569) over P ranks in one process.        */
/* The collectives of sim_comm.hpp:124-156 are order-independent folds, so   */
/* they are restated as loops over ranks. All splitter math in long double.  */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t sample_per_rank; /* 0 -> 32P (sihsort.hpp:512-513) */
    uint64_t bins;            /* 0 -> 8P  (sihsort.hpp:514-515) */
    uint64_t max_refine_rounds;
    double imbalance_tol;
} orc_sih_config;

typedef struct {
    uint64_t rounds_used;
    uint64_t converged;
    double max_deviation;
    uint64_t redistribution_sends;
    uint64_t redistribution_bytes;
    uint64_t collective_ops;
    uint64_t output_count;
} orc_sih_stats;

/* equal_width_edges (sihsort.hpp:76-88); returns edge count */
static uint64_t orc_edges(long double lo, long double hi, uint64_t bins, long double* edges) {
    uint64_t i;
    if (!(lo < hi)) {
        edges[0] = lo;
        edges[1] = lo;
        return 2;
    }
    for (i = 0; i <= bins; ++i)
        edges[i] = lo + (hi - lo) * (long double)i / (long double)bins;
    edges[0] = lo;
    edges[bins] = hi;
    return bins + 1;
}

/* sample positions of sample_local (sihsort.hpp:264-282) */
ORC_API uint64_t orc_sample_positions(uint64_t n, uint64_t k, uint64_t* pos) {
    uint64_t j;
    if (n == 0 || k == 0) return 0;
    if (k > n) k = n;
    if (k == 1) {
        pos[0] = n / 2;
        return 1;
    }
    for (j = 0; j < k; ++j) pos[j] = (2 * j * (n - 1) + (k - 1)) / (2 * (k - 1));
    return k;
}

#define ORC_IS_INT_i32 1
#define ORC_IS_INT_i64 1
#define ORC_IS_INT_u64 1
#define ORC_IS_INT_f32 0
#define ORC_IS_INT_f64 0

#define ORC_DEFINE_SIH(SUF, T, IS_INT, TMIN, TMAX)                                            \
    /* ld_to_key (sihsort.hpp:63-74): ints round half away from zero and saturate */         \
    static T orc_ld_to_key_##SUF(long double x) {                                            \
        if (IS_INT) {                                                                        \
            x = floorl(x + 0.5L);                                                            \
            if (x <= (long double)(TMIN)) return (T)(TMIN);                                  \
            if (x >= (long double)(TMAX)) return (T)(TMAX);                                  \
            return (T)x;                                                                     \
        }                                                                                    \
        return (T)x;                                                                         \
    }                                                                                        \
    /* select_splitters (sihsort.hpp:310-349) */                                             \
    ORC_API void orc_select_splitters_##SUF(const long double* edges, const uint64_t* counts, \
                                            uint64_t k, uint64_t total, uint64_t world,      \
                                            T* out) {                                        \
        uint64_t cum = 0, bin = 0, j;                                                        \
        if (world <= 1) return;                                                              \
        if (total == 0) {                                                                    \
            for (j = 0; j + 1 < world; ++j) out[j] = orc_ld_to_key_##SUF(edges[0]);          \
            return;                                                                          \
        }                                                                                    \
        for (j = 1; j < world; ++j) {                                                        \
            long double target = (long double)total * (long double)j / (long double)world;  \
            long double value;                                                               \
            T key;                                                                           \
            while (bin < k && (long double)(cum + counts[bin]) < target) {                   \
                cum += counts[bin];                                                          \
                ++bin;                                                                       \
            }                                                                                \
            if (bin >= k) {                                                                  \
                value = edges[k];                                                            \
            } else {                                                                         \
                long double frac = counts[bin] == 0                                          \
                                       ? 0.0L                                                \
                                       : (target - (long double)cum) / (long double)counts[bin]; \
                value = edges[bin] + frac * (edges[bin + 1] - edges[bin]);                   \
            }                                                                                \
            key = orc_ld_to_key_##SUF(value);                                                \
            if (j > 1 && key < out[j - 2]) key = out[j - 2];                                 \
            out[j - 1] = key;                                                                \
        }                                                                                    \
    }                                                                                        \
    /* Whole protocol. inputs: P arrays (not modified). out: concatenation of the P outputs  \
       in rank order (capacity = total). out_counts[r]: size of rank r's output.            \
       stats: one per rank. splitters_out: final P-1 splitters (may be NULL). */            \
    ORC_API int orc_sihsort_##SUF(uint64_t P, const T* const* inputs, const uint64_t* counts, \
                                  const orc_sih_config* cfg, T* out, uint64_t* out_counts,   \
                                  orc_sih_stats* stats, T* splitters_out) {                  \
        const uint64_t spr = cfg->sample_per_rank > 0 ? cfg->sample_per_rank : 32 * P;       \
        const uint64_t bins = cfg->bins > 0 ? cfg->bins : 8 * P;                             \
        T** sorted = (T**)calloc(P, sizeof(T*));                                             \
        uint64_t r, j, total = 0, total_samples = 0;                                         \
        T smin = 0, smax = 0, dmin = 0, dmax = 0;                                            \
        int have_s = 0, have_d = 0;                                                          \
        T* spl = (T*)calloc(P > 1 ? P - 1 : 1, sizeof(T));                                   \
        uint64_t* pos = (uint64_t*)malloc((spr + 1) * sizeof(uint64_t));                     \
        uint64_t collectives = 0, rounds_used = 0, converged = 0;                            \
        double max_deviation = 0.0;                                                          \
        if (!sorted || !spl || !pos) return -1;                                              \
        collectives += 1; /* check_consistent_config (sihsort.hpp:518) */                    \
        for (r = 0; r < P; ++r) { /* local sort 1 of 2 (sihsort.hpp:520) */                  \
            sorted[r] = (T*)malloc((counts[r] ? counts[r] : 1) * sizeof(T));                 \
            memcpy(sorted[r], inputs[r], counts[r] * sizeof(T));                             \
            orc_merge_sort_##SUF(sorted[r], counts[r], 0);                                   \
            total += counts[r];                                                              \
        }                                                                                    \
        /* sample_local + global_summary (sihsort.hpp:522-523, :221-238) */                  \
        collectives += 1;                                                                    \
        for (r = 0; r < P; ++r) {                                                            \
            uint64_t k = orc_sample_positions(counts[r], spr, pos);                          \
            if (counts[r] > 0) {                                                             \
                if (!have_d || sorted[r][0] < dmin) dmin = sorted[r][0];                     \
                if (!have_d || dmax < sorted[r][counts[r] - 1]) dmax = sorted[r][counts[r] - 1]; \
                have_d = 1;                                                                  \
            }                                                                                \
            if (k > 0) {                                                                     \
                T s0 = sorted[r][pos[0]], s1 = sorted[r][pos[k - 1]];                        \
                if (!have_s || s0 < smin) smin = s0;                                         \
                if (!have_s || smax < s1) smax = s1;                                         \
                have_s = 1;                                                                  \
            }                                                                                \
            total_samples += k;                                                              \
        }                                                                                    \
        if (total_samples == 0) {                                                            \
            for (j = 0; j + 1 < P; ++j) spl[j] = (T)0;                                       \
        } else {                                                                             \
            /* distributed histogram (sihsort.hpp:526-540) */                                \
            long double* edges = (long double*)malloc((bins + 2) * sizeof(long double));     \
            uint64_t ne = orc_edges((long double)smin, (long double)smax, bins, edges);      \
            uint64_t kb = ne - 1;                                                            \
            uint64_t* hc = (uint64_t*)calloc(kb, sizeof(uint64_t));                          \
            const long double lo = edges[0], hi = edges[ne - 1];                             \
            for (r = 0; r < P; ++r) {                                                        \
                uint64_t k = orc_sample_positions(counts[r], spr, pos), s;                   \
                for (s = 0; s < k; ++s) { /* count_into_bins (sihsort.hpp:91-106) */         \
                    uint64_t bin = 0;                                                        \
                    if (lo < hi) {                                                           \
                        long double frac = ((long double)sorted[r][pos[s]] - lo) / (hi - lo); \
                        long long raw = (long long)floorl(frac * (long double)kb);           \
                        bin = raw <= 0 ? 0 : ((uint64_t)raw < kb - 1 ? (uint64_t)raw : kb - 1); \
                    }                                                                        \
                    ++hc[bin];                                                               \
                }                                                                            \
            }                                                                                \
            collectives += 1;                                                                \
            orc_select_splitters_##SUF(edges, hc, kb, total_samples, P, spl);                \
            free(edges);                                                                     \
            free(hc);                                                                        \
        }                                                                                    \
        /* refine_splitters (sihsort.hpp:364-464) */                                         \
        if (cfg->max_refine_rounds > 0) {                                                    \
            collectives += 1; /* global_summary inside refine (:374) */                      \
            if (P > 1 && total > 0) {                                                        \
                const long double ideal = (long double)total / (long double)P;               \
                T* lo = (T*)malloc((P - 1) * sizeof(T));                                     \
                T* hi = (T*)malloc((P - 1) * sizeof(T));                                     \
                uint64_t* flo = (uint64_t*)malloc((P - 1) * sizeof(uint64_t));               \
                uint64_t* fhi = (uint64_t*)malloc((P - 1) * sizeof(uint64_t));               \
                char* frozen = (char*)calloc(P - 1, 1);                                      \
                uint64_t* le = (uint64_t*)malloc((P - 1) * sizeof(uint64_t));                \
                uint64_t round;                                                              \
                for (j = 0; j + 1 < P; ++j) {                                                \
                    lo[j] = dmin; hi[j] = dmax; flo[j] = 0; fhi[j] = total;                  \
                }                                                                            \
                for (round = 1; round <= cfg->max_refine_rounds; ++round) {                  \
                    long double max_dev = 0.0L;                                              \
                    for (j = 0; j + 1 < P; ++j) {                                            \
                        le[j] = 0;                                                           \
                        for (r = 0; r < P; ++r)                                              \
                            le[j] += orc_upper_##SUF(sorted[r], counts[r], spl[j], 0);       \
                    }                                                                        \
                    collectives += 1;                                                        \
                    for (r = 0; r < P; ++r) {                                                \
                        uint64_t upper = r + 1 < P ? le[r] : total;                          \
                        uint64_t lower = r > 0 ? le[r - 1] : 0;                              \
                        long double bucket = (long double)(upper - lower);                   \
                        long double dev = fabsl(bucket - ideal) / ideal;                     \
                        if (dev > max_dev) max_dev = dev;                                    \
                    }                                                                        \
                    rounds_used = round;                                                     \
                    max_deviation = (double)max_dev;                                         \
                    if (max_dev <= (long double)cfg->imbalance_tol) { converged = 1; break; } \
                    if (round == cfg->max_refine_rounds) break;                              \
                    for (j = 0; j + 1 < P; ++j) {                                            \
                        long double target, frac, cand;                                      \
                        uint64_t measured;                                                   \
                        T key;                                                               \
                        if (frozen[j]) continue;                                             \
                        target = ideal * (long double)(j + 1);                               \
                        measured = le[j];                                                    \
                        if ((long double)measured < target) { lo[j] = spl[j]; flo[j] = measured; } \
                        else if ((long double)measured > target) { hi[j] = spl[j]; fhi[j] = measured; } \
                        else { frozen[j] = 1; continue; }                                    \
                        if (!(lo[j] < hi[j]) || fhi[j] <= flo[j]) { frozen[j] = 1; continue; } \
                        frac = (target - (long double)flo[j]) / (long double)(fhi[j] - flo[j]); \
                        cand = (long double)lo[j] + ((long double)hi[j] - (long double)lo[j]) * frac; \
                        key = orc_ld_to_key_##SUF(cand);                                     \
                        if (IS_INT) {                                                        \
                            if (key <= lo[j]) key = (T)(lo[j] + 1);                          \
                            if (hi[j] < key) key = hi[j];                                    \
                        } else {                                                             \
                            if (!(key > lo[j]) || !(key < hi[j]))                            \
                                key = orc_ld_to_key_##SUF(((long double)lo[j] + (long double)hi[j]) / 2); \
                            if (!(key > lo[j]) || !(key < hi[j])) { frozen[j] = 1; continue; } \
                        }                                                                    \
                        spl[j] = key;                                                        \
                    }                                                                        \
                    for (j = 1; j + 1 < P; ++j)                                              \
                        if (spl[j] < spl[j - 1]) spl[j] = spl[j - 1];                        \
                }                                                                            \
                free(lo); free(hi); free(flo); free(fhi); free(frozen); free(le);            \
            } else {                                                                         \
                converged = 1;                                                               \
            }                                                                                \
        }                                                                                    \
        /* redistribute (sihsort.hpp:472-501) + local sort 2 of 2 (:555) */                  \
        {                                                                                    \
            uint64_t* bounds = (uint64_t*)malloc(P * (P + 1) * sizeof(uint64_t));            \
            uint64_t base = 0;                                                               \
            /* piggyback_tail_mode (sihsort.hpp:129-141) */                                  \
            const int tail = IS_INT ? (total <= (uint64_t)(TMAX)) : 0;                       \
            for (r = 0; r < P; ++r) { /* slice_bounds (sihsort.hpp:110-123) */               \
                bounds[r * (P + 1)] = 0;                                                     \
                for (j = 0; j + 1 < P; ++j)                                                  \
                    bounds[r * (P + 1) + j + 1] = orc_upper_##SUF(sorted[r], counts[r], spl[j], 0); \
                bounds[r * (P + 1) + P] = counts[r];                                         \
            }                                                                                \
            for (r = 0; r < P; ++r) {                                                        \
                uint64_t got = 0, src, sent_bytes = 0, sends = 0;                            \
                for (src = 0; src < P; ++src) {                                              \
                    uint64_t b0 = bounds[src * (P + 1) + r], b1 = bounds[src * (P + 1) + r + 1]; \
                    memcpy(out + base + got, sorted[src] + b0, (b1 - b0) * sizeof(T));       \
                    got += b1 - b0;                                                          \
                }                                                                            \
                for (src = 0; src < P; ++src) { /* what rank r sent */                       \
                    uint64_t len;                                                            \
                    if (src == r) continue;                                                  \
                    len = bounds[r * (P + 1) + src + 1] - bounds[r * (P + 1) + src];         \
                    sends += 1;                                                              \
                    sent_bytes += tail ? (len + 1) * sizeof(T) : 8 + len * sizeof(T);        \
                }                                                                            \
                orc_merge_sort_##SUF(out + base, got, 0);                                    \
                out_counts[r] = got;                                                         \
                if (stats) {                                                                 \
                    stats[r].rounds_used = rounds_used;                                      \
                    stats[r].converged = converged;                                          \
                    stats[r].max_deviation = max_deviation;                                  \
                    stats[r].redistribution_sends = sends;                                   \
                    stats[r].redistribution_bytes = sent_bytes;                              \
                    stats[r].collective_ops = collectives;                                   \
                    stats[r].output_count = got;                                             \
                }                                                                            \
                base += got;                                                                 \
            }                                                                                \
            free(bounds);                                                                    \
        }                                                                                    \
        if (splitters_out) for (j = 0; j + 1 < P; ++j) splitters_out[j] = spl[j];            \
        for (r = 0; r < P; ++r) free(sorted[r]);                                             \
        free(sorted); free(spl); free(pos);                                                  \
        return 0;                                                                            \
    }

ORC_DEFINE_SIH(i32, int32_t, 1, INT32_MIN, INT32_MAX)
ORC_DEFINE_SIH(i64, int64_t, 1, INT64_MIN, INT64_MAX)
ORC_DEFINE_SIH(u64, uint64_t, 1, 0, UINT64_MAX)
ORC_DEFINE_SIH(f32, float, 0, 0, 0)
ORC_DEFINE_SIH(f64, double, 0, 0, 0)
