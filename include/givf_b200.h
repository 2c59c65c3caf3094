/*
 * givf_b200 -- C ABI of the B200-native search path for the grouped inverted
 * index of arXiv 1802.02422 (reference package `givf`).
 *
 * Plain pointers and sizes only.  Every pointer argument of a search call may
 * be host memory or device memory (detected per call); the index arrays of
 * givf_index_create are always host memory and are copied to the device.
 *
 * The entry points replace these reference interfaces
 * (paths under /root/reference/pkg/src/givf/):
 *   givf_index_create    GroupedIndex (index.py:48-85) as produced by
 *                        build_index (index.py:249-380) / load_index
 *                        (storage.py:162-281): the read-only search input.
 *   givf_search_full     search(index, query, params) (search.py:93-163),
 *                        batched: every scanned code, reranked by (dist, id)
 *                        (rerank=True, search.py:156-158) or in scan order
 *                        with group scores (rerank=False, search.py:159-161).
 *   givf_search_topk     the first k entries of search()'s reranked list
 *                        (BASELINE.json k=100; recall_at_r search.py:186-201
 *                        reads only ids[:R]).
 *   givf_probe           _select_regions (search.py:77-90) at
 *                        ef_search == K, i.e. the exact region ranking.
 *   givf_merge_topk      no reference counterpart (single process): merge
 *                        of per-shard top-k lists, SURVEY §8e.
 *   givf_plan            search.py:77-139 alone (probe, group scores,
 *                        prune, budget walk) for a share of the queries,
 *                        emitting each query's begun groups in their global
 *                        form -- the query-sharded planning step of the
 *                        list-sharded layout.
 *   givf_search_planned  search.py:138-158 (scan + rerank, top-k) of plans
 *                        made by givf_plan on any rank, over the rows this
 *                        shard holds.
 *
 * Status codes: GIVF_OK, GIVF_EINVAL (bad argument: givf_last_error() holds
 * the reference's ValueError text, e.g. "need 1 <= nprobe <= 48, got 0"),
 * GIVF_ECUDA, GIVF_ENOMEM, GIVF_EINVARIANT.
 */
#ifndef GIVF_B200_H
#define GIVF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GIVF_OK 0
#define GIVF_EINVAL 1
#define GIVF_ECUDA 2
#define GIVF_ENOMEM 3
#define GIVF_EINVARIANT 4

typedef struct givf_index* givf_index_t;

/* Flat arrays of a GroupedIndex (index.py:48-62).  For a shard of a
 * multi-GPU layout the row arrays (point_ids, codes,
 * const_bytes, region_offsets) hold only this shard's rows, `group_sizes` is
 * the replicated GLOBAL table that drives the budget walk, and
 * local_sizes / local_lo give, per (region, group) slice, how many rows this
 * shard holds and the first global slot it owns.  Both NULL = unsharded. */
typedef struct givf_index_desc {
  int32_t k;               /* regions */
  int32_t dim;             /* vector dimension */
  int32_t groups;          /* groups per region: L, or 1 when grouping is off */
  int32_t m;               /* PQ sub-quantizers (code bytes per point) */
  int32_t grouping;        /* 1 = grouped index (neighbor_ids/norm_terms set) */
  int64_t n;               /* rows stored (in this shard) */
  const float* centroids;      /* (k, dim) */
  const float* alphas;         /* (k) */
  const int32_t* neighbor_ids; /* (k, groups) or NULL */
  const float* norm_terms;     /* (k, groups) or NULL */
  const int32_t* group_sizes;  /* (k, groups) */
  const int64_t* region_offsets; /* (k + 1) row offsets */
  const int32_t* local_sizes;  /* (k, groups) or NULL */
  const int32_t* local_lo;     /* (k, groups) or NULL */
  const int32_t* point_ids;    /* (n) */
  const uint8_t* codes;        /* (n, m) */
  const uint8_t* const_bytes;  /* (n) */
  const float* codewords;      /* (m, 256, dim / m) */
  const float* rotation;       /* (dim, dim) or NULL */
  double const_lo;             /* ConstQuantizer bounds (grouping.py:100-129) */
  double const_hi;
} givf_index_desc;

/* SearchParams (search.py:23-30). */
typedef struct givf_search_params {
  int32_t nprobe;
  double tau;
  int64_t candidates;
  int32_t ef_search;   /* validated like the reference; the probe is exact */
  int32_t rerank;
  int32_t prune;
} givf_search_params;

/* SearchStats (search.py:33-39) without the wall time. */
typedef struct givf_search_stats {
  int64_t regions_visited;
  int64_t subregions_visited;
  int64_t subregions_pruned;
  int64_t codes_scanned;
} givf_search_stats;

const char* givf_last_error(void);
const char* givf_version(void);

int givf_index_create(const givf_index_desc* desc, int device, givf_index_t* out);
int givf_index_destroy(givf_index_t index);
/* bytes of device memory held by the index arrays */
int64_t givf_index_device_bytes(givf_index_t index);
/* Cumulative counts of queries that left the fast path: out[0] = probe
 * candidate sets the float64 re-check could not certify (exhaustive ranking
 * ran instead), out[1] = approximate plans that fell back to the exact
 * planner; out[2..7] split out[1] by reason: 2 = more than 1024 equal
 * approximate keys at the cut, 3 = more than 256 groups in the +-3E window,
 * 4 = exact crossing before the window, 5 = crossing outside +-2E of v*,
 * 6 = walk not ended inside the window, 7 = too many begun groups for the
 * in-CTA rescore.  Synchronises the device. */
int givf_index_counters(givf_index_t index, int64_t* out, int32_t n);

/* queries (nq, dim) f32.  ids (nq, k) int32 padded with -1, dists (nq, k)
 * f32 padded with +inf, stats (nq) -- host or device; stream = cudaStream_t
 * to launch on (NULL = the default stream).  Returns after the results are
 * visible to the caller (host outputs: synchronised; device outputs:
 * enqueued on `stream`).  Page-locked (pinned, mapped) host outputs are
 * written by the kernels in place, so their transfer overlaps the scan;
 * pageable host outputs go through a device buffer and one copy. */
int givf_search_topk(givf_index_t index, const float* queries, int64_t nq,
                     const givf_search_params* params, int32_t k, int32_t* ids,
                     float* dists, givf_search_stats* stats, void* stream);

/* Full reference result per query: row q of ids/dists (width `capacity`)
 * holds stats[q].codes_scanned entries.  capacity must be >= the number of
 * codes any query can scan: min(candidates, rows reachable). */
int givf_search_full(givf_index_t index, const float* queries, int64_t nq,
                     const givf_search_params* params, int64_t capacity, int32_t* ids,
                     float* dists, givf_search_stats* stats, void* stream);

/* K1a alone (parity / accuracy checks): approximate region scores
 * s~[q, c] = |c|^2 - 2 q.c, (nq, k) f32, and the scale of their a-priori
 * error bound: |s~ - exact| <= eps_scale * (max|c|^2 + 2 |q| max|c|). */
int givf_probe_scores(givf_index_t index, const float* queries, int64_t nq, float* scores,
                      float* eps_scale, void* stream);

/* Region probe: region ids (nq, nprobe) int32 and float64 qc2 (nq, nprobe). */
int givf_probe(givf_index_t index, const float* queries, int64_t nq, int32_t nprobe,
               int32_t* regions, double* qc2, void* stream);

/* K7: merge shard lists ids/dists (shards, nq, k) -> (nq, k) by (dist, id). */
int givf_merge_topk(const int32_t* ids, const float* dists, int32_t shards, int64_t nq,
                    int32_t k, int32_t* out_ids, float* out_dists, int device, void* stream);

/* Query-sharded planning.  One record per begun group of a
 * query's plan, in its global form: the group's index region * groups +
 * group (replaces index.py:80-85 group_starts, which is per shard), the
 * number of its rows to scan (search.py:131-139 lengths, global), and the
 * float64 base (1 - a) qc2 + a qs2 (search.py:115-121). */
typedef struct givf_plan_item {
  int32_t group;
  int32_t len;
  double base;
} givf_plan_item;

/* Per-query capacity (records) givf_plan needs: min(ceil(tau P L), candidates). */
int givf_plan_capacity(givf_index_t index, const givf_search_params* params, int64_t* cap);

/* Plans of nq queries from this index's replicated tables (any shard of a
 * sharded index gives the same plans): items (nq, cap) givf_plan_item,
 * nitems (nq) records used, stats (nq) the global SearchStats. */
int givf_plan(givf_index_t index, const float* queries, int64_t nq,
              const givf_search_params* params, int64_t cap, void* items, int32_t* nitems,
              givf_search_stats* stats, void* stream);

/* Top-k of nq queries from their plans (CSR on the device: offsets (nq + 1)
 * into items), scanning this shard's rows of every planned group:
 * clip(len - lo, 0, cnt) rows of the slice this shard holds.  ids / dists
 * (nq, k) as givf_search_topk; merge the shards' lists with givf_merge_topk. */
int givf_search_planned(givf_index_t index, const float* queries, int64_t nq,
                        const givf_search_params* params, const int64_t* offsets,
                        const void* items, int32_t k, int32_t* ids, float* dists, void* stream);

/* Count of kernels this library has launched in the calling process. */
int64_t givf_kernel_launches(void);

/* Per-stage device time: when enabled, every launch is bracketed by CUDA
 * events on its own stream.  Stages: 0 probe_gemm, 1 probe_select,
 * 2 probe_recheck, 3 probe_full, 4 plan, 5 scan, 6 finish (full sort /
 * scan order), 7 merge, 8 lut (per-chunk LUT build).  givf_profile_read
 * synchronises on the recorded
 * events, writes the summed milliseconds and launch counts of the first
 * `nstages` stages, and resets the accumulators. */
int givf_profile_enable(int on);
int givf_profile_read(double* stage_ms, int64_t* stage_launches, int32_t nstages);

#ifdef __cplusplus
}
#endif

#endif /* GIVF_B200_H */
