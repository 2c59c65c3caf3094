/*
 * givf_b200 builder entry points -- the device-resident index build (SURVEY
 * §8f rank 1-2) that produces the arrays givf_index_create consumes.  These
 * replace the numpy build loops of the reference package `givf`
 * (paths under /root/reference/pkg/src/givf/):
 *
 *   givf_assign_nearest  kmeans.py:164-187 assign_exact(top=1) /
 *                        index.py:88-99 _assign_regions: nearest centroid
 *                        per row (tcgen05 GEMM with an arg-min epilogue;
 *                        bf16 products, fp32 accumulation -- the reference
 *                        itself assigns approximately, through its graph, at
 *                        K >= 2^16).
 *   givf_encode_rows     index.py:124-138 _pick_groups, index.py:141-170
 *                        _anchor_rows/_const_terms, pq.py:124-129 pq_encode,
 *                        grouping.py:103-113 ConstQuantizer.quantize: group
 *                        pick, residual PQ codes and constant byte of rows
 *                        grouped by region.
 *   givf_knn_exact       datasets.py:34-61 exact_ground_truth and
 *                        grouping.py:25-41 neighbor_centroids: exact top-k
 *                        by (float64 distance, id), through the search
 *                        path's certified probe.
 *
 * All pointers are DEVICE pointers (the build is device resident); calls are
 * enqueued on `stream` (NULL = default stream).  Status codes as givf_b200.h.
 */
#ifndef GIVF_BUILD_H
#define GIVF_BUILD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* labels (rows) int32: index of the nearest of the k centroids (first on
 * ties of the bf16-product score); dists (rows) f32 or NULL: that score plus
 * |x|^2, clamped at 0.  dim <= 128. */
int givf_assign_nearest(const float* x, int64_t rows, const float* centroids, int32_t k,
                        int32_t dim, int32_t* labels, float* dists, void* stream);

/* Rows grouped by region: order[seg[s] .. seg[s+1]) are the rows of region
 * seg_region[s].  Outputs are indexed by row (order[i]). */
typedef struct givf_encode_desc {
  const float* x;             /* (rows, dim) */
  const int32_t* order;       /* row indices grouped by region */
  const int64_t* seg;         /* (nseg + 1) */
  const int32_t* seg_region;  /* (nseg) */
  int64_t nseg;
  int32_t dim, l, m, grouping;
  const float* centroids;     /* (k, dim) */
  const int32_t* neighbor_ids;/* (k, l) or NULL without grouping */
  const float* alphas;        /* (k) */
  const double* c_sq;         /* (k) float64 |c|^2 */
  const float* codewords;     /* (m, 256, dim / m) */
  const float* cw_sq;         /* (m, 256) float32 |codeword|^2 */
  double const_lo, const_step;/* ConstQuantizer lo, (hi - lo) / 256 */
  int16_t* pick;              /* (rows) group index out, or NULL */
  uint8_t* codes;             /* (rows, m) out */
  uint8_t* const_bytes;       /* (rows) out, or NULL */
  double* consts;             /* (rows) float64 constant terms out, or NULL */
} givf_encode_desc;

int givf_encode_rows(const givf_encode_desc* desc, void* stream);

/* ids (nq, k) int32 and dist (nq, k) float64: the exact k nearest rows of
 * base (nb, dim) for every query, the set by (float64 distance, id); rows
 * ordered by (float32(distance), id). */
int givf_knn_exact(const float* queries, int64_t nq, const float* base, int64_t nb, int32_t dim,
                   int32_t k, int32_t* ids, double* dist, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GIVF_BUILD_H */
