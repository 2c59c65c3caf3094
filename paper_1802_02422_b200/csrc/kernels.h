// Launchers for the search-path kernels (implemented in probe.cu, plan.cu,
// scan.cu).  Host-side orchestration lives in capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace givf {

inline uint32_t next_pow2_host(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// SM count of the current device (cached per device).
int num_sms_cur();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current
// device only: done once per (kernel, device, size) and its status returned.
cudaError_t ensure_max_smem(const void* fn, size_t bytes);

// One scan segment: a run of consecutive code rows of one kept (region,
// group) slice, with the float64 terms the distance needs (search.py:143-148).
struct WorkItem {
  int64_t start;  // first code row (local to this shard)
  int32_t len;    // rows to scan
  int32_t flat;   // pos * G + grp: position in the (score, pos, grp) order key
  double base;    // (1-a) qc2 + a qs2
  double score;   // base + norm term (the pruning key; rerank=False output)
};

struct IndexView {
  int K, d, G, M, grouping;
  int64_t n;
  const float* centroids;     // (K, d)
  const float* c2f;           // (K) f32(|c|^2)
  float cmax;                 // max |c|
  const float* alphas;        // (K)
  const int32_t* nbr;         // (K, G) or null
  const float* norm;          // (K, G) or null
  const float* rneg;          // (K) max(0, max_g -norm[r, g]) or null
  const int32_t* gsize;       // (K, G) global group sizes (budget walk)
  int32_t max_gsize;          // largest group size
  const int64_t* lstart;      // (K, G) first local row of each slice
  const int32_t* lsize;       // (K, G) local rows of each slice (null: = gsize)
  const int32_t* llo;         // (K, G) first global slot held here (null: 0)
  const int32_t* pids;        // (n)
  const uint8_t* codes;       // (n, M)
  const uint8_t* cbytes;      // (n)
  const float* codewords;     // (M, 256, d/M)
  const float* rotation;      // (d, d) or null
  const float* ctab;          // (256) dequantized constants, f32
  const void* csplit;         // (K, tc_kpad_b(d)) bf16 [c_hi | c_lo] or null
  // fused probe (probe_fused.cu): fp16 centroids c 2^-c16e, pitch f16_pitch(d),
  // columns d, d+1: -|c|^2 2^-(1 + ec + T) as an fp16 hi + lo pair
  const void* c16;            // (K, dp) or null
  int c16e;                   // scale exponent ec
  float c16x;                 // 2^ec
  int c16T;                   // T
  const void* c16r;           // (K, f16_row_pitch(d)) the same fp16 coordinates, K3a's rows
  // K3a's rows again, packed per region: chunk c (16 bytes) of neighbour j of
  // region r at ((r DP8 + c) G + j) 16 bytes, DP8 = f16_row_pitch(d) / 8, so a
  // warp reads a region's 64 rows as contiguous 512-byte lines instead of 64
  // random rows; c2p = the neighbours' f32 |c|^2, (K, G).  Null: gather c16r.
  const void* c16p;
  const float* c2p;
  const void* s16;            // (Ks, dp) fp16 rows of a random centroid sample
  const float* sc2;           // (Ks) their f32 |c|^2
  int Ks;
  unsigned long long* counters;  // [0] probe fallbacks, [1] plan fallbacks (device)
};

// Where the probe GEMM puts its scores s~ = |c|^2 - 2 q.c.  The search path
// stores them as fp16 (half the HBM traffic of the GEMM, the select and
// K3a): h = f16((s~ + |q|^2) * qinv), decoded s~ = h * qscale - |q|^2, with
// qscale = 2^e a per-query power of two that keeps (|q| + cmax)^2 / 2^e
// <= 2^15.  The rounding adds at most kHalfRel * (|q| + cmax)^2 to every
// score's error bound.  probe_scores (accuracy checks) keeps fp32.  With fp16
// output the GEMMs' per-tile minima are fp16 codes too (uint16 in the tmin
// buffer); the select compares codes and decodes only its outputs.
constexpr double kHalfRel = 1.0 / 2048.0;  // fp16 half ulp, relative
struct ScoreOut {
  float* D32 = nullptr;           // fp32 scores, or
  uint16_t* D16 = nullptr;        // fp16 encoded scores
  int64_t ld = 0;                 // row pitch (elements)
  const float* q2 = nullptr;      // (nq) f32 |q|^2        (fp16 only)
  const float* qinv = nullptr;    // (nq) 2^-e             (fp16 only)
  const float* qscale = nullptr;  // (nq) 2^e              (fp16 only)
};

// probe_tc.cu: tcgen05 bf16x3 probe GEMM
int tc_kpad(int d);    // row width of the split queries (A')
int tc_kpad_b(int d);  // row width of the split centroids (B')
bool tc_supported(int d);
size_t tc_smem_bytes(int d);
void launch_split_bf16(const float* x, int rows, int d, int centroid, void* out, cudaStream_t s);
bool launch_probe_gemm_tc(const void* Abf, const void* Bbf, const float* c2, int nq, int K, int d,
                          const ScoreOut& o, float* tmin, cudaStream_t s);

// probe_fused.cu: the probe without a score matrix (large K)
int f16_pitch(int d);
bool fused_supported(int d);
float probe_f16_eps(int d);   // GEMM bound, units of cmax^2 + 2 |q| cmax
float direct_f16_eps(int d);  // K3a-from-fp16-rows bound, same units
// dp = row pitch (0: f16_pitch(d), with the |c|^2 columns; d rounded up
// to 32: the coordinates only, for K3a's row reads)
// c16p / c2p of IndexView from c16r, c2f and the neighbour ids
void launch_pack_neighbor_rows(const void* c16r, const float* c2f, const int32_t* nbr, int K, int G,
                               int d, void* c16p, float* c2p, cudaStream_t s);
void launch_rows_f16(const float* x, const int32_t* ids, int64_t rows, int d, int e, int T,
                     const float* c2, void* out, float* c2out, cudaStream_t s, int dp = 0);
__host__ __device__ inline int f16_row_pitch(int d) { return ((d + 31) / 32) * 32; }
void launch_query_f16(const float* Q, int nq, int d, int ec, int T, void* q16, float* ms,
                      float* q2, cudaStream_t s);
cudaError_t launch_probe_sample(const void* q16, const void* s16, int nq, int Ks, int d,
                                const float* ms, float* cmin, cudaStream_t s);
void filter_segments(int nq, int K, int fcap, int* nseg, int* cap_u);
int filter_slots();  // survivor segments per (query, work unit)
cudaError_t launch_probe_filter(const void* q16, const void* c16, int nq, int K, int d,
                                const float* ms, const float* thr, int nseg, int cap_u, int* cnt,
                                int* cid, float* cval, cudaStream_t s);
void launch_probe_thresh(const float* cmin, int nch, int j, const float* q2, float cmax,
                         float eps_scale, int nq, float* thr, cudaStream_t s,
                         const int* qmap = nullptr);
// retry pass of the fused probe: indices of the queries flagged in fail
// (any order) and their count; rows of Q gathered by idx
void launch_collect_failed(const int* fail, int nq, int* idx, int* n, cudaStream_t s);
void launch_gather_rows(const float* Q, const int* idx, int n, int d, float* out, cudaStream_t s);
void launch_add_counter(unsigned long long* c, const int* n, cudaStream_t s);
void launch_probe_pick(const int* cnt, const int* cid, const float* cval, int nseg, int cap_u,
                       int fcap, const float* thr, const float* q2, float cmax, float eps_scale,
                       int P, int cap2, int nq, int* cand, int* cand_n, float* theta,
                       cudaStream_t s);

// probe.cu
int probe_tiles(int K);  // per-query tile minima the GEMM epilogue emits
void launch_query_scale(const float* Q, int nq, int d, float cmax, float* q2, float* qinv,
                        float* qscale, cudaStream_t s);
void launch_probe_gemm(const float* Q, const float* C, const float* c2, int nq, int K, int d,
                       const ScoreOut& o, float* tmin, cudaStream_t s);
void launch_probe_select(const uint16_t* D, int64_t ldD, const float* q2, const float* qscale,
                         int nq, int K, int Tmin, int cap, const float* tmin, int ntiles,
                         uint32_t* tup, int* cand, int* cand_n, float* theta, cudaStream_t s);
size_t probe_recheck_smem(int d, int P, int cap);
void launch_probe_recheck(const float* Q, const float* C, int nq, int K, int d, int P,
                          const int* cand, const int* cand_n, int cap, const float* theta,
                          float cmax, float eps_scale, float half_rel, int* regions, double* qc2,
                          int* fail, unsigned long long* fail_count, cudaStream_t s,
                          const int* qmap = nullptr);
void launch_probe_full(const float* Q, const float* C, int nq, int K, int d, int P, int mode,
                       const int* fail, int nslots, uint64_t* sk, uint32_t* sv, uint64_t* sk2,
                       uint32_t* sv2, double* sdv, int* regions, double* qc2, cudaStream_t s);

// plan.cu
struct PlanArgs {
  IndexView ix;
  const float* Q;
  const int* regions;   // (nq, P)
  const double* qc2;    // (nq, P)
  int nq, P;
  int64_t kept, budget;
  double* sbase;        // (nq, P*G) scratch
  double* sscore;       // (nq, P*G) scratch
  int32_t* ssize;       // (nq, P*G) scratch: global group size of each item
  WorkItem* work;       // (nq, cap_w)
  int64_t cap_w;
  int* nwork;           // (nq)
  int64_t* stats;       // (nq, 4)
  // rerank=False: scan order of the work list
  int sort_work;
  uint64_t* skey;       // (nq, pow2(cap_w)) scratch
  uint32_t* sval;       // (nq, pow2(cap_w)) scratch
  int32_t* order;       // (nq, cap_w)
  // approximate-first path: the probe's fp16-encoded scores (see ScoreOut)
  const uint16_t* D;    // (nq, ldD) or null (exact path only)
  const float* dscale;  // (nq) decode scale 2^e: qs2~ = h * dscale
  int64_t ldD;
  float cmax, eps_scale;
  int* only;            // (nq) fallback flags: exact kernels run where only[b] != 0
  uint32_t* akey;       // (nq, P*G) scratch: float32 order key of the approximate score
  int defer_rescore;    // set by launch_plan_approx: base/score by k_plan_rescore
  // K3a without D: qs2~ from the fp16 centroid rows (ix.c16); half_rel is the
  // relative storage error of the approximate qs2 (kHalfRel for D, 0 here)
  int direct;
  float half_rel;
  // query-sharded planning: emit whole groups (start = global group index
  // region * G + group, len = global length) instead of this shard's rows
  int global_items;
  // K4 window capacity: first pass (0 = the default by staging) and the
  // retry pass for the queries whose certified window overflowed
  int wcap_override;
  int retry;            // 1: only the queries flagged for window overflow
  int* n_overflow;      // (1) device counter of first-pass window overflows
  int approx;           // akey holds K3a's keys: run the approximate-first planner
};
// plan_approx.cu: K3a, the approximate group scores (needs D; may run per
// probe sub-chunk while D is still in L2), then the approximate-first planner
// (sets only[b] for the queries it cannot certify); both return kernels launched.
int launch_plan_scores(const PlanArgs& a, cudaStream_t s);
int launch_plan_approx(const PlanArgs& a, cudaStream_t s);
// Launches the approximate-first planner (when a.approx is set; K3a must have
// run) followed by the exact planner for the queries it could not certify;
// returns kernels launched.
int launch_plan(const PlanArgs& a, cudaStream_t s);

// plan_exchange.cu: plans made on another rank (query-sharded planning,
// SURVEY §8e) as 16-byte records, localized to this shard's rows
struct PlanItem {
  int32_t group;  // region * G + group (global)
  int32_t len;    // rows of the group to scan (global)
  double base;    // (1 - a) qc2 + a qs2
};
// work items (start = global group) -> plan items; nq x cap, counts in nwork
void launch_items_from_work(const WorkItem* work, int64_t cap_w, const int* nwork, int nq,
                            PlanItem* items, int64_t cap, int* nitems, cudaStream_t s);
// CSR plan items -> this shard's work items (empty slices dropped)
void launch_localize(const IndexView& ix, const int64_t* offsets, const PlanItem* items, int nq,
                     WorkItem* work, int64_t cap_w, int* nwork, cudaStream_t s);

// scan.cu
struct ScanArgs {
  IndexView ix;
  const float* Q;
  int nq;
  const WorkItem* work;
  int64_t cap_w;
  const int* nwork;
  int mode;             // 0: top-k, 1: full (all scanned keys)
  int k;
  int32_t* out_ids;     // (nq, k)
  float* out_d;         // (nq, k)
  uint64_t* full_keys;  // (nq, cap_full_p2)
  int64_t cap_full_p2;
  const float* luts;    // (nq, M, 256) built by launch_build_luts, or null: in-kernel
};
// K5 for a whole chunk: the inner-product LUT of every query (pq.py:147-169)
void launch_build_luts(const IndexView& ix, const float* Q, int nq, float* luts, cudaStream_t s);
void launch_scan(const ScanArgs& a, cudaStream_t s);
// scan_warp.cu: warp-independent sweeps (the default); false when the
// configuration is not covered (M > 32, top-k k > 128, n >= 2^32)
bool launch_scan_warp(const ScanArgs& a, cudaStream_t s);
bool scan_warp_ok(const ScanArgs& a);
// full mode: sort each query's keys and split into ids/dists rows of width `ld`
void launch_full_finish(uint64_t* keys, int64_t cap_p2, const int64_t* stats, int nq,
                        int32_t* ids, float* dists, int64_t ld, cudaStream_t s);
// rerank=False: scan-order ids with group scores
void launch_scan_order(const IndexView& ix, const WorkItem* work, int64_t cap_w,
                       const int* nwork, const int32_t* order, int nq, int32_t* ids,
                       float* dists, int64_t ld, cudaStream_t s);
// K7: merge per-shard top-k lists (G, nq, k) into (nq, k)
void launch_merge_topk(const int32_t* ids, const float* dists, int G, int nq, int k,
                       int32_t* out_ids, float* out_d, cudaStream_t s);

// build_tc.cu: index-builder kernels
int assign_kpad(int d);          // bf16 row width of KA's operands
bool assign_supported(int d);    // d <= 128
int assign_nsplit(int64_t rows, int K);
void launch_rows_bf16(const float* x, int64_t rows, int d, void* out, cudaStream_t s);
cudaError_t launch_assign_tc(const void* Xbf, int64_t rows, const void* Cbf, const float* c2, int K,
                             int d, int nsplit, float* part_v, int32_t* part_i, cudaStream_t s);
void launch_assign_reduce(const float* v, const int32_t* idx, int nsplit, int64_t rows,
                          const float* x2, int32_t* out, float* out_d, cudaStream_t s);
struct EncodeArgsC {
  const float* X;
  const int32_t* order;
  const int64_t* seg;
  const int32_t* seg_region;
  int64_t nseg;
  int d, L, M, grouping;
  const float* centroids;
  const int32_t* nbr;
  const float* alphas;
  const double* csq;
  const float* codewords;
  const float* cwsq;
  double lo, step;
  int16_t* pick;
  uint8_t* codes;
  uint8_t* cbytes;
  double* consts;
};
bool encode_supported(int d, int M);
void launch_row_norms(const float* x, int64_t rows, int d, float* out32, double* out64,
                      unsigned int* max_bits, cudaStream_t s);
size_t encode_smem(int d, int L, int M);
cudaError_t launch_encode_rows(const EncodeArgsC& a, cudaStream_t s);

}  // namespace givf
