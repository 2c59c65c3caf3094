// K3 + K4: group scores, tau-pruning and the candidate-budget walk
// (reference: search.py:111-139, util.concat_ranges util.py:58-74,
// GroupedIndex.group_starts index.py:80-85).
//
// One CTA per query.  Scores are float64 with every operation separately
// rounded (no FMA), exactly as numpy evaluates
//     base  = (1 - a) * qc2 + a * qs2,   score = base + f64(norm_term)
// with qs2 = sum((f64(c_s) - f64(q))^2).  The reference then lexsorts all
// P*G items by (score, pos, grp), keeps the first ceil(tau * P*G) and walks
// them until the candidate budget is spent.  Sorting P*G items per query is
// wasteful: only the prefix that ends at min(kept, budget crossing) matters,
// and only its *set* matters for the reranked output.  The CTA therefore
//   1. histograms the order-preserving keys of (score, flat) in <= 2048
//      buckets (counts and group-size weights together),
//   2. finds the first bucket where either the kept count or the budget is
//      reached, refining that bucket with further histogram levels until it
//      holds <= SORTCAP items,
//   3. sorts only that bucket exactly and walks it.
// Everything strictly below the bucket is scanned whole; the walk decides
// the bucket's items (partial last group included).  For rerank=False the
// emitted work list is additionally sorted into the reference scan order.
#include "common.cuh"
#include "kernels.h"

namespace givf {

constexpr int PLAN_THREADS = 256;
constexpr int PLAN_BUCKETS = 1024;
constexpr int SORTCAP = 1024;
constexpr int SORT_SMALL = 128;  // boundary buckets up to this size are sorted directly
constexpr int PLAN_SREG = 2048;  // probed regions staged in shared memory

GIVF_DEV double key_to_f64(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// float64 |c - q|^2 by an 8-lane group (4 centroid rows in flight per warp):
// lanes stride the row in float4 steps, then a 3-level xor tree.
__device__ double group8_sqdist64(const float* __restrict__ c, const double* qd, int d) {
  const int gl = threadIdx.x & 7;
  double s = 0.0;
  if ((d & 3) == 0) {
    const float4* c4 = reinterpret_cast<const float4*>(c);
    for (int j = gl; j < (d >> 2); j += 8) {
      float4 v = __ldg(c4 + j);
      const double* qq = qd + 4 * j;
      double t0 = dsub((double)v.x, qq[0]), t1 = dsub((double)v.y, qq[1]);
      double t2 = dsub((double)v.z, qq[2]), t3 = dsub((double)v.w, qq[3]);
      s = dadd(s, dadd(dadd(dmul(t0, t0), dmul(t1, t1)), dadd(dmul(t2, t2), dmul(t3, t3))));
    }
  } else {
    for (int j = gl; j < d; j += 8) {
      double t = dsub((double)__ldg(c + j), qd[j]);
      s = dadd(s, dmul(t, t));
    }
  }
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}

// U rows at once (d % 4 == 0, d <= 128): all loads issued before any math so
// each lane keeps 4*U float4 requests in flight.
template <int U>
__device__ void group8_sqdist64_multi(const float* const* rows, const double* qd, int d4,
                                      double* out) {
  const int gl = threadIdx.x & 7;
  float4 v[U][4];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int j = gl + 8 * t;
      v[u][t] = j < d4 ? __ldg(reinterpret_cast<const float4*>(rows[u]) + j)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int j = gl + 8 * t;
      if (j < d4) {
        const double* qq = qd + 4 * j;
        double t0 = dsub((double)v[u][t].x, qq[0]), t1 = dsub((double)v[u][t].y, qq[1]);
        double t2 = dsub((double)v[u][t].z, qq[2]), t3 = dsub((double)v[u][t].w, qq[3]);
        s = dadd(s, dadd(dadd(dmul(t0, t0), dmul(t1, t1)), dadd(dmul(t2, t2), dmul(t3, t3))));
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    out[u] = s;
  }
}

// ---- K3: float64 group scores (search.py:111-121), one CTA per query.
__global__ void __launch_bounds__(PLAN_THREADS) k_plan_score(PlanArgs a) {
  __shared__ double qd[1024];
  __shared__ int32_t sreg[PLAN_SREG];
  const IndexView& ix = a.ix;
  const int b = blockIdx.x, tid = threadIdx.x;
  if (a.only && a.only[b] == 0) return;  // fallback mode: flagged queries only
  const int G = ix.G, d = ix.d, P = a.P;
  const int64_t total = (int64_t)P * G;
  const int* reg = a.regions + (int64_t)b * P;
  const double* qc2 = a.qc2 + (int64_t)b * P;
  double* sbase = a.sbase + (int64_t)b * total;
  double* sscore = a.sscore + (int64_t)b * total;
  int32_t* ssize = a.ssize + (int64_t)b * total;

  for (int j = tid; j < d; j += blockDim.x) qd[j] = (double)a.Q[(int64_t)b * d + j];
  if (P <= PLAN_SREG)
    for (int p = tid; p < P; p += blockDim.x) sreg[p] = reg[p];
  __syncthreads();
  if (P <= PLAN_SREG) reg = sreg;

  auto finish = [&](int64_t f, int r, int j, double qs2, int p) {
    double al = (double)ix.alphas[r];
    double base = dadd(dmul(dsub(1.0, al), qc2[p]), dmul(al, qs2));
    sbase[f] = base;
    sscore[f] = dadd(base, (double)ix.norm[(int64_t)r * G + j]);
    ssize[f] = ix.gsize[(int64_t)r * G + j];
  };
  if (!ix.grouping) {
    for (int64_t f = tid; f < total; f += blockDim.x) {
      double v = qc2[f / G];
      sbase[f] = v;
      sscore[f] = v;
      ssize[f] = ix.gsize[(int64_t)reg[f / G] * G + (f % G)];
    }
    return;
  }
  const int grp = tid >> 3, ngrp = blockDim.x >> 3, gl = tid & 7;
  if ((d & 3) == 0 && d <= 128) {
    constexpr int U = 4;
    const int64_t iters = (total + (int64_t)ngrp * U - 1) / ((int64_t)ngrp * U);
    for (int64_t it = 0; it < iters; ++it) {
      const float* rows[U];
      int64_t fs[U];
      int rr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        fs[u] = (it * U + u) * ngrp + grp;
        const int64_t fc = fs[u] < total ? fs[u] : 0;
        rr[u] = reg[fc / G];
        rows[u] = ix.centroids + (int64_t)ix.nbr[(int64_t)rr[u] * G + (fc % G)] * d;
      }
      double qs2[U];
      group8_sqdist64_multi<U>(rows, qd, d >> 2, qs2);
      if (gl == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (fs[u] < total) finish(fs[u], rr[u], (int)(fs[u] % G), qs2[u], (int)(fs[u] / G));
      }
    }
  } else {
    // all 32 lanes of a warp iterate together (shuffles need the full mask)
    const int64_t iters = (total + ngrp - 1) / ngrp;
    for (int64_t it = 0; it < iters; ++it) {
      const int64_t f = it * ngrp + grp;
      const int64_t fc = f < total ? f : 0;
      const int p = (int)(fc / G), j = (int)(fc % G);
      const int r = reg[p];
      double qs2 = group8_sqdist64(ix.centroids + (int64_t)ix.nbr[(int64_t)r * G + j] * d, qd, d);
      if (f < total && gl == 0) finish(f, r, j, qs2, p);
    }
  }
}

// ---- K4: tau-pruning + budget walk + work-list emission, one CTA per query.
__global__ void __launch_bounds__(PLAN_THREADS) k_plan_select(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  unsigned long long* hw = reinterpret_cast<unsigned long long*>(dsm);
  uint64_t* bkey = reinterpret_cast<uint64_t*>(hw + PLAN_BUCKETS);
  uint32_t* hc = reinterpret_cast<uint32_t*>(bkey + SORTCAP);
  uint32_t* bval = hc + PLAN_BUCKETS;
  int32_t* blen = reinterpret_cast<int32_t*>(bval + SORTCAP);
  __shared__ unsigned long long red64[40];
  __shared__ uint32_t red32[40];
  __shared__ int s_b;
  __shared__ uint32_t s_bc_before;
  __shared__ unsigned long long s_bw_before;
  __shared__ int s_nemit;
  __shared__ unsigned long long s_walk_w;
  __shared__ int s_walk_begun;
  __shared__ uint32_t s_nbk;

  const IndexView& ix = a.ix;
  const int b = blockIdx.x, tid = threadIdx.x;
  if (a.only && a.only[b] == 0) return;  // fallback mode: flagged queries only
  const int G = ix.G, P = a.P;
  const int64_t total = (int64_t)P * G;
  const int* reg = a.regions + (int64_t)b * P;
  const double* sbase = a.sbase + (int64_t)b * total;
  const double* sscore = a.sscore + (int64_t)b * total;
  const int32_t* ssize = a.ssize + (int64_t)b * total;

  unsigned long long kmin = ~0ull, kmax = 0ull;
  for (int64_t f = tid; f < total; f += blockDim.x) {
    unsigned long long k = f64_key(sscore[f]);
    kmin = min(kmin, k);
    kmax = max(kmax, k);
  }
  kmin = block_min(kmin, red64);
  kmax = block_max(kmax, red64);

  // ---- 2. locate the end of the scanned prefix (search.py:123-139)
  const uint64_t kept = (uint64_t)a.kept, budget = (uint64_t)a.budget;
  uint64_t taken_c = 0, taken_w = 0;
  int phase = 0;                 // 0: bucket on score key; 1: on flat among score == kx
  uint64_t lo = kmin, hi = kmax, kx = 0;
  uint64_t bucket_lo = 0, bucket_hi = 0;  // final bucket range (phase-dependent key)
  for (int level = 0; level < 16; ++level) {
    uint64_t range = hi - lo;
    int shift = range == 0 ? 0 : max(0, 64 - __clzll((long long)range) - 10);  // <= 1024 buckets
    uint32_t nb = (uint32_t)(range >> shift) + 1;
    for (uint32_t i = tid; i < nb; i += blockDim.x) { hc[i] = 0; hw[i] = 0; }
    __syncthreads();
    for (int64_t f = tid; f < total; f += blockDim.x) {
      uint64_t sk = f64_key(sscore[f]);
      uint64_t key;
      if (phase == 0) {
        if (sk < lo || sk > hi) continue;
        key = sk;
      } else {
        if (sk != kx || (uint64_t)f < lo || (uint64_t)f > hi) continue;
        key = (uint64_t)f;
      }
      uint32_t bk = (uint32_t)((key - lo) >> shift);
      atomicAdd(&hc[bk], 1u);
      atomicAdd(&hw[bk], (unsigned long long)ssize[f]);
    }
    __syncthreads();
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    uint32_t b0 = tid * per, b1 = min(nb, b0 + per);
    uint32_t rc = 0;
    unsigned long long rw = 0;
    for (uint32_t x = b0; x < b1; ++x) { rc += hc[x]; rw += hw[x]; }
    uint32_t totc;
    unsigned long long totw;
    uint32_t pc = block_exclusive_scan(rc, red32, &totc);
    unsigned long long pw = block_exclusive_scan(rw, red64, &totw);
    if (tid == 0) s_b = -1;
    __syncthreads();
    {
      uint64_t c0 = taken_c + pc, w0 = taken_w + pw;
      bool before_ok = c0 < kept && w0 < budget;
      bool after_hit = (c0 + rc >= kept) || (w0 + rw >= budget);
      if (b0 < b1 && before_ok && after_hit) {
        uint64_t cc = c0, ww = w0;
        for (uint32_t x = b0; x < b1; ++x) {
          if (cc + hc[x] >= kept || ww + hw[x] >= budget) {
            s_b = (int)x;
            s_bc_before = (uint32_t)(cc - taken_c);
            s_bw_before = ww - taken_w;
            break;
          }
          cc += hc[x];
          ww += hw[x];
        }
      }
    }
    __syncthreads();
    const int bsel = s_b;
    if (bsel < 0) {  // nothing crosses: the whole range is scanned (cannot happen at level 0)
      bucket_lo = hi + 1;
      bucket_hi = hi;
      taken_c += totc;
      taken_w += totw;
      break;
    }
    const uint32_t cnt_b = hc[bsel];
    const uint64_t bl = lo + ((uint64_t)bsel << shift);
    const uint64_t bspan = bl + ((1ull << shift) - 1);
    const uint64_t bh = bspan < hi ? bspan : hi;
    taken_c += s_bc_before;
    taken_w += s_bw_before;
    __syncthreads();
    // another histogram pass over all items is far cheaper than a large
    // bitonic sort: refine until the boundary bucket is small
    if (cnt_b <= (uint32_t)SORT_SMALL || (shift == 0 && cnt_b <= (uint32_t)SORTCAP)) {
      bucket_lo = bl;
      bucket_hi = bh;
      break;
    }
    if (phase == 0 && shift == 0) {  // many items share one score: order them by flat
      phase = 1;
      kx = bl;
      lo = 0;
      hi = (uint64_t)(total - 1);
      continue;
    }
    lo = bl;
    hi = bh;
  }

  // ---- 3. sort the boundary bucket exactly and walk it
  if (tid == 0) { s_nemit = 0; s_walk_w = 0; s_walk_begun = 0; }
  __syncthreads();
  if (tid == 0) s_nbk = 0;
  __syncthreads();
  auto in_bucket = [&](int64_t f, uint64_t sk) -> bool {
    if (phase == 0) return sk >= bucket_lo && sk <= bucket_hi;
    return sk == kx && (uint64_t)f >= bucket_lo && (uint64_t)f <= bucket_hi;
  };
  auto below = [&](int64_t f, uint64_t sk) -> bool {
    if (phase == 0) return sk < bucket_lo;
    return sk < kx || (sk == kx && (uint64_t)f < bucket_lo);
  };
  for (int64_t f = tid; f < total; f += blockDim.x) {
    uint64_t sk = f64_key(sscore[f]);
    if (in_bucket(f, sk)) {
      uint32_t p = atomicAdd(&s_nbk, 1u);
      bkey[p] = sk;
      bval[p] = (uint32_t)f;
    }
  }
  __syncthreads();
  const uint32_t nbk = s_nbk;
  const uint32_t np2 = next_pow2(max(nbk, 1u));
  for (uint32_t i = nbk + tid; i < np2; i += blockDim.x) { bkey[i] = kKeyPad; bval[i] = 0xffffffffu; }
  __syncthreads();
  bitonic_sort(bkey, bval, np2);
  // walk the sorted bucket in parallel: item i has count prefix taken_c + i
  // and weight prefix taken_w + (exclusive scan of sizes)
  {
    unsigned long long carry = taken_w, my_scanned = 0;
    uint32_t my_begun = 0;
    for (uint32_t t0 = 0; t0 < nbk; t0 += blockDim.x) {
      const uint32_t i = t0 + tid;
      unsigned long long sz = 0;
      if (i < nbk) {
        int64_t f = bval[i];
        sz = (unsigned long long)ssize[f];
      }
      unsigned long long tile;
      unsigned long long excl = block_exclusive_scan(sz, red64, &tile);
      if (i < nbk) {
        const unsigned long long w = carry + excl;
        const bool ok = (taken_c + i < kept) && (w < budget);
        const unsigned long long l = ok ? min(sz, budget - w) : 0ull;
        blen[i] = (int32_t)l;
        my_begun += ok ? 1u : 0u;
        my_scanned += l;
      }
      carry += tile;
    }
    uint32_t tb = block_sum(my_begun, red32);
    unsigned long long ts = block_sum(my_scanned, red64);
    if (tid == 0) { s_walk_begun = (int)tb; s_walk_w = ts; }
  }
  __syncthreads();

  // ---- 4. emit the work list (local rows of this shard)
  auto emit = [&](int64_t f, int64_t len_g) {
    int p = (int)(f / G), j = (int)(f % G);
    int64_t gi = (int64_t)reg[p] * G + j;
    int64_t lo_ = ix.llo ? ix.llo[gi] : 0;
    int64_t cnt_ = ix.lsize ? ix.lsize[gi] : ix.gsize[gi];
    int64_t ll = min(max(len_g - lo_, (int64_t)0), cnt_);
    if (ll <= 0) return;
    int pos = atomicAdd(&s_nemit, 1);
    if (pos >= a.cap_w) return;  // cannot happen: cap_w bounds the begun items
    WorkItem w;
    w.start = ix.lstart[gi];
    w.len = (int32_t)ll;
    w.flat = (int32_t)f;
    w.base = sbase[f];
    w.score = sscore[f];
    a.work[(int64_t)b * a.cap_w + pos] = w;
  };
  for (int64_t f = tid; f < total; f += blockDim.x) {
    uint64_t sk = f64_key(sscore[f]);
    if (below(f, sk)) {
      emit(f, ssize[f]);
    }
  }
  for (uint32_t i = tid; i < nbk; i += blockDim.x)
    if (blen[i] > 0) emit(bval[i], blen[i]);
  __syncthreads();
  const int nemit = min(s_nemit, (int)a.cap_w);
  if (tid == 0) {
    a.nwork[b] = nemit;
    int64_t* st = a.stats + (int64_t)b * 4;
    st[0] = P;
    st[1] = (int64_t)taken_c + s_walk_begun;
    st[2] = total - (int64_t)kept;
    st[3] = (int64_t)taken_w + (int64_t)s_walk_w;
  }

  // ---- 5. rerank=False: reference scan order (score, pos, grp) of the list
  if (a.sort_work) {
    uint32_t wp2 = next_pow2(max(nemit, 1));
    int64_t cp2 = 1;
    while (cp2 < a.cap_w) cp2 <<= 1;
    uint64_t* sk = a.skey + (int64_t)b * cp2;
    uint32_t* sv = a.sval + (int64_t)b * cp2;
    const WorkItem* W = a.work + (int64_t)b * a.cap_w;
    for (uint32_t i = tid; i < wp2; i += blockDim.x) {
      if ((int)i < nemit) {
        // flat is unique per item: (score key, flat) is a total order
        sk[i] = f64_key(W[i].score);
        sv[i] = ((uint32_t)W[i].flat);
      } else {
        sk[i] = kKeyPad;
        sv[i] = 0xffffffffu;
      }
    }
    __syncthreads();
    bitonic_sort(sk, sv, wp2);
    // map sorted flat ids back to work-list positions
    for (int i = tid; i < nemit; i += blockDim.x) {
      // binary search of W's flat in the sorted (sk, sv) list
      uint64_t key = f64_key(W[i].score);
      uint32_t fl = (uint32_t)W[i].flat;
      int lo_i = 0, hi_i = nemit - 1;
      while (lo_i < hi_i) {
        int mid = (lo_i + hi_i) >> 1;
        bool less = sk[mid] < key || (sk[mid] == key && sv[mid] < fl);
        if (less) lo_i = mid + 1; else hi_i = mid;
      }
      a.order[(int64_t)b * a.cap_w + lo_i] = i;
    }
  }
}

// ---- K3+K4 fast path: approximate scores, exact where it matters.
//
// qs2 needs a float64 centroid row per (region, group) item; the probe GEMM
// already holds s~_c = |c|^2 - 2 q.c for every centroid with an a-priori
// error bound eps (probe.cu).  With qs2~ = s~ + |q|^2 every approximate score
// is within E of the exact one (alpha <= 1).  The CTA
//   1. selects on approximate keys exactly like k_plan_select and takes v*,
//      the approximate score of the last begun group;
//   2. splits items into A (score~ < v*-3E: exact < v*-2E), the window W
//      (|score~ - v*| <= 3E) and C (score~ > v*+3E: exact > v*+2E);
//   3. scores W exactly, sorts it and walks it from the prefix of A;
//   4. certifies the walk: the exact last begun group x_c lies in W with
//      v*-2E <= score(x_c) <= v*+2E, and the walk has ended inside W (or at
//      its end).  Then every A item precedes x_c, every C item follows it,
//      and the begun set, lengths and stats equal the exact walk's.
//      Otherwise the query is flagged for the exact planner.
//   5. emits A and the begun W items with float64 base/score recomputed
//      exactly (one centroid row per emitted group only).
constexpr int WCAP = 256;

__global__ void __launch_bounds__(PLAN_THREADS) k_plan_approx(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  unsigned long long* hw = reinterpret_cast<unsigned long long*>(dsm);
  uint64_t* bkey = reinterpret_cast<uint64_t*>(hw + PLAN_BUCKETS);
  uint64_t* wkey = bkey + SORTCAP;
  uint32_t* hc = reinterpret_cast<uint32_t*>(wkey + WCAP);
  uint32_t* bval = hc + PLAN_BUCKETS;
  int32_t* blen = reinterpret_cast<int32_t*>(bval + SORTCAP);
  uint32_t* wval = reinterpret_cast<uint32_t*>(blen + SORTCAP);
  int32_t* wlen = reinterpret_cast<int32_t*>(wval + WCAP);
  double* qd = reinterpret_cast<double*>(wlen + WCAP);
  __shared__ unsigned long long red64[40];
  __shared__ uint32_t red32[40];
  __shared__ double redd[40];
  __shared__ int s_b, s_nemit, s_lastb;
  __shared__ uint32_t s_bc_before, s_nbk, s_nw;
  __shared__ unsigned long long s_bw_before;

  const IndexView& ix = a.ix;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int G = ix.G, d = ix.d, P = a.P;
  const int64_t total = (int64_t)P * G;
  const int* reg = a.regions + (int64_t)b * P;
  const double* qc2 = a.qc2 + (int64_t)b * P;
  double* sscore = a.sscore + (int64_t)b * total;
  int32_t* ssize = a.ssize + (int64_t)b * total;
  const float* Drow = a.D + (int64_t)b * a.ldD;
  const uint64_t kept = (uint64_t)a.kept, budget = (uint64_t)a.budget;

  double q2p = 0.0;
  for (int j = tid; j < d; j += blockDim.x) {
    double x = (double)a.Q[(int64_t)b * d + j];
    qd[j] = x;
    q2p += x * x;
  }
  const double q2 = block_sum(q2p, redd);
  const double qn = sqrt(q2);
  const double E = ix.grouping
      ? 1.0001 * ((double)a.eps_scale * ((double)a.cmax * a.cmax + 2.0 * qn * a.cmax)) +
            1e-12 * ((double)a.cmax + qn) * ((double)a.cmax + qn)
      : 0.0;

  // ---- 1. approximate scores: one warp per probed region, lanes over its
  // groups (region terms loaded once, neighbor/norm/size rows coalesced)
  unsigned long long kmin = ~0ull, kmax = 0ull;
  {
    const int warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
    for (int p = warp; p < P; p += nwarps) {
      const int r = reg[p];
      const double qc = qc2[p];
      const double al = ix.grouping ? (double)ix.alphas[r] : 0.0;
      const double oma_qc = dmul(dsub(1.0, al), qc);
      for (int j = lane; j < G; j += 32) {
        const int64_t gi = (int64_t)r * G + j, f = (int64_t)p * G + j;
        double score = qc;
        if (ix.grouping) {
          const double qs2 = dadd((double)__ldg(Drow + ix.nbr[gi]), q2);
          score = dadd(dadd(oma_qc, dmul(al, qs2)), (double)ix.norm[gi]);
        }
        sscore[f] = score;
        ssize[f] = ix.gsize[gi];
        unsigned long long k = f64_key(score);
        kmin = min(kmin, k);
        kmax = max(kmax, k);
      }
    }
  }
  __syncthreads();
  kmin = block_min(kmin, red64);
  kmax = block_max(kmax, red64);

  // ---- 2. approximate crossing (same bucket refinement as k_plan_select)
  uint64_t taken_c = 0, taken_w = 0;
  uint64_t lo = kmin, hi = kmax, bucket_lo = 0, bucket_hi = 0;
  bool no_cut = false, flag = false;
  for (int level = 0; level < 16; ++level) {
    uint64_t range = hi - lo;
    int shift = range == 0 ? 0 : max(0, 64 - __clzll((long long)range) - 10);
    uint32_t nb = (uint32_t)(range >> shift) + 1;
    for (uint32_t i = tid; i < nb; i += blockDim.x) { hc[i] = 0; hw[i] = 0; }
    __syncthreads();
    for (int64_t f = tid; f < total; f += blockDim.x) {
      uint64_t sk = f64_key(sscore[f]);
      if (sk < lo || sk > hi) continue;
      uint32_t bk = (uint32_t)((sk - lo) >> shift);
      atomicAdd(&hc[bk], 1u);
      atomicAdd(&hw[bk], (unsigned long long)ssize[f]);
    }
    __syncthreads();
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    uint32_t b0 = tid * per, b1 = min(nb, b0 + per);
    uint32_t rc = 0;
    unsigned long long rw = 0;
    for (uint32_t x = b0; x < b1; ++x) { rc += hc[x]; rw += hw[x]; }
    uint32_t totc;
    unsigned long long totw;
    uint32_t pc = block_exclusive_scan(rc, red32, &totc);
    unsigned long long pw = block_exclusive_scan(rw, red64, &totw);
    if (tid == 0) s_b = -1;
    __syncthreads();
    {
      uint64_t c0 = taken_c + pc, w0 = taken_w + pw;
      if (b0 < b1 && c0 < kept && w0 < budget && (c0 + rc >= kept || w0 + rw >= budget)) {
        uint64_t cc = c0, ww = w0;
        for (uint32_t x = b0; x < b1; ++x) {
          if (cc + hc[x] >= kept || ww + hw[x] >= budget) {
            s_b = (int)x;
            s_bc_before = (uint32_t)(cc - taken_c);
            s_bw_before = ww - taken_w;
            break;
          }
          cc += hc[x];
          ww += hw[x];
        }
      }
    }
    __syncthreads();
    const int bsel = s_b;
    if (bsel < 0) {  // never crosses: every group is scanned whole
      no_cut = true;
      break;
    }
    const uint32_t cnt_b = hc[bsel];
    const uint64_t bl = lo + ((uint64_t)bsel << shift);
    const uint64_t bspan = bl + ((1ull << shift) - 1);
    const uint64_t bh = bspan < hi ? bspan : hi;
    taken_c += s_bc_before;
    taken_w += s_bw_before;
    __syncthreads();
    // another histogram pass over all items is far cheaper than a large
    // bitonic sort: refine until the boundary bucket is small
    if (cnt_b <= (uint32_t)SORT_SMALL || (shift == 0 && cnt_b <= (uint32_t)SORTCAP)) {
      bucket_lo = bl;
      bucket_hi = bh;
      break;
    }
    if (shift == 0) {  // > SORTCAP equal approximate scores: leave it to the exact planner
      flag = true;
      break;
    }
    lo = bl;
    hi = bh;
  }

  double vstar = __longlong_as_double(0x7ff0000000000000ll);  // +inf: no cut
  if (!no_cut && !flag) {
    if (tid == 0) s_nbk = 0;
    __syncthreads();
    for (int64_t f = tid; f < total; f += blockDim.x) {
      uint64_t sk = f64_key(sscore[f]);
      if (sk >= bucket_lo && sk <= bucket_hi) {
        uint32_t p = atomicAdd(&s_nbk, 1u);
        bkey[p] = sk;
        bval[p] = (uint32_t)f;
      }
    }
    __syncthreads();
    const uint32_t nbk = s_nbk;
    const uint32_t np2 = next_pow2(max(nbk, 1u));
    for (uint32_t i = nbk + tid; i < np2; i += blockDim.x) { bkey[i] = kKeyPad; bval[i] = 0xffffffffu; }
    __syncthreads();
    bitonic_sort(bkey, bval, np2);
    // approximate walk: index of the last begun item
    if (tid == 0) s_lastb = -1;
    __syncthreads();
    unsigned long long carry = taken_w;
    for (uint32_t t0 = 0; t0 < nbk; t0 += blockDim.x) {
      const uint32_t i = t0 + tid;
      unsigned long long sz = i < nbk ? (unsigned long long)ssize[bval[i]] : 0ull;
      unsigned long long tile;
      unsigned long long excl = block_exclusive_scan(sz, red64, &tile);
      if (i < nbk && taken_c + i < kept && carry + excl < budget) atomicMax(&s_lastb, (int)i);
      carry += tile;
    }
    __syncthreads();
    vstar = key_to_f64(bkey[max(s_lastb, 0)]);
  }

  // ---- 3. window around v*: exact scores, sorted, walked from A's prefix
  const double wlo = vstar - 3.0 * E, whi = vstar + 3.0 * E;
  uint64_t nA = 0, wA = 0;
  if (tid == 0) { s_nw = 0; s_nemit = 0; }
  __syncthreads();
  {
    uint64_t c = 0, w = 0;
    for (int64_t f = tid; f < total; f += blockDim.x) {
      const double sc = sscore[f];
      if (sc < wlo) {
        c += 1;
        w += (uint64_t)ssize[f];
      } else if (sc <= whi && !no_cut) {
        uint32_t p = atomicAdd(&s_nw, 1u);
        if (p < WCAP) wval[p] = (uint32_t)f;
      }
    }
    nA = block_sum((unsigned long long)c, red64);
    wA = block_sum((unsigned long long)w, red64);
  }
  const uint32_t nw = s_nw;
  if (nw > WCAP) flag = true;
  uint32_t lastw = 0;
  bool ended = no_cut;
  if (!flag && !no_cut) {
    // exact float64 scores of the window (8-lane groups)
    const int grp = tid >> 3, ngrp = blockDim.x >> 3, gl = tid & 7;
    for (uint32_t i0 = 0; i0 < nw; i0 += ngrp) {
      const uint32_t i = i0 + grp;
      const int64_t f = i < nw ? wval[i] : 0;
      const int p = (int)(f / G), j = (int)(f % G);
      const int r = reg[p];
      double score = qc2[p];
      if (ix.grouping) {
        const int64_t gi = (int64_t)r * G + j;
        double qs2 = group8_sqdist64(ix.centroids + (int64_t)ix.nbr[gi] * d, qd, d);
        const double al = (double)ix.alphas[r];
        score = dadd(dadd(dmul(dsub(1.0, al), qc2[p]), dmul(al, qs2)), (double)ix.norm[gi]);
      }
      if (i < nw && gl == 0) wkey[i] = f64_key(score);
    }
    const uint32_t np2 = next_pow2(max(nw, 1u));
    for (uint32_t i = nw + tid; i < np2; i += blockDim.x) { wkey[i] = kKeyPad; wval[i] = 0xffffffffu; }
    __syncthreads();
    bitonic_sort(wkey, wval, np2);
    // exact walk over W starting from A's count/weight
    if (tid == 0) s_lastb = -1;
    __syncthreads();
    unsigned long long carry = wA;
    for (uint32_t t0 = 0; t0 < nw; t0 += blockDim.x) {
      const uint32_t i = t0 + tid;
      unsigned long long sz = i < nw ? (unsigned long long)ssize[wval[i]] : 0ull;
      unsigned long long tile;
      unsigned long long excl = block_exclusive_scan(sz, red64, &tile);
      if (i < nw) {
        const unsigned long long w = carry + excl;
        const bool ok = (nA + i < kept) && (w < budget);
        wlen[i] = ok ? (int32_t)min(sz, budget - w) : 0;
        if (ok) atomicMax(&s_lastb, (int)i);
      }
      carry += tile;
    }
    __syncthreads();
    const int xc = s_lastb;
    if (xc < 0) {
      flag = true;  // the exact crossing precedes the window
    } else {
      lastw = (uint32_t)xc;
      const double sx = key_to_f64(wkey[xc]);
      if (!(sx >= vstar - 2.0 * E && sx <= vstar + 2.0 * E)) flag = true;
      // the walk must end at or inside W: the item after x_c is not begun
      if ((uint32_t)xc + 1 == nw) ended = (nA + nw >= kept) || (carry >= budget);
      else ended = true;
      if (!ended) flag = true;
    }
  }
  if (flag) {
    if (tid == 0) {
      a.only[b] = 1;
      if (ix.counters) atomicAdd(&ix.counters[1], 1ull);
    }
    return;
  }
  if (tid == 0) a.only[b] = 0;

  // ---- 4. emit A + begun W with exact base/score (local rows of this shard)
  WorkItem* W = a.work + (int64_t)b * a.cap_w;
  auto emit = [&](int64_t f, int64_t len_g) {
    const int p = (int)(f / G), j = (int)(f % G);
    const int64_t gi = (int64_t)reg[p] * G + j;
    const int64_t lo_ = ix.llo ? ix.llo[gi] : 0;
    const int64_t cnt_ = ix.lsize ? ix.lsize[gi] : ix.gsize[gi];
    const int64_t ll = min(max(len_g - lo_, (int64_t)0), cnt_);
    if (ll <= 0) return;
    const int pos = atomicAdd(&s_nemit, 1);
    if (pos >= a.cap_w) return;
    WorkItem w;
    w.start = ix.lstart[gi];
    w.len = (int32_t)ll;
    w.flat = (int32_t)f;
    w.base = 0.0;
    w.score = 0.0;
    W[pos] = w;
  };
  uint64_t begun_w = 0, scanned_w = 0;
  for (int64_t f = tid; f < total; f += blockDim.x)
    if (sscore[f] < wlo) emit(f, ssize[f]);
  for (uint32_t i = tid; i < nw && !no_cut; i += blockDim.x) {
    if (i <= lastw) {
      begun_w += 1;
      scanned_w += (uint64_t)wlen[i];
      if (wlen[i] > 0) emit(wval[i], wlen[i]);
    }
  }
  begun_w = block_sum((unsigned long long)begun_w, red64);
  scanned_w = block_sum((unsigned long long)scanned_w, red64);
  const int nemit = min(s_nemit, (int)a.cap_w);
  {
    const int grp = tid >> 3, ngrp = blockDim.x >> 3, gl = tid & 7;
    for (int i0 = 0; i0 < nemit; i0 += ngrp) {
      const int i = i0 + grp;
      const int64_t f = i < nemit ? W[i].flat : 0;
      const int p = (int)(f / G), j = (int)(f % G);
      const int r = reg[p];
      double base = qc2[p], score = qc2[p];
      if (ix.grouping) {
        const int64_t gi = (int64_t)r * G + j;
        double qs2 = group8_sqdist64(ix.centroids + (int64_t)ix.nbr[gi] * d, qd, d);
        const double al = (double)ix.alphas[r];
        base = dadd(dmul(dsub(1.0, al), qc2[p]), dmul(al, qs2));
        score = dadd(base, (double)ix.norm[gi]);
      }
      if (i < nemit && gl == 0) { W[i].base = base; W[i].score = score; }
    }
  }
  if (tid == 0) {
    a.nwork[b] = nemit;
    int64_t* st = a.stats + (int64_t)b * 4;
    st[0] = P;
    st[1] = (int64_t)(nA + begun_w);
    st[2] = total - (int64_t)kept;
    st[3] = (int64_t)(wA + scanned_w);
  }
  if (a.sort_work) {
    __syncthreads();
    uint32_t wp2 = next_pow2(max(nemit, 1));
    int64_t cp2 = 1;
    while (cp2 < a.cap_w) cp2 <<= 1;
    uint64_t* sk = a.skey + (int64_t)b * cp2;
    uint32_t* sv = a.sval + (int64_t)b * cp2;
    for (uint32_t i = tid; i < wp2; i += blockDim.x) {
      sk[i] = (int)i < nemit ? f64_key(W[i].score) : kKeyPad;
      sv[i] = (int)i < nemit ? (uint32_t)W[i].flat : 0xffffffffu;
    }
    __syncthreads();
    bitonic_sort(sk, sv, wp2);
    for (int i = tid; i < nemit; i += blockDim.x) {
      uint64_t key = f64_key(W[i].score);
      uint32_t fl = (uint32_t)W[i].flat;
      int lo_i = 0, hi_i = nemit - 1;
      while (lo_i < hi_i) {
        int mid = (lo_i + hi_i) >> 1;
        bool less = sk[mid] < key || (sk[mid] == key && sv[mid] < fl);
        if (less) lo_i = mid + 1; else hi_i = mid;
      }
      a.order[(int64_t)b * a.cap_w + lo_i] = i;
    }
  }
}

size_t plan_smem(int d) {
  (void)d;
  return (size_t)PLAN_BUCKETS * 8 + SORTCAP * 8 + PLAN_BUCKETS * 4 + SORTCAP * 4 + SORTCAP * 4 + 16;
}

size_t plan_approx_smem(int d) {
  return (size_t)PLAN_BUCKETS * 8 + SORTCAP * 8 + WCAP * 8 + PLAN_BUCKETS * 4 + SORTCAP * 4 +
         SORTCAP * 4 + WCAP * 4 + WCAP * 4 + (size_t)d * 8 + 16;
}

int launch_plan(const PlanArgs& a, cudaStream_t s) {
  if (a.D != nullptr && a.only != nullptr) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_plan_approx, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      attr = true;
    }
    k_plan_approx<<<a.nq, PLAN_THREADS, plan_approx_smem(a.ix.d), s>>>(a);
    k_plan_score<<<a.nq, PLAN_THREADS, 0, s>>>(a);
    k_plan_select<<<a.nq, PLAN_THREADS, plan_smem(a.ix.d), s>>>(a);
    return 3;
  }
  PlanArgs e = a;
  e.only = nullptr;
  k_plan_score<<<a.nq, PLAN_THREADS, 0, s>>>(e);
  k_plan_select<<<a.nq, PLAN_THREADS, plan_smem(a.ix.d), s>>>(e);
  return 2;
}

}  // namespace givf
