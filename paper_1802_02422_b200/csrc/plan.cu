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
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "plan_common.cuh"

namespace givf {

constexpr int PLAN_THREADS = 256;
constexpr int PLAN_BUCKETS = 1024;
constexpr int SORTCAP = 1024;
constexpr int SORT_SMALL = 128;  // boundary buckets up to this size are sorted directly
constexpr int PLAN_SREG = 2048;  // probed regions staged in shared memory

// ---- K3: float64 group scores (search.py:111-121), one CTA per query.
__device__ void plan_score_one(const PlanArgs& a, const int b) {
  __shared__ double qd[1024];
  __shared__ int32_t sreg[PLAN_SREG];
  const IndexView& ix = a.ix;
  const int tid = threadIdx.x;
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
__device__ void plan_select_one(const PlanArgs& a, const int b) {
  extern __shared__ __align__(16) unsigned char dsm[];
  unsigned long long* hw = reinterpret_cast<unsigned long long*>(dsm);  // (first 4 KB: u32 weights)
  uint32_t* hw32 = reinterpret_cast<uint32_t*>(dsm);
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
  const int tid = threadIdx.x;
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
    for (uint32_t i = tid; i < nb; i += blockDim.x) { hc[i] = 0; hw32[i] = 0; }
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
      atomicAdd(&hw32[bk], (uint32_t)ssize[f]);  // 32-bit: a 64-bit shared atomic is a CAS loop
    }
    __syncthreads();
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    uint32_t b0 = tid * per, b1 = min(nb, b0 + per);
    uint32_t rc = 0;
    unsigned long long rw = 0;
    for (uint32_t x = b0; x < b1; ++x) { rc += hc[x]; rw += hw32[x]; }
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
          if (cc + hc[x] >= kept || ww + hw32[x] >= budget) {
            s_b = (int)x;
            s_bc_before = (uint32_t)(cc - taken_c);
            s_bw_before = ww - taken_w;
            break;
          }
          cc += hc[x];
          ww += hw32[x];
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
    int64_t lo_ = (ix.llo && !a.global_items) ? ix.llo[gi] : 0;
    int64_t cnt_ = a.global_items ? len_g : (ix.lsize ? ix.lsize[gi] : ix.gsize[gi]);
    int64_t ll = min(max(len_g - lo_, (int64_t)0), cnt_);
    if (ll <= 0) return;
    int pos = atomicAdd(&s_nemit, 1);
    if (pos >= a.cap_w) return;  // cannot happen: cap_w bounds the begun items
    WorkItem w;
    w.start = a.global_items ? gi : ix.lstart[gi];
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

size_t plan_smem(int d) {
  (void)d;
  return (size_t)PLAN_BUCKETS * 8 + SORTCAP * 8 + PLAN_BUCKETS * 4 + SORTCAP * 4 + SORTCAP * 4 + 16;
}

// One CTA per query, or (fallback mode, a.only set) a grid-stride loop over
// the queries that only visits the flagged ones: the approximate planner
// flags few or none, and a 10^4-CTA grid of early exits costs ~20 us.
__global__ void __launch_bounds__(PLAN_THREADS) k_plan_score(PlanArgs a) {
  for (int b = blockIdx.x; b < a.nq; b += gridDim.x) {
    if (a.only && a.only[b] == 0) continue;
    plan_score_one(a, b);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(PLAN_THREADS) k_plan_select(PlanArgs a) {
  for (int b = blockIdx.x; b < a.nq; b += gridDim.x) {
    if (a.only && a.only[b] == 0) continue;
    plan_select_one(a, b);
    __syncthreads();
  }
}

int launch_plan(const PlanArgs& a, cudaStream_t s) {
  int n = 0;
  if (a.approx && a.only != nullptr) {
    n += launch_plan_approx(a, s);  // flags the queries it cannot certify
    int sms = 148;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = std::min(a.nq, 2 * sms);
    k_plan_score<<<grid, PLAN_THREADS, 0, s>>>(a);
    k_plan_select<<<grid, PLAN_THREADS, plan_smem(a.ix.d), s>>>(a);
    return n + 2;
  }
  PlanArgs e = a;
  e.only = nullptr;
  k_plan_score<<<a.nq, PLAN_THREADS, 0, s>>>(e);
  k_plan_select<<<a.nq, PLAN_THREADS, plan_smem(a.ix.d), s>>>(e);
  return 2;
}

}  // namespace givf
