// K3 + K4 fast path: approximate group scores from the probe's fp32 scores,
// float64 only where a decision depends on it (reference: search.py:111-139).
//
// qs2 = |q - c_s|^2 needs a float64 centroid row per (region, group) item;
// the probe GEMM already holds s~_c = |c|^2 - 2 q.c for every centroid with
// an a-priori error bound eps (probe.cu, probe_tc.cu).  With
// qs2~ = s~ + |q|^2 every approximate score is within E of the exact one
// (alpha <= 1; the float32 key adds one more rounding, folded into E).
//
//   K3a k_plan_scores_approx  one warp per (query, probed region), lanes over
//       its groups: gather s~ of the neighbor centroid, form the score, write
//       its float32 order key.
//   K4  k_plan_approx         one CTA per query:
//     1. locates the approximate crossing (kept count / candidate budget) by
//        bucket refinement over the keys, sorts only the boundary bucket and
//        takes v*, the approximate score of the last begun group;
//     2. splits items into A (score~ < v*-3E: exact < v*-2E), the window W
//        (|score~ - v*| <= 3E) and C (score~ > v*+3E: exact > v*+2E);
//     3. scores W exactly, sorts it and walks it from A's count and weight;
//     4. certifies: the exact last begun group x_c lies in W with
//        v*-2E <= score(x_c) <= v*+2E and the walk ends inside W.  Then the
//        groups preceding x_c in the exact order are exactly A and the W
//        groups before it, every C group follows it, and the begun set,
//        lengths and stats are the exact walk's.  Otherwise the query is
//        flagged and the exact planner (plan.cu) redoes it;
//     5. emits A and the begun W groups (compacted, one metadata gather per
//        group) with float64 base/score recomputed exactly from one centroid
//        row per emitted group.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "plan_common.cuh"

namespace givf {

constexpr int PA_THREADS = 256;
constexpr int PA_ITEMS = 4096;    // items staged in shared memory (else read from L2/HBM)
constexpr int PA_BUCKETS = 1024;
constexpr int PA_SORT = 1024;     // boundary-bucket sort capacity
constexpr int PA_SMALL = 128;     // refine further while the bucket is larger
constexpr int PA_WCAP = 256;      // window capacity (items staged in shared memory)
constexpr int PA_WCAP_BIG = 1024; // window capacity when the items are not staged
constexpr int PA_WCAP_RETRY = 2048;  // retry pass for the queries whose window overflowed
constexpr int PA_CAND = 1536;     // begun groups (else the exact planner)
constexpr int PA_PSTAGE = 512;    // probed regions staged in shared memory
constexpr int PA_U = 4;           // centroid rows in flight per 8-lane group
// histogram cells and prefixes carry (count << 40 | weight): weights are group
// sizes summing to at most n < 2^40, counts at most P*G < 2^24
constexpr int CW = 40;
constexpr unsigned long long WMASK = (1ull << CW) - 1;

// ---------------------------------------------------------------- K3a
__global__ void __launch_bounds__(PA_THREADS) k_plan_scores_approx(PlanArgs a) {
  const IndexView& ix = a.ix;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * (PA_THREADS / 32) + (threadIdx.x >> 5);
  const int P = a.P, G = ix.G;
  if (wid >= (int64_t)a.nq * P) return;
  const int b = (int)(wid / P), p = (int)(wid % P);
  const int64_t total = (int64_t)P * G;
  const int r = a.regions[(int64_t)b * P + p];
  const double qc = a.qc2[(int64_t)b * P + p];
  uint32_t* akey = a.akey + (int64_t)b * total + (int64_t)p * G;
  if (!ix.grouping) {
    const uint32_t k = f32_key((float)qc);
    for (int j = lane; j < G; j += 32) akey[j] = k;
    return;
  }
  const uint16_t* Drow = a.D + (int64_t)b * a.ldD;
  const double dsc = (double)a.dscale[b];
  const double al = (double)ix.alphas[r];
  const double oma_qc = dmul(dsub(1.0, al), qc);
  // two groups per lane per step: both gathers in flight at once
  for (int j0 = 0; j0 < G; j0 += 64) {
    const int j1 = j0 + lane, j2 = j0 + 32 + lane;
    const bool v1 = j1 < G, v2 = j2 < G;
    const int64_t g1 = (int64_t)r * G + (v1 ? j1 : 0), g2 = (int64_t)r * G + (v2 ? j2 : 0);
    const int n1 = __ldg(ix.nbr + g1), n2 = __ldg(ix.nbr + g2);
    const float m1 = __ldg(ix.norm + g1), m2 = __ldg(ix.norm + g2);
    const uint16_t h1 = __ldg(Drow + n1), h2 = __ldg(Drow + n2);
    // fp16-encoded |q - c_s|^2 (ScoreOut in kernels.h), decoded exactly
    const double s1 = (double)__half2float(__ushort_as_half(h1)) * dsc;
    const double s2 = (double)__half2float(__ushort_as_half(h2)) * dsc;
    if (v1) akey[j1] = f32_key((float)dadd(dadd(oma_qc, dmul(al, s1)), (double)m1));
    if (v2) akey[j2] = f32_key((float)dadd(dadd(oma_qc, dmul(al, s2)), (double)m2));
  }
}

// K3a without the score matrix (fused probe, probe_fused.cu): qs2~ =
// |q|^2 + |c_s|^2 - 2 q.c~_s from the neighbor's fp16 centroid row (192 B at
// d = 96) and the float32 query, float32 dot product; error bound
// direct_f16_eps (units of cmax^2 + 2 |q| cmax), no storage term (half_rel 0).
// One warp per (query, probed region) as above, a lane per group.
// DP8: 16-byte chunks read per row (d coordinates, zero-padded in the
// query's shared copy); rows from ix.c16r (pitch f16_row_pitch(d))
// PK: rows from the per-region packed copy ix.c16p (contiguous 512-byte
// lines per warp load) instead of gathered from ix.c16r
template <int DP8, bool PK>
__global__ void __launch_bounds__(PA_THREADS) k_plan_scores_direct(PlanArgs a) {
  __shared__ __align__(16) float qsm[PA_THREADS / 32][DP8 * 8];
  const IndexView& ix = a.ix;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t wid = (int64_t)blockIdx.x * (PA_THREADS / 32) + w;
  const int P = a.P, G = ix.G, d = ix.d;
  if (wid >= (int64_t)a.nq * P) return;
  const int b = (int)(wid / P), p = (int)(wid % P);
  const int64_t total = (int64_t)P * G;
  const int r = a.regions[(int64_t)b * P + p];
  const double qc = a.qc2[(int64_t)b * P + p];
  uint32_t* akey = a.akey + (int64_t)b * total + (int64_t)p * G;
  if (!ix.grouping) {
    const uint32_t k = f32_key((float)qc);
    for (int j = lane; j < G; j += 32) akey[j] = k;
    return;
  }
  float* qs = qsm[w];
  double s = 0.0;
  for (int j = lane; j < DP8 * 8; j += 32) {
    const float x = j < d ? a.Q[(int64_t)b * d + j] : 0.f;
    qs[j] = x;
    s += (double)x * x;
  }
  const double q2 = warp_sum(s);
  __syncwarp();
  const double al = (double)ix.alphas[r];
  const double oma_qc = dmul(dsub(1.0, al), qc);
  const double cx2 = 2.0 * (double)ix.c16x;
  const uint4* C16 = reinterpret_cast<const uint4*>(ix.c16r);
  const uint4* P16 = reinterpret_cast<const uint4*>(ix.c16p);
  const int64_t rstride = f16_row_pitch(d) / 8;  // row pitch in 16-byte chunks
  const float4* q4 = reinterpret_cast<const float4*>(qs);
  for (int j = lane; j < G; j += 32) {
    const int64_t g = (int64_t)r * G + j;
    const float m = __ldg(ix.norm + g);
    uint4 u[DP8];
    float c2n;
    if constexpr (PK) {  // the region's packed copy: lanes read consecutive 16-byte chunks
      const uint4* row = P16 + (int64_t)r * DP8 * G + j;
#pragma unroll
      for (int c = 0; c < DP8; ++c) u[c] = __ldg(row + (int64_t)c * G);
      c2n = __ldg(ix.c2p + g);
    } else {
      const int n = __ldg(ix.nbr + g);
      const uint4* row = C16 + (int64_t)n * rstride;
#pragma unroll
      for (int c = 0; c < DP8; ++c) u[c] = __ldg(row + c);
      c2n = __ldg(ix.c2f + n);
    }
    float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
    for (int c = 0; c < DP8; ++c) {
      const float4 qa = q4[2 * c], qb = q4[2 * c + 1];  // shared-memory broadcast
      const float2 h0 = __half22float2(*reinterpret_cast<const __half2*>(&u[c].x));
      const float2 h1 = __half22float2(*reinterpret_cast<const __half2*>(&u[c].y));
      const float2 h2 = __half22float2(*reinterpret_cast<const __half2*>(&u[c].z));
      const float2 h3 = __half22float2(*reinterpret_cast<const __half2*>(&u[c].w));
      acc0 = fmaf(qa.x, h0.x, acc0);
      acc1 = fmaf(qa.y, h0.y, acc1);
      acc0 = fmaf(qa.z, h1.x, acc0);
      acc1 = fmaf(qa.w, h1.y, acc1);
      acc0 = fmaf(qb.x, h2.x, acc0);
      acc1 = fmaf(qb.y, h2.y, acc1);
      acc0 = fmaf(qb.z, h3.x, acc0);
      acc1 = fmaf(qb.w, h3.y, acc1);
    }
    const double qs2 = dsub(dadd(q2, (double)c2n), dmul(cx2, (double)(acc0 + acc1)));
    akey[j] = f32_key((float)dadd(dadd(oma_qc, dmul(al, qs2)), (double)m));
  }
}

// ---------------------------------------------------------------- K4
struct PaSmem {
  // byte offsets into the dynamic shared block
  size_t skey, ssz, pool, wkey, wval, wlen, wrow, wnorm, qd, preg, pqc, pal, bytes;
  int wcap;  // window capacity: larger when the items' staging space is free
  // small: every group size < 2^16, so the staged sizes are 16-bit
  __host__ __device__ PaSmem(int d, int P, int64_t total, bool small, int wcap_override = 0) {
    const bool staged = total <= PA_ITEMS;
    const bool pst = P <= PA_PSTAGE;
    size_t o = 0;
    auto take = [&](size_t n) { size_t r = o; o = (o + n + 15) & ~(size_t)15; return r; };
    pool = take((size_t)3 * PA_CAND * 4 > (size_t)(PA_BUCKETS + PA_SORT) * 8
                    ? (size_t)3 * PA_CAND * 4 : (size_t)(PA_BUCKETS + PA_SORT) * 8);
    wcap = wcap_override > 0 ? wcap_override : (staged ? PA_WCAP : PA_WCAP_BIG);
    wkey = take((size_t)wcap * 8);
    qd = take((size_t)d * 8);
    pqc = take(pst ? (size_t)P * 8 : 0);
    pal = take(pst ? (size_t)P * 8 : 0);
    preg = take(pst ? (size_t)P * 4 : 0);
    wval = take((size_t)wcap * 4);
    wlen = take((size_t)wcap * 4);
    wrow = take((size_t)wcap * 4);
    wnorm = take((size_t)wcap * 4);
    skey = take(staged ? (size_t)PA_ITEMS * 4 : 0);
    ssz = take(staged ? (size_t)PA_ITEMS * (small ? 2 : 4) : 0);
    bytes = o;
  }
};

// INLINE: the emitted groups' exact base/score are computed here (the
// scan-order sort needs them); otherwise k_plan_rescore does it.
template <bool INLINE>
__global__ void __launch_bounds__(PA_THREADS, INLINE ? 3 : 4) k_plan_approx(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const IndexView& ix = a.ix;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int G = ix.G, d = ix.d, P = a.P;
  const int64_t total = (int64_t)P * G;
  const bool staged = total <= PA_ITEMS;
  const bool pst = P <= PA_PSTAGE;
  const bool small = ix.max_gsize < 65536;
  // retry pass: only the queries whose window overflowed in the first pass
  if (a.retry && a.only[b] != 2) return;
  const PaSmem L(d, P, total, small, a.wcap_override);

  // histogram: separate 32-bit counts and weights (a 64-bit shared atomic
  // is a CAS loop); bucket weights are sums of group sizes < 2^32
  uint32_t* hcn = reinterpret_cast<uint32_t*>(dsm + L.pool);
  uint32_t* hwt = hcn + PA_BUCKETS;
  auto HW = [&](uint32_t x) -> unsigned long long {
    return ((unsigned long long)hcn[x] << CW) | hwt[x];
  };
  uint64_t* bkey = reinterpret_cast<uint64_t*>(dsm + L.pool) + PA_BUCKETS;
  uint32_t* cf = reinterpret_cast<uint32_t*>(dsm + L.pool);  // begun groups: flat
  int32_t* cl = reinterpret_cast<int32_t*>(cf + PA_CAND);     //   length; after emission: row
  int32_t* cp = cl + PA_CAND;                                 //   after emission: norm bits | p
  uint64_t* wkey = reinterpret_cast<uint64_t*>(dsm + L.wkey);
  uint32_t* wval = reinterpret_cast<uint32_t*>(dsm + L.wval);
  int32_t* wlen = reinterpret_cast<int32_t*>(dsm + L.wlen);
  int32_t* wrow = reinterpret_cast<int32_t*>(dsm + L.wrow);
  float* wnorm = reinterpret_cast<float*>(dsm + L.wnorm);
  double* qd = reinterpret_cast<double*>(dsm + L.qd);
  uint32_t* skey = reinterpret_cast<uint32_t*>(dsm + L.skey);
  int32_t* ssz = reinterpret_cast<int32_t*>(dsm + L.ssz);
  uint16_t* ssz16 = reinterpret_cast<uint16_t*>(dsm + L.ssz);
  int32_t* preg = reinterpret_cast<int32_t*>(dsm + L.preg);
  double* pqc = reinterpret_cast<double*>(dsm + L.pqc);
  double* pal = reinterpret_cast<double*>(dsm + L.pal);
  __shared__ unsigned long long red64[40];
  __shared__ uint32_t red32[40];
  __shared__ double redd[40];
  __shared__ int s_b, s_lastb;
  __shared__ uint32_t s_nbk, s_nw;
  __shared__ unsigned long long s_before;

  const uint32_t* gkey = a.akey + (int64_t)b * total;
  const int* greg = a.regions + (int64_t)b * P;
  const double* gqc = a.qc2 + (int64_t)b * P;
  const uint64_t kept = (uint64_t)a.kept, budget = (uint64_t)a.budget;
#ifdef GIVF_PHASES
  long long t_phase_ = clock64();
#endif

  // ---- 0. stage the query, the probed regions, the items; key range
  double q2p = 0.0;
  for (int j = tid; j < d; j += PA_THREADS) {
    const double x = (double)a.Q[(int64_t)b * d + j];
    qd[j] = x;
    q2p += x * x;
  }
  double alx = 0.0;  // max |alpha| over the probed regions
  double aln = 0.0;  // min alpha
  double nng = 0.0;  // max -norm term over the probed regions' groups
  for (int p = tid; p < P; p += PA_THREADS) {
    const int r = greg[p];
    const double al = ix.grouping ? (double)ix.alphas[r] : 0.0;
    alx = fmax(alx, fabs(al));
    aln = fmin(aln, al);
    if (ix.rneg) nng = fmax(nng, (double)ix.rneg[r]);
    if (pst) {
      preg[p] = r;
      pqc[p] = gqc[p];
      pal[p] = al;
    }
  }
  __syncthreads();
  auto REG = [&](int p) -> int { return pst ? preg[p] : greg[p]; };
  auto QC = [&](int p) -> double { return pst ? pqc[p] : gqc[p]; };
  auto AL = [&](int p) -> double {
    return pst ? pal[p] : (ix.grouping ? (double)ix.alphas[greg[p]] : 0.0);
  };
  // f / G by multiply-high (exact for f < 2^32 / G; staged f < PA_ITEMS)
  const uint32_t ginv = G > 1 ? (uint32_t)(0xffffffffu / (uint32_t)G) + 1u : 0u;
  auto DIVG = [&](int64_t f) -> int {
    if (G == 1) return (int)f;
    return staged ? (int)__umulhi((uint32_t)f, ginv) : (int)(f / G);
  };
  auto GI = [&](int64_t f) -> int64_t {
    const int p = DIVG(f);
    return (int64_t)REG(p) * G + (f - (int64_t)p * G);
  };
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  if (staged) {
    // all of a thread's loads in flight at once (total <= PA_ITEMS)
    constexpr int PT = PA_ITEMS / PA_THREADS;
    uint32_t kk[PT];
    int32_t zz[PT];
#pragma unroll
    for (int t = 0; t < PT; ++t) {
      const int f = tid + t * PA_THREADS;
      const int p = f < total ? DIVG(f) : 0;
      kk[t] = f < total ? gkey[f] : 0u;
      zz[t] = f < total ? __ldg(ix.gsize + (int64_t)REG(p) * G + (f - p * G)) : 0;
    }
#pragma unroll
    for (int t = 0; t < PT; ++t) {
      const int f = tid + t * PA_THREADS;
      if (f < total) {
        skey[f] = kk[t];
        if (small) ssz16[f] = (uint16_t)zz[t];
        else ssz[f] = zz[t];
        kmin = min(kmin, kk[t]);
        kmax = max(kmax, kk[t]);
      }
    }
  } else {
    for (int64_t f = tid; f < total; f += PA_THREADS) {
      const uint32_t k = gkey[f];
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    }
  }
  PLAN_PHASE(8);
  // the six block reductions in one exchange (one barrier instead of 18);
  // the sum keeps block_sum's order (warp xor tree, then warps in order)
  double q2;
  {
    constexpr int NW = PA_THREADS / 32;
    __shared__ double s_rd[4][NW];
    __shared__ uint32_t s_rk[2][NW];
    const double wq = warp_sum(q2p), wa = warp_max(alx), wn = warp_max(-aln), wg = warp_max(nng);
    const uint32_t w0 = warp_min(kmin), w1 = warp_max(kmax);
    const int lane_ = tid & 31, wid_ = tid >> 5;
    if (lane_ == 0) {
      s_rd[0][wid_] = wq; s_rd[1][wid_] = wa; s_rd[2][wid_] = wn; s_rd[3][wid_] = wg;
      s_rk[0][wid_] = w0; s_rk[1][wid_] = w1;
    }
    __syncthreads();
    q2 = s_rd[0][0];
    double ra = s_rd[1][0], rn = s_rd[2][0], rg = s_rd[3][0];
    uint32_t k0 = s_rk[0][0], k1 = s_rk[1][0];
#pragma unroll
    for (int i = 1; i < NW; ++i) {
      q2 += s_rd[0][i];
      ra = fmax(ra, s_rd[1][i]);
      rn = fmax(rn, s_rd[2][i]);
      rg = fmax(rg, s_rd[3][i]);
      k0 = min(k0, s_rk[0][i]);
      k1 = max(k1, s_rk[1][i]);
    }
    alx = ra;
    aln = -rn;
    nng = rg;
    kmin = k0;
    kmax = k1;
  }
  auto KEY = [&](int64_t f) -> uint32_t { return staged ? skey[f] : gkey[f]; };
  auto SIZE = [&](int64_t f) -> int64_t {
    return staged ? (small ? (int64_t)ssz16[f] : (int64_t)ssz[f]) : (int64_t)ix.gsize[GI(f)];
  };
  const double qn = sqrt(q2);
  const double amax = fmax(fabs((double)key_f32(kmin)), fabs((double)key_f32(kmax)));
  const double cq = (double)a.cmax + qn;
  // Only qs2 is approximate and it enters the score times alpha.  Loose bound
  // (any alpha): alpha_max x (GEMM bound + fp16 storage of the neighbor
  // scores, kHalfRel of at most (|q| + cmax)^2), + the float32 key rounding +
  // slack.  The tight bound (E_tight below, once v* is known) uses that the
  // fp16 error is relative to the stored distance itself.
  const double eps_g = (double)a.eps_scale * ((double)a.cmax * a.cmax + 2.0 * qn * a.cmax);
  const double E_loose = ix.grouping
      ? 1.0001 * alx * (eps_g + 1.001 * (double)a.half_rel * cq * cq) + amax * 1.2e-7 + 1e-12 * cq * cq
      : amax * 1.2e-7;  // float32 key rounding only
  PLAN_PHASE(0);

  // ---- 1. approximate crossing: bucket refinement on the float32 keys
  uint64_t taken_c = 0, taken_w = 0;
  uint32_t lo = kmin, hi = kmax, bucket_lo = 0, bucket_hi = 0;
  bool no_cut = false, flag = false;
  int why = 0;  // fallback reason (counters[2 + why])
  for (int level = 0; level < 4; ++level) {
    const uint32_t range = hi - lo;
    const int shift = range == 0 ? 0 : max(0, 32 - __clz(range) - 10);  // <= 1024 buckets
    const uint32_t nb = (range >> shift) + 1;
    for (uint32_t i = tid; i < nb; i += PA_THREADS) { hcn[i] = 0; hwt[i] = 0; }
    __syncthreads();
    for (int64_t f = tid; f < total; f += PA_THREADS) {
      const uint32_t k = KEY(f);
      if (k < lo || k > hi) continue;
      const uint32_t bk = (k - lo) >> shift;
      atomicAdd(&hcn[bk], 1u);
      atomicAdd(&hwt[bk], (uint32_t)SIZE(f));
    }
    __syncthreads();
    constexpr uint32_t PER = PA_BUCKETS / PA_THREADS;
    const uint32_t b0 = tid * PER, b1 = min(nb, b0 + PER);
    unsigned long long rs = 0;
    for (uint32_t x = b0; x < b1; ++x) rs += HW(x);
    unsigned long long tot;
    const unsigned long long ps = block_exclusive_scan(rs, red64, &tot);
    if (tid == 0) s_b = -1;
    __syncthreads();
    {
      const uint64_t c0 = taken_c + (ps >> CW), w0 = taken_w + (ps & WMASK);
      const uint64_t c1 = c0 + (rs >> CW), w1 = w0 + (rs & WMASK);
      if (b0 < b1 && c0 < kept && w0 < budget && (c1 >= kept || w1 >= budget)) {
        unsigned long long acc = ps;
        for (uint32_t x = b0; x < b1; ++x) {
          const unsigned long long nx = acc + HW(x);
          if (taken_c + (nx >> CW) >= kept || taken_w + (nx & WMASK) >= budget) {
            s_b = (int)x;
            s_before = acc;
            break;
          }
          acc = nx;
        }
      }
    }
    __syncthreads();
    const int bsel = s_b;
    if (bsel < 0) {  // never crosses: every group is scanned whole
      no_cut = true;
      break;
    }
    const uint32_t cnt_b = hcn[bsel];
    const uint32_t bl = lo + ((uint32_t)bsel << shift);
    const uint64_t bspan = (uint64_t)bl + ((1ull << shift) - 1);
    const uint32_t bh = (uint32_t)(bspan < hi ? bspan : hi);
    taken_c += s_before >> CW;
    taken_w += s_before & WMASK;
    __syncthreads();
    if (cnt_b <= (uint32_t)PA_SMALL || (shift == 0 && cnt_b <= (uint32_t)PA_SORT)) {
      bucket_lo = bl;
      bucket_hi = bh;
      break;
    }
    if (shift == 0 || level == 3) {  // > PA_SORT equal approximate keys: exact planner
      flag = true;
      why = 0;
      break;
    }
    lo = bl;
    hi = bh;
  }
  PLAN_PHASE(2);

  double vstar = __longlong_as_double(0x7ff0000000000000ll);  // +inf: no cut
  if (!no_cut && !flag) {
    if (tid == 0) { s_nbk = 0; s_lastb = -1; }
    __syncthreads();
    for (int64_t f = tid; f < total; f += PA_THREADS) {
      const uint32_t k = KEY(f);
      if (k >= bucket_lo && k <= bucket_hi) bkey[atomicAdd(&s_nbk, 1u)] = ((uint64_t)k << 32) | (uint32_t)f;
    }
    __syncthreads();
    const uint32_t nbk = s_nbk;
    const uint32_t np2 = next_pow2(max(nbk, 1u));
    for (uint32_t i = nbk + tid; i < np2; i += PA_THREADS) bkey[i] = kKeyPad;
    __syncthreads();
    bitonic_sort_keys(bkey, np2);
    unsigned long long carry = taken_w;
    for (uint32_t t0 = 0; t0 < nbk; t0 += PA_THREADS) {
      const uint32_t i = t0 + tid;
      const unsigned long long sz = i < nbk ? (unsigned long long)SIZE((uint32_t)bkey[i]) : 0ull;
      unsigned long long tile;
      const unsigned long long excl = block_exclusive_scan(sz, red64, &tile);
      if (i < nbk && taken_c + i < kept && carry + excl < budget) atomicMax(&s_lastb, (int)i);
      carry += tile;
    }
    __syncthreads();
    vstar = (double)key_f32((uint32_t)(bkey[max(s_lastb, 0)] >> 32));
  }
  PLAN_PHASE(3);

  // Tight bound for alpha in [0, 1]: item i's error is at most
  //   alpha_i (eps_g + r |qs2~_i| + 2^-24 dscale (fp16 subnormal step,
  //   dscale < 2^-14 (|q| + cmax)^2))
  //   + float32 key rounding,  r = kHalfRel / (1 - kHalfRel),
  // and alpha_i qs2~_i = s_i - (1 - alpha_i) qc_i - norm_i <= s_i + nng.
  // e(s) = Eabs + r' max(0, s + nng) is increasing and s - e(s) too, so for
  // every item with key <= v* + 3E the error is <= e(v* + 3E) = E, and every
  // item above lies above v* + 2E exactly: the certification below holds.
  double E = E_loose;
  if (ix.grouping && ix.rneg && aln >= 0.0 && alx <= 1.0 && !no_cut) {
    const double rr = 1.001 * (double)a.half_rel;
    const double Eabs = 1.001 * alx * eps_g + alx * 4e-12 * cq * cq +
                        amax * 1.2e-7 * (1.0 + rr) + 1e-12 * cq * cq;
    const double Et = (Eabs + rr * fmax(0.0, vstar + amax * 1.2e-7 + nng)) / (1.0 - 3.0 * rr);
    E = fmin(E, Et);
  }

  // ---- 2./3. window around v*: exact scores, sorted, walked from A's prefix
  const double wlo = vstar - 3.0 * E, whi = vstar + 3.0 * E;
  if (tid == 0) s_nw = 0;
  __syncthreads();
  int my_a = 0;  // A items of this thread (for the compaction below)
  unsigned long long nA, wA;
  // the same tests on the float32 keys: f < wlo <=> f < ru(wlo) and
  // f <= whi <=> f <= rd(whi) for floats f, and f32_key is monotone
  const uint32_t klo = f32_key(__double2float_ru(wlo));
  const uint32_t khi = f32_key(__double2float_rd(whi));
  {
    unsigned long long cw = 0;
    for (int64_t f = tid; f < total; f += PA_THREADS) {
      const uint32_t kf = KEY(f);
      if (kf < klo) {
        ++my_a;
        cw += (1ull << CW) | (unsigned long long)SIZE(f);
      } else if (kf <= khi && !no_cut) {
        const uint32_t p = atomicAdd(&s_nw, 1u);
        if (p < (uint32_t)L.wcap) wval[p] = (uint32_t)f;
      }
    }
    cw = block_sum(cw, red64);
    nA = cw >> CW;
    wA = cw & WMASK;
  }
  const uint32_t nw = s_nw;
  if (nw > (uint32_t)L.wcap && !flag) { flag = true; why = 1; }
  int lastw = -1;
  unsigned long long wsum = 0;  // lengths of the begun window groups
  if (!flag && !no_cut) {
    // one metadata gather per window group, then the centroid rows
    PLAN_PHASE(1);
    for (int i = tid; i < (int)nw; i += PA_THREADS) {
      const int64_t gi = GI(wval[i]);
      wrow[i] = ix.grouping ? ix.nbr[gi] : 0;
      wnorm[i] = ix.grouping ? ix.norm[gi] : 0.f;
    }
    __syncthreads();
    PLAN_PHASE(10);
    const int grp = tid >> 3, gl = tid & 7;
    constexpr int NG = PA_THREADS >> 3;
    // rows in flight per group: no more than the window needs
    const int uw = nw <= (uint32_t)NG ? 1 : (nw <= 2u * NG ? 2 : PA_U);
    for (uint32_t i0 = 0; i0 < nw; i0 += NG * uw) {
      const float* rows[PA_U];
#pragma unroll
      for (int u = 0; u < PA_U; ++u) {
        const uint32_t i = i0 + u * NG + grp;
        rows[u] = ix.centroids + (int64_t)(u < uw && i < nw ? wrow[i] : 0) * d;
      }
      double qs2[PA_U];
      if (ix.grouping) {
        if ((d & 3) == 0 && d <= 128) {
          if (uw == 1) group8_sqdist64_multi<1>(rows, qd, d >> 2, qs2);
          else if (uw == 2) group8_sqdist64_multi<2>(rows, qd, d >> 2, qs2);
          else group8_sqdist64_multi<PA_U>(rows, qd, d >> 2, qs2);
        } else {
#pragma unroll
          for (int u = 0; u < PA_U; ++u)
            if (u < uw) qs2[u] = group8_sqdist64(rows[u], qd, d);
        }
      }
      if (gl == 0) {
#pragma unroll
        for (int u = 0; u < PA_U; ++u) {
          const uint32_t i = i0 + u * NG + grp;
          if (u >= uw || i >= nw) continue;
          const int p = (int)(wval[i] / G);
          double score = QC(p);
          if (ix.grouping) {
            const double al = AL(p);
            score = dadd(dadd(dmul(dsub(1.0, al), QC(p)), dmul(al, qs2[u])), (double)wnorm[i]);
          }
          wkey[i] = f64_key(score);
        }
      }
    }
    const uint32_t np2 = next_pow2(max(nw, 1u));
    for (uint32_t i = nw + tid; i < np2; i += PA_THREADS) { wkey[i] = kKeyPad; wval[i] = 0xffffffffu; }
    __syncthreads();
    PLAN_PHASE(7);
    bitonic_sort(wkey, wval, np2);  // (score, flat): the reference order
    PLAN_PHASE(11);
    if (tid == 0) s_lastb = -1;
    __syncthreads();
    unsigned long long carry = wA, mine = 0;
    for (uint32_t t0 = 0; t0 < nw; t0 += PA_THREADS) {
      const uint32_t i = t0 + tid;
      const unsigned long long sz = i < nw ? (unsigned long long)SIZE(wval[i]) : 0ull;
      unsigned long long tile;
      const unsigned long long excl = block_exclusive_scan(sz, red64, &tile);
      if (i < nw) {
        const unsigned long long w = carry + excl;
        const bool ok = (nA + i < kept) && (w < budget);
        wlen[i] = ok ? (int32_t)min(sz, budget - w) : 0;
        if (ok) {
          atomicMax(&s_lastb, (int)i);
          mine += (unsigned long long)wlen[i];
        }
      }
      carry += tile;
    }
    wsum = block_sum(mine, red64);
    const int xc = s_lastb;
    if (xc < 0) {
      flag = true;  // the exact crossing precedes the window
      why = 2;
    } else {
      lastw = xc;
      const double sx = key_to_f64(wkey[xc]);
      if (!(sx >= vstar - 2.0 * E && sx <= vstar + 2.0 * E)) { flag = true; why = 3; }
      const bool ended = ((uint32_t)xc + 1 < nw) || (nA + nw >= kept) || (carry >= budget);
      if (!ended) { flag = true; why = 4; }
    }
  }
  const uint64_t nbegun = nA + (uint64_t)(lastw + 1);
  // more begun groups than the candidate arrays hold: the deferred variant
  // streams them (below); the inline rescore needs them staged
  const bool big = nbegun > (uint64_t)PA_CAND;
  if (big && INLINE && !flag) { flag = true; why = 5; }
  PLAN_PHASE(4);
#ifdef GIVF_PHASES
  if (tid == 0 && ix.counters) {  // sizes: window items, begun groups
    atomicAdd(&ix.counters[24], (unsigned long long)nw);
    atomicAdd(&ix.counters[25], (unsigned long long)nbegun);
  }
#endif
  if (flag) {
    if (tid == 0) {
      if (why == 1 && !a.retry && a.n_overflow) {
        // window overflow: a second pass with a larger window (only = 2)
        a.only[b] = 2;
        atomicAdd(a.n_overflow, 1);
        if (ix.counters) atomicAdd(&ix.counters[9], 1ull);
      } else {
        a.only[b] = 1;
        if (ix.counters) {
          atomicAdd(&ix.counters[1], 1ull);
          atomicAdd(&ix.counters[2 + why], 1ull);
        }
      }
    }
    return;
  }
  if (tid == 0) a.only[b] = 0;

  // ---- 5. emission: one metadata gather per begun group; positions by block
  // scan (groups with no local rows are dropped)
  WorkItem* Wl = a.work + (int64_t)b * a.cap_w;
  int nemit = 0;
  auto emit_round = [&](bool valid, uint32_t f, int64_t len_g) {  // block-uniform call
    int64_t ll = 0, start = 0;
    int32_t row = 0;
    float nrm = 0.f;
    if (valid) {  // independent loads, issued together
      const int64_t gi = GI(f);
      // global_items (query-sharded planning): the whole group,
      // identified by its global index, for every shard to localize
      const int64_t lo_ = (ix.llo && !a.global_items) ? ix.llo[gi] : 0;
      const int64_t cnt_ = a.global_items ? len_g : (ix.lsize ? ix.lsize[gi] : ix.gsize[gi]);
      start = a.global_items ? gi : ix.lstart[gi];
      if (ix.grouping) {
        row = ix.nbr[gi];
        nrm = ix.norm[gi];
      }
      ll = min(max(len_g - lo_, (int64_t)0), cnt_);
    }
    uint32_t tot;
    const uint32_t pos = nemit + block_exclusive_scan((uint32_t)(ll > 0), red32, &tot);
    if (ll > 0) {
      WorkItem w;
      w.start = start;
      w.len = (int32_t)ll;
      w.flat = (int32_t)f;
      // deferred rescoring (k_plan_rescore): stash (row, p) and (norm, alpha)
      const int p = (int)(f / G);
      w.base = __hiloint2double(p, row);
      w.score = __hiloint2double(__float_as_int((float)AL(p)), __float_as_int(nrm));
      Wl[pos] = w;
      if (!big) {  // in place: slot pos <= candidate index
        cf[pos] = (uint32_t)row;
        cl[pos] = __float_as_int(nrm);
        cp[pos] = p;
      }
    }
    nemit += (int)tot;
  };
  if (!big) {
    // A (compacted in thread order) then W[0..lastw] into the candidate arrays
    {
      uint32_t tot;
      uint32_t pos = block_exclusive_scan((uint32_t)my_a, red32, &tot);
      for (int64_t f = tid; f < total; f += PA_THREADS) {
        if (KEY(f) < klo) {
          cf[pos] = (uint32_t)f;
          cl[pos] = (int32_t)SIZE(f);
          ++pos;
        }
      }
      for (int i = tid; i <= lastw; i += PA_THREADS) {
        cf[nA + i] = wval[i];
        cl[nA + i] = wlen[i];
      }
    }
    __syncthreads();
    PLAN_PHASE(12);
    const int nc = (int)nbegun;
    for (int c0 = 0; c0 < nc; c0 += PA_THREADS) {
      const int c = c0 + tid;
      const bool v = c < nc;
      emit_round(v, v ? cf[c] : 0u, v ? cl[c] : 0);
    }
  } else {
    for (int64_t f0 = 0; f0 < total; f0 += PA_THREADS) {
      const int64_t f = f0 + tid;
      const bool isA = f < total && KEY(f) < klo;
      emit_round(isA, (uint32_t)f, isA ? SIZE(f) : 0);
    }
    for (int i0 = 0; i0 <= lastw; i0 += PA_THREADS) {
      const int i = i0 + tid;
      const bool v = i <= lastw;
      emit_round(v, v ? wval[i] : 0u, v ? wlen[i] : 0);
    }
  }
  __syncthreads();
  PLAN_PHASE(5);
  // exact float64 base / score of the emitted groups (here only when the
  // scan order needs them in this CTA; else k_plan_rescore)
  if (INLINE) {
    const int grp = tid >> 3, gl = tid & 7;
    constexpr int NG = PA_THREADS >> 3;
    const bool vec = (d & 3) == 0 && d <= 128;
    for (int i0 = 0; i0 < nemit; i0 += NG * PA_U) {
      const float* rows[PA_U];
#pragma unroll
      for (int u = 0; u < PA_U; ++u) {
        const int i = i0 + u * NG + grp;
        rows[u] = ix.centroids + (int64_t)(i < nemit ? (int)cf[i] : 0) * d;
      }
      double qs2[PA_U];
      if (ix.grouping) {
        if (vec) {
          group8_sqdist64_multi<PA_U>(rows, qd, d >> 2, qs2);
        } else {
#pragma unroll
          for (int u = 0; u < PA_U; ++u) qs2[u] = group8_sqdist64(rows[u], qd, d);
        }
      }
      if (gl == 0) {
#pragma unroll
        for (int u = 0; u < PA_U; ++u) {
          const int i = i0 + u * NG + grp;
          if (i >= nemit) continue;
          const int p = cp[i];
          double base = QC(p), score = QC(p);
          if (ix.grouping) {
            const double al = AL(p);
            base = dadd(dmul(dsub(1.0, al), QC(p)), dmul(al, qs2[u]));
            score = dadd(base, (double)__int_as_float(cl[i]));
          }
          Wl[i].base = base;
          Wl[i].score = score;
        }
      }
    }
  }
  PLAN_PHASE(6);
  if (tid == 0) {
    a.nwork[b] = nemit;
    int64_t* st = a.stats + (int64_t)b * 4;
    st[0] = P;
    st[1] = (int64_t)nbegun;
    st[2] = total - (int64_t)kept;
    st[3] = (int64_t)(wA + wsum);
  }
  if (INLINE && a.sort_work) {
    __syncthreads();
    const uint32_t wp2 = next_pow2(max(nemit, 1));
    int64_t cp2 = 1;
    while (cp2 < a.cap_w) cp2 <<= 1;
    uint64_t* sk = a.skey + (int64_t)b * cp2;
    uint32_t* sv = a.sval + (int64_t)b * cp2;
    for (uint32_t i = tid; i < wp2; i += PA_THREADS) {
      sk[i] = (int)i < nemit ? f64_key(Wl[i].score) : kKeyPad;
      sv[i] = (int)i < nemit ? (uint32_t)Wl[i].flat : 0xffffffffu;
    }
    __syncthreads();
    bitonic_sort(sk, sv, wp2);
    for (int i = tid; i < nemit; i += PA_THREADS) {
      const uint64_t key = f64_key(Wl[i].score);
      const uint32_t fl = (uint32_t)Wl[i].flat;
      int lo_i = 0, hi_i = nemit - 1;
      while (lo_i < hi_i) {
        const int mid = (lo_i + hi_i) >> 1;
        const bool less = sk[mid] < key || (sk[mid] == key && sv[mid] < fl);
        if (less) lo_i = mid + 1; else hi_i = mid;
      }
      a.order[(int64_t)b * a.cap_w + lo_i] = i;
    }
  }
}

// ---------------------------------------------------------------- K4b
// Exact float64 base / score of the work items k_plan_approx emitted, many
// queries' items in flight per SM (one CTA per (query, slice of its items)).
constexpr int RS_THREADS = 128;
constexpr int RS_SPLIT = 2;
constexpr int RS_U = 2;  // centroid rows in flight per 8-lane group (64 registers: 8 CTAs/SM)

__global__ void __launch_bounds__(RS_THREADS, 6) k_plan_rescore(PlanArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  double* qd = reinterpret_cast<double*>(dsm);
  const IndexView& ix = a.ix;
  const int b = blockIdx.x, tid = threadIdx.x;
  constexpr int NG = RS_THREADS >> 3, PER = NG * RS_U;
  if (a.only[b] != 0) return;  // the exact planner owns this query
  const int n = a.nwork[b];
  if ((int)blockIdx.y * PER >= n) return;
  const int d = ix.d;
  for (int j = tid; j < d; j += RS_THREADS) qd[j] = (double)a.Q[(int64_t)b * d + j];
  __syncthreads();
  WorkItem* Wl = a.work + (int64_t)b * a.cap_w;
  const double* qc2 = a.qc2 + (int64_t)b * a.P;
  const int grp = tid >> 3, gl = tid & 7;
  const bool vec = (d & 3) == 0 && d <= 128;
  for (int i0 = blockIdx.y * PER; i0 < n; i0 += gridDim.y * PER) {
    const float* rows[RS_U];
    double sb[RS_U], ss[RS_U];
#pragma unroll
    for (int u = 0; u < RS_U; ++u) {
      const int i = i0 + u * NG + grp;
      sb[u] = i < n ? Wl[i].base : 0.0;
      ss[u] = i < n ? Wl[i].score : 0.0;
      rows[u] = ix.centroids + (int64_t)__double2loint(sb[u]) * d;
    }
    double qs2[RS_U];
    if (vec) {
      group8_sqdist64_multi<RS_U>(rows, qd, d >> 2, qs2);
    } else {
#pragma unroll
      for (int u = 0; u < RS_U; ++u) qs2[u] = group8_sqdist64(rows[u], qd, d);
    }
    if (gl == 0) {
#pragma unroll
      for (int u = 0; u < RS_U; ++u) {
        const int i = i0 + u * NG + grp;
        if (i >= n) continue;
        const int p = __double2hiint(sb[u]);
        const double al = (double)__int_as_float(__double2hiint(ss[u]));
        const double nrm = (double)__int_as_float(__double2loint(ss[u]));
        const double base = dadd(dmul(dsub(1.0, al), qc2[p]), dmul(al, qs2[u]));
        Wl[i].base = base;
        Wl[i].score = dadd(base, nrm);
      }
    }
  }
}

int launch_plan_approx(const PlanArgs& a0, cudaStream_t s) {
  PlanArgs a = a0;
  // the scan-order sort (rerank=False) needs the scores inside k_plan_approx
  a.defer_rescore = (a.ix.grouping && !a.sort_work) ? 1 : 0;
  static const int wcap_env = getenv("GIVF_PLAN_WCAP") ? atoi(getenv("GIVF_PLAN_WCAP")) : 0;
  a.wcap_override = wcap_env > 0 ? std::min(wcap_env, PA_WCAP_RETRY) : 0;
  a.retry = 0;
  // GIVF_PLAN_RETRY=0 (read per call; tests use it) sends overflowed
  // windows straight to the exact planner
  const char* re = getenv("GIVF_PLAN_RETRY");
  if (re && atoi(re) == 0) a.n_overflow = nullptr;
  const PaSmem L(a.ix.d, a.P, (int64_t)a.P * a.ix.G, a.ix.max_gsize < 65536, a.wcap_override);
  auto kern = a.defer_rescore ? k_plan_approx<false> : k_plan_approx<true>;
  ensure_max_smem((const void*)kern, L.bytes);
  if (a.n_overflow) cudaMemsetAsync(a.n_overflow, 0, sizeof(int), s);
  kern<<<a.nq, PA_THREADS, L.bytes, s>>>(a);
  int n = 1;
  if (a.n_overflow) {
    // queries whose certified window overflowed: one more pass with a
    // 2048-entry window before the exact planner takes what is left
    int nov = 0;
    cudaMemcpyAsync(&nov, a.n_overflow, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (nov > 0) {
      PlanArgs r = a;
      r.retry = 1;
      r.wcap_override = PA_WCAP_RETRY;
      const PaSmem LR(r.ix.d, r.P, (int64_t)r.P * r.ix.G, r.ix.max_gsize < 65536, PA_WCAP_RETRY);
      ensure_max_smem((const void*)kern, LR.bytes);
      kern<<<r.nq, PA_THREADS, LR.bytes, s>>>(r);
      ++n;
    }
  }
  if (!a.defer_rescore) return n;
  static const int split = [] {  // CTAs per query (GIVF_RS_SPLIT)
    const char* e = getenv("GIVF_RS_SPLIT");
    return e ? std::max(1, std::min(64, atoi(e))) : RS_SPLIT;
  }();
  k_plan_rescore<<<dim3(a.nq, split), RS_THREADS, (size_t)a.ix.d * 8, s>>>(a);
  return n + 1;
}

// (K, G) rows of c16r gathered into the per-region chunk-major layout
__global__ void __launch_bounds__(256) k_pack_neighbor_rows(const uint4* __restrict__ c16r,
                                                            const float* __restrict__ c2f,
                                                            const int32_t* __restrict__ nbr, int64_t total,
                                                            int G, int dp8, uint4* __restrict__ out,
                                                            float* __restrict__ c2p) {
  // one thread per (region, chunk, neighbour): out index == thread index
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int j = (int)(i % G);
  const int64_t rc = i / G;
  const int c = (int)(rc % dp8);
  const int64_t r = rc / dp8;
  const int n = __ldg(nbr + r * G + j);
  out[i] = __ldg(c16r + (int64_t)n * dp8 + c);
  if (c == 0) c2p[r * G + j] = __ldg(c2f + n);
}

void launch_pack_neighbor_rows(const void* c16r, const float* c2f, const int32_t* nbr, int K, int G,
                               int d, void* c16p, float* c2p, cudaStream_t s) {
  const int dp8 = f16_row_pitch(d) / 8;
  const int64_t total = (int64_t)K * dp8 * G;
  k_pack_neighbor_rows<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(c16r), c2f, nbr, total, G, dp8, reinterpret_cast<uint4*>(c16p), c2p);
}

int launch_plan_scores(const PlanArgs& a, cudaStream_t s) {
  const int64_t warps = (int64_t)a.nq * a.P;
  const int per = PA_THREADS / 32;
  const unsigned grid = (unsigned)((warps + per - 1) / per);
  if (a.direct) {
    switch ((a.ix.d + 31) / 32) {  // 32-coordinate chunks of a row
      case 1: a.ix.c16p ? k_plan_scores_direct<4, true><<<grid, PA_THREADS, 0, s>>>(a)
                        : k_plan_scores_direct<4, false><<<grid, PA_THREADS, 0, s>>>(a); break;
      case 2: a.ix.c16p ? k_plan_scores_direct<8, true><<<grid, PA_THREADS, 0, s>>>(a)
                        : k_plan_scores_direct<8, false><<<grid, PA_THREADS, 0, s>>>(a); break;
      case 3: a.ix.c16p ? k_plan_scores_direct<12, true><<<grid, PA_THREADS, 0, s>>>(a)
                        : k_plan_scores_direct<12, false><<<grid, PA_THREADS, 0, s>>>(a); break;
      default: a.ix.c16p ? k_plan_scores_direct<16, true><<<grid, PA_THREADS, 0, s>>>(a)
                         : k_plan_scores_direct<16, false><<<grid, PA_THREADS, 0, s>>>(a); break;
    }
    return 1;
  }
  k_plan_scores_approx<<<grid, PA_THREADS, 0, s>>>(a);
  return 1;
}

}  // namespace givf
