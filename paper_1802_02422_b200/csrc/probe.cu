// K1 + K2: region probe (reference: search.py:77-90, graph.py:357-383).
//
// The reference ranks regions by exact float64 squared distance (its
// ef_search == K configuration).  Computing all K*d
// differences in float64 is wasteful, so the probe runs in three steps:
//
//   K1a  probe_gemm    approximate f32 scores  s~ = |c|^2 - 2 q.c  (B x K)
//   K1b  probe_select  per query, a candidate set S = {k : s~_k < theta}
//                      with Tmin <= |S| <= CAP (bucketed radix refinement)
//   K2   probe_recheck exact float64 difference-form distances on S, the
//                      exact top-P by (d64, id), an a-priori error bound check
//                      that nothing outside S can enter the top-P, and the
//                      reference's output order (f32(d64), id) + qc2 = d64.
//
// Queries whose bound check fails (near-ties at the S boundary) and the
// nprobe == K branch go through probe_full, which ranks all K regions
// exactly.  The result is bit-identical to the oracle's probe_exact by
// construction, whatever the approximation error of K1a.
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace givf {

// ----------------------------------------------------------------- scale
// Per query: |q|^2 (f32) and the power-of-two fp16 encoding scale of its
// scores (ScoreOut in kernels.h): 2^e >= (|q| + cmax)^2 / 2^15.
__global__ void k_query_scale(const float* __restrict__ Q, int nq, int d, float cmax,
                              float* __restrict__ q2o, float* __restrict__ qinv,
                              float* __restrict__ qscale) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nq) return;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) s += (double)Q[(int64_t)b * d + j] * Q[(int64_t)b * d + j];
  s = warp_sum(s);
  if (lane == 0) {
    const double m = (sqrt(s) + (double)cmax) * (sqrt(s) + (double)cmax);
    const int e = (m > 0.0 ? ilogb(m) + 1 : 0) - 15;
    q2o[b] = (float)s;
    qinv[b] = ldexpf(1.f, -e);
    qscale[b] = ldexpf(1.f, e);
  }
}

GIVF_DEV float dec_score(uint16_t h, float scale, float q2) {
  return fmaf(__half2float(__ushort_as_half(h)), scale, -q2);
}
// Order-preserving 16-bit key of an fp16 code (-0 folded onto +0): the
// select works on codes directly, decoding only its outputs.
GIVF_DEV uint32_t key16(uint32_t h) {
  h = (h == 0x8000u) ? 0u : h;
  return (h & 0x8000u) ? (~h & 0xffffu) : (h | 0x8000u);
}
GIVF_DEV uint16_t key16_inv(uint32_t k) {
  return (uint16_t)((k & 0x8000u) ? (k & 0x7fffu) : (~k & 0xffffu));
}

// ----------------------------------------------------------------- K1a
// SIMT fp32 tile GEMM: 64 queries x 128 centroids per CTA, 256 threads,
// 4x8 outputs per thread, d in chunks of 16 through shared memory.
constexpr int PG_BM = 64, PG_BN = 128, PG_BK = 16;

template <bool HALF>
__global__ void __launch_bounds__(256)
k_probe_gemm(const float* __restrict__ Q, const float* __restrict__ C,
             const float* __restrict__ c2, int nq, int K, int d, ScoreOut o,
             float* __restrict__ tmin) {
  __shared__ float As[PG_BK][PG_BM + 4];
  __shared__ float Bs[PG_BK][PG_BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int q0 = blockIdx.y * PG_BM, c0 = blockIdx.x * PG_BN;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < d; k0 += PG_BK) {
    // Q tile: 64 x 16 -> 4 per thread; C tile: 128 x 16 -> 8 per thread.
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      int e = tid + t * 256;
      int r = e >> 4, kk = e & 15;
      int qr = q0 + r, dk = k0 + kk;
      As[kk][r] = (qr < nq && dk < d) ? Q[(int64_t)qr * d + dk] : 0.f;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      int e = tid + t * 256;
      int r = e >> 4, kk = e & 15;
      int cr = c0 + r, dk = k0 + kk;
      Bs[kk][r] = (cr < K && dk < d) ? C[(int64_t)cr * d + dk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < PG_BK; ++kk) {
      float a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx * 8 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  // epilogue: scores + the per-(query, 128-centroid tile) minimum that lets
  // k_probe_select bound the T-th smallest score without a histogram pass
  const int ntiles = (K + PG_BN - 1) / PG_BN;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int qr = q0 + ty * 4 + i;
    float q2r = 0.f, ir = 1.f;
    if (HALF && qr < nq) { q2r = o.q2[qr]; ir = o.qinv[qr]; }
    float mn = __int_as_float(0x7f800000);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int cr = c0 + tx * 8 + j;
      if (cr < K) {
        float v = fmaf(-2.f, acc[i][j], c2[cr]);
        if constexpr (HALF) {
          const __half h = __float2half_rn((v + q2r) * ir);
          mn = fminf(mn, __half2float(h));
          if (qr < nq) o.D16[(int64_t)qr * o.ld + cr] = __half_as_ushort(h);
        } else {
          mn = fminf(mn, v);
          if (qr < nq) o.D32[(int64_t)qr * o.ld + cr] = v;
        }
      }
    }
    // 16 threads (tx) share a row: reduce within each half-warp
#pragma unroll
    for (int w = 8; w > 0; w >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, w));
    if (tx == 0 && qr < nq && tmin) {
      if (HALF)  // the tile minimum's fp16 code (mn is a widened fp16 value)
        reinterpret_cast<uint16_t*>(tmin)[(int64_t)qr * ntiles + blockIdx.x] =
            __half_as_ushort(__float2half_rn(mn));
      else
        tmin[(int64_t)qr * ntiles + blockIdx.x] = mn;
    }
  }
}

// ----------------------------------------------------------------- K1b
// Per query: candidate set S = {k : key(s~_k) < boundary}, Tmin <= |S| <= CAP,
// found by <= 3 levels of 2048-bucket histograms over the order-preserving
// u32 keys.  theta = smallest excluded score (+inf when nothing excluded).
constexpr int SEL_THREADS = 512;

// Decoded scores of one fp16 row (ScoreOut in kernels.h).
struct HalfRow {
  const uint16_t* __restrict__ r;
  float scale, q2;
  GIVF_DEV float operator()(int i) const { return dec_score(__ldg(r + i), scale, q2); }
};

// Generic path: bucketed refinement over the whole row (any K, any ties).
template <typename Row>
__device__ void select_bucketed(Row row, int K, int Tmin, int cap,
                                int* __restrict__ out, int* __restrict__ n_out,
                                float* __restrict__ theta_out, uint32_t* hist) {
  __shared__ uint32_t red[40];
  __shared__ uint32_t s_b, s_before, s_through;
  __shared__ uint32_t cnt_lt, cnt_eq;
  const int tid = threadIdx.x;
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int i = tid; i < K; i += blockDim.x) {
    uint32_t k = f32_key(row(i));
    mn = min(mn, k); mx = max(mx, k);
  }
  uint32_t lo = block_min(mn, red), hi = block_max(mx, red);
  uint32_t taken = 0, need = (uint32_t)Tmin;
  uint64_t boundary = (uint64_t)hi + 1;
  bool degenerate = false;
  uint32_t deg_key = 0, deg_before = 0;

  for (int level = 0; level < 4; ++level) {
    uint32_t range = hi - lo;
    int shift = range == 0 ? 0 : max(0, 32 - __clz(range) - 11);
    uint32_t nb = (range >> shift) + 1;
    for (uint32_t i = tid; i < nb; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < K; i += blockDim.x) {
      uint32_t k = f32_key(row(i));
      if (k >= lo && k <= hi) atomicAdd(&hist[(k - lo) >> shift], 1u);
    }
    __syncthreads();
    // each thread owns a contiguous run of buckets; scan run totals
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    uint32_t b0 = tid * per, b1 = min(nb, b0 + per), run = 0;
    for (uint32_t b = b0; b < b1; ++b) run += hist[b];
    uint32_t tot;
    uint32_t pre = block_exclusive_scan(run, red, &tot);
    if (tid == 0) s_b = 0xffffffffu;
    __syncthreads();
    if (b0 < b1 && pre < need && pre + run >= need) {
      uint32_t c = pre;
      for (uint32_t b = b0; b < b1; ++b) {
        if (c + hist[b] >= need) { s_b = b; s_before = c; s_through = c + hist[b]; break; }
        c += hist[b];
      }
    }
    __syncthreads();
    uint32_t b = s_b, before = s_before, through = s_through;
    __syncthreads();
    if (taken + through <= (uint32_t)cap) {
      boundary = (uint64_t)lo + ((uint64_t)(b + 1) << shift);
      break;
    }
    if (shift == 0) {  // one key value holds more than cap elements
      degenerate = true;
      deg_key = lo + b;
      deg_before = taken + before;
      boundary = deg_key;
      break;
    }
    taken += before;
    need -= before;
    lo = lo + (b << shift);
    uint64_t nhi = (uint64_t)lo + ((1ull << shift) - 1);
    hi = (uint32_t)(nhi < (uint64_t)hi ? nhi : (uint64_t)hi);
  }

  if (tid == 0) { cnt_lt = 0; cnt_eq = 0; }
  __syncthreads();
  uint32_t ex = 0xffffffffu;
  for (int i = tid; i < K; i += blockDim.x) {
    uint32_t k = f32_key(row(i));
    if ((uint64_t)k < boundary) {
      out[atomicAdd(&cnt_lt, 1u)] = i;
    } else if (degenerate && k == deg_key) {
      uint32_t p = atomicAdd(&cnt_eq, 1u);
      if (deg_before + p < (uint32_t)cap) out[deg_before + p] = i;
      else ex = min(ex, k);
    } else {
      ex = min(ex, k);
    }
  }
  ex = block_min(ex, red);
  if (tid == 0) {
    uint32_t n = cnt_lt + (degenerate ? min(cnt_eq, (uint32_t)cap - deg_before) : 0u);
    *n_out = (int)n;
    *theta_out = ex == 0xffffffffu ? __int_as_float(0x7f800000) : key_f32(ex);
  }
}

// Fast path: the GEMM epilogue left the minimum of every 128-centroid tile.
// At least Tmin scores are <= the Tmin-th smallest tile minimum theta_up, so
// one pass collecting {s~ <= theta_up} yields a superset of the Tmin smallest;
// theta = the smallest score left out.  Falls back to select_bucketed when
// the collection overflows its buffer.
constexpr int SEL_COLLECT = 4096;

// theta_up for every query: the Tmin-th smallest of its tile minima (fp16
// codes), by a 16-step binary search on the key (one warp per query, no sort).
__global__ void k_tile_theta(const uint16_t* __restrict__ tmin, int nq, int ntiles, int Tmin,
                             uint32_t* __restrict__ up) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nq) return;
  const uint16_t* trow = tmin + (int64_t)b * ntiles;
  constexpr int R = 16;  // keys per lane in registers (ntiles <= 512)
  uint32_t kr[R];
  const bool inreg = ntiles <= 32 * R;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int i = lane + 32 * j;
    kr[j] = (inreg && i < ntiles) ? key16(trow[i]) : 0xffffffffu;
  }
  uint32_t lo = 0, hi = 0xffffu;
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    uint32_t c = 0;
    if (inreg) {
#pragma unroll
      for (int j = 0; j < R; ++j) c += kr[j] <= mid ? 1u : 0u;
    } else {
      for (int i = lane; i < ntiles; i += 32) c += key16(__ldg(trow + i)) <= mid ? 1u : 0u;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= (uint32_t)Tmin) hi = mid; else lo = mid + 1;
  }
  if (lane == 0) up[b] = lo;
}

__global__ void __launch_bounds__(SEL_THREADS)
k_probe_select(const uint16_t* __restrict__ D, int64_t ldD, const float* __restrict__ q2v,
               const float* __restrict__ qscale, int K, int Tmin, int cap,
               const void* __restrict__ tmin, int ntiles, const uint32_t* __restrict__ tup,
               int* __restrict__ cand, int* __restrict__ cand_n, float* __restrict__ theta) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ uint32_t red[40];
  __shared__ uint32_t s_cnt;
  const HalfRow row{D + (int64_t)blockIdx.x * ldD, qscale[blockIdx.x], q2v[blockIdx.x]};
  int* out = cand + (int64_t)blockIdx.x * cap;
  const int tid = threadIdx.x;

  if (K <= cap) {
    for (int i = tid; i < K; i += blockDim.x) out[i] = i;
    if (tid == 0) { cand_n[blockIdx.x] = K; theta[blockIdx.x] = __int_as_float(0x7f800000); }
    return;
  }
  uint32_t* hist = reinterpret_cast<uint32_t*>(dsm);  // 2048 buckets, aliases tk below
  if (tmin == nullptr || ntiles < Tmin) {
    select_bucketed(row, K, Tmin, cap, out, cand_n + blockIdx.x, theta + blockIdx.x, hist);
    return;
  }
  // 1. theta_up = Tmin-th smallest tile minimum (k_tile_theta)
  uint64_t* ck = reinterpret_cast<uint64_t*>(dsm + 8192 * 4);
  const uint32_t up = tup[blockIdx.x];
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  // 2. only tiles whose minimum key is <= up can hold a candidate: list them
  // (the others' minima bound the excluded codes), then read just those
  // tiles, collecting codes with key <= up (key16 order == decoded order)
  // and tracking the smallest key above.
  __shared__ uint32_t s_nt;
  uint16_t* tl = reinterpret_cast<uint16_t*>(dsm);  // <= 8192 tile ids (aliases hist)
  if (tid == 0) s_nt = 0;
  __syncthreads();
  uint32_t ex = 0xffffffffu;
  const uint16_t* trow = reinterpret_cast<const uint16_t*>(tmin) + (int64_t)blockIdx.x * ntiles;
  for (int t = tid; t < ntiles; t += blockDim.x) {
    const uint32_t k = key16(__ldg(trow + t));
    if (k <= up) tl[atomicAdd(&s_nt, 1u)] = (uint16_t)t;
    else ex = min(ex, k);
  }
  __syncthreads();
  const uint32_t nt = s_nt;
  auto take = [&](uint32_t h, int i) {
    const uint32_t k = key16(h);
    if (k <= up) {
      uint32_t p = atomicAdd(&s_cnt, 1u);
      if (p < SEL_COLLECT) ck[p] = ((uint64_t)k << 32) | (uint32_t)i;
    } else {
      ex = min(ex, k);
    }
  };
  if ((K & 7) == 0 && (reinterpret_cast<uintptr_t>(row.r) & 15) == 0) {
    // 16 threads per 128-code tile, one 16-byte load (8 codes) each
    const uint4* r8 = reinterpret_cast<const uint4*>(row.r);
    const int n8 = K >> 3;
    // two 16-byte loads per thread in flight per step
    for (uint32_t e0 = tid; e0 < nt * 16; e0 += 2 * blockDim.x) {
      const uint32_t e1 = e0 + blockDim.x;
      const int i0 = (int)tl[e0 >> 4] * 16 + (int)(e0 & 15);
      const int i1 = e1 < nt * 16 ? (int)tl[e1 >> 4] * 16 + (int)(e1 & 15) : n8;
      const bool ok0 = i0 < n8, ok1 = i1 < n8;
      const uint4 v0 = ok0 ? __ldg(r8 + i0) : make_uint4(0, 0, 0, 0);
      const uint4 v1 = ok1 ? __ldg(r8 + i1) : make_uint4(0, 0, 0, 0);
      if (ok0) {
        const uint32_t w[4] = {v0.x, v0.y, v0.z, v0.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          take(w[k] & 0xffffu, 8 * i0 + 2 * k);
          take(w[k] >> 16, 8 * i0 + 2 * k + 1);
        }
      }
      if (ok1) {
        const uint32_t w[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          take(w[k] & 0xffffu, 8 * i1 + 2 * k);
          take(w[k] >> 16, 8 * i1 + 2 * k + 1);
        }
      }
    }
  } else {
    for (uint32_t e0 = tid; e0 < nt * 128; e0 += blockDim.x) {
      const int i = (int)tl[e0 >> 7] * 128 + (int)(e0 & 127);
      if (i < K) take(__ldg(row.r + i), i);
    }
  }
  ex = block_min(ex, red);  // also orders the collection before its use
  const uint32_t n = s_cnt;
  if (n > (uint32_t)SEL_COLLECT) {
    __syncthreads();
    select_bucketed(row, K, Tmin, cap, out, cand_n + blockIdx.x, theta + blockIdx.x, hist);
    return;
  }
  if (n <= (uint32_t)cap) {
    for (uint32_t i = tid; i < n; i += blockDim.x) out[i] = (int)(uint32_t)ck[i];
    if (tid == 0) {
      cand_n[blockIdx.x] = (int)n;
      theta[blockIdx.x] = ex == 0xffffffffu ? __int_as_float(0x7f800000)
                                            : dec_score(key16_inv(ex), row.scale, row.q2);
    }
    return;
  }
  // 3. more than cap collected: keep the cap smallest, theta = the next one
  const uint32_t np2 = next_pow2(n);
  for (uint32_t i = n + tid; i < np2; i += blockDim.x) ck[i] = kKeyPad;
  __syncthreads();
  bitonic_sort_keys(ck, np2);
  for (int i = tid; i < cap; i += blockDim.x) out[i] = (int)(uint32_t)ck[i];
  if (tid == 0) {
    cand_n[blockIdx.x] = cap;
    theta[blockIdx.x] = dec_score(key16_inv((uint32_t)(ck[cap] >> 32)), row.scale, row.q2);
  }
}

// ----------------------------------------------------------------- K2
GIVF_DEV double key_f64(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// Warp-cooperative float64 squared difference |c - q|^2; lanes stride the
// dimension, then a fixed xor-tree.  f32diff selects the nprobe == K formula
// (difference rounded to f32 first, search.py:82).
GIVF_DEV double warp_sqdist64(const float* __restrict__ c, const double* qd,
                              const float* qf, int d, bool f32diff) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) {
    double t;
    if (f32diff) t = (double)__fsub_rn(c[j], qf[j]);
    else t = dsub((double)c[j], qd[j]);
    s = dadd(s, dmul(t, t));
  }
  return warp_sum(s);
}

// Emit the first P of the (d64, id)-sorted pairs.  f32order reorders them by
// (f32(d64), id) as graph.py:380-382 does for nprobe < K; otherwise the
// (d64, id) order of search.py:83 is kept.  qc2 = the float64 distance.
__device__ void emit_probe(const uint64_t* skey, const uint32_t* sval, int P, bool f32order,
                           uint64_t* k2, uint32_t* v2, double* dv,
                           int* regions_out, double* qc2_out) {
  if (!f32order) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      regions_out[i] = (int)sval[i];
      qc2_out[i] = key_f64(skey[i]);
    }
    __syncthreads();
    return;
  }
  const uint32_t np2 = next_pow2((uint32_t)P);
  for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x) {
    if (i < (uint32_t)P) {
      double d64 = key_f64(skey[i]);
      dv[i] = d64;
      k2[i] = ((uint64_t)f32_key((float)d64) << 32) | sval[i];
      v2[i] = i;
    } else {
      k2[i] = kKeyPad;
      v2[i] = 0xffffffffu;
    }
  }
  __syncthreads();
  bitonic_sort(k2, v2, np2);
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    uint32_t src = v2[i];
    regions_out[i] = (int)sval[src];
    qc2_out[i] = dv[src];
  }
  __syncthreads();
}

// smem: qd[d] f64, qf[d] f32, key[capp2] u64, val[capp2] u32, k2/v2/dv for P.
__global__ void __launch_bounds__(256)
k_probe_recheck(const float* __restrict__ Q, const float* __restrict__ C, int K, int d,
                int P, const int* __restrict__ cand, const int* __restrict__ cand_n,
                int cap, const float* __restrict__ theta, float cmax, float eps_scale,
                float half_rel, int* __restrict__ regions, double* __restrict__ qc2,
                int* __restrict__ fail, unsigned long long* fail_count,
                const int* __restrict__ qmap) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int capp2 = (int)next_pow2((uint32_t)cap);
  const int pp2 = (int)next_pow2((uint32_t)P);
  double* qd = reinterpret_cast<double*>(smem);
  double* dv = qd + d;
  uint64_t* key = reinterpret_cast<uint64_t*>(dv + pp2);
  uint64_t* k2 = key + capp2;
  uint32_t* val = reinterpret_cast<uint32_t*>(k2 + pp2);
  uint32_t* v2 = val + capp2;
  float* qf = reinterpret_cast<float*>(v2 + pp2);
  __shared__ double red[40];

  // b indexes the candidate lists; qb the query (qmap: a re-check of some
  // queries of the chunk, e.g. the fused probe's retry pass)
  const int b = blockIdx.x;
  const int qb = qmap ? qmap[b] : b;
  const float* q = Q + (int64_t)qb * d;
  double q2p = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    qf[j] = q[j];
    qd[j] = (double)q[j];
    q2p += (double)q[j] * (double)q[j];
  }
  double q2 = block_sum(q2p, red);  // also syncs qd/qf
  const int n = cand_n[b];
  const int* cb = cand + (int64_t)b * cap;
  const uint32_t np2 = next_pow2((uint32_t)max(n, 1));
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  if (d <= 128) {
    // two candidates per warp step, every row load issued before the math
    // (same per-candidate arithmetic order as warp_sqdist64)
    constexpr int R = 4;  // d <= 32 * R
    for (int i = warp; i < n; i += 2 * nw) {
      const int i2 = i + nw;
      const int id1 = cb[i], id2 = i2 < n ? cb[i2] : id1;
      const float* c1 = C + (int64_t)id1 * d;
      const float* c2 = C + (int64_t)id2 * d;
      float x1[R], x2[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int j = lane + 32 * r;
        x1[r] = j < d ? __ldg(c1 + j) : 0.f;
        x2[r] = j < d ? __ldg(c2 + j) : 0.f;
      }
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int j = lane + 32 * r;
        if (j < d) {
          const double t1 = dsub((double)x1[r], qd[j]), t2 = dsub((double)x2[r], qd[j]);
          s1 = dadd(s1, dmul(t1, t1));
          s2 = dadd(s2, dmul(t2, t2));
        }
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        key[i] = f64_key(s1);
        val[i] = (uint32_t)id1;
        if (i2 < n) { key[i2] = f64_key(s2); val[i2] = (uint32_t)id2; }
      }
    }
  } else {
    for (int i = warp; i < n; i += nw) {
      int id = cb[i];
      double s = warp_sqdist64(C + (int64_t)id * d, qd, qf, d, false);
      if (lane == 0) { key[i] = f64_key(s); val[i] = (uint32_t)id; }
    }
  }
  for (uint32_t i = n + threadIdx.x; i < np2; i += blockDim.x) { key[i] = kKeyPad; val[i] = 0xffffffffu; }
  __syncthreads();
  bitonic_sort(key, val, np2);

  if (n < K) {
    // a priori bound on |s~ - (|c|^2 - 2 q.c)| for the fp32 GEMM of K1a
    double qn = sqrt(q2);
    double eps = (double)eps_scale * ((double)cmax * cmax + 2.0 * qn * cmax) +
                 1e-12 * ((double)cmax + qn) * ((double)cmax + qn);
    double dp = key_f64(key[P - 1]);
    double th = (double)theta[b];
    // fp16 storage of the scores: the smallest excluded one, decoded, is
    // within half_rel of its encoded distance th + |q|^2 (plus the f32 decode)
    eps += (double)half_rel * 1.001 * fabs(th + q2) + 1.2e-7 * (fabs(th) + q2);
    bool ok = (n >= P) && (dp - q2 < th - eps);
    if (!ok) {
      if (threadIdx.x == 0) {
        fail[qb] = 1;
        if (fail_count) atomicAdd(fail_count, 1ull);
      }
      return;
    }
  }
  if (threadIdx.x == 0) fail[qb] = 0;
  emit_probe(key, val, P, true, k2, v2, dv, regions + (int64_t)qb * P, qc2 + (int64_t)qb * P);
}

// Exhaustive exact ranking of all K regions for one query per loop step:
// mode 0 = nprobe == K branch (f32 differences, order (d, id));
// mode 1 = fallback for queries flagged by k_probe_recheck.
// Scratch per CTA: kp2 u64 keys + kp2 u32 vals (+ P-sized emit buffers).
__global__ void __launch_bounds__(256)
k_probe_full(const float* __restrict__ Q, const float* __restrict__ C, int nq, int K, int d,
             int P, int mode, const int* __restrict__ fail,
             uint64_t* __restrict__ scratch_key, uint32_t* __restrict__ scratch_val,
             uint64_t* __restrict__ scratch_k2, uint32_t* __restrict__ scratch_v2,
             double* __restrict__ scratch_dv,
             int* __restrict__ regions, double* __restrict__ qc2) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* qd = reinterpret_cast<double*>(smem);
  float* qf = reinterpret_cast<float*>(qd + d);
  const uint32_t kp2 = next_pow2((uint32_t)K);
  const uint32_t pp2 = next_pow2((uint32_t)P);
  uint64_t* key = scratch_key + (int64_t)blockIdx.x * kp2;
  uint32_t* val = scratch_val + (int64_t)blockIdx.x * kp2;
  uint64_t* k2 = scratch_k2 + (int64_t)blockIdx.x * pp2;
  uint32_t* v2 = scratch_v2 + (int64_t)blockIdx.x * pp2;
  double* dv = scratch_dv + (int64_t)blockIdx.x * pp2;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const bool f32diff = mode == 0;

  auto one = [&](int b) {
    const float* q = Q + (int64_t)b * d;
    for (int j = threadIdx.x; j < d; j += blockDim.x) { qf[j] = q[j]; qd[j] = (double)q[j]; }
    __syncthreads();
    for (int i = warp; i < K; i += nw) {
      double s = warp_sqdist64(C + (int64_t)i * d, qd, qf, d, f32diff);
      if (lane == 0) { key[i] = f64_key(s); val[i] = (uint32_t)i; }
    }
    for (uint32_t i = K + threadIdx.x; i < kp2; i += blockDim.x) { key[i] = kKeyPad; val[i] = 0xffffffffu; }
    __syncthreads();
    bitonic_sort(key, val, kp2);
    emit_probe(key, val, P, !f32diff, k2, v2, dv, regions + (int64_t)b * P, qc2 + (int64_t)b * P);
    __syncthreads();
  };
  if (mode == 0) {
    for (int b = blockIdx.x; b < nq; b += gridDim.x) one(b);
    return;
  }
  // fallback mode: the flags of blockDim.x queries are read at once and only
  // the flagged ones are redone
  __shared__ int s_list[1024];
  __shared__ int s_n;
  for (int64_t b0 = blockIdx.x; b0 < nq; b0 += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const int64_t b = b0 + (int64_t)threadIdx.x * gridDim.x;
    if (b < nq && fail[b] != 0) s_list[atomicAdd(&s_n, 1)] = (int)b;
    __syncthreads();
    const int n = s_n;
    for (int i = 0; i < n; ++i) one(s_list[i]);
    __syncthreads();
  }
}

// ----------------------------------------------------------------- launchers
int probe_tiles(int K) { return (K + PG_BN - 1) / PG_BN; }

void launch_query_scale(const float* Q, int nq, int d, float cmax, float* q2, float* qinv,
                        float* qscale, cudaStream_t s) {
  k_query_scale<<<(nq + 7) / 8, 256, 0, s>>>(Q, nq, d, cmax, q2, qinv, qscale);
}

void launch_probe_gemm(const float* Q, const float* C, const float* c2, int nq, int K, int d,
                       const ScoreOut& o, float* tmin, cudaStream_t s) {
  dim3 grid((K + PG_BN - 1) / PG_BN, (nq + PG_BM - 1) / PG_BM);
  if (o.D16) k_probe_gemm<true><<<grid, 256, 0, s>>>(Q, C, c2, nq, K, d, o, tmin);
  else k_probe_gemm<false><<<grid, 256, 0, s>>>(Q, C, c2, nq, K, d, o, tmin);
}

void launch_probe_select(const uint16_t* D, int64_t ldD, const float* q2, const float* qscale,
                         int nq, int K, int Tmin, int cap, const float* tmin, int ntiles,
                         uint32_t* tup, int* cand, int* cand_n, float* theta, cudaStream_t s) {
  ensure_max_smem((const void*)k_probe_select, 64 * 1024);
  if (tmin && ntiles >= Tmin && K > cap)
    k_tile_theta<<<(nq + 7) / 8, 256, 0, s>>>(reinterpret_cast<const uint16_t*>(tmin), nq,
                                               ntiles, Tmin, tup);
  k_probe_select<<<nq, SEL_THREADS, 8192 * 4 + SEL_COLLECT * 8, s>>>(
      D, ldD, q2, qscale, K, Tmin, cap, tmin, ntiles, tup, cand, cand_n, theta);
}

size_t probe_recheck_smem(int d, int P, int cap) {
  size_t capp2 = 1, pp2 = 1;
  while (capp2 < (size_t)cap) capp2 <<= 1;
  while (pp2 < (size_t)P) pp2 <<= 1;
  return d * 8 + pp2 * 8 + capp2 * 8 + pp2 * 8 + capp2 * 4 + pp2 * 4 + d * 4 + 16;
}

void launch_probe_recheck(const float* Q, const float* C, int nq, int K, int d, int P,
                          const int* cand, const int* cand_n, int cap, const float* theta,
                          float cmax, float eps_scale, float half_rel, int* regions, double* qc2,
                          int* fail, unsigned long long* fail_count, cudaStream_t s,
                          const int* qmap) {
  size_t sm = probe_recheck_smem(d, P, cap);
  ensure_max_smem((const void*)k_probe_recheck, 200 * 1024);
  k_probe_recheck<<<nq, 256, sm, s>>>(Q, C, K, d, P, cand, cand_n, cap, theta, cmax, eps_scale,
                                      half_rel, regions, qc2, fail, fail_count, qmap);
}

void launch_probe_full(const float* Q, const float* C, int nq, int K, int d, int P, int mode,
                       const int* fail, int nslots, uint64_t* sk, uint32_t* sv, uint64_t* sk2,
                       uint32_t* sv2, double* sdv, int* regions, double* qc2, cudaStream_t s) {
  size_t sm = (size_t)d * 12 + 16;
  k_probe_full<<<nslots, 256, sm, s>>>(Q, C, nq, K, d, P, mode, fail, sk, sv, sk2, sv2, sdv,
                                       regions, qc2);
}

}  // namespace givf
