// K1 without the score matrix: the region probe for large K (reference:
// search.py:77-90, graph.py:357-383 at ef_search == K).
//
// The D-matrix probe (probe_tc.cu + probe.cu) writes an fp16 score for every
// (query, centroid) pair: 2 MB per query at K = 2^20, 20 GB per 10^4-query
// step, and it runs a bf16x3 GEMM (3.3x the MMA work of one product) to keep
// the candidate margin small.  Here the scores never leave TMEM:
//
//   F0  k_query_f16       per query: |q|^2, fp16 row q 2^-eq (eq a power of
//                         two putting max |q_i| in [2^13, 2^14)), epilogue
//                         multiplier -2^(1+eq+ec)
//   F1  k_probe_filter<0> the same tcgen05 GEMM over a random SAMPLE of Ks
//                         centroids (fixed at upload): per (query, 32-centroid
//                         chunk) the smallest approximate score
//   F2  k_probe_thresh    per query: the j-th smallest chunk minimum,
//                         j = ceil(Ttarget Ks / K), + 2 eps -> threshold thr
//   F1' k_probe_filter<1> the GEMM over all K centroids; the epilogue appends
//                         (centroid, s~) with s~ < thr to the query's list
//   F3  k_probe_pick      per query: a_P = the P-th smallest survivor; the
//                         re-check set S = {s~ < min(thr, a_P + 2 eps')}
//   K2  k_probe_recheck   (probe.cu) float64 distances of S, certified top-P
//   K2' k_probe_full      (probe.cu) exhaustive exact ranking of the queries
//                         F3/K2 could not certify
//
// One fp16 product per term (kind::f16, fp32 accumulation): every operand is
// scaled by a power of two into fp16's normal range, so
//   |s~ - (|c|^2 - 2 q.c)| <= eps_f16 (cmax^2 + 2 |q| cmax)   (probe_f16_eps)
// with eps_f16 = 1.25 (2^-10 + (ceil(d/16) + 16) 2^-22 + 2^-23 + 2^-22).
// Correctness does not depend on the sample: F1' appends every centroid
// below thr, F3 only narrows that set, and K2 accepts a query only if the
// exact P-th distance is below min(thr, theta') - eps, which proves no
// excluded centroid can enter the top-P.  A poor threshold costs a fallback
// (counted in givf_index_counters), never a wrong probe list.
//
// GEMM shape (sm_100a, one CTA per SM, persistent), shared with the index
// builder's assignment GEMM (build_tc.cu): a work unit is MB m-blocks of 128
// queries x a slice of the centroid tiles (BN = 256 / MB centroids); the
// A block (MB x 128 queries) stays resident, centroid tiles stream through a
// 4-stage TMA ring (SWIZZLE_64B, 32 fp16 per row chunk), tcgen05.mma
// 128 x BN x 16 per m-block, double-buffered TMEM (2 x 256 columns).  Units
// run slice-major so the CTAs resident together read the same centroid
// tiles (one HBM read, the rest from L2).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace givf {

namespace pf {
constexpr int BM = 128, BK = 32;  // BK fp16 = 64 B = one SWIZZLE_64B row
constexpr int NS_MAX = 4;         // centroid-tile ring depth
// Epilogue warps: EW = 8, two per TMEM lane quarter (a template parameter;
// 16 measured slower, see filter_warps).
__host__ __device__ constexpr int threads_of(int ew) { return 64 + 32 * ew; }
constexpr uint32_t A_CHUNK = BM * BK * 2;  // 8 KB
constexpr int TMEM_COLS = 512;             // 512 / (MB * BN) accumulator buffers
constexpr int NBUF_MAX = 4;
constexpr int KC_MAX = 5;                  // d + 2 <= 160 (the |c|^2 columns)
// kind::f16 instruction descriptor, fp16 x fp16 -> f32, both K-major
constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
struct Smem {
  uint64_t full[NS_MAX], empty[NS_MAX];
  uint64_t a_full, a_empty;
  uint64_t tm_full[NBUF_MAX], tm_empty[NBUF_MAX];
  uint32_t tmem_base;
};
__host__ __device__ constexpr uint32_t b_chunk(int bn) { return (uint32_t)bn * BK * 2; }
// ring depth: 4 stages while they fit beside the A block and the staging
__host__ __device__ constexpr int ring(int mb, int bn, int kc) {
  return (size_t)mb * kc * A_CHUNK + (size_t)NS_MAX * kc * b_chunk(bn) <= 180 * 1024 ? NS_MAX
       : (size_t)mb * kc * A_CHUNK + (size_t)3 * kc * b_chunk(bn) <= 180 * 1024       ? 3
                                                                                       : 2;
}
// [A block][B ring][barriers]
__host__ __device__ constexpr size_t smem_bytes(int mb, int bn, int kc, int ew) {
  return 1024 + (size_t)mb * kc * A_CHUNK + (size_t)ring(mb, bn, kc) * kc * b_chunk(bn) +
         sizeof(Smem) + 64 + 0 * ew;
}
}  // namespace pf

struct FilterArgs {
  int nq, K, KC, d, nsplit;  // d: MMA depth = dim + 2 (the |c|^2 columns)
  const float* ms;   // (nq) -2^(1 + eq + ec): s~ = ms * acc (exact, a power of two)
  // MODE 0: chunk minima
  float* cmin;       // (nq, nch)
  int nch;
  // MODE 1: survivors below thr, in per-(query, unit, epilogue slot)
  // segments of cap_u entries -- no atomics: each segment has one writer
  const float* thr;  // (nq)
  int nseg, cap_u;   // nseg = (EW / 4) * nsplit
  int* cnt;          // (nq, nseg) survivors found (may exceed cap_u)
  int* cid;          // (nq, nseg, cap_u)
  float* cval;       // (nq, nseg, cap_u)
};

GIVF_DEV float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
GIVF_DEV float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
GIVF_DEV float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// Work unit = (MB m-blocks of 128 queries, slice of the BN-centroid tiles).
// The tile's accumulators take MB * BN TMEM columns: 512 / (MB * BN)
// buffers let the MMA run that many tiles ahead of the epilogue.
template <int MB, int BN, int MODE, int EW>
__global__ void __launch_bounds__(pf::threads_of(EW), 1)
k_probe_filter(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
               FilterArgs a) {
  using namespace pf;
  using namespace tcx;
  constexpr uint32_t B_CHUNK = b_chunk(BN);
  constexpr int TC = MB * BN;           // TMEM columns per tile
  constexpr int NBUF = TMEM_COLS / TC;  // accumulator buffers
  constexpr int CPM = BN / 32;          // 32-column chunks per m-block
  constexpr int SLOTS = EW / 4;         // epilogue warps per TMEM lane quarter
  constexpr int CW = TC / (32 * SLOTS);  // chunks per epilogue warp per tile
  constexpr int NR = CW >= CPM ? CW / CPM : 1;  // query rows per thread
  constexpr uint32_t IDESC = idesc_f16(BM, BN);
  static_assert(NBUF >= 2 && NBUF <= NBUF_MAX && CW >= 1, "tile shape");
  extern __shared__ __align__(1024) unsigned char dsm[];
  // offsets from dsm keep the shared address space visible to the compiler
  unsigned char* base = dsm + ((1024u - (smem_u32(dsm) & 1023u)) & 1023u);
  const int KC = a.KC;
  const int NS = ring(MB, BN, KC);
  unsigned char* smA = base;
  unsigned char* smB = base + (size_t)MB * KC * A_CHUNK;
  Smem* sm = reinterpret_cast<Smem*>(smB + (size_t)NS * KC * B_CHUNK);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = (a.nq + MB * BM - 1) / (MB * BM);
  const int n_tiles = (a.K + BN - 1) / BN;
  const int units = groups * a.nsplit;
  const int per_split = (n_tiles + a.nsplit - 1) / a.nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&sm->full[s], 1); mbar_init(&sm->empty[s], 1); }
    mbar_init(&sm->a_full, 1);
    mbar_init(&sm->a_empty, 1);
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&sm->tm_full[i], 1);
      mbar_init(&sm->tm_empty[i], EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm->tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, a_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int g = u % groups, sp = u / groups;  // slice-major
        const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
        if (t0 >= t1) continue;
        mbar_wait(&sm->a_empty, a_phase ^ 1);
        a_phase ^= 1;
        mbar_expect_tx(&sm->a_full, (uint32_t)MB * KC * A_CHUNK);
        for (int mb = 0; mb < MB; ++mb)
          for (int kc = 0; kc < KC; ++kc)
            tma_load_2d(smA + (size_t)(mb * KC + kc) * A_CHUNK, &mapA, &sm->a_full, kc * BK,
                        (g * MB + mb) * BM);
        for (int t = t0; t < t1; ++t) {
          mbar_wait(&sm->empty[stage], phase ^ 1);
          mbar_expect_tx(&sm->full[stage], (uint32_t)KC * B_CHUNK);
          for (int kc = 0; kc < KC; ++kc)
            tma_load_2d(smB + (size_t)(stage * KC + kc) * B_CHUNK, &mapB, &sm->full[stage],
                        kc * BK, t * BN);
          if (++stage == NS) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // k-steps of 16 that hold real dimensions (the rest of the last chunk is
    // zero padding)
    const int ksteps = (a.d + 15) / 16;
    uint32_t stage = 0, phase = 0, a_phase = 0, acc = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int sp = u / groups;
      const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
      if (t0 >= t1) continue;
      mbar_wait(&sm->a_full, a_phase);
      a_phase ^= 1;
      fence_after();
      for (int t = t0; t < t1; ++t) {
        mbar_wait(&sm->tm_empty[acc], acc_phase ^ 1);
        fence_after();
        mbar_wait(&sm->full[stage], phase);
        fence_after();
        if (lane == 0) {
          const uint32_t b0 = smem_u32(smB + (size_t)stage * KC * B_CHUNK);
#pragma unroll
          // k-steps outer, m-blocks inner: consecutive MMAs go to different
          // accumulators, so no MMA waits on the one before it
          for (int ks = 0; ks < ksteps; ++ks) {
            const int kc = ks >> 1, k = ks & 1;
            const uint64_t bd = sw64_desc(b0 + kc * B_CHUNK + k * 32);
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
              const uint32_t a0 = smem_u32(smA + (size_t)mb * KC * A_CHUNK);
              mma_bf16(tmem + acc * TC + mb * BN, sw64_desc(a0 + kc * A_CHUNK + k * 32), bd, IDESC,
                       ks != 0 ? 1u : 0u);
            }
          }
          mma_commit(&sm->empty[stage]);  // the tile's stage is free once these retire
          mma_commit(&sm->tm_full[acc]);  // and its accumulators are ready
        }
        __syncwarp();
        if (++stage == NS) { stage = 0; phase ^= 1; }
        if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
      }
      if (lane == 0) mma_commit(&sm->a_empty);  // the query block may be replaced
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..)
    // Warp e owns lane quarter (warp & 3) and CW 32-column chunks of the
    // tile: flat chunk f = slot * CW + c over (m-block, column chunk).
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int slot = e >> 2;
    uint32_t acc = 0, acc_phase = 0;
    const float kInf = __int_as_float(0x7f800000);
    const uint32_t f0 = (uint32_t)(slot * CW);
    const uint32_t coff = (f0 / CPM) * BN + (f0 % CPM) * 32;  // TMEM column of the warp's first chunk
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int g = u % groups, sp = u / groups;
      const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
      if (t0 >= t1) continue;
      // s~ = ms * acc with ms = -2^k: s~ < thr  <=>  acc > thr / ms (exact)
      int row[NR], kc_[NR];
      float msr[NR], tr[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int mb = (slot * CW + r * CPM) / CPM;
        row[r] = (g * MB + mb) * BM + quarter * 32 + lane;
        const bool ok = row[r] < a.nq;
        msr[r] = ok ? a.ms[row[r]] : -1.f;
        if constexpr (MODE == 1) tr[r] = ok ? a.thr[row[r]] / msr[r] : kInf;
        else tr[r] = 0.f;
        kc_[r] = 0;
      }
      for (int t = t0; t < t1; ++t) {
        const int col0 = t * BN;
        mbar_wait(&sm->tm_full[acc], acc_phase);
        fence_after();
        const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16) + acc * TC;
        // chunk c's TMEM column: a per-warp constant (coff) + a compile-time
        // step when the warp's chunks lie in one m-block, so the tile loop
        // carries no division
        auto chunk_addr = [&](int c) {
          if constexpr (CW <= CPM && CPM % CW == 0) return tq + coff + (uint32_t)c * 32u;
          const uint32_t f = (uint32_t)(slot * CW + c);
          return tq + (f / CPM) * BN + (f % CPM) * 32;
        };
        // columns past K (only a tile that crosses K): -inf, never a maximum
        // or a survivor
        const bool last = col0 + BN > a.K;
        auto clip = [&](uint32_t* r, int cc) {
          const int c0 = col0 + cc * 32;
          if (last && c0 + 32 > a.K) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i >= a.K) r[i] = __float_as_uint(-kInf);
          }
        };
        // maxima of the triples (tt) and of the chunk: depth-4 FMNMX3 tree
        auto maxima = [&](const uint32_t* r, float* tt) -> float {
#pragma unroll
          for (int k = 0; k < 10; ++k)
            tt[k] = fmax3(__uint_as_float(r[3 * k]), __uint_as_float(r[3 * k + 1]),
                          __uint_as_float(r[3 * k + 2]));
          tt[10] = __uint_as_float(r[30]);
          tt[11] = __uint_as_float(r[31]);
          const float u0 = fmax3(tt[0], tt[1], tt[2]), u1 = fmax3(tt[3], tt[4], tt[5]);
          const float u2 = fmax3(tt[6], tt[7], tt[8]), u3 = fmax3(tt[9], tt[10], tt[11]);
          return fmaxf(fmax3(u0, u1, u2), u3);
        };
        // rare: a chunk with survivors for this lane -- walk its triples
        // above tr; values picked out of registers by a switch (no dynamic
        // register indexing, no staging)
        auto append = [&](const uint32_t* r, const float* tt, int cc, int rs) {
          uint32_t tm = 0;
#pragma unroll
          for (int k = 0; k < 12; ++k) tm |= (tt[k] > tr[rs] ? 1u : 0u) << k;
          const int64_t sb = (((int64_t)row[rs] * a.nsplit + sp) * SLOTS + slot) * a.cap_u;
          int kk = kc_[rs];
          while (tm) {
            const int k = __ffs(tm) - 1;
            tm &= tm - 1;
            float x[3];
            int n = 3;
            switch (k) {
#define GIVF_TRIPLE(K)                                                          \
  case K:                                                                       \
    x[0] = __uint_as_float(r[3 * K]); x[1] = __uint_as_float(r[3 * K + 1]);     \
    x[2] = __uint_as_float(r[3 * K + 2]);                                       \
    break;
              GIVF_TRIPLE(0) GIVF_TRIPLE(1) GIVF_TRIPLE(2) GIVF_TRIPLE(3) GIVF_TRIPLE(4)
              GIVF_TRIPLE(5) GIVF_TRIPLE(6) GIVF_TRIPLE(7) GIVF_TRIPLE(8) GIVF_TRIPLE(9)
#undef GIVF_TRIPLE
              case 10: x[0] = __uint_as_float(r[30]); n = 1; break;
              default: x[0] = __uint_as_float(r[31]); n = 1; break;
            }
            const int i0 = k < 10 ? 3 * k : 20 + k;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              if (j < n && x[j] > tr[rs]) {
                if (kk < a.cap_u) {
                  a.cid[sb + kk] = col0 + cc * 32 + i0 + j;
                  a.cval[sb + kk] = x[j] * msr[rs];  // exact: ms is a power of two
                }
                ++kk;
              }
            }
          }
          kc_[rs] = kk;
        };
        float mq[CW];
        // every chunk of this warp into registers, the accumulator buffer
        // released at once (the MMA refills it while the chunks are reduced),
        // then independent max trees; nothing else per score (|c|^2 came
        // through the MMA)
        uint32_t rr[CW][32];
#pragma unroll
        for (int c = 0; c < CW; ++c) tmem_ld32_async(chunk_addr(c), rr[c]);
#pragma unroll
        for (int c = 0; c < CW; ++c) tmem_wait_ld(rr[c]);
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm->tm_empty[acc]);
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const int f = slot * CW + c, cc = f % CPM, rs = NR > 1 ? c / CPM : 0;
          float tt[12];
          clip(rr[c], cc);
          const float m = maxima(rr[c], tt);
          mq[c] = m * msr[rs];  // the chunk's smallest s~
          if constexpr (MODE == 1) {
            if (m > tr[rs]) append(rr[c], tt, cc, rs);
          }
        }
        if constexpr (MODE == 0) {
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const int f = slot * CW + c, cc = f % CPM, rs = NR > 1 ? c / CPM : 0;
            if constexpr (CW == 4 && CPM == 4) {
              if (c == 3 && row[0] < a.nq) {  // one row's whole tile: one 16-byte store
                float* dst = a.cmin + (int64_t)row[0] * a.nch + (col0 >> 5);
                if ((a.nch & 3) == 0 && col0 + BN <= a.K)
                  *reinterpret_cast<float4*>(dst) = make_float4(mq[0], mq[1], mq[2], mq[3]);
                else
                  for (int i = 0; i < 4; ++i)
                    if (col0 + i * 32 < a.K) dst[i] = mq[i];
              }
            } else if (row[rs] < a.nq && col0 + cc * 32 < a.K) {
              a.cmin[(int64_t)row[rs] * a.nch + ((col0 + cc * 32) >> 5)] = mq[c];
            }
          }
        }
        if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
      }
      if constexpr (MODE == 1) {
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if (row[r] < a.nq) a.cnt[((int64_t)row[r] * a.nsplit + sp) * SLOTS + slot] = kc_[r];
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ F0
// One warp per query: q' = q 2^-eq (max |q'_i| in [2^7, 2^8)), then in the
// two |c|^2 columns a = 2^(T - eq); the centroid rows hold there b_hi + b_lo
// = -|c|^2 2^-(1 + ec + T), so the MMA accumulates q'.c' - |c|^2 2^-(1+eq+ec)
// and s~ = ms * acc with ms = -2^(1 + eq + ec).  A query whose a falls
// outside fp16's normal range gets ms = NaN: no survivors, it takes the
// exhaustive probe.
__global__ void k_query_f16(const float* __restrict__ Q, int nq, int d, int dp, int ec, int T,
                            __half* __restrict__ q16, float* __restrict__ ms,
                            float* __restrict__ q2o) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nq) return;
  const float* q = Q + (int64_t)b * d;
  float mx = 0.f;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) {
    const float x = q[j];
    mx = fmaxf(mx, fabsf(x));
    s += (double)x * x;
  }
  mx = warp_max(mx);
  s = warp_sum(s);
  const int eq = mx > 0.f ? ilogbf(mx) - 7 : 0;
  const int ae = T - eq;
  const bool ok = ae >= -14 && ae <= 15;
  for (int j = lane; j < dp; j += 32) {
    float x = 0.f;
    if (j < d) x = ldexpf(q[j], -eq);
    else if (j < d + 2) x = ok ? ldexpf(1.f, ae) : 0.f;
    q16[(int64_t)b * dp + j] = __float2half_rn(x);
  }
  if (lane == 0) {
    ms[b] = ok ? -ldexpf(1.f, eq + ec + 1) : __int_as_float(0x7fc00000);
    if (q2o) q2o[b] = (float)s;
  }
}

// fp16 copy of rows c 2^-ec (zero-padded to dp columns) with the |c|^2
// columns b_hi, b_lo (b = -|c|^2 2^-(1 + ec + T)), optionally of a subset of
// rows (ids) with their |c|^2.
__global__ void k_rows_f16(const float* __restrict__ x, const int32_t* __restrict__ ids,
                           int64_t rows, int d, int dp, int e, int T, const float* __restrict__ c2,
                           __half* __restrict__ out, float* __restrict__ c2out) {
  const int64_t n = rows * dp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / dp;
    const int c = (int)(i % dp);
    const int64_t src = ids ? (int64_t)ids[r] : r;
    __half h = __float2half_rn(0.f);
    if (c < d) {
      h = __float2half_rn(ldexpf(x[src * d + c], -e));
    } else if (c < d + 2 && dp >= d + 2) {
      const double bv = -ldexp((double)c2[src], -(1 + e + T));
      const __half hi = __double2half(bv);
      h = c == d ? hi : __double2half(bv - (double)__half2float(hi));
    }
    out[i] = h;
    if (c == 0 && c2out) c2out[r] = c2[src];
  }
}

// --------------------------------------------------------- block k-th key
// k-th smallest (1-based, k <= n) of n u32 keys in shared memory: four
// 8-bit radix passes with a 256-bin shared histogram.  256 threads.
__device__ uint32_t block_kth_key(const uint32_t* keys, int n, int k, uint32_t* hist,
                                  uint32_t* red) {
  __shared__ uint32_t s_bin, s_k;
  uint32_t prefix = 0, mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    hist[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t key = keys[i];
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    const uint32_t h = hist[threadIdx.x];
    uint32_t tot;
    const uint32_t pre = block_exclusive_scan(h, red, &tot);
    if (pre < (uint32_t)k && (uint32_t)k <= pre + h) { s_bin = threadIdx.x; s_k = k - pre; }
    __syncthreads();
    prefix |= s_bin << shift;
    mask |= 255u << shift;
    k = (int)s_k;
    __syncthreads();
  }
  return prefix;
}

// ------------------------------------------------------------------ F2
// thr = (j-th smallest sample chunk minimum) + 2 eps (+ float slack).
__global__ void __launch_bounds__(256)
k_probe_thresh(const float* __restrict__ cmin, int nch, int j, const float* __restrict__ q2,
               float cmax, float eps_scale, float* __restrict__ thr, const int* __restrict__ qmap) {
  extern __shared__ uint32_t keys[];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t red[40];
  const int b = blockIdx.x;
  const int64_t row = qmap ? qmap[b] : b;  // the sample minima of the chunk's query qmap[b]
  for (int i = threadIdx.x; i < nch; i += blockDim.x)
    keys[i] = f32_key(cmin[row * nch + i]);
  __syncthreads();
  const uint32_t kk = block_kth_key(keys, nch, min(j, nch), hist, red);
  if (threadIdx.x == 0) {
    const double v = (double)key_f32(kk);
    const double qn = sqrt((double)q2[b]);
    const double eps = (double)eps_scale * ((double)cmax * cmax + 2.0 * qn * cmax);
    const double t = v + 2.0 * eps + 1e-6 * (fabs(v) + (double)q2[b]);
    thr[b] = isfinite(v) ? (float)t : __int_as_float(0x7f800000);
  }
}

// ------------------------------------------------------------------ F3
// Re-check set: survivors below min(thr, a_P + 2 eps'), eps' = K2's bound.
// The survivors sit in nseg segments per query (k_probe_filter<1>); they are
// read in place from L2 (four radix passes for a_P, one compaction pass).
// Queries with an overflowing segment, more than fcap or fewer than P
// survivors get cand_n = 0 (K2 then flags them for the exhaustive probe).
__global__ void __launch_bounds__(256)
k_probe_pick(const int* __restrict__ cnt, const int* __restrict__ cid,
             const float* __restrict__ cval, int nseg, int cap_u, int fcap,
             const float* __restrict__ thr, const float* __restrict__ q2, float cmax,
             float eps_scale, int P, int cap2, int* __restrict__ cand, int* __restrict__ cand_n,
             float* __restrict__ theta) {
  constexpr int PICK_SM = 2048;
  __shared__ uint32_t skey[PICK_SM];
  __shared__ int sid[PICK_SM];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t red[40];
  __shared__ uint32_t s_bin, s_k;
  __shared__ int s_n, s_bad;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const int* cb = cnt + (int64_t)b * nseg;
  const int64_t base = (int64_t)b * nseg * cap_u;
  int tot = 0, bad = 0;
  for (int sg = tid; sg < nseg; sg += blockDim.x) {
    const int c = cb[sg];
    tot += c;
    bad |= c > cap_u;
  }
  if (tid == 0) { s_n = 0; s_bad = 0; }
  __syncthreads();
  if (bad) s_bad = 1;
  const int total = (int)block_sum((uint32_t)tot, red);  // also syncs s_bad
  if (s_bad || total < P || total > fcap) {
    if (tid == 0) { cand_n[b] = 0; theta[b] = -__int_as_float(0x7f800000); }
    return;
  }
  // The usual few hundred survivors are first gathered into shared memory
  // (a thread per segment: the segments hold 0-3 entries each, so a warp per
  // segment left 31 lanes idle on every pass); the radix passes and the
  // compaction then run a thread per survivor.
  const bool packed = total <= PICK_SM;
  if (packed) {
    uint32_t all;
    uint32_t o = block_exclusive_scan((uint32_t)tot, red, &all);
    for (int sg = tid; sg < nseg; sg += blockDim.x) {
      const int c = cb[sg];
      for (int i = 0; i < c; ++i) {
        const int64_t at = base + (int64_t)sg * cap_u + i;
        skey[o] = f32_key(cval[at]);
        sid[o] = cid[at];
        ++o;
      }
    }
    __syncthreads();
  }
  // a_P: the P-th smallest survivor (radix select)
  uint32_t prefix = 0, mask = 0;
  int k = P;
  for (int shift = 24; shift >= 0; shift -= 8) {
    hist[tid] = 0;
    __syncthreads();
    if (packed) {
      for (int i = tid; i < total; i += blockDim.x) {
        const uint32_t key = skey[i];
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
    } else {
      for (int sg = warp; sg < nseg; sg += nw) {
        const int c = cb[sg];
        for (int i = lane; i < c; i += 32) {
          const uint32_t key = f32_key(cval[base + (int64_t)sg * cap_u + i]);
          if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
      }
    }
    __syncthreads();
    const uint32_t h = hist[tid];
    uint32_t all;
    const uint32_t pre = block_exclusive_scan(h, red, &all);
    if (pre < (uint32_t)k && (uint32_t)k <= pre + h) { s_bin = tid; s_k = k - pre; }
    __syncthreads();
    prefix |= s_bin << shift;
    mask |= 255u << shift;
    k = (int)s_k;
    __syncthreads();
  }
  const float aP = key_f32(prefix);
  const double qn = sqrt((double)q2[b]);
  // K2's bound (probe.cu: eps + the f32 rounding term at th), doubled, with
  // slack: theta' - eps > a_P + eps >= the exact P-th distance - |q|^2
  const double eps = (double)eps_scale * ((double)cmax * cmax + 2.0 * qn * cmax) +
                     1e-12 * ((double)cmax + qn) * ((double)cmax + qn) +
                     1.2e-7 * (fabs((double)aP) + 4.0 * (double)cmax * qn + (double)q2[b]);
  const float tb = fminf(thr[b], (float)((double)aP + 2.02 * eps));
  if (packed) {
    for (int i = tid; i < total; i += blockDim.x) {
      if (key_f32(skey[i]) < tb) {
        const int p = atomicAdd(&s_n, 1);
        if (p < cap2) cand[(int64_t)b * cap2 + p] = sid[i];
      }
    }
  } else {
    for (int sg = warp; sg < nseg; sg += nw) {
      const int c = cb[sg];
      for (int i = lane; i < c; i += 32) {
        const int64_t at = base + (int64_t)sg * cap_u + i;
        if (cval[at] < tb) {
          const int p = atomicAdd(&s_n, 1);
          if (p < cap2) cand[(int64_t)b * cap2 + p] = cid[at];
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    cand_n[b] = s_n <= cap2 ? s_n : 0;
    theta[b] = tb;
  }
}

// ------------------------------------------------------------- host side
namespace {

bool make_map_f16(CUtensorMap* m, const void* ptr, int64_t rows, int dp, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)dp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)dp * 2};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// GEMM tile shape (m-blocks per unit x centroids per tile); GIVF_FILTER_SHAPE
// = "MBxBN" overrides: 2x128 (default), 4x64, 1x128.  The epilogue's TMEM
// reads bound this kernel (every fp32 score crosses tcgen05.ld once; ~64 B
// per SM clock measured): 2x128 reached 58 B/clk, the narrower-N shapes
// 2x64 / 4x32 lost more to MMA issue overhead than their deeper TMEM
// buffering (4 accumulators) won, and were dropped.
struct FilterShape {
  int mb, bn;
};
FilterShape filter_shape() {
  static const FilterShape fs = [] {
    FilterShape f{1, 256};
    if (const char* e = getenv("GIVF_FILTER_SHAPE")) {
      int m = 0, n = 0;
      if (sscanf(e, "%dx%d", &m, &n) == 2) f = FilterShape{m, n};
    }
    const bool ok = (f.mb == 2 && f.bn == 128) || (f.mb == 4 && f.bn == 64) ||
                    (f.mb == 1 && f.bn == 128) || (f.mb == 1 && f.bn == 256);
    return ok ? f : FilterShape{1, 256};
  }();
  return fs;
}

// Work units = (MB x 128 queries, slice of the centroid tiles), slice-major;
// the slice count minimises the busiest CTA's tiles (+1 tile of overhead
// per unit for its A block).
// epilogue warps of the 1 x 256 shape: 16 (four per TMEM lane quarter, two
// 32-column chunks each).  The epilogue paces this kernel and is bound by
// its own dependent-issue latency: with 8 warps (two per scheduler) each
// tile took ~2000 cycles against an MMA floor of 896; four per scheduler
// bring the GEMM from 2.27 to 1.94 ms (configs[2] shape).  An earlier 16-warp
// variant, before the |c|^2 fold and the early buffer release, had measured
// slower.  GIVF_FILTER_WARPS=8 keeps eight; the other shapes always use 8.
int filter_warps() {
  static const int w = [] {
    const char* e = getenv("GIVF_FILTER_WARPS");
    const FilterShape fs = filter_shape();
    if (!(fs.mb == 1 && fs.bn == 256)) return 8;
    return e && atoi(e) == 8 ? 8 : 16;
  }();
  return w;
}

int filter_nsplit(int nq, int K, int MB, int BN) {
  const int groups = (nq + MB * pf::BM - 1) / (MB * pf::BM);
  const int n_tiles = (K + BN - 1) / BN;
  const int sms = num_sms_cur();
  int nsplit = 1;
  int64_t best = -1;
  for (int ns = 1; ns <= std::min(n_tiles, 1024); ++ns) {
    const int64_t per_cta = ((int64_t)groups * ns + sms - 1) / sms;
    const int64_t cost = per_cta * ((n_tiles + ns - 1) / ns + 1);
    if (best < 0 || cost < best) { best = cost; nsplit = ns; }
  }
  return nsplit;
}

template <int MB, int BN, int MODE, int EW>
cudaError_t launch_filter_w(const CUtensorMap& ma, const CUtensorMap& mb, const FilterArgs& a,
                            cudaStream_t s) {
  const int groups = (a.nq + MB * pf::BM - 1) / (MB * pf::BM);
  const int units = groups * a.nsplit;
  const int grid = std::min(units, num_sms_cur());
  const size_t smem = pf::smem_bytes(MB, BN, a.KC, EW);
  auto fn = k_probe_filter<MB, BN, MODE, EW>;
  cudaError_t e = ensure_max_smem((const void*)fn, smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, pf::threads_of(EW), smem, s>>>(ma, mb, a);
  return cudaGetLastError();
}

template <int MB, int BN, int MODE>
cudaError_t launch_filter_t(const CUtensorMap& ma, const CUtensorMap& mb, const FilterArgs& a,
                            cudaStream_t s) {
  if constexpr (MB == 1 && BN == 256) {
    if (filter_warps() == 16) return launch_filter_w<MB, BN, MODE, 16>(ma, mb, a, s);
  }
  return launch_filter_w<MB, BN, MODE, 8>(ma, mb, a, s);
}

template <int MODE>
cudaError_t launch_filter(const void* q16, const void* c16, int dp, FilterArgs a,
                          cudaStream_t s) {
  const FilterShape fs = filter_shape();
  if (a.nsplit <= 0) a.nsplit = filter_nsplit(a.nq, a.K, fs.mb, fs.bn);
  CUtensorMap ma, mb;
  if (!make_map_f16(&ma, q16, a.nq, dp, pf::BM) || !make_map_f16(&mb, c16, a.K, dp, fs.bn))
    return cudaErrorInvalidValue;
  if (fs.mb == 4 && fs.bn == 64) return launch_filter_t<4, 64, MODE>(ma, mb, a, s);
  if (fs.mb == 1 && fs.bn == 128) return launch_filter_t<1, 128, MODE>(ma, mb, a, s);
  if (fs.mb == 2 && fs.bn == 128) return launch_filter_t<2, 128, MODE>(ma, mb, a, s);
  return launch_filter_t<1, 256, MODE>(ma, mb, a, s);
}

}  // namespace

int f16_pitch(int d) { return ((d + 2 + 31) / 32) * 32; }  // + the two |c|^2 columns
bool fused_supported(int d) { return d >= 1 && d + 2 <= 32 * pf::KC_MAX; }
float probe_f16_eps(int d) {
  const double u2 = std::ldexp(1.0, -10);  // 2u, u = 2^-11
  // fp32 tensor-core accumulation over the d + 2 terms; the b_hi + b_lo
  // split carries |c|^2 to 2^-22 (the separate 2^-22 term below)
  const double acc = (double)((d + 2 + 15) / 16 + 16) * std::ldexp(1.0, -22) * 1.001;
  return (float)(1.25 * (u2 + std::ldexp(1.0, -22) + acc + std::ldexp(1.0, -23)));
}
// K3a from fp16 centroid rows and f32 queries: |qs2~ - qs2| <= eps U with
// 2 (u + (d + 1) 2^-24) |q| cmax + 2^-24 cmax^2 <= (u + (d + 2) 2^-24) U.
float direct_f16_eps(int d) {
  return (float)(1.25 * (std::ldexp(1.0, -11) + (double)(d + 4) * std::ldexp(1.0, -24)));
}

void launch_rows_f16(const float* x, const int32_t* ids, int64_t rows, int d, int e, int T,
                     const float* c2, void* out, float* c2out, cudaStream_t s, int dp) {
  if (dp <= 0) dp = f16_pitch(d);
  const int64_t n = rows * dp;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms_cur() * 16);
  k_rows_f16<<<std::max(blocks, 1), 256, 0, s>>>(x, ids, rows, d, dp, e, T, c2,
                                                  reinterpret_cast<__half*>(out), c2out);
}

void launch_query_f16(const float* Q, int nq, int d, int ec, int T, void* q16, float* ms,
                      float* q2, cudaStream_t s) {
  const int per = 8;
  k_query_f16<<<(nq + per - 1) / per, per * 32, 0, s>>>(
      Q, nq, d, f16_pitch(d), ec, T, reinterpret_cast<__half*>(q16), ms, q2);
}

cudaError_t launch_probe_sample(const void* q16, const void* s16, int nq, int Ks, int d,
                                const float* ms, float* cmin, cudaStream_t s) {
  FilterArgs a{};
  a.nq = nq;
  a.K = Ks;
  a.KC = f16_pitch(d) / 32;
  a.d = d + 2;
  a.ms = ms;
  a.cmin = cmin;
  a.nch = (Ks + 31) / 32;
  return launch_filter<0>(q16, s16, f16_pitch(d), a, s);
}

// Survivor segments of the filter for nq queries: per query nseg segments
// of cap_u entries, cap_u * nseg <= fcap (fixed per-query bytes).
int filter_slots() { return filter_warps() / 4; }

void filter_segments(int nq, int K, int fcap, int* nseg, int* cap_u) {
  const FilterShape fs = filter_shape();
  *nseg = (filter_warps() / 4) * filter_nsplit(nq, K, fs.mb, fs.bn);
  *cap_u = std::max(8, fcap / *nseg);
}

cudaError_t launch_probe_filter(const void* q16, const void* c16, int nq, int K, int d,
                                const float* ms, const float* thr, int nseg, int cap_u, int* cnt,
                                int* cid, float* cval, cudaStream_t s) {
  FilterArgs a{};
  a.nq = nq;
  a.K = K;
  a.KC = f16_pitch(d) / 32;
  a.d = d + 2;
  a.ms = ms;
  a.thr = thr;
  a.nsplit = nseg / (filter_warps() / 4);
  a.nseg = nseg;
  a.cap_u = cap_u;
  a.cnt = cnt;
  a.cid = cid;
  a.cval = cval;
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)nq * nseg, s);
  if (e != cudaSuccess) return e;
  return launch_filter<1>(q16, c16, f16_pitch(d), a, s);
}

void launch_probe_thresh(const float* cmin, int nch, int j, const float* q2, float cmax,
                         float eps_scale, int nq, float* thr, cudaStream_t s, const int* qmap) {
  const size_t sm = (size_t)nch * 4;
  ensure_max_smem((const void*)k_probe_thresh, sm);
  k_probe_thresh<<<nq, 256, sm, s>>>(cmin, nch, j, q2, cmax, eps_scale, thr, qmap);
}

__global__ void k_collect_failed(const int* __restrict__ fail, int nq, int* __restrict__ idx,
                                 int* __restrict__ n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const bool f = b < nq && fail[b] != 0;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if (!bal) return;
  int base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(n, __popc(bal));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (f) idx[base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = b;
}

__global__ void k_gather_rows(const float* __restrict__ Q, const int* __restrict__ idx, int n, int d,
                              float* __restrict__ out) {
  const int64_t total = (int64_t)n * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = Q[(int64_t)idx[e / d] * d + e % d];
}

__global__ void k_add_counter(unsigned long long* c, const int* n) {
  if (threadIdx.x == 0 && *n) atomicAdd(c, (unsigned long long)*n);
}

void launch_collect_failed(const int* fail, int nq, int* idx, int* n, cudaStream_t s) {
  cudaMemsetAsync(n, 0, sizeof(int), s);
  k_collect_failed<<<(nq + 255) / 256, 256, 0, s>>>(fail, nq, idx, n);
}

void launch_gather_rows(const float* Q, const int* idx, int n, int d, float* out, cudaStream_t s) {
  const int64_t total = (int64_t)n * d;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms_cur() * 8);
  if (blocks > 0) k_gather_rows<<<blocks, 256, 0, s>>>(Q, idx, n, d, out);
}

void launch_add_counter(unsigned long long* c, const int* n, cudaStream_t s) {
  k_add_counter<<<1, 32, 0, s>>>(c, n);
}

void launch_probe_pick(const int* cnt, const int* cid, const float* cval, int nseg, int cap_u,
                       int fcap, const float* thr, const float* q2, float cmax, float eps_scale,
                       int P, int cap2, int nq, int* cand, int* cand_n, float* theta,
                       cudaStream_t s) {
  k_probe_pick<<<nq, 256, 0, s>>>(cnt, cid, cval, nseg, cap_u, fcap, thr, q2, cmax, eps_scale, P,
                                  cap2, cand, cand_n, theta);
}

}  // namespace givf
