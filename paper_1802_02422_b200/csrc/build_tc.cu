// Index-builder kernels: the fused sm_100a steps that
// turn a stream of base rows into the GroupedIndex arrays the search path
// reads, so a 1B-row index builds inside one benchmark run.
//
//   KA  k_assign_tc    nearest coarse centroid of every row (kmeans.py
//                      assign_exact top=1 / index.py:88-99 _assign_regions)
//                      as a tcgen05 GEMM rows x centroids whose epilogue
//                      keeps a running arg-min: the rows x K distance matrix
//                      never leaves TMEM.
//   KE  k_encode_rows  per region-run of rows: group pick (index.py:124-138,
//                      grouping.py:77-82 anchors, util.py:24-33 distances),
//                      residual PQ encode (pq.py:56-66 / 124-129), constant
//                      term (index.py:141-170) and its byte (grouping.py:103-
//                      113), one pass over the rows.
//
// KA precision: one bf16 x bf16 product per term, fp32 accumulation (the
// reference itself switches to an approximate graph assignment at
// K >= 2^16, index.py:88-93); the index it produces is a valid GroupedIndex
// and the search path's parity does not depend on how it was built.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace givf {

namespace asg {
constexpr int MB = 4;                      // 128-row m-blocks per work unit
constexpr int BM = 128, BN = 64, BK = 32;  // BK bf16 = 64 B = one SWIZZLE_64B row
constexpr int UNIT_ROWS = MB * BM;         // 512 rows share every centroid tile
constexpr int NS = 4;                      // centroid-tile ring depth
constexpr int EPI_WARPS = 8;               // two per TMEM lane quarter, two m-blocks each
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr uint32_t A_CHUNK = BM * BK * 2;  // 8 KB
constexpr uint32_t B_CHUNK = BN * BK * 2;  // 4 KB
constexpr int TMEM_COLS = 512;             // 2 buffers x 4 m-blocks x 64 columns
constexpr int KC_MAX = 4;                  // d <= 128
constexpr uint32_t IDESC = tcx::make_idesc(BM, BN);
struct Smem {
  uint64_t full[NS], empty[NS];
  uint64_t a_full, a_empty;
  uint64_t tm_full[2], tm_empty[2];
  uint32_t tmem_base;
};
__host__ __device__ constexpr size_t smem_bytes(int kc) {
  return 1024 + (size_t)MB * kc * A_CHUNK + (size_t)NS * kc * B_CHUNK +
         (size_t)EPI_WARPS * BN * 4 + sizeof(Smem) + 64;
}
}  // namespace asg

// Rows of a bf16 operand: x padded with zeros to Kp columns.
__global__ void k_rows_bf16(const float* __restrict__ x, int64_t rows, int d, int Kp,
                            __nv_bfloat16* __restrict__ out) {
  const int64_t n = rows * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Kp;
    const int c = (int)(e % Kp);
    out[e] = __float2bfloat16_rn(c < d ? x[r * d + c] : 0.f);
  }
}

// Work unit u = (group of 512 rows, slice sp of the centroid tiles).  The
// epilogue writes, per row and slice, the smallest c2[j] - 2 x.c_j and its
// first index j.
template <int KC>
__global__ void __launch_bounds__(asg::THREADS, 1)
k_assign_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
            const float* __restrict__ c2, int64_t rows, int K, int nsplit,
            float* __restrict__ out_v, int32_t* __restrict__ out_i) {
  using namespace asg;
  using namespace tcx;
  extern __shared__ __align__(1024) unsigned char dsm[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(dsm) + 1023) & ~(uintptr_t)1023);
  unsigned char* smA = base;
  unsigned char* smB = base + (size_t)MB * KC * A_CHUNK;
  float* c2all = reinterpret_cast<float*>(smB + (size_t)NS * KC * B_CHUNK);
  Smem* sm = reinterpret_cast<Smem*>(c2all + EPI_WARPS * BN);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t groups = (rows + UNIT_ROWS - 1) / UNIT_ROWS;
  const int n_tiles = (K + BN - 1) / BN;
  const int64_t units = groups * nsplit;
  const int per_split = (n_tiles + nsplit - 1) / nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&sm->full[s], 1); mbar_init(&sm->empty[s], 1); }
    mbar_init(&sm->a_full, 1);
    mbar_init(&sm->a_empty, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&sm->tm_full[a], 1);
      mbar_init(&sm->tm_empty[a], EPI_WARPS);
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
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t g = u / nsplit;
        const int sp = (int)(u % nsplit);
        const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
        if (t0 >= t1) continue;
        mbar_wait(&sm->a_empty, a_phase ^ 1);
        a_phase ^= 1;
        mbar_expect_tx(&sm->a_full, (uint32_t)MB * KC * A_CHUNK);
        for (int mb = 0; mb < MB; ++mb)
          for (int kc = 0; kc < KC; ++kc)
            tma_load_2d(smA + (size_t)(mb * KC + kc) * A_CHUNK, &mapA, &sm->a_full, kc * BK,
                        (int)(g * UNIT_ROWS + mb * BM));
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
    uint32_t stage = 0, phase = 0, a_phase = 0, acc = 0, acc_phase = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int sp = (int)(u % nsplit);
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
          for (int mb = 0; mb < MB; ++mb) {
            const uint32_t dcol = tmem + (acc * MB + mb) * BN;
            const uint32_t a0 = smem_u32(smA + (size_t)mb * KC * A_CHUNK);
#pragma unroll
            for (int kc = 0; kc < KC; ++kc)
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                mma_bf16(dcol, sw64_desc(a0 + kc * A_CHUNK + k * 32),
                         sw64_desc(b0 + kc * B_CHUNK + k * 32), IDESC, (kc | k) != 0 ? 1u : 0u);
          }
          mma_commit(&sm->empty[stage]);  // the tile's stage is free once these retire
          mma_commit(&sm->tm_full[acc]);  // and its four accumulators are ready
        }
        __syncwarp();
        if (++stage == NS) { stage = 0; phase ^= 1; }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (lane == 0) mma_commit(&sm->a_empty);  // the row block may be replaced
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..9)
    const int e = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int pair = e >> 2;       // m-blocks {2 pair, 2 pair + 1}
    float* c2w = c2all + e * BN;
    uint32_t acc = 0, acc_phase = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t g = u / nsplit;
      const int sp = (int)(u % nsplit);
      const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
      if (t0 >= t1) continue;
      const int64_t rowA = g * UNIT_ROWS + (2 * pair) * BM + quarter * 32 + lane;
      const int64_t rowB = rowA + BM;
      float bestA = __int_as_float(0x7f800000), bestB = bestA;
      int idxA = -1, idxB = -1;
      for (int t = t0; t < t1; ++t) {
        const int col0 = t * BN;
        const float cA = col0 + lane < K ? __ldg(c2 + col0 + lane) : __int_as_float(0x7f800000);
        const float cB = col0 + 32 + lane < K ? __ldg(c2 + col0 + 32 + lane) : __int_as_float(0x7f800000);
        mbar_wait(&sm->tm_full[acc], acc_phase);
        fence_after();
        c2w[lane] = cA;
        c2w[32 + lane] = cB;
        __syncwarp();
        const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16) + (acc * MB + 2 * pair) * BN;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t ra[32], rb[32];
          tmem_ld32_async(tq + ch * 32, ra);
          tmem_ld32_async(tq + BN + ch * 32, rb);
          tmem_wait_ld(ra);
          tmem_wait_ld(rb);
          float cv[32];
          const float4* c4 = reinterpret_cast<const float4*>(c2w + ch * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 v = c4[i];  // shared-memory broadcast
            cv[4 * i] = v.x; cv[4 * i + 1] = v.y; cv[4 * i + 2] = v.z; cv[4 * i + 3] = v.w;
          }
          float mA = __int_as_float(0x7f800000), mB = mA;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            mA = fminf(mA, fmaf(-2.f, __uint_as_float(ra[i]), cv[i]));
            mB = fminf(mB, fmaf(-2.f, __uint_as_float(rb[i]), cv[i]));
          }
          // rare: a new running minimum -> its first column in this chunk
          if (mA < bestA) {
            int j = 31;
#pragma unroll
            for (int i = 31; i >= 0; --i)
              if (fmaf(-2.f, __uint_as_float(ra[i]), cv[i]) == mA) j = i;
            bestA = mA;
            idxA = col0 + ch * 32 + j;
          }
          if (mB < bestB) {
            int j = 31;
#pragma unroll
            for (int i = 31; i >= 0; --i)
              if (fmaf(-2.f, __uint_as_float(rb[i]), cv[i]) == mB) j = i;
            bestB = mB;
            idxB = col0 + ch * 32 + j;
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm->tm_empty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (rowA < rows) { out_v[sp * rows + rowA] = bestA; out_i[sp * rows + rowA] = idxA; }
      if (rowB < rows) { out_v[sp * rows + rowB] = bestB; out_i[sp * rows + rowB] = idxB; }
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

// Slices -> one (value, first index) per row; out_d (optional) = the value
// plus |x|^2 when x2 is given.
__global__ void k_assign_reduce(const float* __restrict__ v, const int32_t* __restrict__ idx,
                                int nsplit, int64_t rows, const float* __restrict__ x2,
                                int32_t* __restrict__ out, float* __restrict__ out_d) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    float b = v[r];
    int32_t bi = idx[r];
    for (int s = 1; s < nsplit; ++s) {
      const float w = v[s * rows + r];
      const int32_t wi = idx[s * rows + r];
      if (w < b || (w == b && wi < bi) || bi < 0) { b = w; bi = wi; }
    }
    out[r] = bi;
    if (out_d) out_d[r] = x2 ? fmaxf(b + x2[r], 0.f) : b;
  }
}

// ------------------------------------------------------------------- KE
// One CTA per run of rows that share a region (rows sorted by region).
// Shared memory: the region's L anchors t_j = f32(c + a (s_j - c)) with
// stride d + 1 (a lane per anchor reads conflict-free) and |t_j|^2, the PQ
// codebook with stride 256 ds + 1 per sub-quantizer and |codeword|^2 with
// stride 257 (lanes of different sub-quantizers hit distinct banks), and a
// per-warp row / residual staging area.
constexpr int KE_THREADS = 512;
constexpr int KE_WARPS = KE_THREADS / 32;

__host__ __device__ inline size_t ke_smem_bytes(int d, int L, int M) {
  const int ds = d / M;
  return ((size_t)L * (d + 1) + L + (size_t)M * (256 * ds + 1) + (size_t)M * 257 +
          (size_t)KE_WARPS * 2 * d) * 4 + 64;
}

struct EncodeArgs {
  const float* X;          // (n, d) rows (any order)
  const int32_t* order;    // (n) row indices grouped by region
  const int64_t* seg;      // (S + 1) run boundaries into order
  const int32_t* seg_region;  // (S) region of each run
  int64_t nseg;
  int d, L, M, grouping;
  const float* centroids;  // (K, d)
  const int32_t* nbr;      // (K, L)
  const float* alphas;     // (K)
  const double* csq;       // (K) float64 |c|^2
  const float* codewords;  // (M, 256, d / M)
  const float* cwsq;       // (M, 256) f32 |codeword|^2
  double lo, step;         // ConstQuantizer (step <= 0: every byte 0)
  int16_t* pick;           // (n) out, or null
  uint8_t* codes;          // (n, M) out
  uint8_t* cbytes;         // (n) out, or null
  double* consts;          // (n) out, or null
};

template <int M, int DS>
__global__ void __launch_bounds__(KE_THREADS, 1) k_encode_rows(EncodeArgs a) {
  extern __shared__ __align__(16) float ke[];
  constexpr int ds = DS;
  const int d = a.d, L = a.grouping ? a.L : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* T = ke;                                   // [L][d + 1]
  float* Tsq = T + (size_t)L * (d + 1);            // [L]
  float* CW = Tsq + L;                             // [M][256 ds + 1]
  float* CWsq = CW + (size_t)M * (256 * ds + 1);   // [M][257]
  float* stage = CWsq + (size_t)M * 257 + (size_t)warp * 2 * d;  // x row, residual rows
  const int cws = 256 * ds + 1;
  for (int i = threadIdx.x; i < M * 256 * ds; i += KE_THREADS) {
    const int m = i / (256 * ds), r = i % (256 * ds);
    CW[m * cws + r] = a.codewords[i];
  }
  for (int i = threadIdx.x; i < M * 256; i += KE_THREADS) CWsq[(i >> 8) * 257 + (i & 255)] = a.cwsq[i];

  constexpr int R = 32 / M;  // rows encoded per warp step (a lane per sub-quantizer)
  const int rr = lane / M, m = lane % M;
  for (int64_t sg = blockIdx.x; sg < a.nseg; sg += gridDim.x) {
    const int region = a.seg_region[sg];
    const int64_t r0 = a.seg[sg], r1 = a.seg[sg + 1];
    const float* c = a.centroids + (int64_t)region * d;
    const float alpha = a.grouping ? a.alphas[region] : 0.f;
    __syncthreads();  // previous run's readers are done (first: codebook staged)
    for (int i = threadIdx.x; i < L * d; i += KE_THREADS) {
      const int j = i / d, t = i % d;
      float v = c[t];
      if (a.grouping) {
        const float s = a.centroids[(int64_t)a.nbr[(int64_t)region * a.L + j] * d + t];
        v = __fadd_rn(v, __fmul_rn(alpha, __fsub_rn(s, v)));  // grouping.py:77-82, f32 ops
      }
      T[j * (d + 1) + t] = v;
    }
    __syncthreads();
    for (int j = warp; j < L; j += KE_WARPS) {
      float s = 0.f;
      for (int t = lane; t < d; t += 32) s = fmaf(T[j * (d + 1) + t], T[j * (d + 1) + t], s);
      s = warp_sum(s);
      if (lane == 0) Tsq[j] = s;
    }
    __syncthreads();
    const double csq_r = a.csq[region];
    // each warp: R rows at a time, then a lane per (row, sub-quantizer)
    for (int64_t b0 = r0 + (int64_t)warp * R; b0 < r1; b0 += (int64_t)KE_WARPS * R) {
      const int nr = (int)(r1 - b0 < R ? r1 - b0 : R);
      float sub[DS];
      float xsub = 0.f;
      int my_pick = 0;
      int64_t my_row = -1;
      for (int q = 0; q < nr; ++q) {
        const int64_t row = a.order[b0 + q];
        const float* x = a.X + row * d;
        float xsq = 0.f;
        __syncwarp();  // the previous row's readers are done with the stage
        for (int t = lane; t < d; t += 32) {
          const float v = x[t];
          stage[t] = v;
          xsq = fmaf(v, v, xsq);
        }
        xsq = warp_sum(xsq);
        __syncwarp();
        int p = 0;
        if (a.grouping && alpha != 0.f) {
          // nearest anchor, lowest index on ties (index.py:124-138; expanded
          // form clamped at 0, util.py:24-33); alpha == 0: group 0
          float best = __int_as_float(0x7f800000);
          int bi = 0x7fffffff;
          for (int j = lane; j < L; j += 32) {
            const float* tj = T + j * (d + 1);
            float dot = 0.f;
            for (int t = 0; t < d; ++t) dot = fmaf(stage[t], tj[t], dot);
            const float dd = fmaxf(__fsub_rn(__fadd_rn(xsq, Tsq[j]), __fmul_rn(2.f, dot)), 0.f);
            if (dd < best) { best = dd; bi = j; }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
          }
          p = bi;
        }
        // the lanes of row q take their sub-vector of the residual x - t_p
        if (rr == q) {
          my_pick = p;
          my_row = row;
          const float* tp = T + p * (d + 1);
#pragma unroll
          for (int t = 0; t < DS; ++t) {
            const float r = __fsub_rn(stage[m * DS + t], tp[m * DS + t]);
            sub[t] = r;
            xsub = fmaf(r, r, xsub);
          }
        }
      }
      // nearest codeword of the lane's sub-vector, lowest index on ties
      // (expanded form clamped at 0 as util.sq_dists)
      int code = 0;
      double part = 0.0;
      if (my_row >= 0) {
        const float* cwm = CW + m * cws;
        const float* cq = CWsq + m * 257;
        float best = __int_as_float(0x7f800000);
        for (int cidx = 0; cidx < 256; ++cidx) {
          const float* w = cwm + cidx * ds;
          float dot = 0.f;
#pragma unroll
          for (int t = 0; t < DS; ++t) dot = fmaf(sub[t], w[t], dot);
          const float dd = fmaxf(__fsub_rn(__fadd_rn(xsub, cq[cidx]), __fmul_rn(2.f, dot)), 0.f);
          if (dd < best) { best = dd; code = cidx; }
        }
        // |t + recon|^2 over the lane's dimensions in float64 (index.py:141-170)
        const float* tp = T + my_pick * (d + 1);
        const float* w = cwm + code * ds;
#pragma unroll
        for (int t = 0; t < DS; ++t) {
          const double v = (double)__fadd_rn(tp[m * DS + t], w[t]);
          part += v * v;
        }
      }
      // sum over the row's M lanes
#pragma unroll
      for (int o = M / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (my_row >= 0) {
        a.codes[my_row * M + m] = (uint8_t)code;
        if (m == 0) {
          double cst;
          if (a.grouping) {
            const int s = a.nbr[(int64_t)region * a.L + my_pick];
            const double al = (double)alpha;
            cst = part - (1.0 - al) * csq_r - al * a.csq[s];
          } else {
            cst = part - csq_r;
          }
          if (a.consts) a.consts[my_row] = cst;
          if (a.cbytes) {
            uint8_t byte = 0;
            if (a.step > 0.0) {
              const double bq = floor((cst - a.lo) / a.step);
              byte = (uint8_t)fmin(fmax(bq, 0.0), 255.0);
            }
            a.cbytes[my_row] = byte;
          }
          if (a.pick) a.pick[my_row] = (int16_t)my_pick;
        }
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------- host
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// bf16 (rows x cols) in 32-column x box_rows boxes, SWIZZLE_64B
bool make_map64(CUtensorMap* m, const void* ptr, int64_t rows, int cols, int box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int assign_kpad(int d) { return ((d + 31) / 32) * 32; }
bool assign_supported(int d) { return d >= 1 && d <= 32 * asg::KC_MAX; }

void launch_rows_bf16(const float* x, int64_t rows, int d, void* out, cudaStream_t s) {
  const int Kp = assign_kpad(d);
  const int64_t n = rows * Kp;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms_cur() * 16);
  k_rows_bf16<<<std::max(blocks, 1), 256, 0, s>>>(x, rows, d, Kp,
                                                  reinterpret_cast<__nv_bfloat16*>(out));
}

int assign_nsplit(int64_t rows, int K) {
  const int64_t groups = (rows + asg::UNIT_ROWS - 1) / asg::UNIT_ROWS;
  const int n_tiles = (K + asg::BN - 1) / asg::BN;
  const int sms = num_sms_cur();
  int nsplit = 1;
  int64_t best = -1;
  // busiest CTA's tiles, one tile of overhead per unit; at most 64 slices
  for (int ns = 1; ns <= std::min(n_tiles, 64); ++ns) {
    const int64_t per_cta = (groups * ns + sms - 1) / sms;
    const int64_t cost = per_cta * ((n_tiles + ns - 1) / ns + 1);
    if (best < 0 || cost < best) { best = cost; nsplit = ns; }
  }
  return nsplit;
}

cudaError_t launch_assign_tc(const void* Xbf, int64_t rows, const void* Cbf, const float* c2, int K,
                             int d, int nsplit, float* part_v, int32_t* part_i, cudaStream_t s) {
  const int Kp = assign_kpad(d);
  const int KC = Kp / 32;
  CUtensorMap ma, mb;
  if (!make_map64(&ma, Xbf, rows, Kp, asg::BM) || !make_map64(&mb, Cbf, K, Kp, asg::BN))
    return cudaErrorInvalidValue;
  const int64_t groups = (rows + asg::UNIT_ROWS - 1) / asg::UNIT_ROWS;
  const int64_t units = groups * nsplit;
  const int grid = (int)std::min<int64_t>(units, num_sms_cur());
  const size_t smem = asg::smem_bytes(KC);
  const void* fn = nullptr;
  switch (KC) {
    case 1: fn = (const void*)k_assign_tc<1>; break;
    case 2: fn = (const void*)k_assign_tc<2>; break;
    case 3: fn = (const void*)k_assign_tc<3>; break;
    case 4: fn = (const void*)k_assign_tc<4>; break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = ensure_max_smem(fn, smem);
  if (e != cudaSuccess) return e;
  switch (KC) {
    case 1: k_assign_tc<1><<<grid, asg::THREADS, smem, s>>>(ma, mb, c2, rows, K, nsplit, part_v, part_i); break;
    case 2: k_assign_tc<2><<<grid, asg::THREADS, smem, s>>>(ma, mb, c2, rows, K, nsplit, part_v, part_i); break;
    case 3: k_assign_tc<3><<<grid, asg::THREADS, smem, s>>>(ma, mb, c2, rows, K, nsplit, part_v, part_i); break;
    default: k_assign_tc<4><<<grid, asg::THREADS, smem, s>>>(ma, mb, c2, rows, K, nsplit, part_v, part_i); break;
  }
  return cudaGetLastError();
}

void launch_assign_reduce(const float* v, const int32_t* idx, int nsplit, int64_t rows,
                          const float* x2, int32_t* out, float* out_d, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, (int64_t)num_sms_cur() * 8);
  k_assign_reduce<<<std::max(blocks, 1), 256, 0, s>>>(v, idx, nsplit, rows, x2, out, out_d);
}

size_t encode_smem(int d, int L, int M) { return ke_smem_bytes(d, L, M); }

cudaError_t launch_encode_rows(const EncodeArgsC& c, cudaStream_t s) {
  EncodeArgs a;
  a.X = c.X; a.order = c.order; a.seg = c.seg; a.seg_region = c.seg_region; a.nseg = c.nseg;
  a.d = c.d; a.L = c.L; a.M = c.M; a.grouping = c.grouping;
  a.centroids = c.centroids; a.nbr = c.nbr; a.alphas = c.alphas; a.csq = c.csq;
  a.codewords = c.codewords; a.cwsq = c.cwsq; a.lo = c.lo; a.step = c.step;
  a.pick = c.pick; a.codes = c.codes; a.cbytes = c.cbytes; a.consts = c.consts;
  if (a.nseg <= 0) return cudaSuccess;
  const size_t smem = ke_smem_bytes(c.d, c.grouping ? c.L : 1, c.M);
  const int grid = (int)std::min<int64_t>(a.nseg, (int64_t)num_sms_cur() * 8);
  const int ds = c.d / c.M;
#define GIVF_KE(MM, DD)                                                     \
  if (c.M == MM && ds == DD) {                                              \
    cudaError_t e = ensure_max_smem((const void*)k_encode_rows<MM, DD>, smem); \
    if (e != cudaSuccess) return e;                                         \
    k_encode_rows<MM, DD><<<grid, KE_THREADS, smem, s>>>(a);                \
    return cudaGetLastError();                                              \
  }
  GIVF_KE(8, 12)   // d = 96, M = 8
  GIVF_KE(16, 6)   // d = 96, M = 16
  GIVF_KE(8, 16)   // d = 128, M = 8
  GIVF_KE(16, 8)   // d = 128, M = 16
  GIVF_KE(32, 3)   // d = 96, M = 32
  GIVF_KE(32, 4)   // d = 128, M = 32
  GIVF_KE(8, 4)    // d = 32, M = 8 (test shapes)
  GIVF_KE(16, 2)   // d = 32, M = 16
  GIVF_KE(8, 8)    // d = 64, M = 8
  GIVF_KE(16, 4)   // d = 64, M = 16
#undef GIVF_KE
  return cudaErrorInvalidValue;
}

bool encode_supported(int d, int M) {
  if (M <= 0 || d % M) return false;
  const int ds = d / M;
  return (M == 8 && (ds == 12 || ds == 16 || ds == 4 || ds == 8)) ||
         (M == 16 && (ds == 6 || ds == 8 || ds == 2 || ds == 4)) || (M == 32 && (ds == 3 || ds == 4));
}

}  // namespace givf

namespace givf {

// Row norms: f32(sum x^2 accumulated in float64) and, optionally, the
// float64 sum and the largest norm (float bits, atomicMax: norms are >= 0).
__global__ void k_row_norms(const float* __restrict__ x, int64_t rows, int d,
                            float* __restrict__ out32, double* __restrict__ out64,
                            unsigned int* __restrict__ max_bits) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float mx = 0.f;
  for (int64_t r = w0; r < rows; r += nw) {
    double s = 0.0;
    for (int j = lane; j < d; j += 32) {
      const double v = (double)x[r * d + j];
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) {
      if (out32) out32[r] = (float)s;
      if (out64) out64[r] = s;
    }
    mx = fmaxf(mx, (float)sqrt(s));
  }
  if (max_bits) {
    mx = warp_max(mx);
    if (lane == 0) atomicMax(max_bits, __float_as_uint(mx));
  }
}

void launch_row_norms(const float* x, int64_t rows, int d, float* out32, double* out64,
                      unsigned int* max_bits, cudaStream_t s) {
  const int64_t warps = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)num_sms_cur() * 64));
  k_row_norms<<<(int)((warps * 32 + 255) / 256), 256, 0, s>>>(x, rows, d, out32, out64, max_bits);
}

}  // namespace givf
