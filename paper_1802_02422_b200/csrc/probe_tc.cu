// K1a on the 5th-generation tensor cores: s~[q, c] = |c|^2 - 2 q.c for a
// block of queries against all K centroids (reference: search.py:77-90).
//
// Precision: fp32 inputs are split into bf16 pairs x = x_hi + x_lo, and
//   q.c ~ q_hi.c_hi + q_hi.c_lo + q_lo.c_hi
// accumulated in fp32 in TMEM.  The centroid operand is B' = [c_hi | c_lo]
// (2d columns); the query operand A' pairs every 64-column chunk of B' with
// a q_hi chunk and, for the c_hi chunks, a q_lo chunk (k_split_bf16), so each
// B chunk crosses L2 -> shared memory once for its one or two MMAs: 2d
// columns of centroid traffic per tile instead of 3d (this GEMM is bound by
// L2 traffic: the centroid operand is re-read once per 128-query block).
// Its error is bounded a priori (eps_scale in capi.cu) and every decision
// taken from s~ is re-checked in float64 (probe_recheck, k_plan_approx), so
// the result stays exact.
//
// Kernel shape (sm_100a, one CTA per SM, persistent):
//   tile = 128 queries x 256 centroids, UMMA 128x256x16, cta_group::1
//   warp 0  TMA producer: the 128 x K_A A block once per work unit (resident
//           in smem), then B chunks of 256 x 64 through a 3-stage ring
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer; commits free
//           the B stages and publish finished accumulators
//   warps 2-9  epilogue: two warps per TMEM lane quarter, each owning one
//           128-column half of the accumulator (double-buffered: 2 x 256
//           TMEM columns); tcgen05.ld 32x32b.x32 of the next 32 columns is in
//           flight while the current ones become s~ = c2 - 2 acc, go out by
//           TMA store, and fold into the minimum of the 128-centroid tile
// Operands use the SWIZZLE_128B K-major canonical layout written by TMA.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace givf {

namespace tc {

constexpr int BM = 128, BN = 256, BK = 64;  // BK bf16 = 128 B = one swizzle row
constexpr int STAGES = 3;  // B ring depth (2 when the resident A block is 6 chunks)
constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, one 128-column half each
// epilogue smem: TMA-store staging (one 4 KB tile per warp) + per-warp |c|^2
constexpr uint32_t STAGE_OUT = EPI_WARPS * 4096 + EPI_WARPS * 128 * 4;
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr uint32_t A_CHUNK = BM * BK * 2;   // 16 KB
constexpr uint32_t B_CHUNK = BN * BK * 2;   // 32 KB
constexpr int TMEM_COLS = 512;              // two 256-column fp32 accumulators

using namespace tcx;

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major, M x N.
constexpr uint32_t IDESC = make_idesc(BM, BN);

GIVF_DEV void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  tcx::mma_bf16(tmem_d, adesc, bdesc, IDESC, accumulate);
}

struct Smem {
  uint64_t full[STAGES], empty[STAGES];
  uint64_t a_full, a_empty;
  uint64_t tm_full[2], tm_empty[2];
  uint32_t tmem_base;
};

}  // namespace tc

// smem: [A resident: KC x 16 KB][B ring: STAGES x 32 KB][barriers]
// KC = A' chunks (tc_ka), KB = B' chunks per tile (tc_kb), KLO = lo chunks.
// HALF: scores leave as fp16 (ScoreOut in kernels.h), else fp32.  NS: B ring
// depth (tc_stages).
template <bool HALF, int NS>
__global__ void __launch_bounds__(tc::THREADS, 1)
k_probe_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                const __grid_constant__ CUtensorMap mapD, int use_tma_store,
                const float* __restrict__ c2, int nq, int K, int KC, int KB, int KLO, int nsplit,
                float* __restrict__ D, uint16_t* __restrict__ D16, int64_t ldD,
                const float* __restrict__ q2v, const float* __restrict__ qinv,
                const float* __restrict__ qscale, float* __restrict__ tmin) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char dsm[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(dsm) + 1023) & ~(uintptr_t)1023);
  unsigned char* smA = base;
  unsigned char* smB = base + (size_t)KC * A_CHUNK;
  Smem* sm = reinterpret_cast<Smem*>(smB + (size_t)NS * B_CHUNK + STAGE_OUT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_blocks = (nq + BM - 1) / BM;
  const int n_tiles = (K + BN - 1) / BN;
  const int units = m_blocks * nsplit;
  const int per_split = (n_tiles + nsplit - 1) / nsplit;
  // Units run slice-major: the CTAs resident at any moment work on the same
  // centroid slice for different query blocks, so each B tile comes from HBM
  // once and is re-read from L2 by the others (at K = 2^20 the split
  // centroids, 400 MB, do not fit in L2: m-block-major order re-streamed
  // them from HBM once per query block).

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
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int mb = u % m_blocks, sp = u / m_blocks;  // slice-major (see below)
        const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
        if (t0 >= t1) continue;
        mbar_wait(&sm->a_empty, a_phase ^ 1);
        a_phase ^= 1;
        mbar_expect_tx(&sm->a_full, (uint32_t)KC * A_CHUNK);
        for (int kc = 0; kc < KC; ++kc)
          tma_load_2d(smA + (size_t)kc * A_CHUNK, &mapA, &sm->a_full, kc * BK, mb * BM);
        for (int t = t0; t < t1; ++t) {
          for (int kc = 0; kc < KB; ++kc) {
            mbar_wait(&sm->empty[stage], phase ^ 1);
            mbar_expect_tx(&sm->full[stage], B_CHUNK);
            tma_load_2d(smB + (size_t)stage * B_CHUNK, &mapB, &sm->full[stage], kc * BK, t * BN);
            if (++stage == NS) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    uint32_t stage = 0, phase = 0, a_phase = 0, acc = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int sp = u / m_blocks;
      const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
      if (t0 >= t1) continue;
      mbar_wait(&sm->a_full, a_phase);
      a_phase ^= 1;
      fence_after();
      for (int t = t0; t < t1; ++t) {
        mbar_wait(&sm->tm_empty[acc], acc_phase ^ 1);
        fence_after();
        const uint32_t dcol = tmem + acc * BN;
        for (int kc = 0; kc < KB; ++kc) {
          mbar_wait(&sm->full[stage], phase);
          fence_after();
          if (lane == 0) {
            // B chunk kc meets A chunk hi_kc and, while it holds c_hi
            // columns, lo_kc (tc_ka layout: hi_j = j + min(j, KLO))
            const int ahi = kc + min(kc, KLO);
            const uint32_t b0 = smem_u32(smB + (size_t)stage * B_CHUNK);
            const uint32_t a0 = smem_u32(smA + (size_t)ahi * A_CHUNK);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_bf16(dcol, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32),
                       (kc | k) != 0 ? 1u : 0u);
            if (kc < KLO) {
              const uint32_t a1 = a0 + A_CHUNK;
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                mma_bf16(dcol, sw128_desc(a1 + k * 32), sw128_desc(b0 + k * 32), 1u);
            }
            mma_commit(&sm->empty[stage]);  // frees the B stage once these MMAs retire
          }
          __syncwarp();
          if (++stage == NS) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) mma_commit(&sm->tm_full[acc]);  // accumulator ready
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (lane == 0) mma_commit(&sm->a_empty);  // A block may be replaced
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..9)
    const int e = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int half = e >> 2;       // 128-column half of the 256-column tile
    const int ntiles128 = (K + 127) / 128;
    // per-warp 32x32 fp32 staging tile for the TMA store (SWIZZLE_128B: the
    // 16-byte chunk k of row r sits at chunk k ^ (r & 7))
    unsigned char* sb = smB + (size_t)NS * B_CHUNK + (size_t)e * 4096;
    float* c2s = reinterpret_cast<float*>(smB + (size_t)NS * B_CHUNK + EPI_WARPS * 4096) +
                 e * 128;
    uint32_t acc = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int mb = u % m_blocks, sp = u / m_blocks;
      const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
      const int q = mb * BM + quarter * 32 + lane;
      float q2r = 0.f, ir = 1.f;  // fp16 encoding of this row
      if (HALF && q < nq) { q2r = q2v[q]; ir = qinv[q]; }
      const float q2ir = q2r * ir;
      for (int t = t0; t < t1; ++t) {
        const int colh = t * BN + half * 128;
        // this half tile's |c|^2 terms: loaded before the accumulator wait so
        // their latency hides behind it, then kept in a per-warp smem copy
        float c2r[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int col = colh + c * 32 + lane;
          c2r[c] = col < K ? __ldg(c2 + col) : 0.f;
        }
        mbar_wait(&sm->tm_full[acc], acc_phase);
        fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) c2s[c * 32 + lane] = c2r[c];
        __syncwarp();
        float* drow = HALF ? nullptr : D + (int64_t)q * ldD;
        uint16_t* hrow = HALF ? D16 + (int64_t)q * ldD : nullptr;
        float mn = __int_as_float(0x7f800000);
        __half2 mn2 = __floats2half2_rn(mn, mn);  // HALF: minimum in the encoded domain
        const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * 128;
        uint32_t ra[32], rb[32];
        tmem_ld32_async(tb, ra);
        tmem_wait_ld(ra);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t* r = (c & 1) ? rb : ra;
          uint32_t* rn = (c & 1) ? ra : rb;
          if (c < 3) tmem_ld32_async(tb + (c + 1) * 32, rn);  // next chunk in flight
          const int col0 = colh + c * 32;
          float v[32];
          if (col0 + 32 <= K) {
            const float4* c24 = reinterpret_cast<const float4*>(c2s + c * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 cc = c24[i];  // smem broadcast
              v[4 * i] = fmaf(-2.f, __uint_as_float(r[4 * i]), cc.x);
              v[4 * i + 1] = fmaf(-2.f, __uint_as_float(r[4 * i + 1]), cc.y);
              v[4 * i + 2] = fmaf(-2.f, __uint_as_float(r[4 * i + 2]), cc.z);
              v[4 * i + 3] = fmaf(-2.f, __uint_as_float(r[4 * i + 3]), cc.w);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int col = col0 + i;
              v[i] = col < K ? fmaf(-2.f, __uint_as_float(r[i]), __ldg(c2 + col))
                             : __int_as_float(0x7f800000);
            }
          }
          if constexpr (HALF) {
            // (v + |q|^2) * 2^-e as one FMA (exact scaling), packed f16x2
            // conversion and a packed running minimum
            uint32_t hp[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const __half2 h = __floats2half2_rn(fmaf(v[2 * i], ir, q2ir), fmaf(v[2 * i + 1], ir, q2ir));
              mn2 = __hmin2(mn2, h);
              hp[i] = *reinterpret_cast<const uint32_t*>(&h);
            }
            if (use_tma_store) {
              // two 32-column chunks per 32 x 64 staging tile (128 B rows,
              // SWIZZLE_128B: 16-byte chunk k of row r at k ^ (r & 7)), one
              // TMA store per pair of chunks
              if ((c & 1) == 0) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int kk = (c & 1) * 4 + k;
                *reinterpret_cast<uint4*>(sb + lane * 128 + ((kk ^ (lane & 7)) * 16)) =
                    make_uint4(hp[4 * k], hp[4 * k + 1], hp[4 * k + 2], hp[4 * k + 3]);
              }
              if (c & 1) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                  asm volatile(
                      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                          reinterpret_cast<uint64_t>(&mapD)),
                      "r"(col0 - 32), "r"(mb * BM + quarter * 32), "r"(smem_u32(sb))
                      : "memory");
                  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
              }
            } else if (q < nq) {
              if (col0 + 32 <= K && (ldD & 7) == 0) {
                uint4* dst = reinterpret_cast<uint4*>(hrow + col0);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  dst[k] = make_uint4(hp[4 * k], hp[4 * k + 1], hp[4 * k + 2], hp[4 * k + 3]);
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < K) hrow[col0 + i] = (uint16_t)(hp[i >> 1] >> ((i & 1) * 16));
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) mn = fminf(mn, v[i]);
            if (use_tma_store) {
              // the previous store from this staging tile has read it
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
#pragma unroll
              for (int k = 0; k < 8; ++k)
                *reinterpret_cast<float4*>(sb + lane * 128 + ((k ^ (lane & 7)) * 16)) =
                    make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                        reinterpret_cast<uint64_t>(&mapD)),
                    "r"(col0), "r"(mb * BM + quarter * 32), "r"(smem_u32(sb))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              }
            } else if (q < nq) {
              if (col0 + 32 <= K) {
                float4* dst = reinterpret_cast<float4*>(drow + col0);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < K) drow[col0 + i] = v[i];
              }
            }
          }
          if (c < 3) tmem_wait_ld(rn);
        }
        const int h = t * 2 + half;  // this warp's 128-centroid tile
        if (q < nq && tmin && h < ntiles128) {
          if (HALF)  // the tile minimum's fp16 code
            reinterpret_cast<uint16_t*>(tmin)[(int64_t)q * ntiles128 + h] =
                __half_as_ushort(__hmin(__low2half(mn2), __high2half(mn2)));
          else
            tmin[(int64_t)q * ntiles128 + h] = mn;
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm->tm_empty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    if (use_tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// Operand layouts ("reuse" split, 3 bf16 products per score):
//   B' (centroids, row width KB * 64): [c_hi (d) | c_lo (d) | 0 pad]
//   A' (queries, KA * 64): for every 64-column chunk j of B', an A chunk
//     hi_j with q_hi at the dimension of each column (c_hi and c_lo columns
//     alike), then -- when chunk j holds c_hi columns -- a chunk lo_j with
//     q_lo at the c_hi columns and 0 elsewhere.
// So sum_j hi_j . B_j + lo_j . B_j = q_hi.c_hi + q_hi.c_lo + q_lo.c_hi, and
// every B chunk crosses L2 -> SMEM once for its one or two MMAs: 2d columns
// of B per tile instead of 3d.
__host__ __device__ inline int tc_kb(int d) { return (2 * d + 63) / 64; }
__host__ __device__ inline int tc_lo_chunks(int d) { return (d + 63) / 64; }
__host__ __device__ inline int tc_ka(int d) { return tc_kb(d) + tc_lo_chunks(d); }

__global__ void k_split_bf16(const float* __restrict__ x, int rows, int d, int Kp, int centroid,
                             __nv_bfloat16* __restrict__ out) {
  const int64_t n = (int64_t)rows * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Kp;
    const int c = (int)(e % Kp);
    int bc = -1;       // column of B' this element pairs with
    bool lo = false;   // A' lo chunk (q_lo at c_hi columns)
    if (centroid) {
      bc = c;
    } else {
      int a = c >> 6, j = 0;  // A' chunk a -> (B' chunk j, hi / lo)
      for (; j < tc_kb(d); ++j) {
        if (a == 0) break;
        --a;
        if (j < tc_lo_chunks(d)) {
          if (a == 0) { lo = true; break; }
          --a;
        }
      }
      bc = j * 64 + (c & 63);
    }
    float v = 0.f;
    if (bc < 2 * d) {
      const bool chi = bc < d;  // c_hi column (else c_lo)
      const int dim = chi ? bc : bc - d;
      const float f = x[r * d + dim];
      const float hi = __bfloat162float(__float2bfloat16_rn(f));
      const float flo = __bfloat162float(__float2bfloat16_rn(f - hi));
      if (centroid) v = chi ? hi : flo;
      else if (!lo) v = hi;
      else v = chi ? flo : 0.f;
    }
    out[e] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------- host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

// bf16 operand (rows x cols of a pitch-`pitch` matrix) loaded in
// box_cols x box_rows boxes: 64 columns with SWIZZLE_128B or 32 with SWIZZLE_64B.
bool make_map(CUtensorMap* m, const void* ptr, int64_t rows, int cols, int pitch, int box_cols,
              int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Score matrix (rows x cols, pitch ld elements) written in 32 x 32 boxes from
// swizzled staging tiles: fp32 (128 B rows, SWIZZLE_128B) or fp16 (64 B
// rows, SWIZZLE_64B).
bool make_map_out(CUtensorMap* m, void* ptr, int64_t rows, int cols, int64_t ld, bool half,
                  int half_box = 32) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * (half ? 2 : 4)};
  cuuint32_t box[2] = {(cuuint32_t)(half ? half_box : 32), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (half && half_box == 32) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() { return num_sms_cur(); }

}  // namespace

// Row widths of the split operands (tc_ka / tc_kb layout above).
int tc_kpad(int d) { return tc_ka(d) * tc::BK; }    // queries (A')
int tc_kpad_b(int d) { return tc_kb(d) * tc::BK; }  // centroids (B')

size_t tc_smem_bytes(int d);
// A block resident (<= 96 KB) next to the B ring and the epilogue staging
bool tc_supported(int d) { return tc_ka(d) <= 6 && tc_smem_bytes(d) <= 227 * 1024; }

void launch_split_bf16(const float* x, int rows, int d, int centroid, void* out, cudaStream_t s) {
  const int Kp = centroid ? tc_kpad_b(d) : tc_kpad(d);
  int64_t n = (int64_t)rows * Kp;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_split_bf16<<<blocks, 256, 0, s>>>(x, rows, d, Kp, centroid,
                                      reinterpret_cast<__nv_bfloat16*>(out));
}

// B ring depth: 3, or 2 when a 6-chunk resident A block (d > 106) leaves no
// room for the third stage
int tc_stages(int d) { return tc_ka(d) >= 6 ? 2 : tc::STAGES; }
size_t tc_smem_bytes(int d) {
  const int KC = tc_ka(d);
  return 1024 + (size_t)KC * tc::A_CHUNK + (size_t)tc_stages(d) * tc::B_CHUNK + tc::STAGE_OUT +
         sizeof(tc::Smem) + 64;
}

bool launch_probe_gemm_tc(const void* Abf, const void* Bbf, const float* c2, int nq, int K, int d,
                          const ScoreOut& o, float* tmin, cudaStream_t s) {
  const int ka = tc_kpad(d), kb = tc_kpad_b(d);
  const bool half = o.D16 != nullptr;
  CUtensorMap ma, mb, md;
  if (!make_map(&ma, Abf, nq, ka, ka, tc::BK, tc::BM) ||
      !make_map(&mb, Bbf, K, kb, kb, tc::BK, tc::BN))
    return false;
  // scores go out through TMA stores when the row pitch allows it (16 B)
  void* dptr = half ? (void*)o.D16 : (void*)o.D32;
  int use_tma_store = ((o.ld * (half ? 2 : 4)) % 16 == 0) ? 1 : 0;
  if (use_tma_store && !make_map_out(&md, dptr, nq, K, o.ld, half, 64)) use_tma_store = 0;
  if (!use_tma_store) md = ma;  // unused
  const int m_units = (nq + tc::BM - 1) / tc::BM;
  const int n_tiles = (K + tc::BN - 1) / tc::BN;
  const int sms = num_sms();
  // Work units = (m-block, slice of the n-tiles), spread over one CTA per
  // SM.  Pick the slice count that minimises the busiest CTA's tiles, with
  // one tile's worth of overhead per unit (its A-block load):
  //   cost(ns) = ceil(m_units * ns / sms) * (ceil(n_tiles / ns) + 1)
  // (C2: 16 slices -> 9 units of 16 tiles per CTA, 5 % above the even
  // split; a fixed ~2 units per SM left a third of the SMs a unit behind).
  int nsplit = 1;
  {
    int64_t best = -1;
    for (int ns = 1; ns <= n_tiles; ++ns) {
      const int64_t per_cta = ((int64_t)m_units * ns + sms - 1) / sms;
      const int64_t cost = per_cta * ((n_tiles + ns - 1) / ns + 1);
      if (best < 0 || cost < best) { best = cost; nsplit = ns; }
    }
    if (const char* e = getenv("GIVF_GEMM_SPLIT")) nsplit = std::max(1, std::min(n_tiles, atoi(e)));
  }
  const int units = m_units * nsplit;
  const int grid = std::min(units, sms);
  const size_t smem = tc_smem_bytes(d);
  const bool ns2 = tc_stages(d) == 2;
  auto kern = half ? (ns2 ? k_probe_gemm_tc<true, 2> : k_probe_gemm_tc<true, 3>)
                   : (ns2 ? k_probe_gemm_tc<false, 2> : k_probe_gemm_tc<false, 3>);
  if (ensure_max_smem((const void*)kern, smem) != cudaSuccess) return false;
  kern<<<grid, tc::THREADS, smem, s>>>(ma, mb, md, use_tma_store, c2, nq, K, tc_ka(d), tc_kb(d),
                                       tc_lo_chunks(d), nsplit, o.D32, o.D16, o.ld, o.q2, o.qinv,
                                       o.qscale, tmin);
  return true;
}

}  // namespace givf
