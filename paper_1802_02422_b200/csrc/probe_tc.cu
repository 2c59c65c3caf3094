// K1a on the 5th-generation tensor cores: s~[q, c] = |c|^2 - 2 q.c for a
// block of queries against all K centroids (reference: search.py:77-90).
//
// Precision: fp32 inputs are split into bf16 pairs x = x_hi + x_lo, and
//   q.c ~ q_hi.c_hi + q_hi.c_lo + q_lo.c_hi
// is ONE bf16 GEMM over a concatenated K axis: A' = [q_hi | q_hi | q_lo],
// B' = [c_hi | c_lo | c_hi] (3d columns, zero-padded to a multiple of 64),
// accumulated in fp32 in TMEM.  Its error is bounded a priori (eps_scale in
// capi.cu) and every decision taken from s~ is re-checked in float64
// (probe_recheck, k_plan_approx), so the result stays exact.
//
// Kernel shape (sm_100a, one CTA per SM, persistent):
//   tile = 128 queries x 256 centroids, UMMA 128x256x16, cta_group::1
//   warp 0  TMA producer: the 128 x K' A block once per work unit (resident
//           in smem), then B chunks of 256 x 64 through a 4-stage ring
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

#include "common.cuh"
#include "kernels.h"

namespace givf {

namespace tc {

constexpr int BM = 128, BN = 256, BK = 64;  // BK bf16 = 128 B = one swizzle row
constexpr int STAGES = 3;
constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, one 128-column half each
// epilogue smem: TMA-store staging (one 4 KB tile per warp) + per-warp |c|^2
constexpr uint32_t STAGE_OUT = EPI_WARPS * 4096 + EPI_WARPS * 128 * 4;
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr uint32_t A_CHUNK = BM * BK * 2;   // 16 KB
constexpr uint32_t B_CHUNK = BN * BK * 2;   // 32 KB
constexpr int TMEM_COLS = 512;              // two 256-column fp32 accumulators

GIVF_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

GIVF_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
GIVF_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
GIVF_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
GIVF_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

GIVF_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

GIVF_DEV void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
GIVF_DEV void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SWIZZLE_128B K-major operand: 8-row x 128 B atoms, atoms 1024 B apart.
GIVF_DEV uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)1 << 16;                  // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // stride byte offset: next 8-row atom
  d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major, M x N.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

GIVF_DEV void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

GIVF_DEV void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

GIVF_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Asynchronous variant: the registers are valid only after tmem_wait_ld(r),
// which names them so no use can be scheduled before the wait.
GIVF_DEV void tmem_ld32_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
GIVF_DEV void tmem_wait_ld(uint32_t* r) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
        "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
        "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]),
        "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]),
        "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :
      : "memory");
}

struct Smem {
  uint64_t full[STAGES], empty[STAGES];
  uint64_t a_full, a_empty;
  uint64_t tm_full[2], tm_empty[2];
  uint32_t tmem_base;
};

}  // namespace tc

// smem: [A resident: KC x 16 KB][B ring: STAGES x 32 KB][barriers]
// HALF: scores leave as fp16 (ScoreOut in kernels.h), else fp32.
template <bool HALF>
__global__ void __launch_bounds__(tc::THREADS, 1)
k_probe_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                const __grid_constant__ CUtensorMap mapD, int use_tma_store,
                const float* __restrict__ c2, int nq, int K, int KC, int nsplit,
                float* __restrict__ D, uint16_t* __restrict__ D16, int64_t ldD,
                const float* __restrict__ q2v, const float* __restrict__ qinv,
                const float* __restrict__ qscale, float* __restrict__ tmin) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char dsm[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(dsm) + 1023) & ~(uintptr_t)1023);
  unsigned char* smA = base;
  unsigned char* smB = base + (size_t)KC * A_CHUNK;
  Smem* sm = reinterpret_cast<Smem*>(smB + (size_t)STAGES * B_CHUNK + STAGE_OUT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_blocks = (nq + BM - 1) / BM;
  const int n_tiles = (K + BN - 1) / BN;
  const int units = m_blocks * nsplit;
  const int per_split = (n_tiles + nsplit - 1) / nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sm->full[s], 1); mbar_init(&sm->empty[s], 1); }
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
        const int mb = u / nsplit, sp = u % nsplit;
        const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
        if (t0 >= t1) continue;
        mbar_wait(&sm->a_empty, a_phase ^ 1);
        a_phase ^= 1;
        mbar_expect_tx(&sm->a_full, (uint32_t)KC * A_CHUNK);
        for (int kc = 0; kc < KC; ++kc)
          tma_load_2d(smA + (size_t)kc * A_CHUNK, &mapA, &sm->a_full, kc * BK, mb * BM);
        for (int t = t0; t < t1; ++t) {
          for (int kc = 0; kc < KC; ++kc) {
            mbar_wait(&sm->empty[stage], phase ^ 1);
            mbar_expect_tx(&sm->full[stage], B_CHUNK);
            tma_load_2d(smB + (size_t)stage * B_CHUNK, &mapB, &sm->full[stage], kc * BK, t * BN);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    uint32_t stage = 0, phase = 0, a_phase = 0, acc = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int sp = u % nsplit;
      const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
      if (t0 >= t1) continue;
      mbar_wait(&sm->a_full, a_phase);
      a_phase ^= 1;
      fence_after();
      for (int t = t0; t < t1; ++t) {
        mbar_wait(&sm->tm_empty[acc], acc_phase ^ 1);
        fence_after();
        const uint32_t dcol = tmem + acc * BN;
        for (int kc = 0; kc < KC; ++kc) {
          mbar_wait(&sm->full[stage], phase);
          fence_after();
          if (lane == 0) {
            const uint32_t a0 = smem_u32(smA + (size_t)kc * A_CHUNK);
            const uint32_t b0 = smem_u32(smB + (size_t)stage * B_CHUNK);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_bf16(dcol, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32),
                       (kc | k) != 0 ? 1u : 0u);
            mma_commit(&sm->empty[stage]);  // frees the B stage once these MMAs retire
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
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
    unsigned char* sb = smB + (size_t)STAGES * B_CHUNK + (size_t)e * 4096;
    float* c2s = reinterpret_cast<float*>(smB + (size_t)STAGES * B_CHUNK + EPI_WARPS * 4096) +
                 e * 128;
    uint32_t acc = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int mb = u / nsplit, sp = u % nsplit;
      const int t0 = sp * per_split, t1 = min(n_tiles, t0 + per_split);
      const int q = mb * BM + quarter * 32 + lane;
      float q2r = 0.f, ir = 1.f, sr = 1.f;  // fp16 encoding of this row
      if (HALF && q < nq) { q2r = q2v[q]; ir = qinv[q]; sr = qscale[q]; }
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
        float mn = __int_as_float(0x7f800000);  // (HALF: in the encoded domain)
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
            uint32_t hp[16];  // 32 encoded scores, packed in pairs
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const __half h0 = __float2half_rn((v[2 * i] + q2r) * ir);
              const __half h1 = __float2half_rn((v[2 * i + 1] + q2r) * ir);
              mn = fminf(mn, fminf(__half2float(h0), __half2float(h1)));
              hp[i] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
            }
            if (use_tma_store) {
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
              // 32 rows x 64 B, SWIZZLE_64B: chunk k of row r at k ^ ((r >> 1) & 3)
#pragma unroll
              for (int k = 0; k < 4; ++k)
                *reinterpret_cast<uint4*>(sb + lane * 64 + ((k ^ ((lane >> 1) & 3)) * 16)) =
                    make_uint4(hp[4 * k], hp[4 * k + 1], hp[4 * k + 2], hp[4 * k + 3]);
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
        if (HALF) mn = fmaf(mn, sr, -q2r);  // decoded like every stored score
        if (q < nq && tmin && h < ntiles128) tmin[(int64_t)q * ntiles128 + h] = mn;
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

// A' / B' rows: [x_hi | x_hi | x_lo] (queries) or [x_hi | x_lo | x_hi]
// (centroids), bf16, zero-padded to Kp columns.
__global__ void k_split_bf16(const float* __restrict__ x, int rows, int d, int Kp, int centroid,
                             __nv_bfloat16* __restrict__ out) {
  const int64_t n = (int64_t)rows * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Kp;
    const int c = (int)(e % Kp);
    float v = 0.f;
    if (c < 3 * d) {
      const int part = c / d, j = c % d;
      const float f = x[r * d + j];
      const __nv_bfloat16 hi = __float2bfloat16_rn(f);
      const bool take_lo = centroid ? (part == 1) : (part == 2);
      v = take_lo ? __bfloat162float(__float2bfloat16_rn(f - __bfloat162float(hi)))
                  : __bfloat162float(hi);
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

bool make_map(CUtensorMap* m, const void* ptr, int64_t rows, int Kp, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)Kp * 2};
  cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Score matrix (rows x cols, pitch ld elements) written in 32 x 32 boxes from
// swizzled staging tiles: fp32 (128 B rows, SWIZZLE_128B) or fp16 (64 B
// rows, SWIZZLE_64B).
bool make_map_out(CUtensorMap* m, void* ptr, int64_t rows, int cols, int64_t ld, bool half) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * (half ? 2 : 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   half ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

int tc_kpad(int d) { return ((3 * d + tc::BK - 1) / tc::BK) * tc::BK; }

bool tc_supported(int d) { return tc_kpad(d) <= 6 * tc::BK; }  // A block resident (<= 96 KB)

void launch_split_bf16(const float* x, int rows, int d, int centroid, void* out, cudaStream_t s) {
  const int Kp = tc_kpad(d);
  int64_t n = (int64_t)rows * Kp;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_split_bf16<<<blocks, 256, 0, s>>>(x, rows, d, Kp, centroid,
                                      reinterpret_cast<__nv_bfloat16*>(out));
}

size_t tc_smem_bytes(int d) {
  const int KC = tc_kpad(d) / tc::BK;
  return 1024 + (size_t)KC * tc::A_CHUNK + (size_t)tc::STAGES * tc::B_CHUNK + tc::STAGE_OUT +
         sizeof(tc::Smem) + 64;
}

bool launch_probe_gemm_tc(const void* Abf, const void* Bbf, const float* c2, int nq, int K, int d,
                          const ScoreOut& o, float* tmin, cudaStream_t s) {
  const int Kp = tc_kpad(d);
  const bool half = o.D16 != nullptr;
  CUtensorMap ma, mb, md;
  if (!make_map(&ma, Abf, nq, Kp, tc::BM) || !make_map(&mb, Bbf, K, Kp, tc::BN)) return false;
  // scores go out through TMA stores when the row pitch allows it (16 B)
  void* dptr = half ? (void*)o.D16 : (void*)o.D32;
  int use_tma_store = ((o.ld * (half ? 2 : 4)) % 16 == 0) ? 1 : 0;
  if (use_tma_store && !make_map_out(&md, dptr, nq, K, o.ld, half)) use_tma_store = 0;
  if (!use_tma_store) md = ma;  // unused
  const int KC = Kp / tc::BK;
  const int m_blocks = (nq + tc::BM - 1) / tc::BM;
  const int n_tiles = (K + tc::BN - 1) / tc::BN;
  const int sms = num_sms();
  int nsplit = std::max(1, std::min(n_tiles, (2 * sms + m_blocks - 1) / m_blocks));
  const int units = m_blocks * nsplit;
  const int grid = std::min(units, sms);
  const size_t smem = tc_smem_bytes(d);
  auto kern = half ? k_probe_gemm_tc<true> : k_probe_gemm_tc<false>;
  static size_t attr[2] = {0, 0};
  if (attr[half] < smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[half] = smem;
  }
  kern<<<grid, tc::THREADS, smem, s>>>(ma, mb, md, use_tma_store, c2, nq, K, KC, nsplit, o.D32,
                                       o.D16, o.ld, o.q2, o.qinv, o.qscale, tmin);
  return true;
}

}  // namespace givf
