// Device pieces shared by the scan kernels (scan.cu, scan_async.cu): code
// rows in registers, numpy-order LUT sums, and the per-query LUT build.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace givf {

// A code row held in registers as 32-bit words (vector loads for M in
// {4, 8, 16, 32}) so the scan loop can keep the next rows' loads in flight.
template <int M>
struct CodeVec {
  static constexpr int W = (M + 3) / 4;
  uint32_t w[W];
  GIVF_DEV uint32_t byte(int j) const { return (w[j >> 2] >> ((j & 3) * 8)) & 0xffu; }
};

template <int M>
GIVF_DEV CodeVec<M> load_code(const uint8_t* __restrict__ codes, int64_t row) {
  CodeVec<M> v;
  if constexpr (M == 16) {
    uint4 x = __ldg(reinterpret_cast<const uint4*>(codes + row * 16));
    v.w[0] = x.x; v.w[1] = x.y; v.w[2] = x.z; v.w[3] = x.w;
  } else if constexpr (M == 8) {
    uint2 x = __ldg(reinterpret_cast<const uint2*>(codes + row * 8));
    v.w[0] = x.x; v.w[1] = x.y;
  } else if constexpr (M == 4) {
    v.w[0] = __ldg(reinterpret_cast<const uint32_t*>(codes + row * 4));
  } else if constexpr (M == 32) {
    const uint4* p = reinterpret_cast<const uint4*>(codes + row * 32);
    uint4 x = __ldg(p), y = __ldg(p + 1);
    v.w[0] = x.x; v.w[1] = x.y; v.w[2] = x.z; v.w[3] = x.w;
    v.w[4] = y.x; v.w[5] = y.y; v.w[6] = y.z; v.w[7] = y.w;
  } else {
#pragma unroll
    for (int i = 0; i < CodeVec<M>::W; ++i) v.w[i] = 0;
#pragma unroll
    for (int j = 0; j < M; ++j) v.w[j >> 2] |= (uint32_t)__ldg(codes + row * M + j) << ((j & 3) * 8);
  }
  return v;
}

// ip = sum of the M LUT entries in numpy's float32 reduction order: M < 8 a
// left-to-right sum; otherwise 8 running lanes r_j += e_{j+8i}, then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail in order.
// ip = sum of the M LUT entries in numpy's float32 reduction order: M < 8 a
// left-to-right sum; otherwise 8 running lanes r_j += e_{j+8i}, then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail in order.
template <int M>
GIVF_DEV float numpy_sum(const float (&e)[M]) {
  if constexpr (M < 8) {
    float r = e[0];
#pragma unroll
    for (int j = 1; j < M; ++j) r = __fadd_rn(r, e[j]);
    return r;
  } else {
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = e[j];
    constexpr int body = M - (M % 8);
#pragma unroll
    for (int i = 8; i < body; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], e[i + j]);
    float s = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
#pragma unroll
    for (int j = body; j < M; ++j) s = __fadd_rn(s, e[j]);
    return s;
  }
}

template <int M>
GIVF_DEV float code_sum(const CodeVec<M>& code, const float* lut) {
  float e[M];
#pragma unroll
  for (int j = 0; j < M; ++j) e[j] = lut[j * 256 + code.byte(j)];
  return numpy_sum<M>(e);
}

// Bank-conflict-free LUT reads (M in {8, 16}).  The LUT is stored
// "interleaved": xl[code * 32 + c * M + m] = LUT[m][code] for each of the
// 32 / M copies c, so entry (m, code) of copy c sits in bank c * M + m.
// Lane l reads copy c = l / M and, at step s, sub-quantizer m = s ^ x with
// x = l % M: the 32 lanes of a warp hit 32 distinct banks, one wavefront per
// step instead of ~3.1 for random codes in a [m][256] table.
//
// Slot s holds e_{s^x}.  XOR by a constant maps the pairs {t, t^8}, then
// {2t, 2t+1}, {4t..4t+3}, ... onto themselves, so numpy's tree over the
// slots adds exactly the same pairs as over e (in swapped order at most, and
// float addition is commutative): the sum is bit-identical to code_sum.
//
// The row's words are permuted by k ^ (x >> 2) in registers and byte
// (s & 3) ^ (x & 3) of word s >> 2 is extracted with a per-lane PRMT
// selector, so slot s reads byte s ^ x of the row.
// lane_base = shared-window address of the interleaved LUT + the lane's copy
// and column offset (c * M + x) * 4 (LUT base 128-byte aligned).
// xsel[j] = 0x4440 | (j ^ (x & 3)): the PRMT selector that extracts byte
// (j ^ (x & 3)) of a word, so only the words need permuting.
template <int M>
GIVF_DEV float code_sum_xl(const CodeVec<M>& code, uint32_t lane_base, int x,
                           const uint32_t (&xsel)[4]) {
  CodeVec<M> p;  // words by k ^ (x >> 2)
  const int xh = x >> 2;
  if constexpr (M == 16) {
    uint32_t t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = (xh & 1) ? code.w[k ^ 1] : code.w[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) p.w[k] = (xh & 2) ? t[k ^ 2] : t[k];
  } else {
#pragma unroll
    for (int k = 0; k < 2; ++k) p.w[k] = (xh & 1) ? code.w[k ^ 1] : code.w[k];
  }
  float e[M];
#pragma unroll
  for (int s = 0; s < M; ++s) {
    // base + (c*M + (s^x))*4 + byte*128 == (lane_base + byte*128) ^ (s*4):
    // bits 2..5 of lane_base hold x*4 and nothing else touches them
    const uint32_t byte = __byte_perm(p.w[s >> 2], 0, xsel[s & 3]);
    const uint32_t addr = (lane_base + (byte << 7)) ^ ((uint32_t)s << 2);
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e[s]) : "r"(addr));
  }
  return numpy_sum<M>(e);
}

// code_sum_xl with the per-step lane addresses precomputed: bs[s] =
// lane_base ^ (s << 2), so each lookup is PRMT + LEA + LDS.
template <int M, int SHIFT = 7>  // SHIFT = log2(bytes between the rows of consecutive codes)
GIVF_DEV float code_sum_xlb(const CodeVec<M>& code, const uint32_t (&bs)[M], int x,
                            const uint32_t (&xsel)[4]) {
  CodeVec<M> p;  // words by k ^ (x >> 2)
  const int xh = x >> 2;
  if constexpr (M == 16) {
    uint32_t t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) t[k] = (xh & 1) ? code.w[k ^ 1] : code.w[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) p.w[k] = (xh & 2) ? t[k ^ 2] : t[k];
  } else {
#pragma unroll
    for (int k = 0; k < 2; ++k) p.w[k] = (xh & 1) ? code.w[k ^ 1] : code.w[k];
  }
  float e[M];
#pragma unroll
  for (int s = 0; s < M; ++s) {
    const uint32_t byte = __byte_perm(p.w[s >> 2], 0, xsel[s & 3]);
    const uint32_t addr = bs[s] + (byte << SHIFT);
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e[s]) : "r"(addr));
  }
  return numpy_sum<M>(e);
}

// LUT of one query (pq.py:147-169): optional rotation q' = R q, then
// entry[m][i] = <q'_m, codeword[m][i]> accumulated in float64, rounded once;
// plus (ctab != null) the dequantized constants as float64 (grouping.py:123-129).
__device__ inline void build_lut_into(const IndexView& ix, const float* __restrict__ q, float* lut,
                                      double* ctab, float* qrot) {
  const int d = ix.d, M = ix.M, ds = d / M;
  if (ix.rotation) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      const float* r = ix.rotation + (int64_t)i * d;
      double acc = 0.0;
      for (int j = 0; j < d; ++j) acc += (double)r[j] * (double)q[j];
      qrot[i] = (float)acc;
    }
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) qrot[i] = q[i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < M * 256; e += blockDim.x) {
    int m = e >> 8;
    const float* cw = ix.codewords + (int64_t)e * ds;
    const float* qq = qrot + m * ds;
    double acc = 0.0;
    for (int t = 0; t < ds; ++t) acc += (double)cw[t] * (double)qq[t];
    lut[e] = (float)acc;
  }
  if (ctab)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) ctab[i] = (double)ix.ctab[i];
  __syncthreads();
}

}  // namespace givf
