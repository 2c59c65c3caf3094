// Device helpers shared by the planner kernels (plan.cu, plan_approx.cu).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace givf {

// Optional per-phase cycle accounting of k_plan_approx (build with
// -DGIVF_PHASES): thread 0 of every CTA adds clock64 deltas to
// counters[8 + phase].
#ifdef GIVF_PHASES
#define PLAN_PHASE(i)                                                        \
  do {                                                                       \
    if (threadIdx.x == 0 && ix.counters) {                                   \
      long long now_ = clock64();                                            \
      atomicAdd(&ix.counters[8 + (i)], (unsigned long long)(now_ - t_phase_)); \
      t_phase_ = now_;                                                       \
    }                                                                        \
  } while (0)
#else
#define PLAN_PHASE(i) do { } while (0)
#endif

GIVF_DEV double key_to_f64(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// float64 |c - q|^2 by an 8-lane group (4 centroid rows in flight per warp):
// lanes stride the row in float4 steps, then a 3-level xor tree.
__device__ inline double group8_sqdist64(const float* __restrict__ c, const double* qd, int d) {
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
__device__ inline void group8_sqdist64_multi(const float* const* rows, const double* qd, int d4,
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

// The query's float64 coordinates this lane of an 8-lane group needs (float4
// columns gl, gl + 8, gl + 16, gl + 24; d % 4 == 0, d <= 128), held in
// registers across rows.
struct QLane {
  double v[4][4];
};
__device__ inline QLane load_qlane(const double* qd, int d4) {
  const int gl = threadIdx.x & 7;
  QLane q;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int j = gl + 8 * t;
#pragma unroll
    for (int i = 0; i < 4; ++i) q.v[t][i] = j < d4 ? qd[4 * j + i] : 0.0;
  }
  return q;
}

// group8_sqdist64_multi with the query in registers (same arithmetic order).
template <int U>
__device__ inline void group8_sqdist64_multi_q(const float* const* rows, const QLane& q, int d4,
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
        double t0 = dsub((double)v[u][t].x, q.v[t][0]), t1 = dsub((double)v[u][t].y, q.v[t][1]);
        double t2 = dsub((double)v[u][t].z, q.v[t][2]), t3 = dsub((double)v[u][t].w, q.v[t][3]);
        s = dadd(s, dadd(dadd(dmul(t0, t0), dmul(t1, t1)), dadd(dmul(t2, t2), dmul(t3, t3))));
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    out[u] = s;
  }
}

}  // namespace givf
