// Shared device helpers for the grouped-IVF search path (sm_100a).
//
// Order-preserving integer keys, IEEE-exact float64 arithmetic (no FMA
// contraction, matching numpy's separately rounded ops), block-wide
// reductions / scans and a bitonic sorter that works on shared OR global
// memory through generic pointers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define GIVF_DEV __device__ __forceinline__

namespace givf {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- keys
// Monotone float -> unsigned maps: a < b  <=>  key(a) < key(b) for non-NaN.
// -0.0 is folded onto +0.0 first so that, as in numpy's lexsort, the two
// zeros tie and the secondary key (id / position) decides.
GIVF_DEV uint32_t f32_key(float f) {
  uint32_t u = __float_as_uint(f == 0.0f ? 0.0f : f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
GIVF_DEV float key_f32(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
GIVF_DEV uint64_t f64_key(double d) {
  uint64_t u = (uint64_t)__double_as_longlong(d == 0.0 ? 0.0 : d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
// (distance, id) composite used by every top-k / rerank sort: ids are
// non-negative int32, so the low word orders them correctly.
GIVF_DEV uint64_t dist_id_key(float dist, int32_t id) {
  return ((uint64_t)f32_key(dist) << 32) | (uint32_t)id;
}
constexpr uint64_t kKeyPad = 0xffffffffffffffffull;

// ---------------------------------------------------------------- f64 ops
// numpy evaluates every float64 expression one rounded op at a time; the
// intrinsics keep nvcc from contracting a*b+c into an FMA.
GIVF_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
GIVF_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
GIVF_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }

// ---------------------------------------------------------------- warp/block
template <typename T>
GIVF_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
GIVF_DEV T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
template <typename T>
GIVF_DEV T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Block reductions; `red` must hold >= 32 elements of T.  All threads get the
// result.  Callable from uniform control flow only.
template <typename T>
__device__ T block_min(T v, T* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T r = red[0];
  for (int i = 1; i < nw; ++i) r = red[i] < r ? red[i] : r;
  __syncthreads();
  return r;
}
template <typename T>
__device__ T block_max(T v, T* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T r = red[0];
  for (int i = 1; i < nw; ++i) r = red[i] > r ? red[i] : r;
  __syncthreads();
  return r;
}
template <typename T>
__device__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T r = red[0];
  for (int i = 1; i < nw; ++i) r += red[i];
  __syncthreads();
  return r;
}

// Exclusive scan of one value per thread; returns the thread's exclusive
// prefix and writes the block total to *total.  `red` >= 33 elements.
template <typename T>
__device__ T block_exclusive_scan(T v, T* red, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    T acc = 0;
    for (int i = 0; i < nw; ++i) {
      T t = red[i];
      red[i] = acc;
      acc += t;
    }
    red[32] = acc;
  }
  __syncthreads();
  T r = red[wid] + x - v;
  *total = red[32];
  __syncthreads();
  return r;
}

GIVF_DEV uint32_t next_pow2(uint32_t x) {
  return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
}

// ---------------------------------------------------------------- bitonic
// Sort n (power of two) (key, val) pairs ascending by (key, val).  Pointers may
// address shared or global memory.  Block-synchronous.
template <typename K, typename V>
__device__ void bitonic_sort(K* key, V* val, uint32_t n) {
  for (uint32_t k = 2; k <= n; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        uint32_t lo = 2 * i - (i & (j - 1));
        uint32_t hi = lo + j;
        bool up = (lo & k) == 0;
        K ka = key[lo], kb = key[hi];
        V va = val[lo], vb = val[hi];
        bool gt = (ka > kb) || (ka == kb && va > vb);
        if (gt == up) {
          key[lo] = kb; key[hi] = ka;
          val[lo] = vb; val[hi] = va;
        }
      }
      __syncthreads();
    }
  }
}

// Keys only (composite keys that are already unique).
template <typename K>
__device__ void bitonic_sort_keys(K* key, uint32_t n) {
  for (uint32_t k = 2; k <= n; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        uint32_t lo = 2 * i - (i & (j - 1));
        uint32_t hi = lo + j;
        bool up = (lo & k) == 0;
        K ka = key[lo], kb = key[hi];
        if ((ka > kb) == up) { key[lo] = kb; key[hi] = ka; }
      }
      __syncthreads();
    }
  }
}

}  // namespace givf
