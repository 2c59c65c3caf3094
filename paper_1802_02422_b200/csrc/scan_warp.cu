// K6 (default): ADC scan with warp-independent sweeps.
//
// Same results as k_scan (scan.cu): dist = f32(f64(base) - 2 f64(ip) +
// f64(const)) with ip summed in numpy's order, top-k by (dist, id)
// (search.py:142-158).  What changes is how the work is spread:
//
//  * The query's work list is taken in windows of SW_SEGS segments; the CTA
//    stages (start row, base, first position) of a window in shared memory
//    once.  The window's positions are split evenly between the 8 warps, and
//    each warp then runs without block barriers.
//  * A warp handles 32 consecutive positions at a time.  Lane l finds its
//    segment without any per-position table: lane j holds the first position
//    of the j-th following segment, one redux.or turns those into a bitmask
//    of segment starts inside the batch, and popc(mask below l) is the
//    lane's segment offset.  Code rows of consecutive positions are mostly
//    consecutive, so code / constant-byte loads stay coalesced; they are
//    staged by cp.async into a per-warp shared-memory ring (no register
//    copies waiting on loads) while the previous batch is summed.
//  * top-k: each warp keeps its own candidate buffer (dist key, row) and
//    shrinks it with a warp radix select to exactly k by (dist, id).  The
//    smallest k-th key over warps is shared (atomicMin in shared memory) and
//    filters every warp: all keys above it are out of the final top-k.
//  * The final merge takes the <= 8k entries under the shared bound, selects
//    exactly k of them with a block radix select and sorts only those.
//
// Used for M in {4, 8, 12, 16, 24, 32}, k <= SW_KMAX and local row indices
// < 2^32; k_scan covers everything else.
#include "common.cuh"
#include "kernels.h"
#include "scan_common.cuh"

#include <cstdlib>
#include <cstring>

namespace givf {

constexpr int SW_THREADS = 256;
constexpr int SW_WARPS = SW_THREADS / 32;
constexpr int SW_SEGS = 256;   // segments per window
constexpr int SW_WB = 256;     // per-warp candidate buffer (dist key << 32 | row)
constexpr int SW_KMAX = 128;   // SW_WARPS * SW_KMAX merge entries
constexpr unsigned FULL = 0xffffffffu;

// Shared memory: fixed-size parts first so every address is a constant
// offset (M is a template parameter; only qrot depends on the runtime d).
constexpr size_t SW_WBUF = 0;                                     // u64 [WARPS][WB]
constexpr size_t SW_MERGE = SW_WBUF + (size_t)SW_WARPS * SW_WB * 8;  // u64 [WARPS*KMAX]
constexpr size_t SW_SSTART = SW_MERGE + (size_t)SW_WARPS * SW_KMAX * 8;  // u32 [SEGS]
constexpr size_t SW_SBASE = SW_SSTART + (size_t)SW_SEGS * 4;      // f64 [SEGS]
constexpr size_t SW_SOFF = SW_SBASE + (size_t)SW_SEGS * 8;        // i32 [SEGS + 32]
constexpr size_t SW_CTAB = SW_SOFF + (size_t)(SW_SEGS + 32) * 4;  // f32 [256]
constexpr size_t SW_LUT = SW_CTAB + 256 * 4;                      // f32 [M][256]
// cp.async staging (CPA): per warp D slots x 32 lanes x (M code bytes + the
// 4-byte word holding the constant byte)
__host__ __device__ constexpr size_t sw_slot(int M) { return (size_t)32 * (M + 4); }
// LUT: [M][256] f32, or (XL) the interleaved copies of code_sum_xl, 32 KB
// (+128: the interleaved LUT's address is rounded up to 128 bytes, as the
// XOR addressing of code_sum_xl needs; dynamic shared memory is only
// guaranteed 16-byte alignment)
__host__ __device__ constexpr size_t sw_lut_bytes(int M, bool xl) { return xl ? 32768 + 128 : (size_t)M * 1024; }
__host__ __device__ constexpr size_t sw_ring(int M, bool xl) { return SW_LUT + sw_lut_bytes(M, xl); }
__host__ __device__ constexpr size_t sw_qrot(int M, int D, bool cpa, bool xl) {
  return sw_ring(M, xl) + (cpa ? (size_t)SW_WARPS * D * sw_slot(M) : 0);
}
// qrot (in-kernel LUT build) is only needed without prebuilt LUTs (never XL)
__host__ __device__ constexpr size_t sw_bytes(int M, int D, bool cpa, bool xl, int d) {
  return sw_qrot(M, D, cpa, xl) + (xl ? 0 : (((size_t)d * 4 + 15) & ~(size_t)15));
}

GIVF_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int N>
GIVF_DEV void cp_async(void* dst, const void* src) {
  if constexpr (N == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(smem_u32(dst)), "l"(src), "n"(N)
                 : "memory");
}
GIVF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
GIVF_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
template <int M>
constexpr int cp_chunk() { return M % 16 == 0 ? 16 : (M % 8 == 0 ? 8 : 4); }

// code row of M bytes (M % 4 == 0) from shared memory
template <int M>
GIVF_DEV CodeVec<M> smem_code(const uint8_t* p) {
  CodeVec<M> v;
  if constexpr (M % 16 == 0) {
#pragma unroll
    for (int i = 0; i < M / 16; ++i) {
      const uint4 x = reinterpret_cast<const uint4*>(p)[i];
      v.w[4 * i] = x.x; v.w[4 * i + 1] = x.y; v.w[4 * i + 2] = x.z; v.w[4 * i + 3] = x.w;
    }
  } else if constexpr (M % 8 == 0) {
#pragma unroll
    for (int i = 0; i < M / 8; ++i) {
      const uint2 x = reinterpret_cast<const uint2*>(p)[i];
      v.w[2 * i] = x.x; v.w[2 * i + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < M / 4; ++i) v.w[i] = reinterpret_cast<const uint32_t*>(p)[i];
  }
  return v;
}

// Ascending sort of n <= 128 keys by one warp: element e = 4 * lane + r in
// registers, bitonic network (partners inside a lane: register swaps; across
// lanes: xor shuffles), padded with kKeyPad; written back in place.
__device__ __forceinline__ void warp_sort128(uint64_t* keys, int n) {
  const int lane = threadIdx.x & 31;
  uint64_t v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) v[r] = 4 * lane + r < n ? keys[4 * lane + r] : kKeyPad;
#pragma unroll
  for (int size = 2; size <= 128; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j >= 4) {
        const int lj = j >> 2;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int e = 4 * lane + r;
          const bool asc = (e & size) == 0;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[r], lj);
          // the lower element of the pair keeps the min when ascending
          const bool take_min = lower == asc;
          v[r] = take_min ? (o < v[r] ? o : v[r]) : (o > v[r] ? o : v[r]);
        }
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int p = r ^ j;
          if (p > r) {
            const int e = 4 * lane + r;
            const bool asc = (e & size) == 0;
            const uint64_t a = v[r], b = v[p];
            const bool sw = asc ? (a > b) : (a < b);
            v[r] = sw ? b : a;
            v[p] = sw ? a : b;
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (4 * lane + r < n) keys[4 * lane + r] = v[r];
}

// Warp radix select: the digit-by-digit search for the need-th smallest of
// the 32-bit keys key_of(i), i < n, that match `prefix` under `mask` (hist:
// 256 words private to the warp).  Returns the key; *eq = how many of the n
// keys equal it, *need = its rank among those equal keys (1-based).
template <typename KeyOf>
__device__ uint32_t warp_select(int n, KeyOf key_of, uint32_t* hist, uint32_t* need, uint32_t* eq) {
  const int lane = threadIdx.x & 31;
  uint32_t prefix = 0, mask = 0;
  uint32_t last = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) hist[lane * 8 + j] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const uint32_t k = key_of(i);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t h[8], run = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { h[j] = hist[lane * 8 + j]; run += h[j]; }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - run;
    const bool mine = excl < *need && incl >= *need;
    const int src = __ffs(__ballot_sync(FULL, mine)) - 1;
    uint32_t digit = 0, before = 0, cnt = 0;
    if (mine) {
      uint32_t c = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (c + h[j] >= *need) { digit = lane * 8 + j; before = c; cnt = h[j]; break; }
        c += h[j];
      }
    }
    digit = __shfl_sync(FULL, digit, src);
    before = __shfl_sync(FULL, before, src);
    last = __shfl_sync(FULL, cnt, src);
    prefix |= digit << shift;
    mask |= 255u << shift;
    *need -= before;
    __syncwarp();
  }
  *eq = last;
  return prefix;
}

// Block-wide version (hist: 256 shared words; sh: 3 shared words).
template <typename KeyOf>
__device__ uint32_t block_select(int n, KeyOf key_of, uint32_t* hist, uint32_t* sh, uint32_t* need,
                                 uint32_t* eq) {
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t prefix = 0, mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
      const uint32_t k = key_of(i);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      uint32_t h[8], run = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { h[j] = hist[lane * 8 + j]; run += h[j]; }
      uint32_t incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl = incl - run;
      if (excl < *need && incl >= *need) {
        uint32_t c = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (c + h[j] >= *need) { sh[0] = lane * 8 + j; sh[1] = c; sh[2] = h[j]; break; }
          c += h[j];
        }
      }
    }
    __syncthreads();
    prefix |= sh[0] << shift;
    mask |= 255u << shift;
    *need -= sh[1];
    *eq = sh[2];
    __syncthreads();
  }
  return prefix;
}

// One warp's buffer cut to the entries whose distance key is <= T, where T
// is the upper edge of the (range-adaptive, <= 256-bin) histogram bin holding
// the k-th smallest key: >= k entries stay, usually few more.  One or two
// histogram passes and no id loads; T (all ids) becomes the warp's bound and
// is published to s_thr64.  Returns false (nothing changed) when more than
// `room` entries would stay (massive distance ties): use warp_shrink then.
//
// Quota bound (tw, k8 > 0): the first pass's histogram also gives the upper
// edge of the bin holding the k8-th smallest key: this warp holds >= k8
// entries at or below it, and keeps them (every later cut keeps its k-th
// smallest and everything below).  With k8 = ceil(k / WARPS) the largest of
// the warps' edges is a CTA-wide bound (>= k entries at or below it) as
// tight as the k-th of all rows scanned so far, long before any one warp's
// own k-th gets there.
__device__ __forceinline__ bool warp_cut(uint64_t* wb, int* cnt_io, uint32_t* thr, uint64_t* thr64,
                                         uint32_t* hist, int k, int room,
                                         unsigned long long* s_thr64, uint32_t* tw, int k8) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int cnt = *cnt_io;
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int i = lane; i < cnt; i += 32) {
    const uint32_t dk = (uint32_t)(wb[i] >> 32);
    mn = min(mn, dk);
    mx = max(mx, dk);
  }
  uint32_t lo = __reduce_min_sync(FULL, mn), hi = __reduce_max_sync(FULL, mx);
  uint32_t need = (uint32_t)k, taken = 0, T = hi;
  bool found = false;
  for (int pass = 0; pass < 4; ++pass) {
    const uint32_t range = hi - lo;
    const int shift = range == 0 ? 0 : max(0, 32 - __clz(range) - 8);
#pragma unroll
    for (int j = 0; j < 8; ++j) hist[lane * 8 + j] = 0;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
      const uint32_t dk = (uint32_t)(wb[i] >> 32);
      if (dk >= lo && dk <= hi) atomicAdd(&hist[(dk - lo) >> shift], 1u);
    }
    __syncwarp();
    uint32_t h[8], run = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { h[j] = hist[lane * 8 + j]; run += h[j]; }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - run;
    if (pass == 0 && k8 > 0) {  // the quota bound (see above)
      const uint32_t n8 = (uint32_t)k8;
      const bool m8 = excl < n8 && incl >= n8;
      const uint32_t bal8 = __ballot_sync(FULL, m8);
      if (bal8) {
        uint32_t b8 = 0;
        if (m8) {
          uint32_t c = excl;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (c + h[j] >= n8) { b8 = lane * 8 + j; break; }
            c += h[j];
          }
        }
        b8 = __shfl_sync(FULL, b8, __ffs(bal8) - 1);
        const uint64_t e8 = (uint64_t)lo + ((uint64_t)(b8 + 1) << shift) - 1;
        const uint32_t t8 = (uint32_t)(e8 < hi ? e8 : hi);
        if (lane == 0 && t8 < *tw) *(volatile uint32_t*)tw = t8;
      }
    }
    const bool mine = excl < need && incl >= need;
    const int src = __ffs(__ballot_sync(FULL, mine)) - 1;
    uint32_t bin = 0, before = 0, through = 0;
    if (mine) {
      uint32_t c = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (c + h[j] >= need) { bin = lane * 8 + j; before = c; through = c + h[j]; break; }
        c += h[j];
      }
    }
    bin = __shfl_sync(FULL, bin, src);
    before = __shfl_sync(FULL, before, src);
    through = __shfl_sync(FULL, through, src);
    __syncwarp();
    const uint32_t blo = lo + (bin << shift);
    const uint64_t bspan = (uint64_t)blo + ((1ull << shift) - 1);
    const uint32_t bhi = (uint32_t)(bspan < hi ? bspan : hi);
    if (taken + through <= (uint32_t)room) { T = bhi; found = true; break; }
    if (shift == 0) break;  // one distance key holds too many entries
    taken += before;
    need -= before;
    lo = blo;
    hi = bhi;
  }
  if (!found) return false;
  int out = 0;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t v = i < cnt ? wb[i] : kKeyPad;
    const bool keep = i < cnt && (uint32_t)(v >> 32) <= T;
    const uint32_t bal = __ballot_sync(FULL, keep);
    if (keep) wb[out + __popc(bal & lt_mask)] = v;
    out += __popc(bal);
  }
  __syncwarp();
  *cnt_io = out;
  *thr = T;
  *thr64 = ((uint64_t)T << 32) | 0xffffffffu;  // every id at distance key T
  if (lane == 0) atomicMin(s_thr64, (unsigned long long)*thr64);
  return true;
}

// One warp's buffer down to exactly min(cnt, k) entries by (dist key, id);
// the k-th key becomes the warp's threshold and is published to s_thr64.
__device__ __forceinline__ void warp_shrink(uint64_t* wb, int* cnt_io, uint32_t* thr, uint64_t* thr64,
                                         uint32_t* hist, const int32_t* __restrict__ pids, int k,
                                         unsigned long long* s_thr64) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int cnt = *cnt_io;
  uint32_t need = (uint32_t)k, eq = 0;
  const uint32_t kd = warp_select(cnt, [&](int i) { return (uint32_t)(wb[i] >> 32); }, hist, &need, &eq);
  uint32_t kp;  // id of the k-th key among the entries with dist key kd
  if (eq == need) {  // every tie is kept: the largest id among them
    uint32_t mx = 0;
    for (int i = lane; i < cnt; i += 32) {
      const uint64_t v = wb[i];
      if ((uint32_t)(v >> 32) == kd) mx = max(mx, (uint32_t)__ldg(pids + (uint32_t)v));
    }
    kp = __reduce_max_sync(FULL, mx);
  } else {
    uint32_t need2 = need, eq2;
    kp = warp_select(cnt, [&](int i) {
      const uint64_t v = wb[i];
      return (uint32_t)(v >> 32) == kd ? (uint32_t)__ldg(pids + (uint32_t)v) : 0xffffffffu;
    }, hist, &need2, &eq2);
  }
  int out = 0;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t v = i < cnt ? wb[i] : kKeyPad;
    const uint32_t dk = (uint32_t)(v >> 32);
    bool keep = i < cnt && dk <= kd;
    if (keep && dk == kd) keep = (uint32_t)__ldg(pids + (uint32_t)v) <= kp;
    const uint32_t bal = __ballot_sync(FULL, keep);
    if (keep) wb[out + __popc(bal & lt_mask)] = v;
    out += __popc(bal);
  }
  __syncwarp();
  *cnt_io = out;
  *thr = kd;
  *thr64 = ((uint64_t)kd << 32) | kp;
  if (lane == 0) atomicMin(s_thr64, (unsigned long long)*thr64);
}

// The end of a top-k scan: each warp's entries under the shared bound, ids
// resolved, then exactly min(total, k) of them by (dist, id) across the
// warps, written to the outputs.  Called by all threads after the warps'
// final shrink and a block barrier.
__device__ __forceinline__ void scan_final(const ScanArgs& a, int b, int k, uint64_t* wb, int cnt,
                                        unsigned char* dsm, uint64_t* merge, uint32_t* bh,
                                        unsigned long long* s_thr64_p, uint32_t* s_tw, int* s_wcnt,
                                        uint32_t* s_sel, int* s_nout_p) {
  const IndexView& ix = a.ix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  unsigned long long& s_thr64 = *s_thr64_p;
  int& s_nout = *s_nout_p;
  uint64_t T = s_thr64;
  {  // the quota bound (warp_cut) holds as well
    uint32_t qb = 0;
#pragma unroll
    for (int w = 0; w < SW_WARPS; ++w) qb = max(qb, s_tw[w]);
    const uint64_t tq = ((uint64_t)qb << 32) | 0xffffffffull;
    T = T < tq ? T : tq;
  }
  {
    // every id load of the warp in flight at once (cnt <= SW_WB)
    constexpr int R = SW_WB / 32;
    uint64_t vr[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int i = j * 32 + lane;
      uint64_t v = i < cnt ? wb[i] : kKeyPad;
      if (i < cnt && (v >> 32) <= (T >> 32))
        v = (v & 0xffffffff00000000ull) | (uint32_t)__ldg(ix.pids + (uint32_t)v);
      else
        v = kKeyPad;
      vr[j] = v;
    }
    int out = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool keep = vr[j] <= T;
      const uint32_t bal = __ballot_sync(FULL, keep);
      if (keep) wb[out + __popc(bal & lt_mask)] = vr[j];
      out += __popc(bal);
    }
    if (lane == 0) s_wcnt[warp] = out;
  }
  __syncthreads();
  uint64_t* const all = reinterpret_cast<uint64_t*>(dsm + SW_WBUF);
  auto slot_key = [&](int i) -> uint64_t {  // slot i of the warps' buffers
    return (i % SW_WB) < s_wcnt[i / SW_WB] ? all[i] : kKeyPad;
  };
  int nm = 0, myoff = 0;
  for (int w = 0; w < SW_WARPS; ++w) {
    if (w == warp) myoff = nm;
    nm += s_wcnt[w];
  }
  // usually the survivors fit the merge area: gather them there so the
  // selection below touches nm entries, not every buffer slot
  const bool compact = nm <= SW_WARPS * SW_KMAX;
  if (compact) {
    for (int i = lane; i < s_wcnt[warp]; i += 32) merge[myoff + i] = wb[i];
    __syncthreads();
  }
  auto key_at = [&](int i) -> uint64_t { return compact ? merge[i] : slot_key(i); };
  const int n_in = compact ? nm : SW_WARPS * SW_WB;
  uint64_t* fin = compact ? all : merge;
  int nf = 0;
  if (compact && nm <= 128) {  // few survivors: sort them all, keep the first k
    if (warp == 0) warp_sort128(merge, nm);
    __syncthreads();
    fin = merge;
    nf = min(nm, k);
  } else {
    uint64_t lim = kKeyPad;
    if (nm > k) {
      uint32_t need = (uint32_t)k, eq = 0;
      const uint32_t kd = block_select(n_in, [&](int i) { return (uint32_t)(key_at(i) >> 32); },
                                       bh, s_sel, &need, &eq);
      uint32_t kp = 0xffffffffu;
      if (eq != need) {
        uint32_t eq2;
        kp = block_select(n_in, [&](int i) {
          const uint64_t v = key_at(i);
          return (uint32_t)(v >> 32) == kd ? (uint32_t)v : 0xffffffffu;
        }, bh, s_sel, &need, &eq2);
      }
      lim = ((uint64_t)kd << 32) | kp;
    }
    if (tid == 0) s_nout = 0;
    __syncthreads();
    for (int i0 = 0; i0 < n_in; i0 += SW_THREADS) {
      const int i = i0 + tid;
      const uint64_t v = i < n_in ? key_at(i) : kKeyPad;
      const bool keep = v != kKeyPad && v <= lim;
      const uint32_t bal = __ballot_sync(FULL, keep);
      int base = 0;
      if (lane == 0 && bal) base = atomicAdd(&s_nout, __popc(bal));
      base = __shfl_sync(FULL, base, 0);
      if (keep) fin[base + __popc(bal & lt_mask)] = v;
    }
    __syncthreads();
    nf = s_nout;
    if (nf <= 128) {  // k <= SW_KMAX: one warp sorts in registers, no block barriers
      if (warp == 0) warp_sort128(fin, nf);
      __syncthreads();
    } else {
      const uint32_t np2 = next_pow2((uint32_t)max(nf, 1));
      for (uint32_t i = nf + tid; i < np2; i += SW_THREADS) fin[i] = kKeyPad;
      __syncthreads();
      bitonic_sort_keys(fin, np2);
    }
  }
  for (int i = tid; i < k; i += SW_THREADS) {
    int32_t id = -1;
    float dv = __int_as_float(0x7f800000);
    if (i < nf) {
      const uint64_t key = fin[i];
      id = (int32_t)(uint32_t)key;
      dv = key_f32((uint32_t)(key >> 32));
    }
    a.out_ids[(int64_t)b * k + i] = id;
    a.out_d[(int64_t)b * k + i] = dv;
  }
}

// FULLK: every scanned key to full_keys (mode 1), else top-k (mode 0)
template <int M, int U, bool CPA, bool XL, bool FULLK>
__global__ void __launch_bounds__(SW_THREADS, 3) k_scan_warp(ScanArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const IndexView& ix = a.ix;
  float* lut = reinterpret_cast<float*>(dsm + SW_LUT);
  if constexpr (XL)  // 128-byte aligned shared-window address
    lut += ((128u - (smem_u32(lut) & 127u)) & 127u) / 4u;
  float* ctab = reinterpret_cast<float*>(dsm + SW_CTAB);
  float* qrot = reinterpret_cast<float*>(dsm + sw_qrot(M, 2 * U, CPA, XL));
  uint32_t* sstart = reinterpret_cast<uint32_t*>(dsm + SW_SSTART);
  double* sbase = reinterpret_cast<double*>(dsm + SW_SBASE);
  int32_t* soff = reinterpret_cast<int32_t*>(dsm + SW_SOFF);
  uint64_t* merge = reinterpret_cast<uint64_t*>(dsm + SW_MERGE);
  __shared__ int32_t red32[40];
  __shared__ unsigned long long s_thr64;
  __shared__ int s_nmerge, s_nout;
  __shared__ int s_wcnt[SW_WARPS];
  __shared__ uint32_t s_sel[4];
  __shared__ __align__(16) uint32_t s_tw[SW_WARPS];  // per-warp quota bounds (warp_cut)
  static_assert(SW_WARPS == 8, "quota bound read as two uint4");

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int k = a.k;
  if constexpr (XL) {
    // prebuilt [m][256] -> interleaved copies.  Lane (sub, m) = (l / M, l % M)
    // reads 4 codes of row m and writes copy c = cc ^ sub: a warp's stores
    // cover 32 distinct banks
    constexpr int NC = 32 / M;
    const float4* src = reinterpret_cast<const float4*>(a.luts + (int64_t)b * M * 256);
    const int m = lane % M, sub = lane / M;
    // every load (and the constant table's) in flight before any store
    constexpr int IT = M * 64 / 32 / SW_WARPS;
    static_assert(IT * 32 * SW_WARPS == M * 64 && SW_THREADS == 256, "LUT copy shape");
    float4 v[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) v[it] = __ldg(src + m * 64 + NC * (warp + it * SW_WARPS) + sub);
    const float cv = ix.ctab[tid];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int chunk = NC * (warp + it * SW_WARPS) + sub;  // codes 4*chunk .. 4*chunk+3
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        float* dst = lut + (4 * chunk) * 32 + (cc ^ sub) * M + m;
        dst[0] = v[it].x; dst[32] = v[it].y; dst[64] = v[it].z; dst[96] = v[it].w;
      }
    }
    ctab[tid] = cv;
  } else if (a.luts) {  // prebuilt for the chunk (k_build_luts): one coalesced copy
    const uint4* src = reinterpret_cast<const uint4*>(a.luts + (int64_t)b * M * 256);
    uint4* dst = reinterpret_cast<uint4*>(lut);
#pragma unroll 4
    for (int i = tid; i < M * 64; i += SW_THREADS) dst[i] = __ldg(src + i);
  } else {
    build_lut_into(ix, a.Q + (int64_t)b * ix.d, lut, nullptr, qrot);
  }
  if constexpr (!XL)
    for (int i = tid; i < 256; i += SW_THREADS) ctab[i] = ix.ctab[i];
  if (tid == 0) { s_thr64 = kKeyPad; s_nmerge = 0; }
  if (tid < SW_WARPS) s_tw[tid] = 0xffffffffu;
  const int k8 = (k + SW_WARPS - 1) / SW_WARPS;

  uint64_t* wb = reinterpret_cast<uint64_t*>(dsm + SW_WBUF) + warp * SW_WB;
  uint32_t* hist = reinterpret_cast<uint32_t*>(merge) + warp * 256;
  int cnt = 0;
  uint32_t thr = 0xffffffffu;
  uint64_t thr64 = kKeyPad;
  // the bound as a float (+inf while it admits everything)
  auto f_of = [](uint32_t t) -> float {
    const float f = key_f32(t);
    return isnan(f) ? __int_as_float(0x7f800000) : f;
  };
  float thr_f = f_of(thr);
  const WorkItem* W = a.work + (int64_t)b * a.cap_w;
  const int nseg = a.nwork[b];
  uint64_t* fk = FULLK ? a.full_keys + (int64_t)b * a.cap_full_p2 : nullptr;
  // the histogram cut, with the exact id-resolving shrink for heavy ties
  auto shrink = [&](int room) {
    if (!warp_cut(wb, &cnt, &thr, &thr64, hist, k, room, &s_thr64, &s_tw[warp], FULLK ? 0 : k8))
      warp_shrink(wb, &cnt, &thr, &thr64, hist, ix.pids, k, &s_thr64);
  };

  uint8_t* ring = dsm + sw_ring(M, XL) + (size_t)warp * 2 * U * sw_slot(M);
  const int xl_x = lane % M;                                  // XL: column rotation
  // XL: the lane's copy and column inside the interleaved LUT
  const uint32_t xl_base = smem_u32(lut) + (uint32_t)((lane / M) * M + xl_x) * 4u;
  uint32_t xl_sel[4];  // XL: byte selectors (code_sum_xl)
#pragma unroll
  for (int j = 0; j < 4; ++j) xl_sel[j] = 0x4440u | (uint32_t)(j ^ (xl_x & 3));
  struct Slot {  // one batch position of a lane (CPA: code and cb in the ring)
    uint32_t row;
    double base;
    CodeVec<M> code;
    uint32_t cb;
    bool ok;
  };

  int64_t pos_base = 0;
  for (int s0 = 0; s0 < nseg; s0 += SW_SEGS) {
    const int ns = min(SW_SEGS, nseg - s0);
    __syncthreads();  // the previous window's readers are done (first: LUT ready)
    // SW_SEGS / SW_THREADS consecutive segments per thread
    constexpr int SPT = SW_SEGS / SW_THREADS;
    static_assert(SPT * SW_THREADS == SW_SEGS, "window = whole segments per thread");
    int lens[SPT], mine = 0;
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
      const int i = SPT * tid + j;
      lens[j] = 0;
      if (i < ns) {
        const WorkItem w = W[s0 + i];
        sstart[i] = (uint32_t)w.start;
        sbase[i] = w.base;
        lens[j] = w.len;
      }
      mine += lens[j];
    }
    int tot;
    int off = block_exclusive_scan(mine, red32, &tot);
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
      const int i = SPT * tid + j;
      soff[i] = i < ns ? off : INT_MAX;
      if (i < ns) sstart[i] -= (uint32_t)off;  // row of position p = sstart[seg] + p
      off += lens[j];
    }
    if (tid < 32) soff[SW_SEGS + tid] = INT_MAX;
    __syncthreads();
    const int pb = (int)((int64_t)tot * warp / SW_WARPS);
    const int pe = (int)((int64_t)tot * (warp + 1) / SW_WARPS);
    if (pb < pe) {
      int s_cur;
      {
        int lo = 0, hi = ns - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (soff[mid] <= pb) lo = mid; else hi = mid - 1;
        }
        s_cur = lo;
      }
      int s_last;  // segment of the warp's last position pe - 1
      {
        int lo = s_cur, hi = ns - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (soff[mid] <= pe - 1) lo = mid; else hi = mid - 1;
        }
        s_last = lo;
      }
      // positions p0 .. p0+31 -> (segment, row); advances s_cur past the batch
      auto map = [&](int p0, Slot& sl, int slot) {
        const int nxt = soff[s_cur + 1 + lane];
        const int rel = nxt - p0;
        const uint32_t bit = (rel >= 1 && rel <= 31) ? (1u << rel) : 0u;
        const uint32_t starts = __reduce_or_sync(FULL, bit);
        const int seg = s_cur + __popc(starts & (FULL >> (31 - lane)));
        const int p = p0 + lane;
        sl.ok = p < pe;
        // lanes past the end load the warp's last row (their segment is
        // capped the same way), so every load is issued unconditionally
        const int pc = min(p, pe - 1);
        const int sg = pc == p ? seg : s_last;
        sl.row = sstart[sg] + (uint32_t)pc;
        sl.base = sbase[sg];
        if constexpr (CPA) {
          uint8_t* dst = ring + slot * sw_slot(M);
          constexpr int CH = cp_chunk<M>();
          const uint8_t* src = ix.codes + (size_t)sl.row * M;
#pragma unroll
          for (int c = 0; c < M / CH; ++c) cp_async<CH>(dst + lane * M + c * CH, src + c * CH);
          cp_async<4>(dst + 32 * M + lane * 4, ix.cbytes + (sl.row & ~3u));
          cp_async_commit();
        } else {
          sl.code = load_code<M>(ix.codes, sl.row);
          sl.cb = __ldg(ix.cbytes + sl.row);
        }
        const int nst = __popc(starts);
        const int at32 = __shfl_sync(FULL, nxt, nst);
        s_cur += nst + (at32 - p0 == 32 ? 1 : 0);
      };
      auto dist_of = [&](const Slot& cur, int slot) -> float {
        CodeVec<M> code;
        uint32_t cb;
        if constexpr (CPA) {
          const uint8_t* src = ring + slot * sw_slot(M);
          code = smem_code<M>(src + lane * M);
          const uint32_t cw = reinterpret_cast<const uint32_t*>(src + 32 * M)[lane];
          cb = __byte_perm(cw, 0, 0x4440u | (cur.row & 3u));
        } else {
          code = cur.code;
          cb = cur.cb;
        }
        float ip;
        if constexpr (XL) ip = code_sum_xl<M>(code, xl_base, xl_x, xl_sel);
        else ip = code_sum<M>(code, lut);
        return (float)dadd(dsub(cur.base, 2.0 * (double)ip), (double)ctab[cb]);
      };
      auto consider = [&](const Slot& cur, float dist, int p0) {
        if constexpr (FULLK) {
          if (cur.ok) fk[pos_base + p0 + lane] = dist_id_key(dist, __ldg(ix.pids + cur.row));
          return;
        }
        // dist <= thr_f  <=>  f32_key(dist) <= thr (finite distances)
        bool pass = cur.ok && dist <= thr_f;
        // at dk == thr the id decides unless the bound admits every id
        if (pass && dist == thr_f && (uint32_t)thr64 != 0xffffffffu)
          pass = (((uint64_t)f32_key(dist) << 32) | (uint32_t)__ldg(ix.pids + cur.row)) < thr64;
        const uint32_t bal = __ballot_sync(FULL, pass);
        if (bal) {
          if (pass) wb[cnt + __popc(bal & lt_mask)] = ((uint64_t)f32_key(dist) << 32) | cur.row;
          cnt += __popc(bal);
        }
      };
      // Two groups of U batches: one group's loads are in flight while the
      // other's U independent sums are computed (interleaved by the compiler).
      constexpr int D = 2 * U;
      Slot sl[D];
#pragma unroll
      for (int i = 0; i < U; ++i) map(pb + 32 * i, sl[i], i);
      for (int p0 = pb; p0 < pe; p0 += 32 * D) {
        if constexpr (!FULLK) {  // adopt a tighter bound from the other warps
          // the quota bound: the largest of the warps' k8-th edges
          uint32_t q[8];
          asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]) : "r"(smem_u32(&s_tw[0])));
          asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]) : "r"(smem_u32(&s_tw[4])));
          const uint32_t qb = max(max(max(q[0], q[1]), max(q[2], q[3])), max(max(q[4], q[5]), max(q[6], q[7])));
          const uint64_t tq = ((uint64_t)qb << 32) | 0xffffffffull;
          const uint64_t ts = *(volatile unsigned long long*)&s_thr64;
          const uint64_t t = ts < tq ? ts : tq;
          if (t < thr64) { thr64 = t; thr = (uint32_t)(t >> 32); thr_f = f_of(thr); }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // batches past pe are all-invalid no-ops
          const int cur = h * U, nxt = (1 - h) * U;
#pragma unroll
          for (int i = 0; i < U; ++i) map(p0 + 32 * (U * (h + 1) + i), sl[nxt + i], nxt + i);
          if constexpr (CPA) cp_async_wait<U>();  // the current group landed
          float dv[U];
#pragma unroll
          for (int i = 0; i < U; ++i) dv[i] = dist_of(sl[cur + i], cur + i);
#pragma unroll
          for (int i = 0; i < U; ++i) consider(sl[cur + i], dv[i], p0 + 32 * (cur + i));
        }
        // <= D x 32 appends per iteration: room is kept for them
        if (cnt > SW_WB - 32 * D) {
          __syncwarp();
          shrink(SW_WB / 2);
          thr_f = f_of(thr);
        }
      }
      if constexpr (CPA) cp_async_wait<0>();  // prefetches past pe
    }
    pos_base += tot;
  }
  if constexpr (FULLK) return;

  // ---- final: each warp's entries under the shared bound, ids resolved,
  // then exactly min(total, k) of them by (dist, id) across the warps
  __syncwarp();
  if (cnt > k) shrink(k + 32);  // tight final bound: few survivors to merge
  __syncthreads();
  // every warp's bound holds >= k entries: entries above the smallest bound
  // are out; ids are loaded only for the survivors
  scan_final(a, b, k, wb, cnt, dsm, merge, reinterpret_cast<uint32_t*>(sstart), &s_thr64, s_tw,
             s_wcnt, s_sel, &s_nout);
}

// ---------------------------------------------------------------- lean
// k_scan_lean: the default top-k scan for M in {8, 16} (interleaved LUT,
// prebuilt LUTs, local rows < 2^32).  Same arithmetic, candidate buffers,
// bounds and final merge as k_scan_warp; what goes is the block-wide
// segment window (staging + two block barriers per 256 segments, ~25 % of
// the stall samples at configs[2]'s 15-row segments):
//  * every warp sums the query's segment lengths itself (coalesced, from L2)
//    and takes positions [tot w / 8, tot (w + 1) / 8);
//  * the warp's segment window lives in registers: lane j holds segment
//    ws + j (row offset and base); a batch maps lanes to segments with one
//    ballot (segments ending at or before the batch) and one redux.or
//    (segment ends inside it), then two shuffles fetch row and base;
//  * the window re-anchors (one coalesced load of 32 work items and a warp
//    scan) only when a batch runs past its last segment.
// C = LUT copies: 32 / M makes every lookup conflict-free (one bank per
// (copy, sub-quantizer)); fewer copies shrink the LUT (C M KB) at the price of
// bank conflicts between lanes that share a copy.
template <int M, int D, int C = 32 / M>
__global__ void __launch_bounds__(SW_THREADS, C == 32 / M ? 3 : 4) k_scan_lean(ScanArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const IndexView& ix = a.ix;
  float* lut = reinterpret_cast<float*>(dsm + SW_LUT);
  lut += ((128u - (smem_u32(lut) & 127u)) & 127u) / 4u;  // 128-byte aligned
  float* ctab = reinterpret_cast<float*>(dsm + SW_CTAB);
  uint64_t* merge = reinterpret_cast<uint64_t*>(dsm + SW_MERGE);
  __shared__ unsigned long long s_thr64;
  __shared__ int s_nout;
  __shared__ int s_wcnt[SW_WARPS];
  __shared__ uint32_t s_sel[4];
  __shared__ __align__(16) uint32_t s_tw[SW_WARPS];
  static_assert(M == 8 || M == 16, "interleaved LUT");

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int k = a.k;
  // prebuilt [m][256] -> interleaved copies (as in k_scan_warp).  The global
  // loads are issued first and stored to shared memory only after the window
  // setup below, whose own global loads then overlap them.
  constexpr int NC = 32 / M;
  const float4* src = reinterpret_cast<const float4*>(a.luts + (int64_t)b * M * 256);
  const int m = lane % M, sub = lane / M;
  constexpr int IT = M * 64 / 32 / SW_WARPS;
  float4 v[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) v[it] = __ldg(src + m * 64 + NC * (warp + it * SW_WARPS) + sub);
  const float cv = ix.ctab[tid];
  if (tid == 0) s_thr64 = kKeyPad;
  if (tid < SW_WARPS) s_tw[tid] = 0xffffffffu;
  const int k8 = (k + SW_WARPS - 1) / SW_WARPS;
  uint64_t* wb = reinterpret_cast<uint64_t*>(dsm + SW_WBUF) + warp * SW_WB;
  uint32_t* hist = reinterpret_cast<uint32_t*>(merge) + warp * 256;
  int cnt = 0;
  uint32_t thr = 0xffffffffu;
  uint64_t thr64 = kKeyPad;
  auto f_of = [](uint32_t t) -> float {
    const float f = key_f32(t);
    return isnan(f) ? __int_as_float(0x7f800000) : f;
  };
  float thr_f = f_of(thr);
  auto shrink = [&](int room) {
    if (!warp_cut(wb, &cnt, &thr, &thr64, hist, k, room, &s_thr64, &s_tw[warp], k8))
      warp_shrink(wb, &cnt, &thr, &thr64, hist, ix.pids, k, &s_thr64);
  };
  const WorkItem* W = a.work + (int64_t)b * a.cap_w;
  const int nseg = a.nwork[b];

  // ---- this warp's positions.  The lengths are summed window by window
  // (32 segments, one coalesced load); lane l keeps the total of windows
  // [l wpl, (l + 1) wpl), so the window holding the warp's first position is
  // found by one scan instead of a walk from segment 0 (a chain of dependent
  // loads: 11 % of the stall samples at configs[2]'s ~670 segments per query)
  const int nwin = (nseg + 31) >> 5;
  const int wpl = (nwin + 31) >> 5;  // windows per lane: 1 up to 1024 segments
  int csum = 0;
  {
    int owner = 0, left = wpl;
#pragma unroll 4
    for (int t = 0; t < nwin; ++t) {
      const int i = t * 32 + lane;
      const int ws_t = __reduce_add_sync(FULL, i < nseg ? __ldg(&W[i].len) : 0);
      if (lane == owner) csum += ws_t;
      if (--left == 0) { ++owner; left = wpl; }
    }
  }
  int cend = csum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, cend, o);
    if (lane >= o) cend += y;
  }
  const int tot = __shfl_sync(FULL, cend, 31);
  const int pb = (int)((int64_t)tot * warp / SW_WARPS);
  const int pe = (int)((int64_t)tot * (warp + 1) / SW_WARPS);
  const bool active = pb < pe;
  {
    // register window: lane j = segment ws + j; wend = its end position,
    // wadj = first row - first position (row of position p = wadj + p)
    int ws = 0, wend = 0, wlast = 0;
    uint32_t wadj = 0;
    double wbase = 0.0;
    auto fill = [&](int s0, int off0) {
      const int i = s0 + lane;
      int ln = 0;
      uint32_t st = 0;
      double bs = 0.0;
      if (i < nseg) {
        st = (uint32_t)__ldg(&W[i].start);
        ln = __ldg(&W[i].len);
        bs = __ldg(&W[i].base);
      }
      int incl = ln;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      wend = off0 + incl;
      wadj = st - (uint32_t)(wend - ln);
      wbase = bs;
      ws = s0;
      wlast = __shfl_sync(FULL, wend, 31);
    };
    // the window starting at the segment that holds position p (inside or
    // past the current window)
    auto anchor = [&](int p) {
      while (wlast <= p) fill(ws + 32, wlast);
      const int sl = __popc(__ballot_sync(FULL, wend <= p));
      if (sl > 0) fill(ws + sl, __shfl_sync(FULL, wend, sl - 1));
    };
    if (active) {
      const int src = __popc(__ballot_sync(FULL, cend <= pb));  // the lane whose windows hold pb
      fill(src * wpl * 32, __shfl_sync(FULL, cend - csum, src));
      anchor(pb);
    }

    struct Slot {
      uint32_t row;
      double base;
      bool ok;
    };
    uint8_t* ring = dsm + SW_LUT + (size_t)C * M * 1024 + 128 + (size_t)warp * D * sw_slot(M);
    const int xl_x = lane % M;
    const uint32_t xl_base = smem_u32(lut) + (uint32_t)(((lane / M) % C) * M + xl_x) * 4u;
    uint32_t xl_sel[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xl_sel[j] = 0x4440u | (uint32_t)(j ^ (xl_x & 3));
    uint32_t xl_bs[M];  // per-step lane addresses (code_sum_xlb)
#pragma unroll
    for (int s = 0; s < M; ++s) xl_bs[s] = xl_base ^ ((uint32_t)s << 2);

    // batch p0 .. p0 + 31 -> (row, base) per lane; code row + constant-byte
    // word issued by cp.async into ring slot `slot` (one commit group)
    auto map = [&](int p0, Slot& sl, int slot) {
      if (p0 < pe) {
        if (wlast < min(p0 + 32, pe)) anchor(p0);
        const int before = __popc(__ballot_sync(FULL, wend <= p0));
        const int rel = wend - p0;
        const uint32_t bit = (rel >= 1 && rel <= 31) ? (1u << rel) : 0u;
        const uint32_t starts = __reduce_or_sync(FULL, bit);
        const int p = p0 + lane;
        sl.ok = p < pe;
        // lanes past pe take the warp's last position (same row, no new sector)
        const int pc = sl.ok ? p : pe - 1;
        const int seg = before + __popc(starts & (FULL >> (31 - (pc - p0))));
        sl.row = __shfl_sync(FULL, wadj, seg) + (uint32_t)pc;
        sl.base = __shfl_sync(FULL, wbase, seg);
        uint8_t* dst = ring + slot * sw_slot(M);
        const uint8_t* src = ix.codes + (size_t)sl.row * M;
        constexpr int CH = cp_chunk<M>();
#pragma unroll
        for (int c = 0; c < M / CH; ++c) cp_async<CH>(dst + lane * M + c * CH, src + c * CH);
        cp_async<4>(dst + 32 * M + lane * 4, ix.cbytes + (sl.row & ~3u));
      } else {
        sl.ok = false;
      }
      cp_async_commit();
    };
    auto dist_of = [&](const Slot& cur, int slot) -> float {
      const uint8_t* src = ring + slot * sw_slot(M);
      const CodeVec<M> code = smem_code<M>(src + lane * M);
      const uint32_t cw = reinterpret_cast<const uint32_t*>(src + 32 * M)[lane];
      const uint32_t cb = __byte_perm(cw, 0, 0x4440u | (cur.row & 3u));
      constexpr int SHIFT = C * M == 32 ? 7 : (C * M == 16 ? 6 : 5);
      static_assert(C * M == 32 || C * M == 16 || C * M == 8, "row stride");
      const float ip = code_sum_xlb<M, SHIFT>(code, xl_bs, xl_x, xl_sel);
      return (float)dadd(dsub(cur.base, 2.0 * (double)ip), (double)ctab[cb]);
    };
    auto consider = [&](const Slot& cur, float dist) {
      bool pass = cur.ok && dist <= thr_f;
      if (pass && dist == thr_f && (uint32_t)thr64 != 0xffffffffu)
        pass = (((uint64_t)f32_key(dist) << 32) | (uint32_t)__ldg(ix.pids + cur.row)) < thr64;
      const uint32_t bal = __ballot_sync(FULL, pass);
      if (bal) {
        if (pass) wb[cnt + __popc(bal & lt_mask)] = ((uint64_t)f32_key(dist) << 32) | cur.row;
        cnt += __popc(bal);
      }
    };
    // D ring slots: D - 1 batches in flight while one is summed
    Slot sl[D];
    if (active) {
#pragma unroll
      for (int i = 0; i < D - 1; ++i) map(pb + 32 * i, sl[i], i);
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int chunk = NC * (warp + it * SW_WARPS) + sub;
#pragma unroll
      for (int cc = 0; cc < C; ++cc) {
        constexpr int S = C * M;  // floats per code
        float* dst = lut + (4 * chunk) * S + ((cc ^ sub) % C) * M + m;
        dst[0] = v[it].x; dst[S] = v[it].y; dst[2 * S] = v[it].z; dst[3 * S] = v[it].w;
      }
    }
    ctab[tid] = cv;
    __syncthreads();  // LUT, constants and bounds ready
    for (int p0 = pb; p0 < pe; p0 += 32 * D) {
      {  // adopt a tighter bound from the other warps
        uint32_t q[8];
        asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]) : "r"(smem_u32(&s_tw[0])));
        asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]) : "r"(smem_u32(&s_tw[4])));
        const uint32_t qb = max(max(max(q[0], q[1]), max(q[2], q[3])), max(max(q[4], q[5]), max(q[6], q[7])));
        const uint64_t tq = ((uint64_t)qb << 32) | 0xffffffffull;
        const uint64_t ts = *(volatile unsigned long long*)&s_thr64;
        const uint64_t t = ts < tq ? ts : tq;
        if (t < thr64) { thr64 = t; thr = (uint32_t)(t >> 32); thr_f = f_of(thr); }
      }
#pragma unroll
      for (int h = 0; h < D; ++h) {
        const int nx = (h + D - 1) % D;
        map(p0 + 32 * (h + D - 1), sl[nx], nx);
        cp_async_wait<D - 1>();  // this batch's group landed
        const float dv = dist_of(sl[h], h);
        consider(sl[h], dv);
      }
      if (cnt > SW_WB - 32 * D) {
        __syncwarp();
        shrink(SW_WB / 2);
        thr_f = f_of(thr);
      }
    }
    cp_async_wait<0>();
  }
  __syncwarp();
  if (cnt > k) shrink(k + 32);
  __syncthreads();
  scan_final(a, b, k, wb, cnt, dsm, merge, reinterpret_cast<uint32_t*>(dsm + SW_SSTART), &s_thr64,
             s_tw, s_wcnt, s_sel, &s_nout);
}

// LUTs of QB queries for one sub-quantizer m per CTA (grid (ceil(nq/QB), M)):
// the m-th codebook and the queries' m-th (rotated) sub-vectors are staged in
// shared memory; thread e owns codeword e.  Same arithmetic as
// build_lut_into (float64 accumulation, one rounding).
constexpr int LUT_QB = 32;

template <int DS>  // DS > 0: the sub-vector length as a constant (codeword in registers)
__global__ void __launch_bounds__(256)
k_build_luts(IndexView ix, const float* __restrict__ Q, int nq, float* __restrict__ luts) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int d = ix.d, M = ix.M, ds = DS > 0 ? DS : d / M;
  const int m = blockIdx.y, q0 = blockIdx.x * LUT_QB;
  const int nqb = min(LUT_QB, nq - q0);
  float* cw = reinterpret_cast<float*>(dsm);               // 256 x ds
  double* qs = reinterpret_cast<double*>(cw + 256 * ds);  // LUT_QB x ds (1024*ds B: aligned)
  for (int i = threadIdx.x; i < 256 * ds; i += blockDim.x)
    cw[i] = ix.codewords[(int64_t)m * 256 * ds + i];
  for (int i = threadIdx.x; i < nqb * ds; i += blockDim.x) {
    const int qb = i / ds, t = i % ds;
    const float* q = Q + (int64_t)(q0 + qb) * d;
    float v;
    if (ix.rotation) {  // (R q)[m*ds + t], float64 accumulation rounded once
      const float* r = ix.rotation + (int64_t)(m * ds + t) * d;
      double acc = 0.0;
      for (int j = 0; j < d; ++j) acc += (double)r[j] * (double)q[j];
      v = (float)acc;
    } else {
      v = q[m * ds + t];
    }
    qs[i] = (double)v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 256; e += blockDim.x) {
    const float* c = cw + e * ds;
    if constexpr (DS > 0) {
      double cr[DS];  // this codeword, held across the queries
#pragma unroll
      for (int t = 0; t < DS; ++t) cr[t] = (double)c[t];
      for (int qb = 0; qb < nqb; ++qb) {
        const double* qq = qs + qb * DS;
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < DS; ++t) acc += cr[t] * qq[t];
        luts[((int64_t)(q0 + qb) * M + m) * 256 + e] = (float)acc;
      }
    } else {
      for (int qb = 0; qb < nqb; ++qb) {
        const double* qq = qs + qb * ds;
        double acc = 0.0;
        for (int t = 0; t < ds; ++t) acc += (double)c[t] * qq[t];
        luts[((int64_t)(q0 + qb) * M + m) * 256 + e] = (float)acc;
      }
    }
  }
}

void launch_build_luts(const IndexView& ix, const float* Q, int nq, float* luts, cudaStream_t s) {
  const int ds = ix.d / ix.M;
  const size_t smem = (size_t)256 * ds * 4 + (size_t)LUT_QB * ds * 8 + 16;
  dim3 grid((nq + LUT_QB - 1) / LUT_QB, ix.M);
  auto go = [&](auto kern) {
    ensure_max_smem((const void*)kern, smem);
    kern<<<grid, 256, smem, s>>>(ix, Q, nq, luts);
  };
  switch (ds) {
    case 4: go(k_build_luts<4>); break;
    case 6: go(k_build_luts<6>); break;
    case 8: go(k_build_luts<8>); break;
    case 12: go(k_build_luts<12>); break;
    case 16: go(k_build_luts<16>); break;
    default: go(k_build_luts<0>); break;
  }
}

template <int M, int U, bool CPA, bool XL, bool FULLK>
static void launch_warp_mdxf(const ScanArgs& a, cudaStream_t s) {
  const size_t bytes = sw_bytes(M, 2 * U, CPA, XL, a.ix.d);
  ensure_max_smem((const void*)k_scan_warp<M, U, CPA, XL, FULLK>, bytes);
  k_scan_warp<M, U, CPA, XL, FULLK><<<a.nq, SW_THREADS, bytes, s>>>(a);
}

template <int M, int U, bool CPA, bool XL>
static void launch_warp_mdx(const ScanArgs& a, cudaStream_t s) {
  if constexpr (XL) launch_warp_mdxf<M, U, CPA, true, false>(a, s);  // XL: top-k only
  else if (a.mode == 1) launch_warp_mdxf<M, U, CPA, false, true>(a, s);
  else launch_warp_mdxf<M, U, CPA, false, false>(a, s);
}

// Interleaved (bank-conflict-free) LUT for M in {8, 16} with prebuilt LUTs
// (GIVF_SCAN_LUT=plain keeps the [m][256] table)
static bool scan_xl() {
  static bool x = [] {
    const char* e = getenv("GIVF_SCAN_LUT");
    return !(e && strcmp(e, "plain") == 0);
  }();
  return x;
}

// GIVF_SCAN=warp keeps k_scan_warp's block-wide segment windows
static bool scan_lean() {
  static bool x = [] {
    const char* e = getenv("GIVF_SCAN");
    return !(e && strcmp(e, "warp") == 0);
  }();
  return x;
}

template <int M, int U, bool CPA>
static void launch_warp_md(const ScanArgs& a, cudaStream_t s) {
  if constexpr (M == 8 || M == 16) {
    if (a.luts && a.mode == 0 && scan_xl()) {
      if (scan_lean()) {
        // two ring slots: deeper rings (3, 4) cost a CTA per SM of shared
        // memory and measured slower (configs[2] shape: 1.20 -> 1.60 / 1.85 ms)
        // default: half the conflict-free copies -- a 16 KB LUT and 64
        // registers fit 4 CTAs per SM, and 32 resident warps beat the bank
        // conflicts they cost (configs[2] shape: M = 16 1.19 -> 1.13 ms,
        // M = 8 1.09 -> 0.99 ms; GIVF_SCAN_COPIES=full keeps 32 / M copies)
        static const bool full = [] {
          const char* e = getenv("GIVF_SCAN_COPIES");
          return e && strcmp(e, "full") == 0;
        }();
        constexpr int CH = 16 / M;
        if (!full) {
          const size_t bytes = SW_LUT + (size_t)CH * M * 1024 + 128 + (size_t)SW_WARPS * 2 * sw_slot(M);
          ensure_max_smem((const void*)k_scan_lean<M, 2, CH>, bytes);
          k_scan_lean<M, 2, CH><<<a.nq, SW_THREADS, bytes, s>>>(a);
          return;
        }
        const size_t bytes = sw_bytes(M, 2, true, true, a.ix.d);
        ensure_max_smem((const void*)k_scan_lean<M, 2>, bytes);
        k_scan_lean<M, 2><<<a.nq, SW_THREADS, bytes, s>>>(a);
        return;
      }
      launch_warp_mdx<M, U, CPA, true>(a, s);
      return;
    }
  }
  launch_warp_mdx<M, U, CPA, false>(a, s);
}

// One batch summed per group, code rows staged by cp.async (measured
// fastest on C2; the register-staged and two-batch variants were dropped).
template <int M>
static void launch_warp_m(const ScanArgs& a, cudaStream_t s) {
  launch_warp_md<M, 1, true>(a, s);
}

bool scan_warp_ok(const ScanArgs& a) {
  if (a.mode == 0 && (a.k > SW_KMAX || a.k < 1)) return false;
  if (a.ix.n >= (int64_t)1 << 32) return false;
  const int M = a.ix.M;
  return M == 4 || M == 8 || M == 12 || M == 16 || M == 24 || M == 32;
}

bool launch_scan_warp(const ScanArgs& a, cudaStream_t s) {
  if (!scan_warp_ok(a)) return false;
  switch (a.ix.M) {  // M a multiple of 4: cp.async-able code rows
    case 4: launch_warp_m<4>(a, s); return true;
    case 8: launch_warp_m<8>(a, s); return true;
    case 12: launch_warp_m<12>(a, s); return true;
    case 16: launch_warp_m<16>(a, s); return true;
    case 24: launch_warp_m<24>(a, s); return true;
    case 32: launch_warp_m<32>(a, s); return true;
    default: return false;
  }
}

}  // namespace givf
