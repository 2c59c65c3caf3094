// K5 + K6 + K7 + K8: LUT, ADC scan with top-k, full rerank, scan-order
// output, and the multi-shard top-k merge.
//
// Reference: pq.build_lookup_table (pq.py:147-169, inner mode, rotation at
// pq.py:37-41), pq.lookup_code_sums (pq.py:172-177), the distance of
// search.py:142-148 and the rerank of search.py:156-161.
//
//  * LUT: M x 256 float32 in shared memory, built per query by the same CTA
//    that scans (entries accumulated in float64, rounded once).
//  * ip = sum of M LUT entries in float32 in numpy's reduction order
//    (8 running lanes, r_j = e_j + e_{j+8} + ..., then
//    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), tail added in order; M < 8 is a
//    plain left-to-right sum) -- verified against numpy in tests.
//  * dist = f32( f64(base) - 2*f64(ip) + f64(const) ), separately rounded.
//  * The work list is consumed in windows of <= 256 segments / CHUNK codes;
//    lanes map to consecutive code rows, so code (M-byte) and constant
//    (1-byte) loads are coalesced 16/8/4-byte vectors.
//  * top-k: a shared-memory candidate buffer filtered by a running
//    (dist, id) threshold; ids are loaded only for candidates.
#include "common.cuh"
#include "kernels.h"
#include "scan_common.cuh"

namespace givf {

constexpr int SCAN_THREADS = 256;
constexpr int CHUNK = 1024;
constexpr int WIN = SCAN_THREADS;

// Shared memory layout of k_scan (dynamic):
//   lut f32[M*256] | ctab f64[256] | qrot f32[d] | wstart i64[WIN] | wbase f64[WIN]
//   | woff i32[WIN] | wlen i32[WIN] | rowv i64[CHUNK] | segv u16[CHUNK]
//   | buf u64[bufcap] | rowbuf i64[bufcap]
struct ScanSmem {
  float* lut;
  double* ctab;
  float* qrot;
  int64_t* wstart;
  double* wbase;
  int32_t* woff;
  int32_t* wlen;
  int64_t* rowv;
  uint16_t* segv;
  uint64_t* buf;
  int64_t* rowbuf;
};

GIVF_DEV ScanSmem carve(unsigned char* p, int M, int d, int bufcap) {
  ScanSmem s;
  s.lut = reinterpret_cast<float*>(p);
  s.ctab = reinterpret_cast<double*>(s.lut + M * 256);
  s.qrot = reinterpret_cast<float*>(s.ctab + 256);
  size_t off = (size_t)M * 256 * 4 + 256 * 8 + (((size_t)d * 4 + 15) & ~(size_t)15);
  s.wstart = reinterpret_cast<int64_t*>(p + off);
  s.wbase = reinterpret_cast<double*>(s.wstart + WIN);
  s.woff = reinterpret_cast<int32_t*>(s.wbase + WIN);
  s.wlen = s.woff + WIN;
  s.rowv = reinterpret_cast<int64_t*>(s.wlen + WIN);
  s.segv = reinterpret_cast<uint16_t*>(s.rowv + CHUNK);
  s.buf = reinterpret_cast<uint64_t*>(s.segv + CHUNK);
  s.rowbuf = reinterpret_cast<int64_t*>(s.buf + bufcap);
  return s;
}

static size_t scan_smem_bytes(int M, int d, int bufcap) {
  return (size_t)M * 256 * 4 + 256 * 8 + (((size_t)d * 4 + 15) & ~(size_t)15) + WIN * 8 + WIN * 8 +
         WIN * 4 + WIN * 4 + CHUNK * 8 + CHUNK * 2 + (size_t)bufcap * 16 + 64;
}

__device__ void build_lut(const IndexView& ix, const float* __restrict__ q, ScanSmem& s) {
  build_lut_into(ix, q, s.lut, s.ctab, s.qrot);
}

template <int M>
__global__ void __launch_bounds__(SCAN_THREADS, (M <= 16 ? 3 : 1)) k_scan(ScanArgs a, int bufcap) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const IndexView& ix = a.ix;
  ScanSmem s = carve(dsm, M, ix.d, bufcap);
  __shared__ int32_t red32[40];
  __shared__ int s_count;
  __shared__ int s_nfit;
  const int b = blockIdx.x, tid = threadIdx.x;

  build_lut(ix, a.Q + (int64_t)b * ix.d, s);
  if (tid == 0) s_count = 0;
  __syncthreads();

  const WorkItem* W = a.work + (int64_t)b * a.cap_w;
  const int nseg = a.nwork[b];
  uint64_t* fk = a.mode == 1 ? a.full_keys + (int64_t)b * a.cap_full_p2 : nullptr;
  int64_t code_base = 0;
  // shrink the candidate buffer as soon as it holds 2k keys (cheap radix
  // select) so the threshold tightens early, and always before it can
  // overflow during the next chunk
  const int shrink_at = min(bufcap - CHUNK, max(2 * a.k, 128));

  // top-k: candidates are appended while their distance key is <= thr (the
  // k-th smallest key kept so far, ties included).  Only the key and the row
  // are stored; ids are read for the final buffer (and for exact-tie
  // decisions once thr64 is set).
  uint32_t thr = 0xffffffffu;
  uint64_t thr64 = kKeyPad;
  auto dist_of = [&](float ip, double base, uint8_t cb) -> float {
    return (float)dadd(dsub(base, 2.0 * (double)ip), s.ctab[cb]);
  };
  auto consider = [&](int64_t row, float dist, int64_t pos) {
    if (a.mode == 1) {
      fk[pos] = dist_id_key(dist, __ldg(ix.pids + row));
      return;
    }
    const uint32_t dk = f32_key(dist);
    if (dk > thr) return;
    if (dk == thr && thr64 != kKeyPad &&
        (((uint64_t)dk << 32) | (uint32_t)__ldg(ix.pids + row)) >= thr64)
      return;
    const int slot = atomicAdd(&s_count, 1);
    s.buf[slot] = (uint64_t)dk << 32;
    s.rowbuf[slot] = row;
  };
  // Software-pipelined sweep over n codes: each thread owns codes v, v+T,
  // ...; the loads of its next two codes are in flight while the current two
  // are summed (4 code rows + 4 constant bytes outstanding per thread).
  struct Slot {
    int64_t row;
    double base;
    CodeVec<M> code;
    uint8_t cb;
    bool ok;
  };
  auto sweep = [&](int n, int64_t pos0, auto row_of, auto base_of) {
    auto fetch = [&](Slot& sl, int vv) {
      sl.ok = vv < n;
      if (sl.ok) {
        sl.row = row_of(vv);
        sl.base = base_of(vv);
        sl.code = load_code<M>(ix.codes, sl.row);
        sl.cb = __ldg(ix.cbytes + sl.row);
      }
    };
    Slot cur;
    fetch(cur, tid);
    for (int v = tid; v < n; v += SCAN_THREADS) {
      Slot nxt;
      fetch(nxt, v + SCAN_THREADS);  // next row's loads overlap this row's sums
      consider(cur.row, dist_of(code_sum<M>(cur.code, s.lut), cur.base, cur.cb), pos0 + v);
      cur = nxt;
    }
  };
  auto maybe_shrink = [&]() {
    __syncthreads();
    const int cnt = s_count;
    if (a.mode != 0 || cnt <= shrink_at) return;
    uint32_t* hist = reinterpret_cast<uint32_t*>(s.rowv);  // free between chunks
    uint32_t prefix = 0, mask = 0, need = (uint32_t)a.k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < cnt; i += blockDim.x) {
        uint32_t dk = (uint32_t)(s.buf[i] >> 32);
        if ((dk & mask) == prefix) atomicAdd(&hist[(dk >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid < 32) {  // warp 0: find the digit holding the need-th key
        uint32_t h[8], run = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { h[j] = hist[tid * 8 + j]; run += h[j]; }
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += y;
        }
        uint32_t excl = incl - run;
        if (excl < need && incl >= need) {
          uint32_t c = excl;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (c + h[j] >= need) { s_nfit = (int)(tid * 8 + j); red32[32] = (int32_t)c; break; }
            c += h[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint32_t)s_nfit << shift;
      mask |= 255u << shift;
      need -= (uint32_t)red32[32];
      __syncthreads();
    }
    // in-place stable compaction (output index <= input index, tile by tile)
    int base = 0;
    for (int t0 = 0; t0 < cnt; t0 += blockDim.x) {
      const int i = t0 + tid;
      uint64_t v = i < cnt ? s.buf[i] : kKeyPad;
      int64_t rw = i < cnt ? s.rowbuf[i] : 0;
      int keep = (i < cnt && (uint32_t)(v >> 32) <= prefix) ? 1 : 0;
      int tot;
      int pos = block_exclusive_scan(keep, red32, &tot);
      if (keep) { s.buf[base + pos] = v; s.rowbuf[base + pos] = rw; }
      base += tot;
      __syncthreads();
    }
    if (tid == 0) s_count = base;
    thr = prefix;
    __syncthreads();
    if (base > bufcap - CHUNK) {  // > CHUNK exact distance ties: order them by id
      const uint32_t np2 = next_pow2((uint32_t)base);
      for (uint32_t i = tid; i < np2; i += blockDim.x) {
        uint64_t v = kKeyPad;
        if (i < (uint32_t)base) {
          v = s.buf[i];
          if (s.rowbuf[i] >= 0) v |= (uint32_t)__ldg(ix.pids + s.rowbuf[i]);
        }
        s.buf[i] = v;
      }
      __syncthreads();
      // rows are no longer needed for these: keys now carry the ids
      bitonic_sort_keys(s.buf, np2);
      thr64 = s.buf[a.k - 1];
      thr = (uint32_t)(thr64 >> 32);
      if (tid == 0) s_count = a.k;
      // mark the kept keys as resolved: rowbuf = -1
      for (int i = tid; i < a.k; i += blockDim.x) s.rowbuf[i] = -1;
      __syncthreads();
    }
  };

  for (int seg0 = 0; seg0 < nseg;) {
    const bool valid = seg0 + tid < nseg;
    int len = 0;
    WorkItem w;
    if (valid) { w = W[seg0 + tid]; len = w.len; }
    int tot;
    int off = block_exclusive_scan(len, red32, &tot);
    const bool fits = valid && off + len <= CHUNK;
    if (fits) { s.wstart[tid] = w.start; s.wbase[tid] = w.base; s.woff[tid] = off; s.wlen[tid] = len; }
    if (tid == 0) s_nfit = 0;
    __syncthreads();
    if (fits) atomicAdd(&s_nfit, 1);
    if (tid == 0 && !fits && valid && off == 0) {  // first segment alone exceeds CHUNK
      s.wstart[0] = w.start; s.wbase[0] = w.base; s.wlen[0] = len;
    }
    __syncthreads();
    const int nfit = s_nfit;
    if (nfit == 0) {
      const int64_t st = s.wstart[0];
      const double bs = s.wbase[0];
      const int ln = s.wlen[0];
      for (int piece = 0; piece < ln; piece += CHUNK) {
        const int n = min(CHUNK, ln - piece);
        sweep(n, code_base + piece, [&](int vv) { return st + piece + vv; },
              [&](int) { return bs; });
        maybe_shrink();
      }
      code_base += ln;
      seg0 += 1;
      continue;
    }
    const int chunk_total = s.woff[nfit - 1] + s.wlen[nfit - 1];
    {
      const int warp = tid >> 5, nw = blockDim.x >> 5, lane = tid & 31;
      for (int sg = warp; sg < nfit; sg += nw) {
        const int o = s.woff[sg], l = s.wlen[sg];
        const int64_t st = s.wstart[sg];
        for (int i = lane; i < l; i += 32) { s.rowv[o + i] = st + i; s.segv[o + i] = (uint16_t)sg; }
      }
    }
    __syncthreads();
    sweep(chunk_total, code_base, [&](int vv) { return s.rowv[vv]; },
          [&](int vv) { return s.wbase[s.segv[vv]]; });
    maybe_shrink();
    code_base += chunk_total;
    seg0 += nfit;
  }

  if (a.mode == 0) {
    __syncthreads();
    const int cnt = s_count;
    uint32_t np2 = next_pow2((uint32_t)max(cnt, 1));
    for (uint32_t i = tid; i < np2; i += blockDim.x) {
      uint64_t v = kKeyPad;
      if ((int)i < cnt) {
        v = s.buf[i];
        const int64_t rw = s.rowbuf[i];
        if (rw >= 0) v |= (uint32_t)__ldg(ix.pids + rw);  // resolve the id
      }
      s.buf[i] = v;
    }
    __syncthreads();
    bitonic_sort_keys(s.buf, np2);
    for (int i = tid; i < a.k; i += blockDim.x) {
      int32_t id = -1;
      float dv = __int_as_float(0x7f800000);
      if (i < cnt) {
        uint64_t key = s.buf[i];
        id = (int32_t)(uint32_t)key;
        dv = key_f32((uint32_t)(key >> 32));
      }
      a.out_ids[(int64_t)b * a.k + i] = id;
      a.out_d[(int64_t)b * a.k + i] = dv;
    }
  }
}

template <int M>
static void launch_scan_m(const ScanArgs& a, cudaStream_t s) {
  int bufcap = (int)next_pow2_host((uint32_t)((a.mode == 0 ? a.k : 0) + CHUNK));
  size_t sm = scan_smem_bytes(M, a.ix.d, bufcap);
  ensure_max_smem((const void*)k_scan<M>, sm);
  k_scan<M><<<a.nq, SCAN_THREADS, sm, s>>>(a, bufcap);
}

void launch_scan(const ScanArgs& a, cudaStream_t s) {
  switch (a.ix.M) {
    case 1: launch_scan_m<1>(a, s); break;
    case 2: launch_scan_m<2>(a, s); break;
    case 3: launch_scan_m<3>(a, s); break;
    case 4: launch_scan_m<4>(a, s); break;
    case 6: launch_scan_m<6>(a, s); break;
    case 8: launch_scan_m<8>(a, s); break;
    case 12: launch_scan_m<12>(a, s); break;
    case 16: launch_scan_m<16>(a, s); break;
    case 24: launch_scan_m<24>(a, s); break;
    case 32: launch_scan_m<32>(a, s); break;
    case 48: launch_scan_m<48>(a, s); break;
    case 64: launch_scan_m<64>(a, s); break;
    default: break;  // rejected at index creation
  }
}

// ------------------------------------------------------------ full rerank
// Sort one query's (dist, id) keys (search.py:156-158) and split them.
constexpr int FULL_SMEM_KEYS = 4096;

__global__ void __launch_bounds__(512)
k_full_finish(uint64_t* __restrict__ keys, int64_t cap_p2, const int64_t* __restrict__ stats,
              int32_t* __restrict__ ids, float* __restrict__ dists, int64_t ld) {
  __shared__ uint64_t sk[FULL_SMEM_KEYS];
  const int b = blockIdx.x;
  const int64_t n = stats[(int64_t)b * 4 + 3];
  uint64_t* k = keys + (int64_t)b * cap_p2;
  uint32_t np2 = next_pow2((uint32_t)(n > 1 ? n : 1));
  uint64_t* work = np2 <= FULL_SMEM_KEYS ? sk : k;
  for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x) work[i] = i < n ? k[i] : kKeyPad;
  __syncthreads();
  bitonic_sort_keys(work, np2);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    uint64_t key = work[i];
    ids[(int64_t)b * ld + i] = (int32_t)(uint32_t)key;
    dists[(int64_t)b * ld + i] = key_f32((uint32_t)(key >> 32));
  }
}

void launch_full_finish(uint64_t* keys, int64_t cap_p2, const int64_t* stats, int nq,
                        int32_t* ids, float* dists, int64_t ld, cudaStream_t s) {
  k_full_finish<<<nq, 512, 0, s>>>(keys, cap_p2, stats, ids, dists, ld);
}

// ------------------------------------------------------------ rerank=False
// Scan order: kept groups by (score, pos, grp), each group's rows in stored
// (ascending id) order, every code carrying f32(score) (search.py:159-161).
__global__ void __launch_bounds__(256)
k_scan_order(IndexView ix, const WorkItem* __restrict__ work, int64_t cap_w,
             const int* __restrict__ nwork, const int32_t* __restrict__ order,
             int32_t* __restrict__ ids, float* __restrict__ dists, int64_t ld) {
  __shared__ int32_t red[40];
  __shared__ int64_t s_base;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int n = nwork[b];
  const WorkItem* W = work + (int64_t)b * cap_w;
  const int32_t* O = order + (int64_t)b * cap_w;
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += blockDim.x) {
    int i = i0 + tid;
    WorkItem w;
    int len = 0;
    if (i < n) { w = W[O[i]]; len = w.len; }
    int tot;
    int off = block_exclusive_scan(len, red, &tot);
    int64_t base = s_base;
    for (int t = 0; t < len; ++t) {
      int64_t row = w.start + t;
      ids[(int64_t)b * ld + base + off + t] = ix.pids[row];
      dists[(int64_t)b * ld + base + off + t] = (float)w.score;
    }
    __syncthreads();
    if (tid == 0) s_base = base + tot;
    __syncthreads();
  }
}

void launch_scan_order(const IndexView& ix, const WorkItem* work, int64_t cap_w,
                       const int* nwork, const int32_t* order, int nq, int32_t* ids,
                       float* dists, int64_t ld, cudaStream_t s) {
  k_scan_order<<<nq, 256, 0, s>>>(ix, work, cap_w, nwork, order, ids, dists, ld);
}

// ------------------------------------------------------------ K7 merge
// Per query, the k smallest (dist, id) over G shard lists.
__global__ void __launch_bounds__(256)
k_merge_topk(const int32_t* __restrict__ ids, const float* __restrict__ dists, int G, int nq,
             int k, int32_t* __restrict__ out_ids, float* __restrict__ out_d) {
  extern __shared__ __align__(16) unsigned char dsm[];
  uint64_t* key = reinterpret_cast<uint64_t*>(dsm);
  const int b = blockIdx.x;
  const uint32_t n = (uint32_t)G * k;
  const uint32_t np2 = next_pow2(n);
  for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x) {
    uint64_t v = kKeyPad;
    if (i < n) {
      int g = i / k, j = i % k;
      int64_t src = ((int64_t)g * nq + b) * k + j;
      int32_t id = ids[src];
      if (id >= 0) v = dist_id_key(dists[src], id);
    }
    key[i] = v;
  }
  __syncthreads();
  bitonic_sort_keys(key, np2);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    uint64_t v = key[i];
    bool ok = v != kKeyPad;
    out_ids[(int64_t)b * k + i] = ok ? (int32_t)(uint32_t)v : -1;
    out_d[(int64_t)b * k + i] = ok ? key_f32((uint32_t)(v >> 32)) : __int_as_float(0x7f800000);
  }
}

void launch_merge_topk(const int32_t* ids, const float* dists, int G, int nq, int k,
                       int32_t* out_ids, float* out_d, cudaStream_t s) {
  uint32_t np2 = next_pow2_host((uint32_t)(G * k));
  size_t sm = (size_t)np2 * 8;
  ensure_max_smem((const void*)k_merge_topk, sm);
  k_merge_topk<<<nq, 256, sm, s>>>(ids, dists, G, nq, k, out_ids, out_d);
}

}  // namespace givf
