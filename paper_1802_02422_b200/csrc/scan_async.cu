// K5 + K6, top-k mode, with cp.async-staged code tiles (M in {4, 8, 16, 32}).
//
// Same arithmetic as k_scan (scan.cu): per-query LUT in shared memory, numpy
// pairwise float32 sums, dist = f32(f64(base) - 2 f64(ip) + f64(const)),
// running-threshold candidate buffer.  What changes is how code bytes reach
// the SM: the work list is cut into chunks of SA_CHUNK code rows, and while
// chunk i is summed out of shared memory, every thread already has chunk
// i+1's rows (M bytes each) and constant-byte words in flight as cp.async
// copies -- the latency of the random segment starts is hidden without
// holding loads in registers, and the LUT lookups are the only per-code
// shared-memory traffic besides one vector read of the staged row.
#include "common.cuh"
#include "kernels.h"
#include "scan_common.cuh"

namespace givf {

constexpr int SA_THREADS = 256;
constexpr int SA_CHUNK = 512;   // code rows per pipeline stage
constexpr int SA_WIN = 256;     // at most one segment per thread per chunk

template <int B>
GIVF_DEV void cp_async(uint32_t saddr, const void* g) {
  if constexpr (B == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(saddr), "l"(g), "n"(B)
                 : "memory");
}
GIVF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
GIVF_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct SaBuf {  // one pipeline stage
  int64_t* wstart;
  double* wbase;
  int32_t* woff;
  uint16_t* segv;
  uint8_t* stage;   // SA_CHUNK x M code bytes
  uint32_t* cword;  // SA_CHUNK aligned words holding the constant byte
};

template <int M>
struct SaLayout {
  __host__ __device__ static constexpr size_t buf_bytes() {
    return (size_t)SA_WIN * (8 + 8 + 4) + SA_CHUNK * 2 + ((SA_CHUNK * M + 15) & ~15) + SA_CHUNK * 4 +
           16;
  }
  static size_t bytes(int d, int bufcap) {
    return (size_t)M * 256 * 4 + 256 * 8 + (((size_t)d * 4 + 15) & ~(size_t)15) + 2 * buf_bytes() +
           (size_t)bufcap * 16 + 64;
  }
};

template <int M>
__global__ void __launch_bounds__(SA_THREADS, 3) k_scan_async(ScanArgs a, int bufcap) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const IndexView& ix = a.ix;
  float* lut = reinterpret_cast<float*>(dsm);
  double* ctab = reinterpret_cast<double*>(lut + M * 256);
  float* qrot = reinterpret_cast<float*>(ctab + 256);
  unsigned char* p = reinterpret_cast<unsigned char*>(qrot) + (((size_t)ix.d * 4 + 15) & ~(size_t)15);
  SaBuf bufs[2];
  for (int i = 0; i < 2; ++i) {
    bufs[i].wstart = reinterpret_cast<int64_t*>(p);
    bufs[i].wbase = reinterpret_cast<double*>(bufs[i].wstart + SA_WIN);
    bufs[i].woff = reinterpret_cast<int32_t*>(bufs[i].wbase + SA_WIN);
    bufs[i].segv = reinterpret_cast<uint16_t*>(bufs[i].woff + SA_WIN);
    bufs[i].stage = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(bufs[i].segv + SA_CHUNK) + 15) & ~(uintptr_t)15);
    bufs[i].cword = reinterpret_cast<uint32_t*>(bufs[i].stage + ((SA_CHUNK * M + 15) & ~15));
    p += SaLayout<M>::buf_bytes();
  }
  uint64_t* buf = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~(uintptr_t)15);
  int64_t* rowbuf = reinterpret_cast<int64_t*>(buf + bufcap);
  __shared__ int32_t red32[40];
  __shared__ int s_count, s_nin, s_nseg0, s_noff0, s_digit;

  const int b = blockIdx.x, tid = threadIdx.x;
  build_lut_into(ix, a.Q + (int64_t)b * ix.d, lut, ctab, qrot);
  if (tid == 0) s_count = 0;
  __syncthreads();

  const WorkItem* W = a.work + (int64_t)b * a.cap_w;
  const int nseg = a.nwork[b];
  const int shrink_at = min(bufcap - SA_CHUNK, max(2 * a.k, 128));
  uint32_t thr = 0xffffffffu;
  uint64_t thr64 = kKeyPad;
  int seg0 = 0, off0 = 0;  // next unconsumed work item and rows already taken from it

  // Cut the next chunk out of the work list into stage `bi` and issue its copies.
  auto build_chunk = [&](int bi) -> int {
    SaBuf& B = bufs[bi];
    const int s = seg0 + tid;
    const bool valid = s < nseg;
    int64_t start = 0;
    double base = 0.0;
    int len = 0;
    if (valid) {
      const WorkItem w = W[s];
      const int skip = tid == 0 ? off0 : 0;
      start = w.start + skip;
      len = w.len - skip;
      base = w.base;
    }
    int tot;
    const int off = block_exclusive_scan(len, red32, &tot);
    const int take = valid ? max(0, min(len, SA_CHUNK - off)) : 0;
    const int chunk_total = min(tot, SA_CHUNK);
    if (take > 0) {
      B.wstart[tid] = start;
      B.wbase[tid] = base;
      B.woff[tid] = off;
      if (off + take == chunk_total) {  // the last segment of this chunk
        s_nin = tid + 1;
        if (take < len) { s_nseg0 = s; s_noff0 = (tid == 0 ? off0 : 0) + take; }
        else { s_nseg0 = s + 1; s_noff0 = 0; }
      }
    }
    __syncthreads();
    const int nin = s_nin;
    seg0 = s_nseg0;
    off0 = s_noff0;
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int sg = warp; sg < nin; sg += SA_THREADS / 32) {
        const int o = B.woff[sg];
        const int l = (sg + 1 < nin ? B.woff[sg + 1] : chunk_total) - o;
        for (int i = lane; i < l; i += 32) B.segv[o + i] = (uint16_t)sg;
      }
    }
    __syncthreads();
    for (int v = tid; v < chunk_total; v += SA_THREADS) {
      const int sg = B.segv[v];
      const int64_t row = B.wstart[sg] + (v - B.woff[sg]);
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(B.stage + v * M);
      if constexpr (M == 32) {
        cp_async<16>(dst, ix.codes + row * M);
        cp_async<16>(dst + 16, ix.codes + row * M + 16);
      } else {
        cp_async<M>(dst, ix.codes + row * M);
      }
      cp_async<4>((uint32_t)__cvta_generic_to_shared(B.cword + v), ix.cbytes + (row & ~(int64_t)3));
    }
    cp_async_commit();
    return chunk_total;
  };

  auto consider = [&](int64_t row, float dist) {
    const uint32_t dk = f32_key(dist);
    if (dk > thr) return;
    if (dk == thr && thr64 != kKeyPad &&
        (((uint64_t)dk << 32) | (uint32_t)__ldg(ix.pids + row)) >= thr64)
      return;
    const int slot = atomicAdd(&s_count, 1);
    buf[slot] = (uint64_t)dk << 32;
    rowbuf[slot] = row;
  };

  // radix-select the k-th smallest distance key of the buffer, keep <= it
  auto maybe_shrink = [&](uint32_t* hist) {
    __syncthreads();
    const int cnt = s_count;
    if (cnt <= shrink_at) return;
    uint32_t prefix = 0, mask = 0, need = (uint32_t)a.k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += SA_THREADS) hist[i] = 0;
      __syncthreads();
      for (int i = tid; i < cnt; i += SA_THREADS) {
        const uint32_t dk = (uint32_t)(buf[i] >> 32);
        if ((dk & mask) == prefix) atomicAdd(&hist[(dk >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid < 32) {
        uint32_t h[8], run = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { h[j] = hist[tid * 8 + j]; run += h[j]; }
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += y;
        }
        const uint32_t excl = incl - run;
        if (excl < need && incl >= need) {
          uint32_t c = excl;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (c + h[j] >= need) { s_digit = tid * 8 + j; red32[32] = (int32_t)c; break; }
            c += h[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint32_t)s_digit << shift;
      mask |= 255u << shift;
      need -= (uint32_t)red32[32];
      __syncthreads();
    }
    int basei = 0;
    for (int t0 = 0; t0 < cnt; t0 += SA_THREADS) {
      const int i = t0 + tid;
      const uint64_t v = i < cnt ? buf[i] : kKeyPad;
      const int64_t rw = i < cnt ? rowbuf[i] : 0;
      const int keep = (i < cnt && (uint32_t)(v >> 32) <= prefix) ? 1 : 0;
      int tot;
      const int pos = block_exclusive_scan(keep, red32, &tot);
      if (keep) { buf[basei + pos] = v; rowbuf[basei + pos] = rw; }
      basei += tot;
      __syncthreads();
    }
    if (tid == 0) s_count = basei;
    thr = prefix;
    __syncthreads();
    if (basei > bufcap - SA_CHUNK) {  // > SA_CHUNK exact distance ties: order by id
      const uint32_t np2 = next_pow2((uint32_t)basei);
      for (uint32_t i = tid; i < np2; i += SA_THREADS) {
        uint64_t v = kKeyPad;
        if (i < (uint32_t)basei) {
          v = buf[i];
          if (rowbuf[i] >= 0) v |= (uint32_t)__ldg(ix.pids + rowbuf[i]);
        }
        buf[i] = v;
      }
      __syncthreads();
      bitonic_sort_keys(buf, np2);
      thr64 = buf[a.k - 1];
      thr = (uint32_t)(thr64 >> 32);
      if (tid == 0) s_count = a.k;
      for (int i = tid; i < a.k; i += SA_THREADS) rowbuf[i] = -1;
      __syncthreads();
    }
  };

  int cur = 0;
  int tot_cur = seg0 < nseg ? build_chunk(0) : 0;
  while (tot_cur > 0) {
    const int tot_next = seg0 < nseg ? build_chunk(cur ^ 1) : 0;
    if (tot_next > 0) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();
    const SaBuf& B = bufs[cur];
    for (int v = tid; v < tot_cur; v += SA_THREADS) {
      const int sg = B.segv[v];
      const int64_t row = B.wstart[sg] + (v - B.woff[sg]);
      CodeVec<M> code;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(B.stage + v * M);
      if constexpr (M == 16) {
        const uint4 x = *reinterpret_cast<const uint4*>(src);
        code.w[0] = x.x; code.w[1] = x.y; code.w[2] = x.z; code.w[3] = x.w;
      } else {
#pragma unroll
        for (int i = 0; i < CodeVec<M>::W; ++i) code.w[i] = src[i];
      }
      const uint32_t cb = (B.cword[v] >> ((row & 3) * 8)) & 0xffu;
      const float ip = code_sum<M>(code, lut);
      consider(row, (float)dadd(dsub(B.wbase[sg], 2.0 * (double)ip), ctab[cb]));
    }
    // the staging area of the chunk just summed is free for the histogram
    maybe_shrink(reinterpret_cast<uint32_t*>(B.stage));
    __syncthreads();
    cur ^= 1;
    tot_cur = tot_next;
  }

  __syncthreads();
  const int cnt = s_count;
  const uint32_t np2 = next_pow2((uint32_t)max(cnt, 1));
  for (uint32_t i = tid; i < np2; i += SA_THREADS) {
    uint64_t v = kKeyPad;
    if ((int)i < cnt) {
      v = buf[i];
      if (rowbuf[i] >= 0) v |= (uint32_t)__ldg(ix.pids + rowbuf[i]);
    }
    buf[i] = v;
  }
  __syncthreads();
  bitonic_sort_keys(buf, np2);
  for (int i = tid; i < a.k; i += SA_THREADS) {
    int32_t id = -1;
    float dv = __int_as_float(0x7f800000);
    if (i < cnt) {
      const uint64_t key = buf[i];
      id = (int32_t)(uint32_t)key;
      dv = key_f32((uint32_t)(key >> 32));
    }
    a.out_ids[(int64_t)b * a.k + i] = id;
    a.out_d[(int64_t)b * a.k + i] = dv;
  }
}

template <int M>
static void launch_m(const ScanArgs& a, cudaStream_t s) {
  const int bufcap = (int)next_pow2_host((uint32_t)(a.k + SA_CHUNK));
  const size_t sm = SaLayout<M>::bytes(a.ix.d, bufcap);
  static size_t attr = 0;
  if (attr < sm) {
    cudaFuncSetAttribute(k_scan_async<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = sm;
  }
  k_scan_async<M><<<a.nq, SA_THREADS, sm, s>>>(a, bufcap);
}

bool launch_scan_async(const ScanArgs& a, cudaStream_t s) {
  if (a.mode != 0 || a.k > 2048) return false;
  switch (a.ix.M) {
    case 4: launch_m<4>(a, s); return true;
    case 8: launch_m<8>(a, s); return true;
    case 16: launch_m<16>(a, s); return true;
    case 32: launch_m<32>(a, s); return true;
    default: return false;
  }
}

}  // namespace givf
