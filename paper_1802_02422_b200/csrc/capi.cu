// C ABI (include/givf_b200.h): device-resident index handle, workspace and
// the per-batch kernel pipeline probe -> plan -> scan.
#include <cuda_runtime.h>

#include <algorithm>
#include <random>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "givf_b200.h"
#include "kernels.h"

using namespace givf;

namespace givf {

int num_sms_cur() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 148;
  }
  cache[dev] = n;
  return n;
}

cudaError_t ensure_max_smem(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{fn, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

}  // namespace givf

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

// Per-stage device timing: CUDA events around every launch, on its stream.
enum Stage { ST_GEMM, ST_SELECT, ST_RECHECK, ST_FULL, ST_PLAN, ST_SCAN, ST_FINISH, ST_MERGE, ST_LUT,
             ST_SAMPLE, ST_K3A, ST_N };
struct Profiler {
  std::mutex mu;
  std::atomic<bool> on{false};
  struct Rec {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[ST_N] = {};
  int64_t cnt[ST_N] = {};
  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
Profiler g_prof;

template <class F>
void staged(int stage, cudaStream_t st, F&& launch, int kernels = 1) {
  g_launches += kernels;
  if (!g_prof.on.load()) {
    launch();
    return;
  }
  std::lock_guard<std::mutex> lk(g_prof.mu);
  cudaEvent_t a = g_prof.ev(), b = g_prof.ev();
  cudaEventRecord(a, st);
  launch();
  cudaEventRecord(b, st);
  g_prof.pending.push_back({stage, a, b});
}

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                             \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      return fail(_e == cudaErrorMemoryAllocation ? GIVF_ENOMEM : GIVF_ECUDA,      \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));             \
    }                                                                              \
  } while (0)

#define ARENA_CHECK(ar)                                                          \
  do {                                                                           \
    if ((ar).over) return fail(GIVF_ENOMEM, "workspace estimate exceeded (internal)"); \
  } while (0)

#define KCHECK()                                                                   \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess)                                                         \
      return fail(GIVF_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Output pointers kernels may write directly: device / managed memory, or
// page-locked host memory mapped into the device's address space (written
// over the bus by the kernels themselves, so the device-to-host transfer of
// the results overlaps the scan instead of following it).  Null otherwise.
template <typename T>
T* kernel_writable(T* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return p;
  if (at.type == cudaMemoryTypeHost && at.devicePointer) return static_cast<T*>(at.devicePointer);
  return nullptr;
}

// Grow-only scratch arena carved per call.
struct Arena {
  void* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (base) cudaFree(base);
    base = nullptr;
    cap = 0;
    size_t want = std::max(bytes, (size_t)1 << 20);
    cudaError_t e = cudaMalloc(&base, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  bool over = false;  // a take() ran past cap: nothing taken may be used
  void reset() { off = 0; over = false; }
  template <typename T>
  T* take(size_t count) {
    size_t bytes = ((count * sizeof(T)) + 255) & ~(size_t)255;
    if (off + bytes > cap) {
      over = true;
      return static_cast<T*>(base);
    }
    T* p = reinterpret_cast<T*>(static_cast<char*>(base) + off);
    off += bytes;
    return p;
  }
};

template <typename T>
size_t aligned_bytes(size_t count) {
  return ((count * sizeof(T)) + 255) & ~(size_t)255;
}

}  // namespace

struct givf_index {
  int device = 0;
  IndexView v{};
  double const_lo = 0, const_hi = 0;
  bool sharded = false;
  cudaStream_t stream = nullptr;
  std::vector<void*> allocs;
  int64_t dev_bytes = 0;
  Arena arena;
  std::mutex mu;

  cudaStream_t side = nullptr;  // LUT builds overlap the probe / planner
  cudaEvent_t ev_q = nullptr, ev_lut = nullptr;
  cudaError_t ensure_side() {
    if (side) return cudaSuccess;
    cudaError_t e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_q, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_lut, cudaEventDisableTiming);
    return e;
  }

};

namespace {

template <typename T>
cudaError_t upload(givf_index* ix, const T* host, size_t count, const T** out) {
  void* d = nullptr;
  // padded: vector loads (the scan's 4-byte constant-byte words) may read up
  // to 15 bytes past the last element
  size_t bytes = ((count * sizeof(T) + 15) & ~(size_t)15) + 16;
  cudaError_t e = cudaMalloc(&d, bytes);
  if (e != cudaSuccess) return e;
  ix->allocs.push_back(d);
  ix->dev_bytes += (int64_t)bytes;
  if (count) {
    e = cudaMemcpy(d, host, count * sizeof(T), cudaMemcpyDefault);  // host or device source
    if (e != cudaSuccess) return e;
  }
  *out = static_cast<const T*>(d);
  return cudaSuccess;
}

const char* kSupportedM = "1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64";
bool supported_m(int m) {
  switch (m) {
    case 1: case 2: case 3: case 4: case 6: case 8: case 12: case 16: case 24: case 32:
    case 48: case 64:
      return true;
    default:
      return false;
  }
}

// ConstQuantizer.table() (grouping.py:123-129): float64 (b + 0.5) * step + lo,
// each op rounded separately, then float32.
void const_table(double lo, double hi, float* out) {
  volatile double step = (hi - lo) / 256.0;
  for (int b = 0; b < 256; ++b) {
    volatile double t = ((double)b + 0.5) * step;
    volatile double v = t + lo;
    out[b] = (float)v;
  }
}

int check_params(const givf_index* ix, const givf_search_params* p) {
  char buf[160];
  if (!(1 <= p->nprobe && p->nprobe <= ix->v.K)) {
    snprintf(buf, sizeof buf, "need 1 <= nprobe <= %d, got %d", ix->v.K, p->nprobe);
    return fail(GIVF_EINVAL, buf);
  }
  if (!(0.0 < p->tau && p->tau <= 1.0)) {
    snprintf(buf, sizeof buf, "need 0 < tau <= 1, got %g", p->tau);
    return fail(GIVF_EINVAL, buf);
  }
  if (p->candidates < 1) {
    snprintf(buf, sizeof buf, "need candidates >= 1, got %lld", (long long)p->candidates);
    return fail(GIVF_EINVAL, buf);
  }
  if (p->ef_search < 1) {
    snprintf(buf, sizeof buf, "need ef_search >= 1, got %d", p->ef_search);
    return fail(GIVF_EINVAL, buf);
  }
  return GIVF_OK;
}

size_t l2_budget() {
  const char* s = getenv("GIVF_L2_CHUNK_MB");
  // measured on C2: per-chunk launch/tail costs outweigh L2 residency, so the
  // cap is off unless requested
  return (size_t)(s ? atoll(s) : (1ll << 20)) << 20;
}

size_t workspace_budget() {
  const char* s = getenv("GIVF_WORKSPACE_MB");
  size_t mb = s ? (size_t)atoll(s) : 8192;
  return std::max<size_t>(mb, 64) << 20;
}

// Probe tuning: candidate-set target and capacity (K1b / K2).
struct ProbeShape {
  int Tmin, cap;
  bool exhaustive;  // rank all K regions exactly (nprobe == K or P too large)
  // fused probe (probe_fused.cu): survivors targeted by the sample
  // threshold, the sample order statistic that estimates it, the survivor
  // list capacity and the re-check set capacity
  int ftarget, fj, fcap, fcap2;
};
ProbeShape probe_shape(int K, int P) {
  ProbeShape s;
  s.exhaustive = (P == K);
  static const int extra = getenv("GIVF_TMIN_EXTRA") ? atoi(getenv("GIVF_TMIN_EXTRA")) : 16;
  static const int capmin = getenv("GIVF_CAP_MIN") ? atoi(getenv("GIVF_CAP_MIN")) : 128;
  s.Tmin = std::min(K, P + std::max(extra, P / 4));
  s.cap = std::min(K, std::max(2 * s.Tmin, capmin));
  if (s.cap > 4096) s.exhaustive = true;  // recheck sorts in <= 4096-entry smem
  s.ftarget = s.fj = s.fcap = s.fcap2 = 0;
  return s;
}

// Fused-probe sizes for a sample of Ks of the K centroids: aim the
// threshold at ~2P + 128 survivors (the sample's j-th smallest chunk minimum
// estimates the ftarget-th smallest score; with j >= 16 the chance that it
// falls below the P-th is negligible), list capacity 6x that.
void fused_shape(ProbeShape* s, int K, int Ks, int P) {
  static const int mul = getenv("GIVF_FUSED_TARGET") ? atoi(getenv("GIVF_FUSED_TARGET")) : 2;
  const int64_t target = std::min<int64_t>(K, (int64_t)mul * P + 128);
  s->ftarget = (int)target;
  s->fj = (int)std::max<int64_t>(1, (target * Ks + K - 1) / K);
  s->fcap = (int)std::min<int64_t>(65536, std::max<int64_t>(8192, 8 * target));
  s->fcap2 = (int)std::min<int64_t>(4096, std::max<int64_t>(256, 4 * (int64_t)P));
  if (s->fcap2 < P) s->exhaustive = true;
}

constexpr int kFullSlots = 32;

struct Plan {
  int P, G, K, d;
  bool fused;  // probe_fused.cu (no score matrix), K3a from fp16 rows
  int Ks;
  int64_t total, kept, budget, cap_w;
  ProbeShape ps;
};

// A-priori bounds on |s~ - (|c|^2 - 2 q.c)| in units of (cmax^2 + 2|q| cmax):
//  SIMT fp32 FMA chain: ~(d + 4) ulp, x3 margin;
//  tcgen05 bf16x3: q.c - (q_hi c_hi + q_hi c_lo + q_lo c_hi) <= 3 x 2^-18
//  |q||c| (two bf16 terms carry 16 bits) + fp32 tensor-core accumulation
//  over 3d/16 k-steps with alignment truncation (~2^-22 each, 2d/16 + 16
//  within-step terms) -> s~ error <= ~1.6e-5 units; x5 margin.  Measured
//  worst case over adversarial families (tools/eps_probe.py: aligned
//  positive, bf16 rounding-boundary mantissas, 2^+-6 exponent spread,
//  d = 32..128): 6.6e-6 units, 12x below the bound.
constexpr float kEpsScaleUlp = 5.9604645e-8f;  // 2^-24
float probe_eps_scale(int d) { return 3.0f * (float)(d + 4) * kEpsScaleUlp; }
constexpr float kEpsScaleTC = 8e-5f;

bool use_tensor_cores(const IndexView& v) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("GIVF_PROBE");
    mode = (e && strcmp(e, "simt") == 0) ? 0 : 1;
  }
  return mode == 1 && v.csplit != nullptr;
}

// The fused probe (no score matrix) from K = 2^17 up, where the fp16 score
// matrix (2 K bytes per query) costs more HBM traffic than K3a's direct
// reads of the probed regions' neighbor rows (P G 2 d bytes); GIVF_PROBE =
// fused | dmat | simt overrides.
bool use_fused(const IndexView& v) {
  static const int mode = [] {  // 1 forced, 0 off, -1 by K
    const char* e = getenv("GIVF_PROBE");
    return !e ? -1 : strcmp(e, "fused") == 0 ? 1 : 0;
  }();
  if (!v.c16) return false;
  return mode == 1 || (mode == -1 && v.K >= (1 << 17));
}

// Probe for one chunk of queries: regions (nq, P) and qc2 (nq, P).  *D_out
// receives the fp16-encoded score matrix (nq, K) when the GEMM path ran, else
// null, *scale_out its per-query decode scale and *eps_out the GEMM's
// error-bound scale.
int run_probe(givf_index* ix, const Plan& pl, const float* dQ, int nq, int* regions,
              double* qc2, Arena& ar, cudaStream_t st, const uint16_t** D_out = nullptr,
              const float** scale_out = nullptr, float* eps_out = nullptr,
              bool* fused_out = nullptr) {
  const IndexView& v = ix->v;
  const int P = pl.P, K = v.K, d = v.d;
  if (D_out) *D_out = nullptr;
  if (fused_out) *fused_out = false;
  int* failf = ar.take<int>(nq);
  const uint32_t kp2 = next_pow2_host((uint32_t)K), pp2 = next_pow2_host((uint32_t)P);
  uint64_t* sk = ar.take<uint64_t>((size_t)kFullSlots * kp2);
  uint32_t* sv = ar.take<uint32_t>((size_t)kFullSlots * kp2);
  uint64_t* sk2 = ar.take<uint64_t>((size_t)kFullSlots * pp2);
  uint32_t* sv2 = ar.take<uint32_t>((size_t)kFullSlots * pp2);
  double* sdv = ar.take<double>((size_t)kFullSlots * pp2);
  ARENA_CHECK(ar);
  const int slots = std::min(kFullSlots, nq);
  if (pl.ps.exhaustive) {
    // nprobe == K: search.py:80-84 formula; larger P: exact f64 ranking of all.
    int mode = (P == K) ? 0 : 1;
    if (mode == 1) {
      CUDA_TRY(cudaMemsetAsync(failf, 0xff, sizeof(int) * nq, st));  // all "failed"
    }
    staged(ST_FULL, st, [&] {
      launch_probe_full(dQ, v.centroids, nq, K, d, P, mode, failf, slots, sk, sv, sk2, sv2, sdv,
                        regions, qc2, st);
    });
    KCHECK();
    return GIVF_OK;
  }
  if (pl.fused) {
    // F0-F3 + K2 (probe_fused.cu): no score matrix
    const ProbeShape& ps = pl.ps;
    const int dp = f16_pitch(d);
    const int nch = (v.Ks + 31) / 32;
    uint16_t* q16 = ar.take<uint16_t>((size_t)nq * dp);
    float* ms = ar.take<float>(nq);
    float* q2f = ar.take<float>(nq);
    float* cmin = ar.take<float>((size_t)nq * nch);
    float* thr = ar.take<float>(nq);
    int nseg = 0, cap_u = 0;
    filter_segments(nq, K, ps.fcap, &nseg, &cap_u);
    int* cnt = ar.take<int>((size_t)nq * nseg);
    int* cid = ar.take<int>((size_t)nq * nseg * cap_u);
    float* cval = ar.take<float>((size_t)nq * nseg * cap_u);
    int* cand = ar.take<int>((size_t)nq * ps.fcap2);
    int* cand_n = ar.take<int>(nq);
    float* theta = ar.take<float>(nq);
    ARENA_CHECK(ar);
    const float eps = probe_f16_eps(d);
    cudaError_t ce = cudaSuccess;
    staged(ST_SAMPLE, st, [&] {
      launch_query_f16(dQ, nq, d, v.c16e, v.c16T, q16, ms, q2f, st);
      ce = launch_probe_sample(q16, v.s16, nq, v.Ks, d, ms, cmin, st);
      launch_probe_thresh(cmin, nch, ps.fj, q2f, v.cmax, eps, nq, thr, st);
    }, 3);
    if (ce != cudaSuccess) return fail(GIVF_ECUDA, std::string("probe sample: ") + cudaGetErrorString(ce));
    staged(ST_GEMM, st, [&] {
      ce = launch_probe_filter(q16, v.c16, nq, K, d, ms, thr, nseg, cap_u, cnt, cid, cval,
                               st);
    });
    if (ce != cudaSuccess) return fail(GIVF_ECUDA, std::string("probe filter: ") + cudaGetErrorString(ce));
    staged(ST_SELECT, st, [&] {
      launch_probe_pick(cnt, cid, cval, nseg, cap_u, ps.fcap, thr, q2f, v.cmax, eps, P, ps.fcap2,
                        nq, cand, cand_n, theta, st);
    });
    if (eps_out) *eps_out = direct_f16_eps(d);  // K3a's bound (direct rows)
    if (fused_out) *fused_out = true;
    staged(ST_RECHECK, st, [&] {
      launch_probe_recheck(dQ, v.centroids, nq, K, d, P, cand, cand_n, ps.fcap2, theta, v.cmax,
                           eps, 0.f, regions, qc2, failf, nullptr, st);
    });
    // Retry pass for the queries the sampled threshold missed (too few
    // survivors, an overflowing segment, or no certificate): the P-th
    // smallest sample chunk minimum bounds the P-th smallest score of all K
    // from above, so the second threshold always admits the true top-P;
    // only what still fails takes the exhaustive float64 probe (K2').
    int* fidx = ar.take<int>(nq);
    int* fcnt = ar.take<int>(1);
    ARENA_CHECK(ar);
    launch_collect_failed(failf, nq, fidx, fcnt, st);
    int nfail = 0;
    CUDA_TRY(cudaMemcpyAsync(&nfail, fcnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    g_launches += 1;
    if (nfail > 0) {
      launch_add_counter(v.counters + 8, fcnt, st);  // retried queries
      // up to 64k survivors per retried query, in groups that fit the first
      // pass's survivor buffers (nq x nseg counters, nq x nseg x cap_u records)
      const int64_t room = (int64_t)nq * nseg * cap_u;
      const int fcap_r = (int)std::min<int64_t>(65536, (int64_t)K);
      int g = (int)std::max<int64_t>(1, std::min<int64_t>(nfail, room / fcap_r));
      int nseg_r = 0, cap_u_r = 0;
      for (;;) {  // shrink the group until its segment counters fit
        filter_segments(g, K, fcap_r, &nseg_r, &cap_u_r);
        cap_u_r = (int)std::min<int64_t>(cap_u_r, room / ((int64_t)g * nseg_r));
        if ((int64_t)g * nseg_r <= (int64_t)nq * nseg || g == 1) break;
        g = std::max(1, g / 2);
      }
      float* qr = ar.take<float>((size_t)std::min(nfail, g) * d);
      ARENA_CHECK(ar);
      if ((int64_t)g * nseg_r > (int64_t)nq * nseg || cap_u_r < 8) {
        launch_add_counter(v.counters, fcnt, st);  // no room: straight to K2'
      } else {
        for (int f0 = 0; f0 < nfail; f0 += g) {
          const int gn = std::min(g, nfail - f0);
          const int* gidx = fidx + f0;
          staged(ST_SAMPLE, st, [&] {
            launch_gather_rows(dQ, gidx, gn, d, qr, st);
            launch_query_f16(qr, gn, d, v.c16e, v.c16T, q16, ms, q2f, st);
            launch_probe_thresh(cmin, nch, P, q2f, v.cmax, eps, gn, thr, st, gidx);
          }, 3);
          staged(ST_GEMM, st, [&] {
            ce = launch_probe_filter(q16, v.c16, gn, K, d, ms, thr, nseg_r, cap_u_r, cnt,
                                     cid, cval, st);
          });
          if (ce != cudaSuccess)
            return fail(GIVF_ECUDA, std::string("probe retry: ") + cudaGetErrorString(ce));
          staged(ST_SELECT, st, [&] {
            launch_probe_pick(cnt, cid, cval, nseg_r, cap_u_r, nseg_r * cap_u_r, thr, q2f, v.cmax,
                              eps, P, ps.fcap2, gn, cand, cand_n, theta, st);
          });
          staged(ST_RECHECK, st, [&] {
            launch_probe_recheck(dQ, v.centroids, gn, K, d, P, cand, cand_n, ps.fcap2, theta,
                                 v.cmax, eps, 0.f, regions, qc2, failf, v.counters, st, gidx);
          });
        }
      }
    }
    if (nfail > 0) {
      staged(ST_FULL, st, [&] {
        launch_probe_full(dQ, v.centroids, nq, K, d, P, 1, failf, slots, sk, sv, sk2, sv2, sdv,
                          regions, qc2, st);
      });
    }
    KCHECK();
    return GIVF_OK;
  }
  ScoreOut so;
  so.D16 = ar.take<uint16_t>((size_t)nq * K);
  so.ld = K;
  float* q2f = ar.take<float>(nq);
  float* qinv = ar.take<float>(nq);
  float* qscale = ar.take<float>(nq);
  so.q2 = q2f;
  so.qinv = qinv;
  so.qscale = qscale;
  if (D_out) *D_out = so.D16;
  if (scale_out) *scale_out = qscale;
  int* cand = ar.take<int>((size_t)nq * pl.ps.cap);
  int* cand_n = ar.take<int>(nq);
  float* theta = ar.take<float>(nq);
  const int ntiles = probe_tiles(K);
  float* tmin = ar.take<float>((size_t)nq * ntiles);
  const bool tc = use_tensor_cores(v);
  uint32_t* tup = ar.take<uint32_t>(nq);
  void* abf = tc ? ar.take<uint16_t>((size_t)nq * tc_kpad(d)) : nullptr;
  ARENA_CHECK(ar);
  if (tc) {
    staged(ST_GEMM, st, [&] {
      launch_query_scale(dQ, nq, d, v.cmax, q2f, qinv, qscale, st);
      launch_split_bf16(dQ, nq, d, 0, abf, st);
      launch_probe_gemm_tc(abf, v.csplit, v.c2f, nq, K, d, so, tmin, st);
    }, 3);
  } else {
    staged(ST_GEMM, st, [&] {
      launch_query_scale(dQ, nq, d, v.cmax, q2f, qinv, qscale, st);
      launch_probe_gemm(dQ, v.centroids, v.c2f, nq, K, d, so, tmin, st);
    }, 2);
  }
  staged(ST_SELECT, st, [&] {
    launch_probe_select(so.D16, K, q2f, qscale, nq, K, pl.ps.Tmin, pl.ps.cap, tmin, ntiles, tup,
                        cand, cand_n, theta, st);
  }, 2);
  const float eps_scale = tc ? kEpsScaleTC : probe_eps_scale(d);
  if (eps_out) *eps_out = eps_scale;
  staged(ST_RECHECK, st, [&] {
    launch_probe_recheck(dQ, v.centroids, nq, K, d, P, cand, cand_n, pl.ps.cap, theta, v.cmax,
                         eps_scale, (float)kHalfRel, regions, qc2, failf, v.counters, st);
  });
  staged(ST_FULL, st, [&] {
    launch_probe_full(dQ, v.centroids, nq, K, d, P, 1, failf, slots, sk, sv, sk2, sv2, sdv,
                      regions, qc2, st);
  });
  KCHECK();
  return GIVF_OK;
}

size_t probe_bytes_per_query(const Plan& pl) {
  size_t b = aligned_bytes<int>(1) * 4 + aligned_bytes<int>(pl.P) + aligned_bytes<double>(pl.P);
  if (!pl.ps.exhaustive && pl.fused)
    b += (size_t)f16_pitch(pl.d) * 2 + 8 * aligned_bytes<float>(1) +
         (size_t)((pl.Ks + 31) / 32) * 4 + (size_t)pl.ps.fcap * 8 + 2048 * 4 +
         (size_t)pl.ps.fcap2 * 4 + (size_t)pl.d * 4 + 512;  // + the retry's gathered rows
  else if (!pl.ps.exhaustive)
    b += (size_t)pl.K * 2 + 4 * aligned_bytes<float>(1) + (size_t)pl.ps.cap * 4 +
         aligned_bytes<float>(probe_tiles(pl.K)) +
         (size_t)tc_kpad(pl.d) * 2 + 256;
  return b;
}
size_t probe_fixed_bytes(const Plan& pl) {
  const size_t kp2 = next_pow2_host((uint32_t)pl.K), pp2 = next_pow2_host((uint32_t)pl.P);
  return kFullSlots * (kp2 * 12 + pp2 * 20) + 16 * 256;
}

int build_plan(givf_index* ix, const givf_search_params* p, Plan* pl) {
  int rc = check_params(ix, p);
  if (rc) return rc;
  pl->P = p->nprobe;
  pl->G = ix->v.G;
  pl->K = ix->v.K;
  pl->d = ix->v.d;
  pl->total = (int64_t)pl->P * pl->G;
  pl->kept = p->prune ? (int64_t)std::ceil(p->tau * (double)pl->total) : pl->total;
  pl->kept = std::min(std::max<int64_t>(pl->kept, 1), pl->total);
  pl->budget = p->candidates;
  pl->cap_w = std::max<int64_t>(1, std::min(pl->kept, pl->budget));
  pl->ps = probe_shape(pl->K, pl->P);
  pl->fused = !pl->ps.exhaustive && use_fused(ix->v);
  pl->Ks = ix->v.Ks;
  if (pl->fused) fused_shape(&pl->ps, pl->K, pl->Ks, pl->P);
  if (pl->ps.exhaustive) pl->fused = false;
  return GIVF_OK;
}

enum OutMode { OUT_TOPK = 0, OUT_FULL = 1, OUT_PLAN = 2 };

// OUT_PLAN (givf_plan): the planner's global work lists, no scan
struct PlanOut {
  PlanItem* items;  // (nq, cap)
  int32_t* nitems;  // (nq)
  int64_t cap;
};

int run_search(givf_index* ix, const float* queries, int64_t nq, const givf_search_params* p,
               OutMode om, int64_t width, int32_t* ids, float* dists, givf_search_stats* stats,
               void* stream, const PlanOut* po = nullptr) {
  Plan pl;
  int rc = build_plan(ix, p, &pl);
  if (rc) return rc;
  if (om == OUT_PLAN && (!po || !po->items || !po->nitems || po->cap < pl.cap_w))
    return fail(GIVF_EINVAL, "plan output capacity must be >= givf_plan_capacity()");
  if (om == OUT_TOPK && (width < 1 || width > 4096))
    return fail(GIVF_EINVAL, "need 1 <= k <= 4096");
  if (om == OUT_FULL) {
    if (ix->sharded) return fail(GIVF_EINVAL, "full results need an unsharded index");
    int64_t need = std::min<int64_t>(p->candidates, ix->v.n);
    if (width < need)
      return fail(GIVF_EINVAL, "capacity must be >= min(candidates, n)");
  }
  if (nq == 0) return GIVF_OK;
  if (!queries || !stats || (om != OUT_PLAN && (!ids || !dists)))
    return fail(GIVF_EINVAL, "null output pointer");

  std::lock_guard<std::mutex> lock(ix->mu);
  CUDA_TRY(cudaSetDevice(ix->device));
  cudaStream_t st = (cudaStream_t)stream;  // NULL = the default stream
  const IndexView& v = ix->v;
  const bool q_dev = is_device_ptr(queries);
  // outputs the kernels write in place (device or pinned host memory)
  int32_t* const ids_w = kernel_writable(ids);
  float* const dists_w = kernel_writable(dists);
  int64_t* const stats_w = reinterpret_cast<int64_t*>(kernel_writable(stats));
  const bool out_dev = om == OUT_PLAN || (ids_w && dists_w);
  const bool st_dev = stats_w != nullptr;
  // results in host memory: the call returns once they have landed
  const bool host_out = om == OUT_PLAN
      ? !(is_device_ptr(po->items) && is_device_ptr(po->nitems) && is_device_ptr(stats))
      : !(is_device_ptr(ids) && is_device_ptr(dists) && is_device_ptr(stats));
  const bool plan_dev = om == OUT_PLAN && is_device_ptr(po->items) && is_device_ptr(po->nitems);
  const bool rerank = p->rerank != 0;
  const int64_t full_p2 = om == OUT_FULL ? (int64_t)next_pow2_host((uint32_t)std::max<int64_t>(width, 1)) : 0;

  // per-query workspace (the probe's part is sized by probe sub-chunk below)
  const size_t probe_q = probe_bytes_per_query(pl);
  size_t per_q = aligned_bytes<float>(v.d) +
                 2 * aligned_bytes<double>(pl.total) + aligned_bytes<int32_t>(pl.total) +
                 aligned_bytes<WorkItem>(pl.cap_w) + aligned_bytes<int>(1) +
                 aligned_bytes<int>(1) + aligned_bytes<int64_t>(4);
  if (om == OUT_FULL && !rerank) {
    size_t cp2 = next_pow2_host((uint32_t)std::min<int64_t>(pl.cap_w, 1 << 30));
    per_q += aligned_bytes<int32_t>(pl.cap_w) + cp2 * 12;
  }
  if (om == OUT_FULL && rerank) per_q += (size_t)full_p2 * 8;
  if (!out_dev) per_q += (size_t)width * 8 + 512;
  if (om == OUT_PLAN && !plan_dev) per_q += (size_t)po->cap * sizeof(PlanItem) + 64;
  per_q += aligned_bytes<float>((size_t)v.M * 256);  // prebuilt LUTs
  per_q += probe_q;
  const size_t fixed = probe_fixed_bytes(pl) + (1 << 16);
  const size_t budget = workspace_budget();
  int64_t chunk = budget > fixed ? (int64_t)((budget - fixed) / per_q) : 1;
  // Keep one chunk's probe scores + plan scratch resident in the 126 MB L2:
  // they are written and re-read by the select / plan kernels right away.
  const size_t hot = (pl.ps.exhaustive ? 0 : (size_t)pl.K * 4) + (size_t)pl.total * 20 +
                     (size_t)pl.cap_w * 32;
  chunk = std::min<int64_t>(chunk, std::max<int64_t>(128, (int64_t)(l2_budget() / hot)));
  if (const char* e = getenv("GIVF_CHUNK_QUERIES")) chunk = std::max<int64_t>(1, atoll(e));
  chunk = std::max<int64_t>(1, std::min<int64_t>(chunk, nq));
  chunk = std::min<int64_t>(chunk, 65535);
  // equal chunks (no small tail chunk that leaves the GPU half empty)
  chunk = (nq + (nq + chunk - 1) / chunk - 1) / ((nq + chunk - 1) / chunk);
  const size_t slice = ((fixed + per_q * (size_t)chunk + (1 << 20)) + 4095) & ~(size_t)4095;
  CUDA_TRY(ix->arena.reserve(slice));
  // Chunks run in order on the caller's stream, each reusing the arena
  // (stream order makes the reuse safe without host synchronisation).
  for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
    const int bq = (int)std::min<int64_t>(chunk, nq - q0);
    Arena ar;
    ar.base = ix->arena.base;
    ar.cap = slice;
    ar.reset();
    const float* dQ;
    if (q_dev) {
      dQ = queries + q0 * v.d;
    } else {
      float* tmp = ar.take<float>((size_t)bq * v.d);
      ARENA_CHECK(ar);
      CUDA_TRY(cudaMemcpyAsync(tmp, queries + q0 * v.d, sizeof(float) * bq * v.d,
                               cudaMemcpyHostToDevice, st));
      dQ = tmp;
    }
    // K5 (LUTs) depends only on the queries: it runs on a side stream while
    // the probe and the planner run here (measured: launching it next to the
    // GEMM, to K3a or to K4 costs the same device time; this placement gives
    // the best end-to-end time).  The event is recorded after the
    // previous chunk's scan (stream order), so the buffer is free to rewrite.
    float* luts = nullptr;
    {
      ScanArgs la{};
      la.ix = v;
      la.mode = om == OUT_TOPK ? 0 : 1;
      la.k = (int)(om == OUT_TOPK ? width : 0);
      if (om == OUT_TOPK && scan_warp_ok(la)) {  // (OUT_PLAN: no LUTs)
        luts = ar.take<float>((size_t)bq * v.M * 256);
        CUDA_TRY(ix->ensure_side());
      }
    }
    auto launch_luts = [&]() -> int {
      if (!luts) return GIVF_OK;
      CUDA_TRY(cudaEventRecord(ix->ev_q, st));
      CUDA_TRY(cudaStreamWaitEvent(ix->side, ix->ev_q, 0));
      staged(ST_LUT, ix->side, [&] { launch_build_luts(v, dQ, bq, luts, ix->side); });
      CUDA_TRY(cudaEventRecord(ix->ev_lut, ix->side));
      return GIVF_OK;
    };
    int* regions = ar.take<int>((size_t)bq * pl.P);
    double* qc2 = ar.take<double>((size_t)bq * pl.P);

    PlanArgs pa{};
    pa.ix = v;
    pa.Q = dQ;
    pa.regions = regions;
    pa.qc2 = qc2;
    pa.nq = bq;
    pa.P = pl.P;
    pa.kept = pl.kept;
    pa.budget = pl.budget;
    pa.sbase = ar.take<double>((size_t)bq * pl.total);
    pa.sscore = ar.take<double>((size_t)bq * pl.total);
    pa.ssize = ar.take<int32_t>((size_t)bq * pl.total);
    pa.cap_w = pl.cap_w;
    pa.work = ar.take<WorkItem>((size_t)bq * pl.cap_w);
    pa.nwork = ar.take<int>(bq);
    int64_t* dstats = st_dev ? stats_w + q0 * 4 : ar.take<int64_t>((size_t)bq * 4);
    pa.stats = dstats;
    pa.sort_work = (om == OUT_FULL && !rerank) ? 1 : 0;
    if (pa.sort_work) {
      int64_t cp2 = next_pow2_host((uint32_t)pl.cap_w);
      pa.skey = ar.take<uint64_t>((size_t)bq * cp2);
      pa.sval = ar.take<uint32_t>((size_t)bq * cp2);
      pa.order = ar.take<int32_t>((size_t)bq * pl.cap_w);
    }
    pa.ldD = v.K;
    pa.cmax = v.cmax;
    pa.half_rel = (float)kHalfRel;
    pa.n_overflow = ar.take<int>(1);
    pa.global_items = om == OUT_PLAN ? 1 : 0;
    pa.only = ar.take<int>(bq);
    ARENA_CHECK(ar);
    // the approximate planner's keys alias the exact scratch, which the exact
    // kernels only write after the approximate planner has finished
    pa.akey = reinterpret_cast<uint32_t*>(pa.sbase);

    // probe + K3a; the probe workspace (D included) is dead afterwards
    const size_t mark = ar.off;
    bool approx = true;
    rc = launch_luts();
    if (rc) return rc;
    {
      const uint16_t* Dmat = nullptr;
      const float* dscale = nullptr;
      float eps_scale = 0.f;
      bool fused = false;
      rc = run_probe(ix, pl, dQ, bq, regions, qc2, ar, st, &Dmat, &dscale, &eps_scale, &fused);
      if (rc) return rc;
      pa.eps_scale = eps_scale;
      if (!Dmat && !fused) {  // exhaustive probe (nprobe == K or too wide): exact planner only
        approx = false;
      } else {
        PlanArgs sa = pa;
        sa.D = Dmat;
        sa.dscale = dscale;
        if (fused) {
          sa.direct = 1;
          sa.half_rel = 0.f;
          pa.half_rel = 0.f;
        }
        int nk = 0;
        staged(ST_K3A, st, [&] { nk = launch_plan_scores(sa, st); }, 0);
        g_launches += nk;
        KCHECK();
      }
    }
    ar.off = mark;  // the probe workspace is dead once K3a has run (stream order)
    pa.approx = approx ? 1 : 0;
    pa.D = nullptr;
    int nk = 0;
    staged(ST_PLAN, st, [&] { nk = launch_plan(pa, st); }, 0);
    g_launches += nk;
    KCHECK();

    if (om == OUT_PLAN) {
      PlanItem* pi = plan_dev ? po->items + q0 * po->cap : ar.take<PlanItem>((size_t)bq * po->cap);
      int32_t* pn = plan_dev ? po->nitems + q0 : ar.take<int32_t>(bq);
      ARENA_CHECK(ar);
      staged(ST_FINISH, st, [&] {
        launch_items_from_work(pa.work, pl.cap_w, pa.nwork, bq, pi, po->cap, pn, st);
      });
      KCHECK();
      if (!plan_dev) {
        CUDA_TRY(cudaMemcpyAsync(po->items + q0 * po->cap, pi, sizeof(PlanItem) * bq * po->cap,
                                 cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(po->nitems + q0, pn, sizeof(int32_t) * bq, cudaMemcpyDeviceToHost, st));
      }
      if (!st_dev)
        CUDA_TRY(cudaMemcpyAsync(stats + q0, dstats, sizeof(int64_t) * 4 * bq,
                                 cudaMemcpyDeviceToHost, st));
      continue;
    }

    int32_t* oid;
    float* od;
    if (out_dev) {
      oid = ids_w + q0 * width;
      od = dists_w + q0 * width;
    } else {
      oid = ar.take<int32_t>((size_t)bq * width);
      od = ar.take<float>((size_t)bq * width);
    }
    if (om == OUT_TOPK || rerank) {
      ScanArgs sa{};
      sa.ix = v;
      sa.Q = dQ;
      sa.nq = bq;
      sa.work = pa.work;
      sa.cap_w = pl.cap_w;
      sa.nwork = pa.nwork;
      sa.mode = om == OUT_TOPK ? 0 : 1;
      sa.k = (int)(om == OUT_TOPK ? width : 0);
      sa.out_ids = oid;
      sa.out_d = od;
      if (om == OUT_FULL) {
        sa.full_keys = ar.take<uint64_t>((size_t)bq * full_p2);
        sa.cap_full_p2 = full_p2;
      }
      if (luts) {  // prebuilt on the side stream
        CUDA_TRY(cudaStreamWaitEvent(st, ix->ev_lut, 0));
        sa.luts = luts;
      }
      ARENA_CHECK(ar);
      staged(ST_SCAN, st, [&] {
        if (!launch_scan_warp(sa, st)) launch_scan(sa, st);  // k_scan: full mode, other M / k
      });
      KCHECK();
      if (om == OUT_FULL) {
        staged(ST_FINISH, st, [&] {
          launch_full_finish(sa.full_keys, full_p2, dstats, bq, oid, od, width, st);
        });
        KCHECK();
      }
    } else {
      ARENA_CHECK(ar);
      staged(ST_FINISH, st, [&] {
        launch_scan_order(v, pa.work, pl.cap_w, pa.nwork, pa.order, bq, oid, od, width, st);
      });
      KCHECK();
    }
    if (!out_dev) {
      CUDA_TRY(cudaMemcpyAsync(ids + q0 * width, oid, sizeof(int32_t) * bq * width,
                               cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(dists + q0 * width, od, sizeof(float) * bq * width,
                               cudaMemcpyDeviceToHost, st));
    }
    if (!st_dev) {
      CUDA_TRY(cudaMemcpyAsync(stats + q0, dstats, sizeof(int64_t) * 4 * bq,
                               cudaMemcpyDeviceToHost, st));
    }
  }
  if (host_out || !q_dev) CUDA_TRY(cudaStreamSynchronize(st));
  return GIVF_OK;
}

}  // namespace

extern "C" {

const char* givf_last_error(void) { return g_err.c_str(); }
const char* givf_version(void) { return "givf_b200 0.1 (sm_100a)"; }
int64_t givf_kernel_launches(void) { return g_launches.load(); }

int givf_profile_enable(int on) {
  g_prof.on.store(on != 0);
  return GIVF_OK;
}

int givf_profile_read(double* stage_ms, int64_t* stage_launches, int32_t nstages) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  for (auto& r : g_prof.pending) {
    CUDA_TRY(cudaEventSynchronize(r.b));
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    g_prof.ms[r.stage] += t;
    g_prof.cnt[r.stage] += 1;
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.pending.clear();
  for (int i = 0; i < nstages && i < ST_N; ++i) {
    if (stage_ms) stage_ms[i] = g_prof.ms[i];
    if (stage_launches) stage_launches[i] = g_prof.cnt[i];
  }
  for (int i = 0; i < ST_N; ++i) { g_prof.ms[i] = 0; g_prof.cnt[i] = 0; }
  return GIVF_OK;
}

int givf_index_create(const givf_index_desc* ds, int device, givf_index_t* out) {
  if (!ds || !out) return fail(GIVF_EINVAL, "null argument");
  *out = nullptr;
  const int K = ds->k, d = ds->dim, G = ds->groups, M = ds->m;
  if (K < 1 || d < 1 || G < 1 || M < 1) return fail(GIVF_EINVAL, "k, dim, groups, m must be >= 1");
  if (d % M != 0) return fail(GIVF_EINVAL, "m must divide dim");
  if (!supported_m(M)) return fail(GIVF_EINVAL, std::string("m must be one of ") + kSupportedM);
  if (d > 1024) return fail(GIVF_EINVAL, "dim must be <= 1024");
  if (ds->grouping && (!ds->neighbor_ids || !ds->norm_terms))
    return fail(GIVF_EINVAL, "grouping needs neighbor_ids and norm_terms");
  if (!ds->grouping && G != 1) return fail(GIVF_EINVAL, "groups must be 1 without grouping");
  if (!ds->centroids || !ds->alphas || !ds->group_sizes || !ds->region_offsets ||
      !ds->codewords || (ds->n > 0 && (!ds->point_ids || !ds->codes || !ds->const_bytes)))
    return fail(GIVF_EINVAL, "null index array");
  if ((ds->local_sizes == nullptr) != (ds->local_lo == nullptr))
    return fail(GIVF_EINVAL, "local_sizes and local_lo go together");
  if (ds->n >= (int64_t)1 << 40) return fail(GIVF_EINVAL, "too many rows");

  // host-side layout checks and derived tables
  const int32_t* lsz = ds->local_sizes ? ds->local_sizes : ds->group_sizes;
  std::vector<int64_t> lstart((size_t)K * G);
  for (int r = 0; r < K; ++r) {
    int64_t o = ds->region_offsets[r];
    for (int j = 0; j < G; ++j) {
      int32_t s = lsz[(size_t)r * G + j];
      if (s < 0 || ds->group_sizes[(size_t)r * G + j] < 0)
        return fail(GIVF_EINVAL, "negative group size");
      lstart[(size_t)r * G + j] = o;
      o += s;
    }
    if (o != ds->region_offsets[r + 1]) return fail(GIVF_EINVAL, "region_offsets disagree with group sizes");
  }
  if (ds->region_offsets[0] != 0 || ds->region_offsets[K] != ds->n)
    return fail(GIVF_EINVAL, "region_offsets must span [0, n]");
  if (ds->grouping) {
    for (size_t i = 0; i < (size_t)K * G; ++i)
      if (ds->neighbor_ids[i] < 0 || ds->neighbor_ids[i] >= K)
        return fail(GIVF_EINVAL, "neighbor id out of range");
  }
  std::vector<float> c2f(K);
  double cmax = 0.0;
  for (int r = 0; r < K; ++r) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
      double x = ds->centroids[(size_t)r * d + j];
      s += x * x;
    }
    c2f[r] = (float)s;
    cmax = std::max(cmax, std::sqrt(s));
  }
  float ctab[256];
  const_table(ds->const_lo, ds->const_hi, ctab);

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(GIVF_ECUDA, "no CUDA device");
  }
  if (device < 0 || device >= ndev) return fail(GIVF_EINVAL, "bad device ordinal");
  CUDA_TRY(cudaSetDevice(device));

  givf_index* ix = new givf_index();
  ix->device = device;
  ix->const_lo = ds->const_lo;
  ix->const_hi = ds->const_hi;
  ix->sharded = ds->local_sizes != nullptr;
  IndexView& v = ix->v;
  v.K = K; v.d = d; v.G = G; v.M = M; v.grouping = ds->grouping ? 1 : 0; v.n = ds->n;
  v.cmax = (float)(cmax * (1.0 + 1e-6));
  {
    int32_t mg = 0;
    for (size_t i = 0; i < (size_t)K * (ds->grouping ? G : 1); ++i)
      mg = std::max(mg, ds->group_sizes[i]);
    v.max_gsize = mg;
  }
  const size_t KG = (size_t)K * G;
  cudaError_t e = cudaSuccess;
#define UP(host, count, field) \
  if (e == cudaSuccess) e = upload(ix, host, count, &v.field)
  UP(ds->centroids, (size_t)K * d, centroids);
  UP(c2f.data(), (size_t)K, c2f);
  UP(ds->alphas, (size_t)K, alphas);
  std::vector<float> rneg;
  if (ds->grouping) {
    UP(ds->neighbor_ids, KG, nbr);
    UP(ds->norm_terms, KG, norm);
    // per region, the most negative norm term (the planner's window width)
    rneg.assign((size_t)K, 0.f);
    for (size_t r = 0; r < (size_t)K; ++r) {
      float m = 0.f;
      for (size_t g = 0; g < (size_t)G; ++g) m = std::max(m, -ds->norm_terms[r * G + g]);
      rneg[r] = m;
    }
    UP(rneg.data(), (size_t)K, rneg);
  }
  UP(ds->group_sizes, KG, gsize);
  UP(lstart.data(), KG, lstart);
  if (ds->local_sizes) {
    UP(ds->local_sizes, KG, lsize);
    UP(ds->local_lo, KG, llo);
  }
  UP(ds->point_ids, (size_t)ds->n, pids);
  UP(ds->codes, (size_t)ds->n * M, codes);
  UP(ds->const_bytes, (size_t)ds->n, cbytes);
  UP(ds->codewords, (size_t)M * 256 * (d / M), codewords);
  if (ds->rotation) UP(ds->rotation, (size_t)d * d, rotation);
  UP(ctab, (size_t)256, ctab);
#undef UP
  if (e == cudaSuccess) {
    unsigned long long* cnt = nullptr;
    e = cudaMalloc(&cnt, 256);
    if (e == cudaSuccess) {
      ix->allocs.push_back(cnt);
      e = cudaMemset(cnt, 0, 256);
      v.counters = cnt;
    }
  }
  if (e == cudaSuccess && tc_supported(d)) {
    // bf16 split of the centroids for the tensor-core probe (probe_tc.cu)
    void* cs = nullptr;
    const size_t bytes = (size_t)K * tc_kpad_b(d) * 2;
    e = cudaMalloc(&cs, bytes);
    if (e == cudaSuccess) {
      ix->allocs.push_back(cs);
      ix->dev_bytes += (int64_t)bytes;
      launch_split_bf16(v.centroids, K, d, 1, cs, 0);
      e = cudaDeviceSynchronize();
      v.csplit = cs;
    }
  }
  if (e == cudaSuccess && fused_supported(d)) {
    // fused probe (probe_fused.cu): fp16 centroids scaled by 2^-ec (max
    // |c_ij| in [2^7, 2^8)) with the |c|^2 columns scaled by 2^-T so that
    // the largest b = |c|^2 2^-(1 + ec + T) is below 2^14, and a seeded
    // random sample of the rows
    float amax = 0.f;
    double c2max = 0.0;
    for (size_t i = 0; i < (size_t)K * d; ++i) amax = std::max(amax, std::fabs(ds->centroids[i]));
    for (int r = 0; r < K; ++r) c2max = std::max(c2max, (double)c2f[r]);
    const int ec = amax > 0.f ? std::ilogb(amax) - 7 : 0;
    const double bmax = std::ldexp(c2max, -(1 + ec));
    const int T = bmax > 0.0 ? std::ilogb(bmax) + 1 - 14 : 0;
    v.c16e = ec;
    v.c16x = std::ldexp(1.0f, ec);
    v.c16T = T;
    const int dp = f16_pitch(d);
    // sample: every centroid up to 8192, else K/16 (at most 2^16); its
    // j-th smallest chunk minimum aims the threshold at ~2P + 128 survivors
    // (j >= 20 at nprobe 64: a sample that lands below the P-th smallest
    // score of all K is a > 5 sigma event, and costs only a fallback)
    const int Ks = K <= 8192 ? K : std::min(1 << 16, std::max(8192, K / 16));
    std::vector<int32_t> ids((size_t)K);
    for (int i = 0; i < K; ++i) ids[i] = i;
    if (Ks < K) {
      std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
      for (int i = 0; i < Ks; ++i) {
        std::uniform_int_distribution<int> pick(i, K - 1);
        std::swap(ids[i], ids[pick(rng)]);
      }
      std::sort(ids.begin(), ids.begin() + Ks);
    }
    void *c16 = nullptr, *s16 = nullptr, *c16r = nullptr;
    float* sc2 = nullptr;
    const int32_t* dids = nullptr;
    const size_t cb = (size_t)K * dp * 2, sb = (size_t)Ks * dp * 2;
    const size_t rb = (size_t)K * f16_row_pitch(d) * 2;
    e = cudaMalloc(&c16r, rb);
    if (e == cudaSuccess) { ix->allocs.push_back(c16r); ix->dev_bytes += (int64_t)rb; }
    if (e == cudaSuccess) e = cudaMalloc(&c16, cb);
    if (e == cudaSuccess) { ix->allocs.push_back(c16); ix->dev_bytes += (int64_t)cb; e = cudaMalloc(&s16, sb); }
    if (e == cudaSuccess) { ix->allocs.push_back(s16); ix->dev_bytes += (int64_t)sb; e = cudaMalloc(&sc2, (size_t)Ks * 4 + 16); }
    if (e == cudaSuccess) { ix->allocs.push_back(sc2); e = upload(ix, ids.data(), (size_t)Ks, &dids); }
    if (e == cudaSuccess) {
      launch_rows_f16(v.centroids, nullptr, K, d, ec, T, v.c2f, c16, nullptr, 0);
      launch_rows_f16(v.centroids, nullptr, K, d, ec, T, v.c2f, c16r, nullptr, 0, f16_row_pitch(d));
      launch_rows_f16(v.centroids, dids, Ks, d, ec, T, v.c2f, s16, sc2, 0);
      e = cudaDeviceSynchronize();
    }
    if (e == cudaSuccess) {
      v.c16 = c16;
      v.c16r = c16r;
      v.s16 = s16;
      v.sc2 = sc2;
      v.Ks = Ks;
    }
    // K3a's per-region packed neighbour rows (K G row bytes: 12.9 GB at
    // configs[2]): taken when the fused probe will run (K >= 2^17 or forced)
    // and the device keeps >= 32 GB free after it (workspace, caller's
    // tensors); GIVF_PACK_NEIGHBORS=0 / 1 overrides
    if (e == cudaSuccess && v.grouping && v.nbr) {
      const char* pk = getenv("GIVF_PACK_NEIGHBORS");
      const size_t pb = (size_t)K * v.G * f16_row_pitch(d) * 2, p2 = (size_t)K * v.G * 4;
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      const bool want = pk ? atoi(pk) != 0 : (use_fused(v) && fr > pb + p2 + ((size_t)32 << 30));
      if (want) {
        void* c16p = nullptr;
        float* c2p = nullptr;
        if (cudaMalloc(&c16p, pb) == cudaSuccess) {
          if (cudaMalloc(&c2p, p2) == cudaSuccess) {
            launch_pack_neighbor_rows(c16r, v.c2f, v.nbr, K, v.G, d, c16p, c2p, 0);
            e = cudaDeviceSynchronize();
            ix->allocs.push_back(c16p);
            ix->allocs.push_back(c2p);
            ix->dev_bytes += (int64_t)(pb + p2);
            v.c16p = c16p;
            v.c2p = c2p;
          } else {
            cudaFree(c16p);
            cudaGetLastError();
          }
        } else {
          cudaGetLastError();
        }
      }
    }
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    givf_index_destroy(ix);
    return fail(e == cudaErrorMemoryAllocation ? GIVF_ENOMEM : GIVF_ECUDA,
                std::string("index upload: ") + cudaGetErrorString(e));
  }
  *out = ix;
  return GIVF_OK;
}

int givf_index_destroy(givf_index_t ix) {
  if (!ix) return GIVF_OK;
  cudaSetDevice(ix->device);
  if (ix->stream) cudaStreamSynchronize(ix->stream);
  for (void* p : ix->allocs) cudaFree(p);
  if (ix->arena.base) cudaFree(ix->arena.base);
  if (ix->stream) cudaStreamDestroy(ix->stream);
  if (ix->side) cudaStreamDestroy(ix->side);
  if (ix->ev_q) cudaEventDestroy(ix->ev_q);
  if (ix->ev_lut) cudaEventDestroy(ix->ev_lut);
  delete ix;
  return GIVF_OK;
}

int64_t givf_index_device_bytes(givf_index_t ix) { return ix ? ix->dev_bytes : 0; }

int givf_index_counters(givf_index_t ix, int64_t* out, int32_t n) {
  if (!ix || !out) return fail(GIVF_EINVAL, "null argument");
  unsigned long long h[32] = {};
  CUDA_TRY(cudaSetDevice(ix->device));
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(h, ix->v.counters, sizeof h, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < 32; ++i) out[i] = (int64_t)h[i];
  return GIVF_OK;
}

int givf_search_topk(givf_index_t ix, const float* queries, int64_t nq,
                     const givf_search_params* params, int32_t k, int32_t* ids, float* dists,
                     givf_search_stats* stats, void* stream) {
  if (!ix || !params) return fail(GIVF_EINVAL, "null argument");
  return run_search(ix, queries, nq, params, OUT_TOPK, k, ids, dists, stats, stream);
}

int givf_search_full(givf_index_t ix, const float* queries, int64_t nq,
                     const givf_search_params* params, int64_t capacity, int32_t* ids,
                     float* dists, givf_search_stats* stats, void* stream) {
  if (!ix || !params) return fail(GIVF_EINVAL, "null argument");
  return run_search(ix, queries, nq, params, OUT_FULL, capacity, ids, dists, stats, stream);
}

int givf_plan_capacity(givf_index_t ix, const givf_search_params* params, int64_t* cap) {
  if (!ix || !params || !cap) return fail(GIVF_EINVAL, "null argument");
  Plan pl;
  int rc = build_plan(ix, params, &pl);
  if (rc) return rc;
  *cap = pl.cap_w;
  return GIVF_OK;
}

int givf_plan(givf_index_t ix, const float* queries, int64_t nq, const givf_search_params* params,
              int64_t cap, void* items, int32_t* nitems, givf_search_stats* stats, void* stream) {
  if (!ix || !params) return fail(GIVF_EINVAL, "null argument");
  static_assert(sizeof(PlanItem) == sizeof(givf_plan_item), "plan item layout");
  PlanOut po{reinterpret_cast<PlanItem*>(items), nitems, cap};
  return run_search(ix, queries, nq, params, OUT_PLAN, 0, nullptr, nullptr, stats, stream, &po);
}

int givf_search_planned(givf_index_t ix, const float* queries, int64_t nq,
                        const givf_search_params* params, const int64_t* offsets, const void* items,
                        int32_t k, int32_t* ids, float* dists, void* stream) {
  if (!ix || !params) return fail(GIVF_EINVAL, "null argument");
  Plan pl;
  int rc = build_plan(ix, params, &pl);
  if (rc) return rc;
  if (k < 1 || k > 4096) return fail(GIVF_EINVAL, "need 1 <= k <= 4096");
  if (nq == 0) return GIVF_OK;
  if (!queries || !offsets || !items || !ids || !dists) return fail(GIVF_EINVAL, "null argument");
  if (!is_device_ptr(offsets) || !is_device_ptr(items))
    return fail(GIVF_EINVAL, "planned search expects device offsets / items");
  std::lock_guard<std::mutex> lock(ix->mu);
  CUDA_TRY(cudaSetDevice(ix->device));
  cudaStream_t st = (cudaStream_t)stream;
  const IndexView& v = ix->v;
  const bool q_dev = is_device_ptr(queries);
  int32_t* const ids_w = kernel_writable(ids);
  float* const dists_w = kernel_writable(dists);
  const bool out_dev = ids_w && dists_w;
  const bool host_out = !(is_device_ptr(ids) && is_device_ptr(dists));
  size_t per_q = aligned_bytes<float>(v.d) + aligned_bytes<WorkItem>(pl.cap_w) +
                 aligned_bytes<int>(1) + aligned_bytes<float>((size_t)v.M * 256) + 256;
  if (!out_dev) per_q += (size_t)k * 8 + 512;
  const size_t budget = workspace_budget();
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>({nq, 65535, (int64_t)(budget / per_q)}));
  chunk = (nq + (nq + chunk - 1) / chunk - 1) / ((nq + chunk - 1) / chunk);
  const size_t slice = ((per_q * (size_t)chunk + (1 << 20)) + 4095) & ~(size_t)4095;
  CUDA_TRY(ix->arena.reserve(slice));
  for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
    const int bq = (int)std::min<int64_t>(chunk, nq - q0);
    Arena ar;
    ar.base = ix->arena.base;
    ar.cap = slice;
    ar.reset();
    const float* dQ;
    if (q_dev) {
      dQ = queries + q0 * v.d;
    } else {
      float* tmp = ar.take<float>((size_t)bq * v.d);
      ARENA_CHECK(ar);
      CUDA_TRY(cudaMemcpyAsync(tmp, queries + q0 * v.d, sizeof(float) * bq * v.d,
                               cudaMemcpyHostToDevice, st));
      dQ = tmp;
    }
    WorkItem* work = ar.take<WorkItem>((size_t)bq * pl.cap_w);
    int* nwork = ar.take<int>(bq);
    float* luts = ar.take<float>((size_t)bq * v.M * 256);
    ARENA_CHECK(ar);
    staged(ST_PLAN, st, [&] {
      launch_localize(v, offsets + q0, reinterpret_cast<const PlanItem*>(items), bq, work, pl.cap_w,
                      nwork, st);
    });
    staged(ST_LUT, st, [&] { launch_build_luts(v, dQ, bq, luts, st); });
    KCHECK();
    int32_t* oid;
    float* od;
    if (out_dev) {
      oid = ids_w + q0 * k;
      od = dists_w + q0 * k;
    } else {
      oid = ar.take<int32_t>((size_t)bq * k);
      od = ar.take<float>((size_t)bq * k);
      ARENA_CHECK(ar);
    }
    ScanArgs sa{};
    sa.ix = v;
    sa.Q = dQ;
    sa.nq = bq;
    sa.work = work;
    sa.cap_w = pl.cap_w;
    sa.nwork = nwork;
    sa.mode = 0;
    sa.k = k;
    sa.out_ids = oid;
    sa.out_d = od;
    sa.luts = luts;
    staged(ST_SCAN, st, [&] {
      if (!launch_scan_warp(sa, st)) launch_scan(sa, st);
    });
    KCHECK();
    if (!out_dev) {
      CUDA_TRY(cudaMemcpyAsync(ids + q0 * k, oid, sizeof(int32_t) * bq * k, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(dists + q0 * k, od, sizeof(float) * bq * k, cudaMemcpyDeviceToHost, st));
    }
  }
  if (host_out || !q_dev) CUDA_TRY(cudaStreamSynchronize(st));
  return GIVF_OK;
}

int givf_probe_scores(givf_index_t ix, const float* queries, int64_t nq, float* scores,
                      float* eps_scale_out, void* stream) {
  if (!ix || !queries || !scores) return fail(GIVF_EINVAL, "null argument");
  if (nq == 0) return GIVF_OK;
  std::lock_guard<std::mutex> lock(ix->mu);
  CUDA_TRY(cudaSetDevice(ix->device));
  cudaStream_t st = (cudaStream_t)stream;
  const IndexView& v = ix->v;
  const int K = v.K, d = v.d;
  const bool q_dev = is_device_ptr(queries), o_dev = is_device_ptr(scores);
  const bool fz = use_fused(v);
  int nseg = 0, cap_u = 0;
  if (fz) {  // every centroid survives thr = +inf: segments sized for a whole slice
    filter_segments((int)nq, K, K, &nseg, &cap_u);
    const int ns = nseg / filter_slots();
    cap_u = (K + ns - 1) / ns + 256;
  }
  const size_t bytes = (size_t)nq * (d * 4 + (size_t)K * 4 + (size_t)nseg * cap_u * 8 + nseg * 4 +
                                     tc_kpad(d) * 2 + probe_tiles(K) * 4 + f16_pitch(d) * 2 + 64) +
                       (1 << 20);
  CUDA_TRY(ix->arena.reserve(bytes));
  Arena& ar = ix->arena;
  ar.reset();
  const float* dQ = queries;
  if (!q_dev) {
    float* t = ar.take<float>((size_t)nq * d);
    CUDA_TRY(cudaMemcpyAsync(t, queries, sizeof(float) * nq * d, cudaMemcpyHostToDevice, st));
    dQ = t;
  }
  float* D = o_dev ? scores : ar.take<float>((size_t)nq * K);
  if (fz) {
    // the fused GEMM's own fp32 scores: its filter with thr = +inf keeps all
    uint16_t* q16 = ar.take<uint16_t>((size_t)nq * f16_pitch(d));
    float* ms = ar.take<float>(nq);
    float* thr = ar.take<float>(nq);
    int* cnt = ar.take<int>((size_t)nq * nseg);
    int* cid = ar.take<int>((size_t)nq * nseg * cap_u);
    float* cval = ar.take<float>((size_t)nq * nseg * cap_u);
    ARENA_CHECK(ar);
    std::vector<float> inf((size_t)nq, INFINITY);
    CUDA_TRY(cudaMemcpyAsync(thr, inf.data(), sizeof(float) * nq, cudaMemcpyHostToDevice, st));
    launch_query_f16(dQ, (int)nq, d, v.c16e, v.c16T, q16, ms, nullptr, st);
    cudaError_t ce = launch_probe_filter(q16, v.c16, (int)nq, K, d, ms, thr, nseg, cap_u,
                                         cnt, cid, cval, st);
    if (ce != cudaSuccess) return fail(GIVF_ECUDA, std::string("probe filter: ") + cudaGetErrorString(ce));
    g_launches += 2;
    const size_t ne = (size_t)nq * nseg * cap_u;
    std::vector<int> hc((size_t)nq * nseg), hi(ne);
    std::vector<float> hv(ne), out((size_t)nq * K, NAN);
    CUDA_TRY(cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * nq * nseg, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(hi.data(), cid, sizeof(int) * ne, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(hv.data(), cval, sizeof(float) * ne, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int64_t b = 0; b < nq; ++b)
      for (int sg = 0; sg < nseg; ++sg) {
        const size_t o = ((size_t)b * nseg + sg) * cap_u;
        for (int i = 0; i < std::min(hc[(size_t)b * nseg + sg], cap_u); ++i)
          out[(size_t)b * K + hi[o + i]] = hv[o + i];
      }
    CUDA_TRY(cudaMemcpy(scores, out.data(), sizeof(float) * nq * K,
                        o_dev ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost));
    if (eps_scale_out) *eps_scale_out = probe_f16_eps(d);
    return GIVF_OK;
  }
  float* tmin = ar.take<float>((size_t)nq * probe_tiles(K));
  const bool tc = use_tensor_cores(v);
  ScoreOut so;  // the GEMM's own fp32 scores (the search path stores fp16)
  so.D32 = D;
  so.ld = K;
  if (tc) {
    void* abf = ar.take<uint16_t>((size_t)nq * tc_kpad(d));
    launch_split_bf16(dQ, (int)nq, d, 0, abf, st);
    launch_probe_gemm_tc(abf, v.csplit, v.c2f, (int)nq, K, d, so, tmin, st);
    g_launches += 2;
  } else {
    launch_probe_gemm(dQ, v.centroids, v.c2f, (int)nq, K, d, so, tmin, st);
    g_launches += 1;
  }
  KCHECK();
  if (!o_dev)
    CUDA_TRY(cudaMemcpyAsync(scores, D, sizeof(float) * nq * K, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (eps_scale_out) *eps_scale_out = tc ? kEpsScaleTC : probe_eps_scale(d);
  return GIVF_OK;
}

int givf_probe(givf_index_t ix, const float* queries, int64_t nq, int32_t nprobe,
               int32_t* regions, double* qc2, void* stream) {
  if (!ix) return fail(GIVF_EINVAL, "null argument");
  givf_search_params p{nprobe, 1.0, 1, 1, 1, 1};
  Plan pl;
  int rc = build_plan(ix, &p, &pl);
  if (rc) return rc;
  if (nq == 0) return GIVF_OK;
  std::lock_guard<std::mutex> lock(ix->mu);
  CUDA_TRY(cudaSetDevice(ix->device));
  cudaStream_t st = (cudaStream_t)stream;  // NULL = the default stream
  const bool q_dev = is_device_ptr(queries), o_dev = is_device_ptr(regions) && is_device_ptr(qc2);
  const int d = ix->v.d;
  size_t per_q = aligned_bytes<float>(d) + probe_bytes_per_query(pl) + (size_t)pl.P * 12 + 1024;
  size_t fixed = probe_fixed_bytes(pl) + (1 << 16);
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nq, (workspace_budget() - std::min(workspace_budget() - 1, fixed)) / per_q));
  chunk = std::min<int64_t>(chunk, 65535);
  CUDA_TRY(ix->arena.reserve(fixed + per_q * (size_t)chunk + (1 << 20)));
  for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
    const int bq = (int)std::min<int64_t>(chunk, nq - q0);
    Arena& ar = ix->arena;
    ar.reset();
    const float* dQ = queries + q0 * d;
    if (!q_dev) {
      float* tmp = ar.take<float>((size_t)bq * d);
      CUDA_TRY(cudaMemcpyAsync(tmp, queries + q0 * d, sizeof(float) * bq * d, cudaMemcpyHostToDevice, st));
      dQ = tmp;
    }
    int* r = o_dev ? regions + q0 * pl.P : ar.take<int>((size_t)bq * pl.P);
    double* c = o_dev ? qc2 + q0 * pl.P : ar.take<double>((size_t)bq * pl.P);
    rc = run_probe(ix, pl, dQ, bq, r, c, ar, st);
    if (rc) return rc;
    if (!o_dev) {
      CUDA_TRY(cudaMemcpyAsync(regions + q0 * pl.P, r, sizeof(int) * bq * pl.P, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaMemcpyAsync(qc2 + q0 * pl.P, c, sizeof(double) * bq * pl.P, cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  return GIVF_OK;
}

int givf_merge_topk(const int32_t* ids, const float* dists, int32_t shards, int64_t nq, int32_t k,
                    int32_t* out_ids, float* out_dists, int device, void* stream) {
  if (shards < 1 || k < 1 || (int64_t)shards * k > 65536) return fail(GIVF_EINVAL, "bad shards/k");
  if (nq == 0) return GIVF_OK;
  if (!is_device_ptr(ids) || !is_device_ptr(dists) || !is_device_ptr(out_ids) || !is_device_ptr(out_dists))
    return fail(GIVF_EINVAL, "merge expects device pointers");
  CUDA_TRY(cudaSetDevice(device));
  for (int64_t q0 = 0; q0 < nq; q0 += 65535) {
    int bq = (int)std::min<int64_t>(65535, nq - q0);
    // shard lists are (shards, nq, k): offset rows of every shard
    if (q0 == 0 && bq == nq) {
      staged(ST_MERGE, (cudaStream_t)stream, [&] {
        launch_merge_topk(ids, dists, shards, (int)nq, k, out_ids, out_dists, (cudaStream_t)stream);
      });
    } else {
      return fail(GIVF_EINVAL, "merge supports nq <= 65535 per call");
    }
  }
  KCHECK();
  return GIVF_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ builder
#include "givf_build.h"

namespace {

// Per-device scratch of the builder entry points (grow-only arena, device
// counters for the certified probe).
givf_index* builder_ctx(int device) {
  static std::mutex mu;
  static std::map<int, givf_index*> ctx;
  std::lock_guard<std::mutex> lk(mu);
  auto it = ctx.find(device);
  if (it != ctx.end()) return it->second;
  givf_index* ix = new givf_index();
  ix->device = device;
  unsigned long long* cnt = nullptr;
  if (cudaMalloc(&cnt, 256) != cudaSuccess || cudaMemset(cnt, 0, 256) != cudaSuccess) {
    cudaGetLastError();
    delete ix;
    return nullptr;
  }
  ix->allocs.push_back(cnt);
  ix->v.counters = cnt;
  ctx[device] = ix;
  return ix;
}

int device_of(const void* p, int* dev) {
  cudaPointerAttributes at;
  if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return fail(GIVF_EINVAL, "expected a device pointer");
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(GIVF_EINVAL, "expected a device pointer");
  *dev = at.device;
  return GIVF_OK;
}

}  // namespace

extern "C" {

int givf_assign_nearest(const float* x, int64_t rows, const float* centroids, int32_t k,
                        int32_t dim, int32_t* labels, float* dists, void* stream) {
  if (rows < 0 || k < 1 || dim < 1) return fail(GIVF_EINVAL, "bad shape");
  if (!assign_supported(dim)) return fail(GIVF_EINVAL, "assign needs dim <= 128");
  if (rows == 0) return GIVF_OK;
  int dev = 0, rc;
  if ((rc = device_of(x, &dev)) || (rc = device_of(centroids, &dev)) || (rc = device_of(labels, &dev)))
    return rc;
  CUDA_TRY(cudaSetDevice(dev));
  givf_index* ix = builder_ctx(dev);
  if (!ix) return fail(GIVF_ENOMEM, "builder context");
  std::lock_guard<std::mutex> lock(ix->mu);
  cudaStream_t st = (cudaStream_t)stream;
  const int Kp = assign_kpad(dim);
  const int64_t chunk = std::min<int64_t>(rows, (int64_t)1 << 24);
  const int nsplit = assign_nsplit(chunk, k);
  const size_t need = aligned_bytes<uint16_t>((size_t)k * Kp) + aligned_bytes<float>(k) +
                      aligned_bytes<uint16_t>((size_t)chunk * Kp) +
                      (size_t)nsplit * (aligned_bytes<float>(chunk) + aligned_bytes<int32_t>(chunk)) +
                      aligned_bytes<float>(chunk) + (1 << 16);
  CUDA_TRY(ix->arena.reserve(need));
  Arena& ar = ix->arena;
  ar.reset();
  void* cbf = ar.take<uint16_t>((size_t)k * Kp);
  float* c2 = ar.take<float>(k);
  void* xbf = ar.take<uint16_t>((size_t)chunk * Kp);
  float* pv = ar.take<float>((size_t)nsplit * chunk);
  int32_t* pi = ar.take<int32_t>((size_t)nsplit * chunk);
  float* x2 = dists ? ar.take<float>(chunk) : nullptr;
  ARENA_CHECK(ar);
  launch_rows_bf16(centroids, k, dim, cbf, st);
  launch_row_norms(centroids, k, dim, c2, nullptr, nullptr, st);
  g_launches += 2;
  for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
    const int64_t n = std::min<int64_t>(chunk, rows - r0);
    const int ns = nsplit > 1 ? assign_nsplit(n, k) : 1;
    launch_rows_bf16(x + r0 * dim, n, dim, xbf, st);
    cudaError_t e = launch_assign_tc(xbf, n, cbf, c2, k, dim, ns, pv, pi, st);
    if (e != cudaSuccess) return fail(GIVF_ECUDA, std::string("assign: ") + cudaGetErrorString(e));
    if (x2) launch_row_norms(x + r0 * dim, n, dim, x2, nullptr, nullptr, st);
    launch_assign_reduce(pv, pi, ns, n, x2, labels + r0, dists ? dists + r0 : nullptr, st);
    g_launches += 3 + (x2 ? 1 : 0);
    KCHECK();
  }
  return GIVF_OK;
}

int givf_encode_rows(const givf_encode_desc* ds, void* stream) {
  if (!ds) return fail(GIVF_EINVAL, "null argument");
  if (!encode_supported(ds->dim, ds->m))
    return fail(GIVF_EINVAL, "encode supports dim / m in {2..16} for m in {8, 16, 32}");
  if (ds->grouping && (!ds->neighbor_ids || ds->l < 1 || ds->l > 64))
    return fail(GIVF_EINVAL, "grouping needs neighbor_ids and 1 <= l <= 64");
  if (ds->nseg == 0) return GIVF_OK;
  int dev = 0, rc;
  if ((rc = device_of(ds->x, &dev)) || (rc = device_of(ds->codes, &dev))) return rc;
  if (encode_smem(ds->dim, ds->grouping ? ds->l : 1, ds->m) > 227 * 1024)
    return fail(GIVF_EINVAL, "encode: shared memory for dim / l / m exceeds 227 KB");
  CUDA_TRY(cudaSetDevice(dev));
  EncodeArgsC a;
  a.X = ds->x; a.order = ds->order; a.seg = ds->seg; a.seg_region = ds->seg_region;
  a.nseg = ds->nseg; a.d = ds->dim; a.L = ds->l; a.M = ds->m; a.grouping = ds->grouping;
  a.centroids = ds->centroids; a.nbr = ds->neighbor_ids; a.alphas = ds->alphas; a.csq = ds->c_sq;
  a.codewords = ds->codewords; a.cwsq = ds->cw_sq; a.lo = ds->const_lo; a.step = ds->const_step;
  a.pick = ds->pick; a.codes = ds->codes; a.cbytes = ds->const_bytes; a.consts = ds->consts;
  cudaError_t e = launch_encode_rows(a, (cudaStream_t)stream);
  g_launches += 1;
  if (e != cudaSuccess) return fail(GIVF_ECUDA, std::string("encode: ") + cudaGetErrorString(e));
  return GIVF_OK;
}

int givf_knn_exact(const float* queries, int64_t nq, const float* base, int64_t nb, int32_t dim,
                   int32_t k, int32_t* ids, double* dist, void* stream) {
  if (nq < 0 || nb < 1 || dim < 1 || dim > 1024) return fail(GIVF_EINVAL, "bad shape");
  if (k < 1 || k > nb) return fail(GIVF_EINVAL, "need 1 <= k <= nb");
  if (nb >= ((int64_t)1 << 31)) return fail(GIVF_EINVAL, "nb must be < 2^31");
  if (nq == 0) return GIVF_OK;
  int dev = 0, rc;
  if ((rc = device_of(queries, &dev)) || (rc = device_of(base, &dev)) || (rc = device_of(ids, &dev)) ||
      (rc = device_of(dist, &dev)))
    return rc;
  CUDA_TRY(cudaSetDevice(dev));
  givf_index* ix = builder_ctx(dev);
  if (!ix) return fail(GIVF_ENOMEM, "builder context");
  std::lock_guard<std::mutex> lock(ix->mu);
  cudaStream_t st = (cudaStream_t)stream;
  IndexView& v = ix->v;
  v.K = (int)nb; v.d = dim; v.G = 1; v.M = 1; v.grouping = 0; v.n = 0;
  v.centroids = base;
  Plan pl{};
  pl.P = k; pl.G = 1; pl.K = (int)nb; pl.d = dim;
  pl.total = k; pl.kept = k; pl.budget = 1; pl.cap_w = 1;
  pl.ps = probe_shape((int)nb, k);
  const bool tc = tc_supported(dim);
  const size_t persist = aligned_bytes<float>(nb) + aligned_bytes<unsigned int>(1) +
                         (tc ? aligned_bytes<uint16_t>((size_t)nb * tc_kpad_b(dim)) : 0);
  const size_t per_q = aligned_bytes<float>(dim) + probe_bytes_per_query(pl) + (size_t)k * 12 + 1024;
  const size_t fixed = probe_fixed_bytes(pl) + (1 << 16);
  const size_t budget = workspace_budget();
  int64_t chunk = budget > fixed + persist ? (int64_t)((budget - fixed - persist) / per_q) : 1;
  chunk = std::max<int64_t>(1, std::min<int64_t>({chunk, nq, (int64_t)65535}));
  const size_t slice = fixed + per_q * (size_t)chunk + (1 << 20);
  CUDA_TRY(ix->arena.reserve(persist + slice));
  Arena& top = ix->arena;
  top.reset();
  float* c2f = top.take<float>(nb);
  unsigned int* mx = top.take<unsigned int>(1);
  void* cs = tc ? top.take<uint16_t>((size_t)nb * tc_kpad_b(dim)) : nullptr;
  ARENA_CHECK(top);
  CUDA_TRY(cudaMemsetAsync(mx, 0, sizeof(unsigned int), st));
  launch_row_norms(base, nb, dim, c2f, nullptr, mx, st);
  if (tc) launch_split_bf16(base, (int)nb, dim, 1, cs, st);
  g_launches += tc ? 2 : 1;
  KCHECK();
  unsigned int mxh = 0;
  CUDA_TRY(cudaMemcpyAsync(&mxh, mx, sizeof mxh, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float cmaxf;
  std::memcpy(&cmaxf, &mxh, sizeof cmaxf);
  v.c2f = c2f;
  v.cmax = (float)((double)cmaxf * (1.0 + 1e-6));
  v.csplit = cs;
  for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
    const int bq = (int)std::min<int64_t>(chunk, nq - q0);
    Arena ar;
    ar.base = static_cast<char*>(top.base) + top.off;
    ar.cap = top.cap - top.off;
    ar.reset();
    rc = run_probe(ix, pl, queries + q0 * dim, bq, ids + q0 * k, dist + q0 * k, ar, st);
    if (rc) return rc;
  }
  v.centroids = nullptr;
  v.c2f = nullptr;
  v.csplit = nullptr;
  return GIVF_OK;
}

}  // extern "C"
