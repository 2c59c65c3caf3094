// Plans that cross ranks (list-sharded layout with query-sharded
// planning).  Rank r probes and plans its share of the queries with the
// replicated GLOBAL group sizes (k_plan_approx / k_plan with global_items),
// and the plans -- one 16-byte PlanItem per begun group: global group index,
// global scan length, float64 base (search.py:131-148) -- are all-gathered.
// Every rank then localizes every query's plan to the rows it holds: the
// slice [lo, lo + cnt) of group gi scans clip(len - lo, 0, cnt) rows from
// its local start, exactly the emission rule of the unsharded planner
// (plan_approx.cu emit_round), so the per-rank top-k lists merge (K7) to the
// single-GPU result.
#include "common.cuh"
#include "kernels.h"

namespace givf {

// one warp per query
__global__ void k_items_from_work(const WorkItem* __restrict__ work, int64_t cap_w,
                                  const int* __restrict__ nwork, int nq, PlanItem* __restrict__ items,
                                  int64_t cap, int* __restrict__ nitems) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nq) return;
  const int n = nwork[b];
  const int m = (int)min((int64_t)n, cap);
  for (int i = lane; i < m; i += 32) {
    const WorkItem& w = work[(int64_t)b * cap_w + i];
    PlanItem it;
    it.group = (int32_t)w.start;
    it.len = w.len;
    it.base = w.base;
    items[(int64_t)b * cap + i] = it;
  }
  if (lane == 0) nitems[b] = n;  // > cap: the caller's buffer was too small
}

__global__ void k_localize(IndexView ix, const int64_t* __restrict__ offsets,
                           const PlanItem* __restrict__ items, int nq, WorkItem* __restrict__ work,
                           int64_t cap_w, int* __restrict__ nwork) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nq) return;
  const int64_t i0 = offsets[b], i1 = offsets[b + 1];
  WorkItem* W = work + (int64_t)b * cap_w;
  int out = 0;
  for (int64_t i = i0; i < i1; i += 32) {
    const int64_t j = i + lane;
    int64_t ll = 0, start = 0;
    double base = 0.0;
    if (j < i1) {
      const PlanItem it = items[j];
      const int64_t gi = it.group;
      const int64_t lo = ix.llo ? ix.llo[gi] : 0;
      const int64_t cnt = ix.lsize ? ix.lsize[gi] : ix.gsize[gi];
      ll = min(max((int64_t)it.len - lo, (int64_t)0), cnt);
      start = ix.lstart[gi];
      base = it.base;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, ll > 0);
    if (ll > 0) {
      const int pos = out + __popc(bal & ((1u << lane) - 1u));
      if (pos < cap_w) {
        WorkItem w;
        w.start = start;
        w.len = (int32_t)ll;
        w.flat = 0;
        w.base = base;
        w.score = base;
        W[pos] = w;
      }
    }
    out += __popc(bal);
  }
  if (lane == 0) nwork[b] = (int)min((int64_t)out, cap_w);
}

void launch_items_from_work(const WorkItem* work, int64_t cap_w, const int* nwork, int nq,
                            PlanItem* items, int64_t cap, int* nitems, cudaStream_t s) {
  const int per = 8;
  k_items_from_work<<<(nq + per - 1) / per, per * 32, 0, s>>>(work, cap_w, nwork, nq, items, cap,
                                                               nitems);
}

void launch_localize(const IndexView& ix, const int64_t* offsets, const PlanItem* items, int nq,
                     WorkItem* work, int64_t cap_w, int* nwork, cudaStream_t s) {
  const int per = 8;
  k_localize<<<(nq + per - 1) / per, per * 32, 0, s>>>(ix, offsets, items, nq, work, cap_w, nwork);
}

}  // namespace givf
