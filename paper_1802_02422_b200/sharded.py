"""Multi-GPU layout: one process per GPU, every rank owns a
slice of EVERY inverted list.

  * Rank g of G keeps rows [floor(g*s/G), floor((g+1)*s/G)) of each (region,
    group) slice of size s (`device_index.shard_rows`), in stored order.
  * Centroids, alphas, neighbor ids, norm terms and the GLOBAL group-size
    table are replicated.
  * `search_topk` (default): query-sharded planning.  Rank g probes and plans
    only its share of the queries (search.py:77-139, global group sizes) and
    emits each query's begun groups in global form (givf_plan: group index,
    global scan length, float64 base).  The plans are all-gathered over NCCL
    (one 16-byte record per begun group), every rank localizes every query's
    plan to its own rows -- clip(len - lo_g, 0, cnt_g) rows of each planned
    slice -- and scans them (givf_search_planned); the per-rank top-k lists
    are all-gathered and merged by K7 with the (dist, id) tie rule, which
    reproduces the single-GPU top-k.  Probe, planner and scan all shrink
    with the rank count.
  * `search_topk_replicated`: every rank plans every query (no plan
    exchange; only the scan shrinks with the rank count).

The per-rank compute and the merge are injectable so the host-side protocol
can be exercised on CPU ranks (gloo) with the oracle standing in.
"""

from __future__ import annotations

import ctypes

from . import _native
from .device_index import DeviceIndex


def merge_topk(ids, dists, k: int):
    """K7 on the GPU: (G, B, k) CUDA tensors -> (B, k) by (dist, id)."""
    import torch

    g, b, kk = ids.shape
    assert kk == k and dists.shape == ids.shape
    ids = ids.contiguous()
    dists = dists.contiguous()
    out_i = torch.empty((b, k), dtype=torch.int32, device=ids.device)
    out_d = torch.empty((b, k), dtype=torch.float32, device=ids.device)
    stream = torch.cuda.current_stream(ids.device).cuda_stream
    _native.check(_native.load().givf_merge_topk(
        ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(dists.data_ptr()), g, b, k,
        ctypes.c_void_p(out_i.data_ptr()), ctypes.c_void_p(out_d.data_ptr()),
        ids.device.index or 0, ctypes.c_void_p(stream)))
    return out_i, out_d


class ShardedIndex:
    """This rank's shard plus the exchange protocols."""

    def __init__(self, index, rank: int, world: int, device: int = 0, group=None,
                 local_search=None, local_merge=None, local_plan=None, local_scan=None):
        self.rank, self.world, self.group = int(rank), int(world), group
        self._local_search = local_search
        self._local_merge = local_merge
        self._local_plan = local_plan
        self._local_scan = local_scan
        self.dev = None
        if local_search is None and local_plan is None:
            self.dev = DeviceIndex(index, device=device, shard=(rank, world))

    # ------------------------------------------------------------ collectives
    def _gather(self, t):
        """(world,) + t.shape: every rank's t (same shape on every rank)."""
        import torch
        import torch.distributed as dist

        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if hasattr(dist, "all_gather_into_tensor") and t.is_cuda:
            dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        else:
            dist.all_gather(list(out.unbind(0)), t.contiguous(), group=self.group)
        return out

    def _merge(self, ids, dists, k):
        if self.world == 1:
            return ids, dists
        merge = self._local_merge or merge_topk
        return merge(self._gather(ids), self._gather(dists), k)

    # ------------------------------------------------------------- protocols
    def search_topk(self, queries, params, k: int):
        """Global top-k of every query with query-sharded planning: (ids,
        dists, stats), identical on all ranks.  Every rank passes the same
        queries; stats are the global SearchStats of the planning rank."""
        import torch

        from .query import compact_plans, plan_batch, search_planned

        if self.world == 1 and self._local_plan is None:  # nothing to exchange
            from .query import search_batch

            return search_batch(self.dev, queries, params, k=k)
        b = int(queries.shape[0])
        share = -(-b // self.world)  # ceil
        lo, hi = min(b, self.rank * share), min(b, (self.rank + 1) * share)
        mine = queries[lo:hi]
        if self._local_plan is None:
            items, nitems, stats = plan_batch(self.dev, mine, params)
        else:
            items, nitems, stats = self._local_plan(mine, params)
        dev = items.device
        offs, flat = compact_plans(items, nitems)
        # pad the per-rank pieces to common shapes for the all-gathers
        tot = torch.tensor([flat.shape[0]], dtype=torch.int64, device=dev)
        n_pad = torch.zeros(share, dtype=torch.int32, device=dev)
        n_pad[: hi - lo] = nitems
        s_pad = torch.zeros((share, 4), dtype=torch.int64, device=dev)
        s_pad[: hi - lo] = stats
        if self.world > 1:
            tots = self._gather(tot).view(-1)
            tmax = int(tots.max())
            f_pad = torch.zeros((max(tmax, 1), 4), dtype=torch.int32, device=dev)
            f_pad[: flat.shape[0]] = flat
            all_f, all_n, all_s = self._gather(f_pad), self._gather(n_pad), self._gather(s_pad)
            cnt = [max(0, min(b, (w + 1) * share) - min(b, w * share)) for w in range(self.world)]
            flat = torch.cat([all_f[w, : int(tots[w])] for w in range(self.world)])
            nitems = torch.cat([all_n[w, : cnt[w]] for w in range(self.world)])
            stats = torch.cat([all_s[w, : cnt[w]] for w in range(self.world)])
            offs = torch.zeros(b + 1, dtype=torch.int64, device=dev)
            offs[1:] = torch.cumsum(nitems.to(torch.int64), 0)
        if self._local_scan is None:
            ids, dists = search_planned(self.dev, queries, params, offs, flat, k)
        else:
            ids, dists = self._local_scan(queries, params, offs, flat, k)
        mi, md = self._merge(ids, dists, k)
        return mi, md, stats

    def search_topk_replicated(self, queries, params, k: int):
        """Every rank plans every query (no plan exchange), scans its rows;
        the per-rank top-k lists are all-gathered and merged."""
        if self._local_search is None:
            from .query import search_batch

            ids, dists, stats = search_batch(self.dev, queries, params, k=k)
        else:
            ids, dists, stats = self._local_search(queries, params, k)
        mi, md = self._merge(ids, dists, k)
        return mi, md, stats
