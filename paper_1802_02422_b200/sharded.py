"""Multi-GPU layout: one process per GPU, every rank owns a
slice of EVERY inverted list.

  * Rank g of G keeps rows [floor(g*s/G), floor((g+1)*s/G)) of each (region,
    group) slice of size s (`device_index.shard_rows`), in stored order.
  * Centroids, alphas, neighbor ids, norm terms and the GLOBAL group-size
    table are replicated, so every rank computes the identical probe, kept
    order and budget crossing with no communication; its local scan length of
    a kept group is clip(len_global - lo_g, 0, cnt_g).
  * The only exchange is an all-gather of the per-rank top-k (dist f32,
    id i32) over NCCL, followed by the K7 merge kernel; ties resolve by
    (dist, id), so the merged list equals the single-GPU top-k.

The per-rank search and the merge are injectable so the host-side protocol
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
    """This rank's shard plus the gather/merge protocol."""

    def __init__(self, index, rank: int, world: int, device: int = 0, group=None,
                 local_search=None, local_merge=None):
        self.rank, self.world, self.group = int(rank), int(world), group
        self._local_search = local_search
        self._local_merge = local_merge
        self.dev = None
        if local_search is None:
            self.dev = DeviceIndex(index, device=device, shard=(rank, world))

    def search_topk(self, queries, params, k: int):
        """Global top-k of every query: (ids, dists, stats), identical on all
        ranks.  stats are the global SearchStats (every rank computes them)."""
        import torch
        import torch.distributed as dist

        if self._local_search is None:
            from .query import search_batch

            ids, dists, stats = search_batch(self.dev, queries, params, k=k)
        else:
            ids, dists, stats = self._local_search(queries, params, k)
        if self.world == 1:
            return ids, dists, stats
        all_i = torch.empty((self.world,) + tuple(ids.shape), dtype=ids.dtype, device=ids.device)
        all_d = torch.empty((self.world,) + tuple(dists.shape), dtype=dists.dtype, device=dists.device)
        if hasattr(dist, "all_gather_into_tensor") and ids.is_cuda:
            dist.all_gather_into_tensor(all_i, ids.contiguous(), group=self.group)
            dist.all_gather_into_tensor(all_d, dists.contiguous(), group=self.group)
        else:
            dist.all_gather(list(all_i.unbind(0)), ids.contiguous(), group=self.group)
            dist.all_gather(list(all_d.unbind(0)), dists.contiguous(), group=self.group)
        merge = self._local_merge or merge_topk
        mi, md = merge(all_i, all_d, k)
        return mi, md, stats
