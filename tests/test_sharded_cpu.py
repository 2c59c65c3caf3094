"""Multi-rank protocol on CPU ranks (gloo, world_size 2): shard layout,
all-gather of per-rank top-k and the (dist, id) merge reproduce the
single-index result.  The oracle stands in for the per-rank CUDA search."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_io
from oracle import search_oracle as so


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows_match_oracle_layout():
    from paper_1802_02422_b200.device_index import IndexArrays, shard_rows

    fx = golden_io.load("c1like_m8")
    arr = IndexArrays.from_any(fx.index)
    for shards in (1, 2, 3, 8):
        seen = []
        for g in range(shards):
            rows, lo, cnt = shard_rows(arr, g, shards)
            ref = so.shard_index(fx.index, g, shards)
            np.testing.assert_array_equal(arr.point_ids[rows], ref.point_ids)
            np.testing.assert_array_equal(cnt, ref.group_sizes)
            np.testing.assert_array_equal(lo, ref.lo)
            seen.append(rows)
        allr = np.sort(np.concatenate(seen))
        np.testing.assert_array_equal(allr, np.arange(arr.n))


def _rank_main(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_02422_b200.sharded import ShardedIndex

        fx = golden_io.load("c1like_m8")
        shard = so.shard_index(fx.index, rank, world)
        p = so.Params(nprobe=24, tau=0.5, candidates=2500)

        def local_search(queries, params, k):
            i, d, s = so.search_shard_topk(shard, queries, params, k)
            return torch.from_numpy(i), torch.from_numpy(d), torch.from_numpy(s)

        def local_merge(all_i, all_d, k):
            mi, md = so.merge_topk(list(all_i.numpy()), list(all_d.numpy()), k)
            return torch.from_numpy(mi), torch.from_numpy(md)

        sx = ShardedIndex(None, rank, world, local_search=local_search, local_merge=local_merge)
        ids, d, st = sx.search_topk_replicated(fx.queries, p, 40)
        if rank == 0:
            np.savez(out_path, ids=ids.numpy(), d=d.numpy(), st=st.numpy())
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_merge_equals_single(tmp_path):
    out = str(tmp_path / "r0.npz")
    mp.spawn(_rank_main, args=(2, _free_port(), out), nprocs=2, join=True)
    z = np.load(out)
    fx = golden_io.load("c1like_m8")
    p = so.Params(nprobe=24, tau=0.5, candidates=2500)
    want_i, want_d, want_s = so.search_topk(fx.index, fx.queries, p, 40)
    np.testing.assert_array_equal(z["ids"], want_i)
    np.testing.assert_array_equal(z["d"], want_d)
    np.testing.assert_array_equal(z["st"], want_s)


def _rank_main_planned(rank, world, port, out_path):
    """Query-sharded planning: each rank plans its share of the queries, the
    plans (global group, length, base) are all-gathered, every rank scans its
    rows of every plan, the top-k lists are all-gathered and merged."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_02422_b200.sharded import ShardedIndex

        fx = golden_io.load("c1like_m8")
        shard = so.shard_index(fx.index, rank, world)
        p = so.Params(nprobe=24, tau=0.5, candidates=2500)
        k = 40

        def local_plan(queries, params):
            plans = [so.plan_items(shard, q, params, sizes=shard.global_sizes) for q in queries]
            cap = max([len(x[0]) for x in plans] + [1])
            items = np.zeros((len(plans), cap, 4), np.int32)
            nitems = np.zeros(len(plans), np.int32)
            stats = np.zeros((len(plans), 4), np.int64)
            for i, (gi, ln, base, st) in enumerate(plans):
                n = len(gi)
                items[i, :n, 0] = gi
                items[i, :n, 1] = ln
                items[i, :n, 2:] = np.ascontiguousarray(base, np.float64).view(np.int32).reshape(n, 2)
                nitems[i], stats[i] = n, st
            return torch.from_numpy(items), torch.from_numpy(nitems), torch.from_numpy(stats)

        def local_scan(queries, params, offs, flat, k):
            offs, flat = offs.numpy(), flat.numpy()
            ids = np.full((len(queries), k), -1, np.int32)
            d = np.full((len(queries), k), np.inf, np.float32)
            for b, q in enumerate(queries):
                it = flat[offs[b]:offs[b + 1]]
                base = np.ascontiguousarray(it[:, 2:]).view(np.float64).ravel()
                pi, pd = so.scan_items_topk(shard, q, it[:, 0].astype(np.int64),
                                            it[:, 1].astype(np.int64), base, k)
                ids[b, : len(pi)], d[b, : len(pi)] = pi, pd
            return torch.from_numpy(ids), torch.from_numpy(d)

        def local_merge(all_i, all_d, k):
            mi, md = so.merge_topk(list(all_i.numpy()), list(all_d.numpy()), k)
            return torch.from_numpy(mi), torch.from_numpy(md)

        sx = ShardedIndex(None, rank, world, local_plan=local_plan, local_scan=local_scan,
                          local_merge=local_merge)
        # 33 queries: the last rank's share is shorter (padding in the exchange)
        ids, d, st = sx.search_topk(fx.queries[:33], p, k)
        np.savez(out_path + f".{rank}.npz", ids=ids.numpy(), d=d.numpy(), st=st.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_query_sharded_planning_equals_single(tmp_path, world):
    out = str(tmp_path / "r")
    mp.spawn(_rank_main_planned, args=(world, _free_port(), out), nprocs=world, join=True)
    fx = golden_io.load("c1like_m8")
    p = so.Params(nprobe=24, tau=0.5, candidates=2500)
    want_i, want_d, want_s = so.search_topk(fx.index, fx.queries[:33], p, 40)
    for r in range(world):  # every rank holds the merged result
        z = np.load(out + f".{r}.npz")
        np.testing.assert_array_equal(z["ids"], want_i)
        np.testing.assert_array_equal(z["d"], want_d)
        np.testing.assert_array_equal(z["st"], want_s)
