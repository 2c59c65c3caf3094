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
        ids, d, st = sx.search_topk(fx.queries, p, 40)
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
