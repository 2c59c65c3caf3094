"""The multi-GPU layout on one device: every shard of every
(region, group) slice searched as its own DeviceIndex, the per-shard top-k
lists merged by the K7 kernel, must equal the single-index top-k exactly.
The shards run one after the other (no rank waits on another); the
all-gather between them is the only step a real multi-GPU run adds, and its
protocol is covered on CPU ranks by test_sharded_cpu.py."""

import numpy as np
import pytest

import golden_io

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1like_m16", "c1like_m8"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_merge_to_single_device_topk(name, world):
    import torch

    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex
    from paper_1802_02422_b200.sharded import merge_topk

    fx = golden_io.load(name)
    k = 100
    p = SearchParams(nprobe=32, tau=0.5, candidates=5000, ef_search=256)
    q = torch.from_numpy(np.ascontiguousarray(fx.queries, np.float32)).cuda()
    want_i, want_d, want_s = search_batch(DeviceIndex(fx.index, device=0), q, p, k=k)
    parts_i, parts_d = [], []
    for g in range(world):
        dev = DeviceIndex(fx.index, device=0, shard=(g, world))
        i, d, st = search_batch(dev, q, p, k=k)
        # every shard walks the same global budget: identical global stats
        torch.testing.assert_close(st, want_s, rtol=0, atol=0)
        parts_i.append(i)
        parts_d.append(d)
    mi, md = merge_topk(torch.stack(parts_i), torch.stack(parts_d), k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(mi.cpu().numpy(), want_i.cpu().numpy())
    np.testing.assert_array_equal(md.cpu().numpy(), want_d.cpu().numpy())


@pytest.mark.parametrize("name,probe", [("c1like_m16", None), ("c1like_m8", None),
                                        ("c1like_m16", "fused")])
@pytest.mark.parametrize("world", [2, 3])
def test_query_sharded_plans_scan_to_single_device_topk(name, probe, world, monkeypatch):
    """Query-sharded planning on one device: each 'rank' plans its share of
    the queries (givf_plan, global group sizes), the plans are concatenated
    as the all-gather would, every shard scans its rows of every plan
    (givf_search_planned) and K7 merges: ids, distances and stats equal the
    single-index top-k, and a shard's plans equal the full index's."""
    import subprocess
    import sys

    if probe is not None:  # the probe mode is read once per process
        code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r);"
                "import test_gpu_sharded as t; t._planned_case(%r, %d)")
        here = __import__("os").path.dirname(__file__)
        subprocess.check_call([sys.executable, "-c", code % (here + "/..", here, name, world)],
                              env=dict(__import__("os").environ, GIVF_PROBE=probe))
        return
    _planned_case(name, world)


def _planned_case(name, world):
    import torch

    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex
    from paper_1802_02422_b200.query import compact_plans, plan_batch, search_planned
    from paper_1802_02422_b200.sharded import merge_topk

    fx = golden_io.load(name)
    k = 100
    p = SearchParams(nprobe=32, tau=0.5, candidates=5000, ef_search=256)
    q = torch.from_numpy(np.ascontiguousarray(fx.queries, np.float32)).cuda()
    full = DeviceIndex(fx.index, device=0)
    want_i, want_d, want_s = search_batch(full, q, p, k=k)
    shards = [DeviceIndex(fx.index, device=0, shard=(g, world)) for g in range(world)]
    b = q.shape[0]
    share = -(-b // world)
    items, nitems, stats = [], [], []
    for g in range(world):  # rank g plans queries [g*share, (g+1)*share)
        it, n, st = plan_batch(shards[g], q[g * share:(g + 1) * share], p)
        it_f, n_f, st_f = plan_batch(full, q[g * share:(g + 1) * share], p)
        torch.testing.assert_close(n, n_f, rtol=0, atol=0)
        torch.testing.assert_close(st, st_f, rtol=0, atol=0)
        for i in range(n.shape[0]):
            torch.testing.assert_close(it[i, : n[i]], it_f[i, : n[i]], rtol=0, atol=0)
        items.append(it)
        nitems.append(n)
        stats.append(st)
    cap = max(x.shape[1] for x in items)
    items = torch.cat([torch.nn.functional.pad(x, (0, 0, 0, cap - x.shape[1])) for x in items])
    offs, flat = compact_plans(items, torch.cat(nitems))
    torch.testing.assert_close(torch.cat(stats), want_s, rtol=0, atol=0)
    parts_i, parts_d = [], []
    for g in range(world):
        i, d = search_planned(shards[g], q, p, offs, flat, k)
        parts_i.append(i)
        parts_d.append(d)
    mi, md = merge_topk(torch.stack(parts_i), torch.stack(parts_d), k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(mi.cpu().numpy(), want_i.cpu().numpy())
    np.testing.assert_array_equal(md.cpu().numpy(), want_d.cpu().numpy())
