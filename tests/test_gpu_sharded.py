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
