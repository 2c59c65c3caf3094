"""Parity in the BASELINE configs[2] regime and at configs[0]'s own shape.

* K = 2^20 regions, L = 64, M = 16, d = 96 with ~1.4 rows per (region,
  group) slice -- the C3 index's shape at a size the CPU oracle can check --
  at nprobe 32 / 128 / 512 and tau 0.25 / 0.5 (search.py:77-163): stats and
  probe lists bit-exact, top-100 equal outside 1e-4 tie runs, full-mode
  candidate-id sets equal, and no query leaving the certified fast paths.
* A GPU-built C1 index (1M x 96, K = 4096, L = 64, M = 8) at C1's search
  parameters with 200 queries, top-k and full-mode candidate sets.

Synthetic arrays are enough at K = 2^20: the search path reads the index as
given, so parity does not depend on how it was trained.
"""

import numpy as np
import pytest

from parity import assert_ranked_equal, assert_topk_equal

pytestmark = pytest.mark.gpu


def _k20_arrays():
    """The K = 2^20 index and 100 queries (deterministic)."""
    import torch

    from paper_1802_02422_b200.builder import neighbor_centroids, norm_terms
    from paper_1802_02422_b200.device_index import DeviceIndex, IndexArrays

    g = torch.Generator(device="cuda").manual_seed(20)
    k, l, m, d, n = 1 << 20, 64, 16, 96, 96_000_000
    cent = torch.randn(k, d, device="cuda", generator=g)
    cent /= cent.norm(dim=1, keepdim=True)
    nbr = neighbor_centroids(cent, l)
    alphas = 0.05 + 0.55 * torch.rand(k, device="cuda", generator=g)
    nt = norm_terms(cent, nbr, alphas)
    key = torch.randint(0, k * l, (n,), device="cuda", generator=g, dtype=torch.int64)
    order = torch.sort(key, stable=True).indices
    gsize = torch.bincount(key, minlength=k * l).reshape(k, l).int()
    offs = torch.zeros(k + 1, dtype=torch.int64, device="cuda")
    offs[1:] = torch.cumsum(gsize.sum(1).long(), 0)
    codes = torch.randint(0, 256, (n, m), device="cuda", generator=g, dtype=torch.uint8)
    cbytes = torch.randint(0, 256, (n,), device="cuda", generator=g, dtype=torch.uint8)
    cw = 0.05 * torch.randn(m, 256, d // m, device="cuda", generator=g)
    qsrc = torch.randint(0, k, (100,), device="cuda", generator=g)
    q = cent[qsrc] + 0.04 * torch.randn(100, d, device="cuda", generator=g)
    q /= q.norm(dim=1, keepdim=True)
    arr = IndexArrays(
        centroids=cent.cpu().numpy(), alphas=alphas.cpu().numpy(), neighbor_ids=nbr.int().cpu().numpy(),
        norm_terms=nt.cpu().numpy(), group_sizes=gsize.cpu().numpy(), region_offsets=offs.cpu().numpy(),
        point_ids=order.int().cpu().numpy(), codes=codes.cpu().numpy(), const_bytes=cbytes.cpu().numpy(),
        codewords=cw.cpu().numpy(), rotation=None, const_lo=-0.5, const_hi=0.5, grouping=True)
    del key, order, codes, cbytes
    torch.cuda.empty_cache()
    return arr, q.cpu().numpy()


@pytest.fixture(scope="module")
def k20():
    from paper_1802_02422_b200.device_index import DeviceIndex

    arr, q = _k20_arrays()
    return arr, DeviceIndex(arr), q


_RETRY_CODE = """
import sys, json, numpy as np
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
import test_gpu_parity_scale as t
from paper_1802_02422_b200 import SearchParams, search_batch
from paper_1802_02422_b200.device_index import DeviceIndex
arr, q = t._k20_arrays()
dev = DeviceIndex(arr)
ids, d, st = search_batch(dev, q, SearchParams(nprobe=512, tau=0.5, candidates=10_000), k=100)
np.savez(%(out)r, ids=ids, d=d, st=st, fb=dev.fallback_counts()["probe"], retry=dev.probe_retries())
"""


def test_k20_fused_retry_pass(tmp_path):
    """A sampled threshold aimed at 128 survivors (GIVF_FUSED_TARGET=0) is
    below the 512th score for every query: all of them take the fused
    probe's retry pass (guaranteed threshold) instead of the exhaustive
    float64 probe, with results identical to the default run."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    outs = {}
    for name, env in (("default", {}), ("retry", {"GIVF_FUSED_TARGET": "0"})):
        out = str(tmp_path / f"{name}.npz")
        code = _RETRY_CODE % dict(root=os.path.dirname(here), tests=here, out=out)
        subprocess.check_call([sys.executable, "-c", code], env=dict(os.environ, **env))
        outs[name] = np.load(out)
    a, b = outs["default"], outs["retry"]
    assert int(a["retry"]) == 0 and int(a["fb"]) == 0
    assert int(b["retry"]) == b["ids"].shape[0] and int(b["fb"]) == 0
    np.testing.assert_array_equal(a["ids"], b["ids"])
    np.testing.assert_array_equal(a["d"], b["d"])
    np.testing.assert_array_equal(a["st"], b["st"])


@pytest.mark.parametrize("nprobe,tau", [(32, 0.5), (32, 0.25), (128, 0.5), (128, 0.25),
                                        (512, 0.5), (512, 0.25)])
def test_k20_topk_and_stats(k20, nprobe, tau):
    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch

    arr, dev, q = k20
    q = q[:40]  # the CPU oracle takes ~0.5 s per query at K = 2^20
    p = SearchParams(nprobe=nprobe, tau=tau, candidates=10_000)
    fb0 = dev.fallback_counts()
    ids, d, st = search_batch(dev, q, p, k=100)
    fb1 = dev.fallback_counts()
    c_sq = np.einsum("kd,kd->k", arr.centroids.astype(np.float64), arr.centroids.astype(np.float64))
    cmax = float(np.sqrt(c_sq.max()))
    probe = lambda c, qq, P: so.probe_exact_fast(c, qq, P, c_sq=c_sq, cmax=cmax)  # noqa: E731
    wi, wd, ws = so.search_topk(arr, q, so.Params(**vars(p)), 100, probe=probe)
    np.testing.assert_array_equal(st, ws)
    for i in range(q.shape[0]):
        assert_topk_equal(ids[i], d[i], wi[i], wd[i])
    # the certified fast paths held: no exhaustive probe, no exact planner
    assert fb1["probe"] == fb0["probe"], (fb0, fb1)
    assert fb1["plan"] == fb0["plan"], (fb0, fb1, dev.plan_fallback_reasons())
    if nprobe >= 128:  # walks that begin more groups than K4 stages
        assert (st[:, 1] > 1536).any()


def test_k20_probe_lists_bit_exact(k20):
    from oracle import search_oracle as so
    from paper_1802_02422_b200.query import probe

    arr, dev, q = k20
    for nprobe in (32, 512):
        regions, qc2 = probe(dev, q[:16], nprobe)
        for i in range(16):
            want_r, want_c = so.probe_exact(arr.centroids, q[i], nprobe)
            np.testing.assert_array_equal(regions[i], want_r)
            # float64 sums of 96 terms in another order: a few ulps
            np.testing.assert_allclose(qc2[i], want_c, rtol=4e-15, atol=0)


def test_k20_full_mode_candidate_sets(k20):
    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch

    arr, dev, q = k20
    p = SearchParams(nprobe=128, tau=0.5, candidates=10_000)
    res = search_batch(dev, q[:12], p)
    for i, r in enumerate(res):
        wi, wd, ws = so.search_one(arr, q[i], so.Params(**vars(p)))
        assert (r.stats.regions_visited, r.stats.subregions_visited, r.stats.subregions_pruned,
                r.stats.codes_scanned) == tuple(ws)
        assert_ranked_equal(r.ids, r.distances, wi, wd)


@pytest.fixture(scope="module")
def c1_built():
    import torch

    from paper_1802_02422_b200.builder import BuildSpec, SynthSpec, build_synthetic

    torch.manual_seed(0)
    data = SynthSpec(d=96, n_clusters=4096, sigma=0.3, noise="total", seed=0)
    spec = BuildSpec(n=1_000_000, k=4096, l=64, m=8, n_learn=100_000, kmeans_iters=10,
                     pq_iters=15, seed=0)
    return build_synthetic(data, spec, 200, device="cuda", log=lambda *_: None)


def test_c1_shape_topk_and_full(c1_built):
    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex

    arr, q, gt = c1_built
    dev = DeviceIndex(arr)
    p = SearchParams(nprobe=32, tau=0.5, candidates=10_000)
    ids, d, st = search_batch(dev, q, p, k=100)
    wi, wd, ws = so.search_topk(arr, q, so.Params(**vars(p)), 100)
    np.testing.assert_array_equal(st, ws)
    for i in range(q.shape[0]):
        assert_topk_equal(ids[i], d[i], wi[i], wd[i])
    assert so.recall_at_r(list(ids), gt, 10) == so.recall_at_r(list(wi), gt, 10)
    res = search_batch(dev, q[:50], p)
    for i, r in enumerate(res):
        fi, fd, fs = so.search_one(arr, q[i], so.Params(**vars(p)))
        assert_ranked_equal(r.ids, r.distances, fi, fd)
    assert dev.fallback_counts() == {"probe": 0, "plan": 0}
