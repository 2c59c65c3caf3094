"""GPU checks of individual kernels and of the certified fast paths:
tensor-core probe accuracy vs its a-priori bound, SIMT/tensor-core
equivalence, forced fallbacks, and parity on a GPU-built index."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import golden_io
from parity import assert_ranked_equal, assert_topk_equal

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _arrays(centroids, seed=0, m=8):
    from paper_1802_02422_b200.device_index import IndexArrays

    k, d = centroids.shape
    rng = np.random.default_rng(seed)
    return IndexArrays(
        centroids=np.ascontiguousarray(centroids, np.float32), alphas=np.zeros(k, np.float32),
        neighbor_ids=None, norm_terms=None, group_sizes=np.zeros((k, 1), np.int32),
        region_offsets=np.zeros(k + 1, np.int64), point_ids=np.zeros(0, np.int32),
        codes=np.zeros((0, m), np.uint8), const_bytes=np.zeros(0, np.uint8),
        codewords=rng.standard_normal((m, 256, d // m)).astype(np.float32), rotation=None,
        const_lo=0.0, const_hi=1.0, grouping=False)


@pytest.mark.parametrize("scale,d", [(1.0, 96), (37.0, 96), (1.0, 128), (1.0, 64), (1.0, 24)])
def test_probe_scores_within_bound(scale, d):
    from paper_1802_02422_b200.query import probe_scores

    rng = np.random.default_rng(1)
    c = (rng.standard_normal((5000, d)) * scale).astype(np.float32)
    q = (rng.standard_normal((300, d)) * scale).astype(np.float32)
    s, eps_scale = probe_scores(_arrays(c), q)
    c64, q64 = c.astype(np.float64), q.astype(np.float64)
    exact = (c64 * c64).sum(1)[None, :] - 2.0 * q64 @ c64.T
    cmax = np.sqrt((c64 * c64).sum(1).max())
    bound = eps_scale * (cmax**2 + 2.0 * np.linalg.norm(q64, axis=1) * cmax)
    ratio = np.abs(s - exact) / bound[:, None]
    print(f"max |err| / bound = {ratio.max():.3e}")
    assert ratio.max() < 0.25  # the bound holds with a 4x margin


@pytest.mark.parametrize("family", ["aligned", "boundary", "wide"])
@pytest.mark.parametrize("d", [32, 96, 128])
def test_probe_bound_adversarial(family, d):
    """Inputs that maximise the bf16-split residual and the accumulation error
    (all products one sign, mantissas just below a bf16 rounding boundary,
    a 2^+-6 exponent spread across columns) stay 4x inside the a-priori
    bound the certified fast paths rely on (tools/eps_probe.py)."""
    from paper_1802_02422_b200.query import probe_scores

    rng = np.random.default_rng(7)
    if family == "aligned":
        c = rng.uniform(0.5, 1.0, (4096, d))
    elif family == "boundary":
        c = 1.0 + (2.0**-8 - 2.0**-17) * rng.integers(1, 127, (4096, d))
    else:
        c = rng.uniform(0.5, 1.0, (4096, d)) * 2.0 ** rng.integers(-6, 6, (1, d))
    c = c.astype(np.float32)
    q = c[:256].copy()
    s, eps_scale = probe_scores(_arrays(c), q)
    c64, q64 = c.astype(np.float64), q.astype(np.float64)
    exact = (c64 * c64).sum(1)[None, :] - 2.0 * q64 @ c64.T
    cmax = np.sqrt((c64 * c64).sum(1).max())
    unit = cmax**2 + 2.0 * np.linalg.norm(q64, axis=1)[:, None] * cmax
    ratio = np.abs(s - exact) / (eps_scale * unit)
    print(f"{family} d={d}: max |err| / bound = {ratio.max():.3e}")
    assert ratio.max() < 0.25


_MODE_CODE = (
    "import sys, json, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r);"
    "import golden_io; from paper_1802_02422_b200 import SearchParams, search_batch;"
    "fx = golden_io.load('c1like_m16');"
    "p = SearchParams(nprobe=32, tau=0.5, candidates=3000);"
    "i, d, s = search_batch(fx.index, fx.queries, p, k=50);"
    "full = search_batch(fx.index, fx.queries, p);"
    "print(json.dumps([i.tolist(), d.tolist(), s.tolist(),"
    " [r.ids.tolist() for r in full], [r.distances.tolist() for r in full]]))")


def _run_mode(env_over):
    code = _MODE_CODE % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, **env_over)
    out = subprocess.check_output([sys.executable, "-c", code], env=env, cwd=ROOT)
    return json.loads(out.decode().strip().splitlines()[-1])


@pytest.fixture(scope="module")
def default_mode_result():
    return _run_mode({})


@pytest.mark.parametrize("env_over", [
    {"GIVF_PROBE": "simt"},                        # SIMT fp32 probe GEMM
    {"GIVF_CHUNK_QUERIES": "3"},                   # many small chunks (arena reuse)
    {"GIVF_SCAN_LUT": "plain"},                    # warp scan, [m][256] LUT (bank conflicts)
    {"GIVF_SCAN": "warp"},                         # block-wide segment windows (k_scan_warp)
    {"GIVF_SCAN_COPIES": "full"},                  # 32 / M LUT copies, 3 CTAs/SM (conflict-free lookups)
    {"GIVF_GEMM_SPLIT": "3"},                      # probe GEMM work units: 3 slices per m-block
    {"GIVF_RS_SPLIT": "5"},                        # K4b: 5 CTAs per query
    {"GIVF_PLAN_WCAP": "8"},                       # K4 windows overflow: the 2048-entry retry pass
    {"GIVF_PROBE": "fused"},                       # fused probe, 128 queries x 256 centroids
    {"GIVF_PROBE": "fused", "GIVF_FILTER_SHAPE": "2x128"},  # 2 x 128 queries x 128 centroids
    {"GIVF_PROBE": "fused", "GIVF_FILTER_SHAPE": "4x64"},  # 4 x 128 queries x 64 centroids
    {"GIVF_PROBE": "fused", "GIVF_FILTER_SHAPE": "1x128"},  # 128 queries, rows shared by 2 warps
    {"GIVF_PROBE": "fused", "GIVF_FUSED_TARGET": "0"},  # threshold at ~128 survivors
    {"GIVF_PROBE": "fused", "GIVF_PACK_NEIGHBORS": "0"},  # K3a gathers rows instead of the packed copy
    {"GIVF_PROBE": "fused", "GIVF_FILTER_WARPS": "8"},  # 8 epilogue warps instead of 16
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_execution_modes_agree(env_over, default_mode_result):
    """Every tuning knob changes how the work is scheduled, never the result:
    top-k ids / distances / stats and the full reranked lists are identical."""
    got = _run_mode(env_over)
    want = default_mode_result
    assert got[0] == want[0]
    assert got[2] == want[2]
    np.testing.assert_array_equal(np.array(got[1]), np.array(want[1]))
    assert got[3] == want[3]
    for a, b in zip(got[4], want[4]):
        np.testing.assert_array_equal(np.array(a), np.array(b))


def test_near_duplicate_centroids_take_the_fallback_and_stay_exact():
    """Pairs of centroids 1e-7 apart make the fp32 scores unable to certify
    the probe boundary or the pruning cut; the exhaustive / exact paths must
    take over and the results must still equal the oracle."""
    from types import SimpleNamespace

    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex

    fx = golden_io.load("c1like_m8")
    ix = SimpleNamespace(**vars(fx.index))
    c = ix.centroids.copy()
    c[1::2] = c[0::2] + np.float32(1e-7)
    ix.centroids = c
    dev = DeviceIndex(ix)
    for p in (SearchParams(nprobe=31, tau=0.5, candidates=4000),
              SearchParams(nprobe=16, tau=0.7, candidates=1500)):
        ids, d, st = search_batch(dev, fx.queries, p, k=60)
        wi, wd, ws = so.search_topk(ix, fx.queries, so.Params(**vars(p)), 60)
        np.testing.assert_array_equal(st, ws)
        for i in range(len(fx.queries)):
            assert_topk_equal(ids[i], d[i], wi[i], wd[i])
    print("fallbacks", dev.fallback_counts())


def _sphere_index(seed=0, k=4096, d=96, g=8, m=16, on_sphere=1024):
    """Regions whose centroids are all (numerically) equidistant from the
    query origin, alpha = 0.5 (the neighbor distances count) and zero norm
    terms: no fp32 / fp16 score can separate them, so both certified fast
    paths must hand over."""
    from paper_1802_02422_b200.device_index import IndexArrays

    rng = np.random.default_rng(seed)
    u = rng.standard_normal((k, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    c = np.where(np.arange(k)[:, None] < on_sphere, 0.5 * u, 3.0 * u).astype(np.float32)
    sizes = rng.integers(0, 5, (k, g)).astype(np.int32)
    offs = np.zeros(k + 1, np.int64)
    np.cumsum(sizes.sum(1), out=offs[1:])
    n = int(offs[-1])
    return IndexArrays(
        centroids=c, alphas=np.full(k, 0.5, np.float32),
        neighbor_ids=rng.integers(0, k, (k, g)).astype(np.int32),
        norm_terms=np.zeros((k, g), np.float32), group_sizes=sizes, region_offsets=offs,
        point_ids=rng.permutation(n).astype(np.int32),
        codes=rng.integers(0, 256, (n, m)).astype(np.uint8),
        const_bytes=rng.integers(0, 256, n).astype(np.uint8),
        codewords=(0.1 * rng.standard_normal((m, 256, d // m))).astype(np.float32),
        rotation=None, const_lo=-0.5, const_hi=0.5, grouping=True)


@pytest.mark.parametrize("retry", [True, False])
def test_equidistant_regions_force_both_fallbacks(retry, monkeypatch):
    """Tied group scores overflow the planner's certified window: with the
    retry pass its 2048-entry window takes them; without it (GIVF_PLAN_RETRY=0)
    the queries go to the exact planner."""
    monkeypatch.setenv("GIVF_PLAN_RETRY", "1" if retry else "0")
    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex

    arr = _sphere_index()
    rng = np.random.default_rng(9)
    q = (1e-3 * rng.standard_normal((6, arr.dim))).astype(np.float32)
    dev = DeviceIndex(arr)
    p = SearchParams(nprobe=100, tau=0.5, candidates=600)
    ids, d, st = search_batch(dev, q, p, k=50)
    wi, wd, ws = so.search_topk(arr, q, so.Params(**vars(p)), 50)
    np.testing.assert_array_equal(st, ws)
    for i in range(q.shape[0]):
        assert_topk_equal(ids[i], d[i], wi[i], wd[i])
    counts = dev.fallback_counts()
    print("fallbacks", counts, "plan retries", dev.plan_retries())
    assert counts["probe"] > 0
    if retry:
        assert dev.plan_retries() > 0
    else:
        assert dev.plan_retries() == 0 and counts["plan"] > 0


@pytest.fixture(scope="module")
def built_index():
    import torch

    from paper_1802_02422_b200.builder import BuildSpec, SynthSpec, build_synthetic

    torch.manual_seed(0)
    data = SynthSpec(d=96, n_clusters=1500, sigma=0.3, noise="total", seed=3)
    spec = BuildSpec(n=300_000, k=2048, l=32, m=16, n_learn=60_000, kmeans_iters=6, pq_iters=6, seed=3)
    arr, q, gt = build_synthetic(data, spec, 120, device="cuda", log=lambda *_: None)
    return arr, q, gt


@pytest.mark.parametrize("nprobe,tau,cand", [(64, 0.5, 10_000), (128, 0.25, 3000), (16, 1.0, 100_000)])
def test_parity_on_gpu_built_index(built_index, nprobe, tau, cand):
    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch

    arr, q, gt = built_index
    p = SearchParams(nprobe=nprobe, tau=tau, candidates=cand)
    ids, d, st = search_batch(arr, q, p, k=100)
    wi, wd, ws = so.search_topk(arr, q, so.Params(**vars(p)), 100)
    np.testing.assert_array_equal(st, ws)
    for i in range(q.shape[0]):
        assert_topk_equal(ids[i], d[i], wi[i], wd[i])
    r10 = so.recall_at_r(list(ids), gt, 10)
    assert r10 == so.recall_at_r(list(wi), gt, 10)


def test_many_begun_groups_stream_without_fallback(built_index):
    """A budget walk that begins more groups than the planner's staging arrays
    hold (≈4.6 rows per group here, 60k-candidate budget ⇒ >10k groups) is
    emitted by streaming, not by the exact fallback; results equal the oracle."""
    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.device_index import DeviceIndex

    arr, q, _ = built_index
    dev = DeviceIndex(arr)
    p = SearchParams(nprobe=512, tau=1.0, candidates=60_000)
    ids, d, st = search_batch(dev, q[:24], p, k=100)
    wi, wd, ws = so.search_topk(arr, q[:24], so.Params(**vars(p)), 100)
    np.testing.assert_array_equal(st, ws)
    assert (st[:, 1] > 1536).all()
    for i in range(24):
        assert_topk_equal(ids[i], d[i], wi[i], wd[i])
    assert dev.fallback_counts()["plan"] == 0


def test_parity_sift_u8_d128():
    """BASELINE config 3's data family at small scale: d = 128 uint8-valued
    rows (unnormalised, distances ~1e5), M = 16; the 2-stage tensor-core
    probe (d > 106) and the full pipeline against the oracle."""
    import torch

    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.builder import BuildSpec, SynthSpec, build_synthetic

    torch.manual_seed(0)
    data = SynthSpec(d=128, n_clusters=700, kind="sift_u8", seed=5)
    spec = BuildSpec(n=200_000, k=1024, l=32, m=16, n_learn=50_000, kmeans_iters=5, pq_iters=5,
                     seed=5)
    arr, q, gt = build_synthetic(data, spec, 64, device="cuda", log=lambda *_: None)
    assert float(q.min()) >= 0.0 and float(q.max()) <= 255.0 and np.all(q == np.round(q))
    for nprobe, tau, cand in [(32, 0.5, 10_000), (96, 0.25, 3_000)]:
        p = SearchParams(nprobe=nprobe, tau=tau, candidates=cand)
        ids, d, st = search_batch(arr, q, p, k=100)
        wi, wd, ws = so.search_topk(arr, q, so.Params(**vars(p)), 100)
        np.testing.assert_array_equal(st, ws)
        for i in range(q.shape[0]):
            assert_topk_equal(ids[i], d[i], wi[i], wd[i])


def test_parity_c2_family_at_10m():
    """BASELINE configs[1]'s index shape except n: K = 2^16 regions, L = 64,
    M = 16, per-coordinate noise, 10M rows built on the GPU; the full path at
    the C2 search parameters against the oracle (stats bit-exact, top-100
    equal outside 1e-4 tie runs), plus a wide-probe setting."""
    import torch

    from oracle import search_oracle as so
    from paper_1802_02422_b200 import SearchParams, search_batch
    from paper_1802_02422_b200.builder import BuildSpec, SynthSpec, build_synthetic
    from paper_1802_02422_b200.device_index import DeviceIndex

    torch.manual_seed(0)
    data = SynthSpec(d=96, n_clusters=65536, sigma=0.3, noise="per_coord", seed=11)
    spec = BuildSpec(n=10_000_000, k=65536, l=64, m=16, n_learn=1_000_000, kmeans_iters=4,
                     pq_iters=6, seed=11)
    arr, q, gt = build_synthetic(data, spec, 40, device="cuda", log=lambda *_: None)
    dev = DeviceIndex(arr)
    for nprobe, tau, cand in ((64, 0.5, 10_000), (256, 0.25, 30_000)):
        p = SearchParams(nprobe=nprobe, tau=tau, candidates=cand)
        ids, d, st = search_batch(dev, q, p, k=100)
        wi, wd, ws = so.search_topk(arr, q, so.Params(**vars(p)), 100)
        np.testing.assert_array_equal(st, ws)
        for i in range(q.shape[0]):
            assert_topk_equal(ids[i], d[i], wi[i], wd[i])
    assert dev.fallback_counts()["probe"] == 0
    # full reference semantics (every scanned code): candidate-id sets
    # bit-exact, ranked lists equal outside tie runs
    p = SearchParams(nprobe=64, tau=0.5, candidates=10_000)
    for i, r in enumerate(search_batch(dev, q[:16], p)):
        fi, fd, fs = so.search_one(arr, q[i], so.Params(**vars(p)))
        assert (r.stats.regions_visited, r.stats.subregions_visited, r.stats.subregions_pruned,
                r.stats.codes_scanned) == tuple(fs)
        assert_ranked_equal(r.ids, r.distances, fi, fd)
