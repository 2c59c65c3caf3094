"""Pin the CPU oracle against the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

import golden_io
from oracle import search_oracle as so


@pytest.fixture(scope="module", params=golden_io.NAMES)
def fx(request):
    return golden_io.load(request.param)


def test_oracle_reproduces_reference(fx):
    for run in golden_io.exact_runs(fx):
        p = so.Params(**vars(run.params))
        for qi, q in enumerate(fx.queries):
            ids, d, st = so.search_one(fx.index, q, p)
            want_ids, want_d = run.results[qi]
            assert tuple(run.stats[qi]) == st, (fx.name, vars(run.params), qi)
            np.testing.assert_array_equal(ids, want_ids)
            # same numpy calls: equal to float32 rounding of SIMD-order LUTs
            np.testing.assert_allclose(d, want_d, rtol=1e-6, atol=1e-6)


def test_code_sums_is_pairwise8():
    rng = np.random.default_rng(0)
    for m in (8, 16):
        lut = rng.standard_normal((m, 256)).astype(np.float32)
        codes = rng.integers(0, 256, (5000, m)).astype(np.uint8)
        np.testing.assert_array_equal(so.code_sums(lut, codes), so.code_sums_pairwise8(lut, codes))


def test_ranges_to_rows_matches_loop():
    rng = np.random.default_rng(1)
    starts = rng.integers(0, 1000, 50)
    lens = rng.integers(0, 7, 50)
    want = np.concatenate([np.arange(s, s + n) for s, n in zip(starts, lens)])
    np.testing.assert_array_equal(so.ranges_to_rows(starts, lens), want)


def test_topk_is_prefix_of_full(fx):
    run = golden_io.exact_runs(fx)[0]
    if not run.params.rerank:
        pytest.skip("scan-order run")
    p = so.Params(**vars(run.params))
    nq = min(6, fx.queries.shape[0])
    ids, d, st = so.search_topk(fx.index, fx.queries[:nq], p, k=25)
    for qi in range(nq):
        want_ids, want_d = run.results[qi]
        n = min(25, want_ids.shape[0])
        np.testing.assert_array_equal(ids[qi, :n], want_ids[:n])
        assert np.all(ids[qi, n:] == -1)


def test_param_messages(fx):
    q = fx.queries[0]
    k = fx.index.centroids.shape[0]
    for kw, msg in [(dict(nprobe=0), "nprobe"), (dict(nprobe=k + 1), "nprobe"),
                    (dict(tau=0.0), "tau"), (dict(tau=1.5), "tau"),
                    (dict(candidates=0), "candidates"), (dict(ef_search=0), "ef_search")]:
        with pytest.raises(ValueError, match=msg):
            so.search_one(fx.index, q, so.Params(**kw))
    with pytest.raises(ValueError, match="query dim"):
        so.search_one(fx.index, q[:-1], so.Params())


@pytest.mark.parametrize("shards", [2, 3])
def test_sharded_oracle_equals_unsharded(shards):
    fx = golden_io.load("c1like_m8")
    p = so.Params(nprobe=32, tau=0.5, candidates=3000)
    want_i, want_d, want_s = so.search_topk(fx.index, fx.queries[:8], p, k=50)
    parts = [so.shard_index(fx.index, g, shards) for g in range(shards)]
    outs = [so.search_shard_topk(s, fx.queries[:8], p, k=50) for s in parts]
    for o in outs:
        np.testing.assert_array_equal(o[2], want_s)
    got_i, got_d = so.merge_topk([o[0] for o in outs], [o[1] for o in outs], 50)
    np.testing.assert_array_equal(got_i, want_i)
    np.testing.assert_array_equal(got_d, want_d)


def test_fast_probe_equals_exact_probe():
    rng = np.random.default_rng(5)
    for fxn in ("c1like_m8", "small_grouped", "rot_m8"):
        fx = golden_io.load(fxn)
        c = fx.index.centroids
        k = c.shape[0]
        for nprobe in (1, 7, 32, k // 2, k):
            nprobe = max(1, min(k, nprobe))
            for q in fx.queries[:6]:
                a = so.probe_exact(c, q, nprobe)
                b = so.probe_exact_fast(c, q, nprobe)
                np.testing.assert_array_equal(a[0], b[0])
                np.testing.assert_array_equal(a[1], b[1])
    # many near-duplicate centroids exercise the fallback
    c = rng.standard_normal((3000, 24)).astype(np.float32)
    c[1000:2000] = c[:1000] + 1e-7
    for _ in range(10):
        q = rng.standard_normal(24).astype(np.float32)
        a, b = so.probe_exact(c, q, 40), so.probe_exact_fast(c, q, 40)
        np.testing.assert_array_equal(a[0], b[0])


def _xl_sum(lut, code, x):
    """Host model of scan_common.cuh:code_sum_xl for one lane with column
    rotation x: slot s holds entry m = s ^ x, and numpy's tree is applied to
    the slots (float32, one rounding per add)."""
    m = lut.shape[0]
    v = [lut[s ^ x, code[s ^ x]] for s in range(m)]
    f = np.float32
    if m == 16:
        r = [f(v[t] + v[t + 8]) for t in range(8)]
    else:
        r = v
    return f(f(f(r[0] + r[1]) + f(r[2] + r[3])) + f(f(r[4] + r[5]) + f(r[6] + r[7])))


def test_interleaved_lut_order_is_bit_identical():
    """The bank-conflict-free scan reads sub-quantizer s ^ x at step s; the
    XOR only permutes the leaves of numpy's pairwise tree inside pairs,
    quads and octets, so every lane's sum equals lookup_code_sums bit for
    bit (pq.py:172-177)."""
    rng = np.random.default_rng(7)
    for m in (8, 16):
        lut = (rng.standard_normal((m, 256)) * rng.choice([1e-3, 1.0, 1e3], (m, 1))).astype(np.float32)
        codes = rng.integers(0, 256, (400, m)).astype(np.uint8)
        want = so.code_sums(lut, codes)
        for x in range(m):
            got = np.array([_xl_sum(lut, c, x) for c in codes], np.float32)
            np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_interleaved_lut_banks_are_distinct():
    """Entry (m, code) of copy c sits at word code * 32 + c * M + m; lane l
    reads copy l // M, column m = s ^ (l % M): 32 distinct banks per step
    for any codes."""
    rng = np.random.default_rng(3)
    for m in (8, 16):
        for s in range(m):
            codes = rng.integers(0, 256, 32)
            banks = {((int(codes[l]) * 32 + (l // m) * m + (s ^ (l % m))) % 32) for l in range(32)}
            assert len(banks) == 32
