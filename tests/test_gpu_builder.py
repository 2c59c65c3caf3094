"""Builder kernels (include/givf_build.h) against numpy restatements of the
reference build formulas: KA nearest centroid (kmeans.py:164-187 /
index.py:88-99), KE group pick + PQ encode + constant (index.py:124-170,
pq.py:56-66, grouping.py:77-82, 103-113) and the exact k-NN
(datasets.py:34-61, grouping.py:25-41)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _sq(x, c):
    """util.py:24-33: expanded f32 form clamped at 0."""
    x = x.astype(np.float32)
    c = c.astype(np.float32)
    d = (x * x).sum(1, dtype=np.float32)[:, None] + (c * c).sum(1, dtype=np.float32)[None, :] - \
        np.float32(2.0) * (x @ c.T)
    return np.maximum(d, 0.0)


@pytest.mark.parametrize("n,k,d", [(20_000, 3000, 96), (700, 50_000, 96), (5000, 1000, 128),
                                   (3000, 257, 32), (4000, 300, 6)])
def test_assign_nearest_matches_exact_within_bf16(n, k, d):
    torch = _torch()
    from paper_1802_02422_b200.builder import assign_nearest

    g = torch.Generator(device="cuda").manual_seed(n + k)
    x = torch.randn(n, d, device="cuda", generator=g)
    c = torch.randn(k, d, device="cuda", generator=g)
    lab, dist = assign_nearest(x, c, want_dist=True)
    x64, c64 = x.double(), c.double()
    dd = (x64 * x64).sum(1)[:, None] + (c64 * c64).sum(1)[None, :] - 2 * x64 @ c64.T
    best = dd.min(1).values
    got = dd.gather(1, lab.long()[:, None])[:, 0]
    # bf16 products: |error| <= ~2 * 2^-8 |x| |c| per score (both operands rounded)
    tol = 2.0 * 2.0 ** -8 * x64.norm(dim=1) * c64.norm(dim=1).max() + 1e-6
    assert bool(((got - best) <= 2 * tol).all())
    agree = float((lab.long() == dd.argmin(1)).float().mean())
    assert agree > 0.9, agree
    assert bool((dist.double() - got).abs().le(2 * tol + 1e-3 * got.abs()).all())


def test_assign_nearest_picks_first_of_equal_scores():
    torch = _torch()
    from paper_1802_02422_b200.builder import assign_nearest

    c = torch.zeros(300, 32, device="cuda")
    c[:, 0] = 1.0  # every centroid identical: the first index wins
    x = torch.randn(1000, 32, device="cuda")
    lab, _ = assign_nearest(x, c)
    assert bool((lab == 0).all())
    c2 = torch.randn(300, 32, device="cuda")
    c2[200] = 0.0
    x2 = c2[[5, 17, 299]].clone()
    lab2, _ = assign_nearest(x2, c2)
    np.testing.assert_array_equal(lab2.cpu().numpy(), [5, 17, 299])


@pytest.mark.parametrize("nq,nb,d,k", [(300, 50_000, 96, 10), (64, 4096, 128, 65), (50, 700, 32, 1)])
def test_knn_exact_is_the_float64_ranking(nq, nb, d, k):
    torch = _torch()
    from paper_1802_02422_b200.builder import knn_exact, lexsort_rows

    rng = np.random.default_rng(nq)
    q = rng.standard_normal((nq, d)).astype(np.float32)
    b = rng.standard_normal((nb, d)).astype(np.float32)
    b[7] = b[3]  # a duplicate row: tie broken by id
    q[0] = b[3]
    ids, dd = knn_exact(torch.from_numpy(q).cuda(), torch.from_numpy(b).cuda(), k)
    ids, dd = ids.cpu().numpy(), dd.cpu().numpy()
    d64 = ((q.astype(np.float64)[:, None, :] - b.astype(np.float64)[None, :, :]) ** 2).sum(-1)
    for i in range(nq):
        want = np.lexsort((np.arange(nb), d64[i]))[:k]
        assert sorted(ids[i]) == sorted(want), i
        np.testing.assert_allclose(dd[i], d64[i, ids[i]], rtol=1e-12, atol=1e-12)
    assert ids[0, 0] == 3 and (k == 1 or ids[0, 1] == 7)
    # (d64, id) order after lexsort_rows
    sd, si = lexsort_rows(torch.from_numpy(dd), torch.from_numpy(ids.astype(np.int64)))
    for i in range(nq):
        np.testing.assert_array_equal(si[i].numpy(), np.lexsort((np.arange(nb), d64[i]))[:k])


def test_neighbor_centroids_exact():
    torch = _torch()
    from paper_1802_02422_b200.builder import neighbor_centroids

    rng = np.random.default_rng(3)
    c = rng.standard_normal((2000, 96)).astype(np.float32)
    c[10] = c[4]  # duplicate: each still excludes itself
    nb = neighbor_centroids(torch.from_numpy(c).cuda(), 16).cpu().numpy()
    d64 = ((c.astype(np.float64)[:, None, :] - c.astype(np.float64)[None, :, :]) ** 2).sum(-1)
    for j in range(c.shape[0]):
        order = np.lexsort((np.arange(c.shape[0]), d64[j]))
        want = order[order != j][:16]
        assert sorted(nb[j]) == sorted(want), j
        assert j not in nb[j]
    assert nb[4][0] == 10 and nb[10][0] == 4


def _encode_reference(x, region, cent, nbr, alphas, cw, lo, hi, grouping):
    """numpy restatement of index.py:124-170 + pq.py:56-66 + grouping.py:103-113."""
    n, d = x.shape
    m = cw.shape[0]
    sub = d // m
    pick = np.zeros(n, np.int64)
    t = np.empty_like(x)
    for r in np.unique(region):
        rows = np.flatnonzero(region == r)
        if grouping:
            a = np.float32(alphas[r])
            anchors = (cent[r][None, :] + a * (cent[nbr[r]] - cent[r][None, :])).astype(np.float32)
            if alphas[r] != 0.0:
                pick[rows] = np.argmin(_sq(x[rows], anchors), axis=1)
            t[rows] = anchors[pick[rows]]
        else:
            t[rows] = cent[r]
    disp = x - t
    codes = np.empty((n, m), np.int64)
    for j in range(m):
        codes[:, j] = np.argmin(_sq(disp[:, j * sub:(j + 1) * sub], cw[j]), axis=1)
    recon = np.concatenate([cw[j][codes[:, j]] for j in range(m)], axis=1)
    tpr = (t + recon).astype(np.float64)
    c64 = cent[region].astype(np.float64)
    if grouping:
        s64 = cent[nbr[region, pick]].astype(np.float64)
        a = alphas[region].astype(np.float64)
        const = (tpr * tpr).sum(1) - (1 - a) * (c64 * c64).sum(1) - a * (s64 * s64).sum(1)
    else:
        const = (tpr * tpr).sum(1) - (c64 * c64).sum(1)
    step = (hi - lo) / 256.0
    b = np.clip(np.floor((const - lo) / step), 0, 255).astype(np.uint8)
    return pick, codes, b, const


@pytest.mark.parametrize("d,m,grouping", [(96, 16, True), (96, 8, True), (128, 16, True),
                                          (96, 16, False), (32, 8, True)])
def test_encode_rows_matches_reference_formulas(d, m, grouping):
    torch = _torch()
    from paper_1802_02422_b200.builder import Model, encode_rows

    rng = np.random.default_rng(d + m)
    k, l, n = 300, 24, 20_000
    cent = rng.standard_normal((k, d)).astype(np.float32)
    nbr = np.stack([rng.choice(np.delete(np.arange(k), r), l, replace=False) for r in range(k)]).astype(np.int32)
    alphas = rng.uniform(0, 1, k).astype(np.float32)
    alphas[:5] = 0.0  # alpha 0: group 0
    region = rng.integers(0, k, n).astype(np.int32)
    x = (cent[region] + 0.3 * rng.standard_normal((n, d))).astype(np.float32)
    cw = (0.3 * rng.standard_normal((m, 256, d // m))).astype(np.float32)
    lo, hi = -2.0, 3.0
    dv = lambda a: torch.from_numpy(a).cuda()
    md = Model(dv(cent), dv(nbr), dv(alphas), dv(cw), lo, hi, grouping, l)
    p, cd, cb, cs = encode_rows(dv(x), dv(region), md, want_consts=True)
    p, cd, cb, cs = p.cpu().numpy(), cd.cpu().numpy(), cb.cpu().numpy(), cs.cpu().numpy()
    wp, wc, wb, wcs = _encode_reference(x, region, cent, nbr, alphas, cw, lo, hi, grouping)
    # float32 dot products may be summed in another order than BLAS: only
    # near-ties can resolve differently
    assert np.mean(p == wp) > 0.999
    same = (p == wp)
    assert np.mean(np.all(cd[same] == wc[same], axis=1)) > 0.995
    ok = same & np.all(cd == wc, axis=1)
    np.testing.assert_allclose(cs[ok], wcs[ok], rtol=1e-6, atol=1e-6)
    assert np.mean(cb[ok] == wb[ok]) > 0.999
    assert (p[np.isin(region, np.arange(5))] == 0).all() or not grouping
