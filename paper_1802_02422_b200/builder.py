"""GPU index builder and synthetic data for the benchmark shapes (SURVEY §8f
rank 1-2): builds the read-only `GroupedIndex` arrays the search path
consumes, following the semantics of the reference `build_index`
(/root/reference/pkg/src/givf/index.py:249-380), and exact ground truth
(datasets.py:34-61 semantics: float64 ranking, ties by id).

This is offline tooling on PyTorch (cuBLAS GEMMs); it is not on the query
path.  Deviations from the reference build, all outside the searched data
semantics:
  * k-means is seeded with a random sample instead of k-means++
    (kmeans.py:80-104): k-means++ is K sequential passes, hours at K=2^16.
  * region assignment is exact (f32 expanded form, first minimum) for every
    K; the reference switches to approximate graph assignment at K >= 2^16
    (kmeans.py:18, index.py:88-99).
Every quantity the query path reads -- alphas (grouping.py:44-74), group
picks (index.py:124-138), PQ codes of displacements (index.py:213-246),
constant bytes (index.py:160-170, grouping.py:132-145), norm terms
(index.py:173-192) and the (region, group, id) layout (index.py:326-337) --
is computed with the reference's formulas.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np
import torch

from .device_index import IndexArrays

CHUNK_ROWS = 1 << 20  # generator chunk: any row range can be regenerated


def derive_seed(seed: int, tag: str) -> int:
    """Stable sub-stream seed (same construction as util.py:102-104)."""
    h = hashlib.blake2b(f"{seed}:{tag}".encode(), digest_size=8).digest()
    return int.from_bytes(h, "little") & 0x7FFFFFFF


# ---------------------------------------------------------------- synthetic data


@dataclass(frozen=True)
class SynthSpec:
    """kind='gauss' (BASELINE.json configs 0-2): isotropic Gaussian mixture
    around unit-norm means, rows L2-normalised; noise='per_coord': sigma per
    coordinate (the literal reading), 'total': sigma/sqrt(d) per coordinate.

    kind='sift_u8' (config 3, SIFT-like uint8): cluster profiles
    mu_c = U8_SCALE * Gamma(0.5) per coordinate (nonnegative, heavy-tailed,
    many near-zero coordinates); a row is clip(round(mu_c * Gamma(4)/4),
    0, 255) -- multiplicative noise of mean 1, zeros stay zero -- stored as
    uint8 values and widened to float32 as vecio does (vecio.py:70-71)."""

    d: int
    n_clusters: int
    sigma: float = 0.3
    noise: str = "per_coord"
    seed: int = 0
    kind: str = "gauss"

    def coord_sigma(self) -> float:
        return self.sigma if self.noise == "per_coord" else self.sigma / math.sqrt(self.d)


U8_SCALE = 32.0  # sift_u8 profile scale (mean coordinate 16, tail clipped at 255)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def cluster_means(spec: SynthSpec, device="cuda") -> torch.Tensor:
    g = _gen(derive_seed(spec.seed, "means"), device)
    if spec.kind == "sift_u8":
        a = torch.full((spec.n_clusters, spec.d), 0.5, device=device, dtype=torch.float32)
        return U8_SCALE * torch._standard_gamma(a, generator=g)
    m = torch.randn(spec.n_clusters, spec.d, generator=g, device=device, dtype=torch.float32)
    return m / m.norm(dim=1, keepdim=True)


def synth_rows(spec: SynthSpec, tag: str, start: int, count: int, means=None,
               device="cuda") -> torch.Tensor:
    """Rows [start, start+count) of stream `tag` ('base', 'learn', 'query').
    Chunked counter-style seeding: row r lives in chunk r // CHUNK_ROWS whose
    generator is seeded by (seed, tag, chunk)."""
    if means is None:
        means = cluster_means(spec, device)
    out = torch.empty(count, spec.d, device=device, dtype=torch.float32)
    s = spec.coord_sigma()
    c0, c1 = start // CHUNK_ROWS, (start + count - 1) // CHUNK_ROWS if count else -1
    for c in range(c0, c1 + 1):
        g = _gen(derive_seed(spec.seed, f"{tag}:{c}"), device)
        lab = torch.randint(0, spec.n_clusters, (CHUNK_ROWS,), generator=g, device=device)
        if spec.kind == "sift_u8":
            a = torch.full((CHUNK_ROWS, spec.d), 4.0, device=device, dtype=torch.float32)
            x = (means[lab] * (torch._standard_gamma(a, generator=g) * 0.25)).round_().clamp_(0, 255)
        else:
            noise = torch.randn(CHUNK_ROWS, spec.d, generator=g, device=device, dtype=torch.float32)
            x = means[lab] + s * noise
            x = x / x.norm(dim=1, keepdim=True).clamp_min(1e-30)
        lo = max(start, c * CHUNK_ROWS)
        hi = min(start + count, (c + 1) * CHUNK_ROWS)
        out[lo - start: hi - start] = x[lo - c * CHUNK_ROWS: hi - c * CHUNK_ROWS]
    return out


# ---------------------------------------------------------------- primitives


# Fast builds (1B-row benchmark indexes) let the nearest-centroid matmuls use
# TF32 tensor cores; assignments may then differ from exact fp32 ones at
# near-ties.  The index is still a valid GroupedIndex -- the search path and
# its parity do not depend on how the index was built.
FAST_BUILD = False


class _NoTF32:
    def __enter__(self):
        self.a = torch.backends.cuda.matmul.allow_tf32
        self.b = torch.backends.cudnn.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = FAST_BUILD
        torch.backends.cudnn.allow_tf32 = FAST_BUILD

    def __exit__(self, *exc):
        torch.backends.cuda.matmul.allow_tf32 = self.a
        torch.backends.cudnn.allow_tf32 = self.b


def sq_dists(x: torch.Tensor, c: torch.Tensor, c_sq=None) -> torch.Tensor:
    """f32 expanded-form squared distances, clamped at 0 (util.py:24-33)."""
    if c_sq is None:
        c_sq = (c * c).sum(1)
    d = (x * x).sum(1, keepdim=True) + c_sq[None, :] - 2.0 * (x @ c.T)
    return d.clamp_min_(0.0)


def assign_top1(x: torch.Tensor, c: torch.Tensor, budget_elems=1 << 30):
    """Nearest centroid (first minimum) and its distance, chunked."""
    c_sq = (c * c).sum(1)
    rows = max(1, budget_elems // max(c.shape[0], 1))
    labels = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
    dists = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    with _NoTF32():
        for s in range(0, x.shape[0], rows):
            d = sq_dists(x[s:s + rows], c, c_sq)
            v, i = d.min(dim=1)
            labels[s:s + rows], dists[s:s + rows] = i, v
    return labels, dists


def kmeans(x: torch.Tensor, k: int, iters: int, seed: int) -> torch.Tensor:
    """Lloyd iterations (kmeans.py:132-142) from a random-sample seeding;
    empty clusters take the farthest point of the largest cluster
    (kmeans.py:115-126)."""
    n = x.shape[0]
    g = _gen(seed, x.device)
    cent = x[torch.randperm(n, generator=g, device=x.device)[:k]].clone()
    for _ in range(iters):
        labels, dists = assign_top1(x, cent)
        sums = torch.zeros(k, x.shape[1], dtype=torch.float64, device=x.device)
        sums.index_add_(0, labels, x.double())
        counts = torch.bincount(labels, minlength=k)
        cent = (sums / counts.clamp_min(1)[:, None]).float()
        if FAST_BUILD:  # re-seed empty clusters at random points, vectorised
            empty = torch.nonzero(counts == 0).flatten()
            if empty.numel():
                cent[empty] = x[torch.randint(0, n, (empty.numel(),), generator=g,
                                              device=x.device)]
            continue
        empty = torch.nonzero(counts == 0).flatten().tolist()
        for e in empty:
            donor = int(torch.argmax(counts))
            members = torch.nonzero(labels == donor).flatten()
            far = members[torch.argmax(dists[members])]
            cent[e] = x[far]
            labels[far] = e
            dists[far] = 0.0
            counts[donor] -= 1
            counts[e] = 1
    return cent


def neighbor_centroids(c: torch.Tensor, l: int) -> torch.Tensor:
    """l nearest other centroids per centroid, (distance, id) order
    (grouping.py:25-41), via f32 expanded distances."""
    k = c.shape[0]
    out = torch.empty(k, l, dtype=torch.int64, device=c.device)
    c_sq = (c * c).sum(1)
    rows = max(1, (1 << 28) // k)
    ar = torch.arange(k, device=c.device)
    with _NoTF32():
        for s in range(0, k, rows):
            d = sq_dists(c[s:s + rows], c, c_sq)
            d[torch.arange(d.shape[0], device=c.device), ar[s:s + rows]] = float("inf")
            v, i = torch.topk(d, l + 1, dim=1, largest=False, sorted=False)
            # (distance, id) order: stable sort by id, then stable by distance
            o = torch.argsort(i, dim=1, stable=True)
            v, i = v.gather(1, o), i.gather(1, o)
            o = torch.argsort(v, dim=1, stable=True)
            i = i.gather(1, o)
            out[s:s + rows] = i[:, :l]
    return out


def learn_alphas(x, labels, c, nbr, k) -> torch.Tensor:
    """Per-region interpolation factor (grouping.py:44-74), float64."""
    num = torch.zeros(k, dtype=torch.float64, device=x.device)
    den = torch.zeros(k, dtype=torch.float64, device=x.device)
    c64 = c.double()
    rows = max(1, (1 << 27) // (nbr.shape[1] * c.shape[1]))
    for s in range(0, x.shape[0], rows):
        lab = labels[s:s + rows]
        xc = x[s:s + rows].double() - c64[lab]
        dirs = c64[nbr[lab]] - c64[lab][:, None, :]          # (n, L, d)
        nsq = (dirs * dirs).sum(-1)                          # (n, L)
        dots = torch.einsum("nd,nld->nl", xc, dirs)
        xc_sq = (xc * xc).sum(-1, keepdim=True)
        usable = nsq > 0
        t = torch.where(usable, dots / torch.where(usable, nsq, torch.ones_like(nsq)),
                        torch.zeros_like(nsq)).clamp(0.0, 1.0)
        resid = xc_sq - 2.0 * t * dots + t * t * nsq
        resid = torch.where(usable, resid, torch.full_like(resid, float("inf")))
        pick = torch.argmin(resid, dim=1)
        ok = usable.any(dim=1)
        num.index_add_(0, lab[ok], dots.gather(1, pick[:, None])[:, 0][ok])
        den.index_add_(0, lab[ok], nsq.gather(1, pick[:, None])[:, 0][ok])
    alpha = torch.where(den > 0, num / torch.where(den > 0, den, torch.ones_like(den)),
                        torch.zeros_like(den)).clamp(0.0, 1.0)
    return alpha.float()


def anchors_of(c, nbr, alphas, region, pick=None):
    """Anchor t = c + a (s - c) in float32 (grouping.py:77-82, index.py:141-157).
    pick=None returns all L anchors (n, L, d)."""
    cr = c[region]
    a = alphas[region]
    if pick is None:
        s = c[nbr[region]]
        return cr[:, None, :] + a[:, None, None] * (s - cr[:, None, :])
    s = c[nbr[region, pick]]
    return cr + a[:, None] * (s - cr)


def pick_groups(x, region, c, nbr, alphas):
    """Nearest anchor per point, lowest group on ties, 0 when alpha == 0
    (index.py:124-138)."""
    out = torch.zeros(x.shape[0], dtype=torch.int64, device=x.device)
    rows = max(1, (1 << 27) // (nbr.shape[1] * c.shape[1]))
    with _NoTF32():
        for s in range(0, x.shape[0], rows):
            xs, rs = x[s:s + rows], region[s:s + rows]
            t = anchors_of(c, nbr, alphas, rs)                     # (n, L, d)
            d = (xs * xs).sum(1, keepdim=True) + (t * t).sum(-1) - 2.0 * torch.einsum("nd,nld->nl", xs, t)
            d.clamp_min_(0.0)
            p = torch.argmin(d, dim=1)
            p[alphas[rs] == 0.0] = 0
            out[s:s + rows] = p
    return out


def pq_train(disp: torch.Tensor, m: int, iters: int, seed: int) -> torch.Tensor:
    n, d = disp.shape
    sub = d // m
    cw = torch.empty(m, 256, sub, dtype=torch.float32, device=disp.device)
    for j in range(m):
        cw[j] = kmeans(disp[:, j * sub:(j + 1) * sub].contiguous(), 256, iters,
                       derive_seed(seed, f"pq{j}"))
    return cw


def pq_encode(disp: torch.Tensor, cw: torch.Tensor) -> torch.Tensor:
    """Nearest codeword per subspace, lowest index on ties (pq.py:56-66)."""
    m, _, sub = cw.shape
    out = torch.empty(disp.shape[0], m, dtype=torch.uint8, device=disp.device)
    with _NoTF32():
        for j in range(m):
            x = disp[:, j * sub:(j + 1) * sub]
            for s in range(0, x.shape[0], 1 << 21):
                out[s:s + (1 << 21), j] = sq_dists(x[s:s + (1 << 21)], cw[j]).argmin(1).to(torch.uint8)
    return out


def pq_decode(codes: torch.Tensor, cw: torch.Tensor) -> torch.Tensor:
    m = cw.shape[0]
    return torch.cat([cw[j][codes[:, j].long()] for j in range(m)], dim=1)


def const_terms(c, nbr, alphas, region, pick, codes, cw, grouping=True) -> torch.Tensor:
    """|t + r|^2 - (1-a)|c|^2 - a|s|^2 in float64 (index.py:141-170)."""
    c64 = c.double()
    if grouping:
        t = anchors_of(c, nbr, alphas, region, pick)
        s64 = c64[nbr[region, pick]]
        s_sq = (s64 * s64).sum(1)
        a = alphas[region].double()
    else:
        t = c[region]
        s_sq = torch.zeros(region.shape[0], dtype=torch.float64, device=c.device)
        a = torch.zeros(region.shape[0], dtype=torch.float64, device=c.device)
    tpr = (t + pq_decode(codes, cw)).double()
    cr = c64[region]
    return (tpr * tpr).sum(1) - (1.0 - a) * (cr * cr).sum(1) - a * s_sq


def norm_terms(c, nbr, alphas) -> torch.Tensor:
    """Per-group constants that turn scores into anchor distances
    (index.py:173-192), float64 then float32."""
    c64 = c.double()
    c_sq = (c64 * c64).sum(1)
    a = alphas.double()[:, None, None]
    cc = c64[:, None, :]
    ss = c64[nbr]
    t = cc + a * (ss - cc)
    t_sq = (t * t).sum(-1)
    return (t_sq - (1.0 - a[:, :, 0]) * c_sq[:, None] - a[:, :, 0] * c_sq[nbr]).float()


# ---------------------------------------------------------------- ground truth


class TopT:
    """Running exact top-t (float64 distance, id) per query over base chunks."""

    def __init__(self, queries: torch.Tensor, t: int = 10, pre: int = 16):
        self.q = queries
        self.q64 = queries.double()
        self.t, self.pre = t, max(pre, t)
        nq = queries.shape[0]
        self.d = torch.full((nq, self.t), float("inf"), dtype=torch.float64, device=queries.device)
        self.i = torch.full((nq, self.t), -1, dtype=torch.int64, device=queries.device)

    def update(self, x: torch.Tensor, first_id: int):
        with _NoTF32():
            for s in range(0, x.shape[0], 1 << 16):
                xs = x[s:s + (1 << 16)]
                d = sq_dists(self.q, xs)
                v, j = torch.topk(d, min(self.pre, xs.shape[0]), dim=1, largest=False)
                cand = xs[j]                                     # (nq, pre, d)
                d64 = ((cand.double() - self.q64[:, None, :]) ** 2).sum(-1)
                ids = j + (first_id + s)
                alld = torch.cat([self.d, d64], 1)
                alli = torch.cat([self.i, ids], 1)
                # (d64, id) lexicographic: sort by id then stable by distance
                o = torch.argsort(alli, dim=1, stable=True)
                alld, alli = alld.gather(1, o), alli.gather(1, o)
                o = torch.argsort(alld, dim=1, stable=True)[:, : self.t]
                self.d, self.i = alld.gather(1, o), alli.gather(1, o)

    def result(self) -> np.ndarray:
        return self.i.to(torch.int32).cpu().numpy()


# ---------------------------------------------------------------- build


@dataclass
class BuildSpec:
    n: int
    k: int
    l: int = 64
    m: int = 16
    grouping: bool = True
    n_learn: int = 0            # default max(100k, 32 K)
    kmeans_iters: int = 10
    pq_iters: int = 15
    seed: int = 0
    fast: bool = False          # TF32 assignment matmuls (1B-scale builds)

    def learn_rows(self) -> int:
        return self.n_learn or max(100_000, 32 * self.k)


def build_synthetic(data: SynthSpec, spec: BuildSpec, n_queries: int, gt_t: int = 10,
                    device="cuda", log=print):
    """Generate, train, encode and lay out a grouped index on the GPU.

    Returns (IndexArrays on host, queries (nq, d) f32 numpy, gt (nq, gt_t) i32).
    """
    import time

    global FAST_BUILD
    FAST_BUILD = spec.fast
    t0 = time.perf_counter()
    means = cluster_means(data, device)
    learn = synth_rows(data, "learn", 0, spec.learn_rows(), means, device)
    queries = synth_rows(data, "query", 0, n_queries, means, device)
    k, l = spec.k, spec.l
    cent = kmeans(learn, k, spec.kmeans_iters, derive_seed(spec.seed, "kmeans"))
    log(f"[build] kmeans K={k} on {learn.shape[0]} learn rows: {time.perf_counter()-t0:.1f}s")

    lr, _ = assign_top1(learn, cent)
    if spec.grouping:
        nbr = neighbor_centroids(cent, l)
        alphas = learn_alphas(learn, lr, cent, nbr, k)
        lp = pick_groups(learn, lr, cent, nbr, alphas)
        t_learn = anchors_of(cent, nbr, alphas, lr, lp)
    else:
        nbr = torch.zeros(k, 1, dtype=torch.int64, device=device)
        alphas = torch.zeros(k, dtype=torch.float32, device=device)
        lp = torch.zeros_like(lr)
        t_learn = cent[lr]
    cw = pq_train(learn - t_learn, spec.m, spec.pq_iters, derive_seed(spec.seed, "pq"))
    lcodes = pq_encode(learn - t_learn, cw)
    lconst = const_terms(cent, nbr, alphas, lr, lp, lcodes, cw, spec.grouping)
    # grouping.py:132-145: percentile bounds rounded through float32
    qlo, qhi = (float(np.float32(v)) for v in np.percentile(lconst.cpu().numpy(), [0.1, 99.9]))
    lo_, hi_ = min(qlo, qhi), max(qlo, qhi)
    step = (hi_ - lo_) / 256.0
    log(f"[build] grouping + PQ(M={spec.m}) trained: {time.perf_counter()-t0:.1f}s")
    del learn, t_learn, lcodes, lconst

    n = spec.n
    region = torch.empty(n, dtype=torch.int32, device=device)
    pick = torch.empty(n, dtype=torch.int16, device=device)
    codes = torch.empty(n, spec.m, dtype=torch.uint8, device=device)
    cbytes = torch.empty(n, dtype=torch.uint8, device=device)
    gt = TopT(queries, gt_t)
    for s in range(0, n, CHUNK_ROWS):
        e = min(n, s + CHUNK_ROWS)
        x = synth_rows(data, "base", s, e - s, means, device)
        r, _ = assign_top1(x, cent)
        p = pick_groups(x, r, cent, nbr, alphas) if spec.grouping else torch.zeros_like(r)
        t = anchors_of(cent, nbr, alphas, r, p) if spec.grouping else cent[r]
        cd = pq_encode(x - t, cw)
        ct = const_terms(cent, nbr, alphas, r, p, cd, cw, spec.grouping)
        if step > 0:
            b = torch.floor((ct - lo_) / step).clamp(0, 255).to(torch.uint8)
        else:
            b = torch.zeros_like(ct, dtype=torch.uint8)
        region[s:e], pick[s:e], codes[s:e], cbytes[s:e] = r.int(), p.short(), cd, b
        gt.update(x, s)
        del x, t
        if n >= 100 * CHUNK_ROWS and (s // CHUNK_ROWS) % 100 == 99:
            log(f"[build]   {e} rows encoded: {time.perf_counter()-t0:.1f}s")
    log(f"[build] {n} base rows assigned/encoded + ground truth: {time.perf_counter()-t0:.1f}s")

    groups = l if spec.grouping else 1
    key = region.long() * groups + pick.long()
    order = torch.sort(key, stable=True).indices                # ties keep id order
    gsize = torch.bincount(key, minlength=k * groups).reshape(k, groups).int()
    offs = torch.zeros(k + 1, dtype=torch.int64, device=device)
    offs[1:] = torch.cumsum(gsize.sum(1).long(), 0)
    arr = IndexArrays(
        centroids=cent.cpu().numpy(),
        alphas=alphas.cpu().numpy(),
        neighbor_ids=nbr.int().cpu().numpy() if spec.grouping else None,
        norm_terms=norm_terms(cent, nbr, alphas).cpu().numpy() if spec.grouping else None,
        group_sizes=gsize.cpu().numpy(),
        region_offsets=offs.cpu().numpy(),
        point_ids=order.int().cpu().numpy(),
        codes=codes[order].cpu().numpy(),
        const_bytes=cbytes[order].cpu().numpy(),
        codewords=cw.cpu().numpy(),
        rotation=None,
        const_lo=lo_,
        const_hi=hi_,
        grouping=spec.grouping,
    )
    log(f"[build] layout done: {time.perf_counter()-t0:.1f}s")
    return arr, queries.cpu().numpy(), gt.result()
