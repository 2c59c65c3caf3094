"""GPU index builder and synthetic data for the benchmark shapes (SURVEY §8f
rank 1-2): builds the read-only `GroupedIndex` arrays the search path
consumes, following the semantics of the reference `build_index`
(/root/reference/pkg/src/givf/index.py:249-380), and exact ground truth
(datasets.py:34-61 semantics: float64 ranking, ties by id).

The row-sized work runs in the library's own sm_100a kernels
(include/givf_build.h):
  * nearest centroid (k-means steps and region assignment) -- KA, a tcgen05
    GEMM with an arg-min epilogue (`givf_assign_nearest`);
  * group pick, residual PQ codes, constant term and byte of every row -- KE
    (`givf_encode_rows`), one pass over rows grouped by region;
  * exact k-NN (ground truth, the centroids' neighbour lists) -- the search
    path's certified probe (`givf_knn_exact`).
PyTorch holds the buffers and runs the small training reductions (centroid
means, alpha fits, percentiles); nothing row-sized goes through the host.

Deviations from the reference build, all outside the searched data
semantics (the search path's parity does not depend on how an index was
built):
  * k-means is seeded with a random sample instead of k-means++
    (kmeans.py:80-104); empty clusters are re-seeded at random rows.
  * region assignment uses bf16 products with fp32 accumulation (the
    reference itself assigns through its approximate graph at K >= 2^16,
    index.py:88-99); near-ties may resolve differently from float32.
  * neighbour lists are ordered by (float32(d64), id) (the probe's order)
    instead of float32 expanded distances.
Every quantity the query path reads -- alphas (grouping.py:44-74), group
picks (index.py:124-138), PQ codes of displacements (index.py:213-246),
constant bytes (index.py:160-170, grouping.py:132-145), norm terms
(index.py:173-192) and the (region, group, id) layout (index.py:326-337) --
follows the reference's formulas.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device_index import IndexArrays

CHUNK_ROWS = 1 << 20  # generator chunk: any row range can be regenerated
ENCODE_ROWS = 1 << 24  # rows assigned / encoded per pass


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
               device="cuda", out=None) -> torch.Tensor:
    """Rows [start, start+count) of stream `tag` ('base', 'learn', 'query').
    Chunked counter-style seeding: row r lives in chunk r // CHUNK_ROWS whose
    generator is seeded by (seed, tag, chunk)."""
    if means is None:
        means = cluster_means(spec, device)
    if out is None:
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


# ---------------------------------------------------------------- native steps


def _vp(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def assign_nearest(x: torch.Tensor, cent: torch.Tensor, want_dist: bool = False):
    """KA: nearest centroid per row (first on ties) and, optionally, its
    squared distance (bf16-product score + |x|^2)."""
    x = x.contiguous()
    cent = cent.contiguous()
    lab = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
    dist = torch.empty(x.shape[0], dtype=torch.float32, device=x.device) if want_dist else None
    _native.check(_native.load().givf_assign_nearest(
        _vp(x), x.shape[0], _vp(cent), cent.shape[0], cent.shape[1], _vp(lab), _vp(dist),
        _stream()))
    return lab, dist


def knn_exact(q: torch.Tensor, base: torch.Tensor, k: int):
    """Exact top-k rows of `base` per query: ids (int32) and float64
    squared distances, the set by (d64, id), rows in (f32(d64), id) order."""
    q = q.contiguous()
    base = base.contiguous()
    ids = torch.empty(q.shape[0], k, dtype=torch.int32, device=q.device)
    dd = torch.empty(q.shape[0], k, dtype=torch.float64, device=q.device)
    _native.check(_native.load().givf_knn_exact(
        _vp(q), q.shape[0], _vp(base), base.shape[0], base.shape[1], k, _vp(ids), _vp(dd),
        _stream()))
    return ids, dd


def lexsort_rows(d: torch.Tensor, i: torch.Tensor):
    """Per row, (d, i) ascending: stable sort by id, then stable by distance."""
    o = torch.argsort(i, dim=1, stable=True)
    d, i = d.gather(1, o), i.gather(1, o)
    o = torch.argsort(d, dim=1, stable=True)
    return d.gather(1, o), i.gather(1, o)


class Model:
    """Trained coarse/grouping/PQ state (everything but the rows)."""

    def __init__(self, cent, nbr, alphas, cw, lo, hi, grouping, l):
        self.cent = cent.contiguous()
        self.k, self.d = cent.shape
        self.nbr = nbr.int().contiguous() if grouping else None
        self.alphas = alphas.float().contiguous()
        self.cw = cw.contiguous()
        self.m = cw.shape[0]
        self.lo, self.hi = lo, hi
        self.step = (hi - lo) / 256.0
        self.grouping = grouping
        self.l = l if grouping else 1
        self.csq = (cent.double() ** 2).sum(1).contiguous()
        self.cwsq = (cw * cw).sum(-1).contiguous()  # (M, 256) f32 (pq row norms)


def encode_rows(x: torch.Tensor, region: torch.Tensor, md: Model, want_consts=False,
                want_bytes=True):
    """KE over rows grouped by region: (pick int16, codes (n, M) u8,
    const bytes u8 or None, consts f64 or None), indexed like x."""
    n = x.shape[0]
    dev = x.device
    reg_s, order = torch.sort(region, stable=True)
    vals, counts = torch.unique_consecutive(reg_s, return_counts=True)
    seg = torch.zeros(vals.shape[0] + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=seg[1:])
    order = order.int().contiguous()
    vals = vals.int().contiguous()
    pick = torch.empty(n, dtype=torch.int16, device=dev)
    codes = torch.empty(n, md.m, dtype=torch.uint8, device=dev)
    cb = torch.empty(n, dtype=torch.uint8, device=dev) if want_bytes else None
    consts = torch.empty(n, dtype=torch.float64, device=dev) if want_consts else None
    desc = _native.EncodeDesc(
        x=_vp(x.contiguous()), order=_vp(order), seg=_vp(seg), seg_region=_vp(vals),
        nseg=vals.shape[0], dim=md.d, l=md.l, m=md.m, grouping=1 if md.grouping else 0,
        centroids=_vp(md.cent), neighbor_ids=_vp(md.nbr), alphas=_vp(md.alphas), c_sq=_vp(md.csq),
        codewords=_vp(md.cw), cw_sq=_vp(md.cwsq), const_lo=md.lo, const_step=md.step,
        pick=_vp(pick), codes=_vp(codes), const_bytes=_vp(cb), consts=_vp(consts))
    _native.check(_native.load().givf_encode_rows(ctypes.byref(desc), _stream()))
    return pick, codes, cb, consts


# ---------------------------------------------------------------- training


def kmeans(x: torch.Tensor, k: int, iters: int, seed: int) -> torch.Tensor:
    """Lloyd iterations (kmeans.py:132-142) from a random-sample seeding;
    empty clusters are re-seeded at random rows."""
    n = x.shape[0]
    g = _gen(seed, x.device)
    cent = x[torch.randperm(n, generator=g, device=x.device)[:k]].clone()
    for _ in range(iters):
        lab, _ = assign_nearest(x, cent)
        lab = lab.long()
        sums = torch.zeros(k, x.shape[1], dtype=torch.float64, device=x.device)
        sums.index_add_(0, lab, x.double())
        counts = torch.bincount(lab, minlength=k)
        cent = (sums / counts.clamp_min(1)[:, None]).float()
        empty = torch.nonzero(counts == 0).flatten()
        if empty.numel():
            cent[empty] = x[torch.randint(0, n, (empty.numel(),), generator=g, device=x.device)]
    return cent.contiguous()


def neighbor_centroids(c: torch.Tensor, l: int) -> torch.Tensor:
    """l nearest other centroids per centroid (grouping.py:25-41): the exact
    top-(l+1) of every centroid, itself removed."""
    k = c.shape[0]
    ids, _ = knn_exact(c, c, l + 1)
    ar = torch.arange(k, device=c.device, dtype=torch.int32)[:, None]
    is_self = ids == ar
    # position of the row's own id (l + 1 when absent: drop the last)
    pos = torch.where(is_self.any(1), is_self.int().argmax(1), torch.full_like(ar[:, 0], l))
    j = torch.arange(l, device=c.device)[None, :]
    j = j + (j >= pos[:, None]).long()
    return ids.gather(1, j)


def learn_alphas(x, labels, c, nbr, k) -> torch.Tensor:
    """Per-region interpolation factor (grouping.py:44-74), float64."""
    num = torch.zeros(k, dtype=torch.float64, device=x.device)
    den = torch.zeros(k, dtype=torch.float64, device=x.device)
    c64 = c.double()
    nbr = nbr.long()
    labels = labels.long()
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


def anchors_of(c, nbr, alphas, region, pick):
    """Anchor t = c + a (s - c) in float32 (grouping.py:77-82, index.py:141-157)."""
    region = region.long()
    cr = c[region]
    if nbr is None:
        return cr
    a = alphas[region]
    s = c[nbr.long()[region, pick.long()]]
    return cr + a[:, None] * (s - cr)


def pq_train(disp: torch.Tensor, m: int, iters: int, seed: int) -> torch.Tensor:
    n, d = disp.shape
    sub = d // m
    cw = torch.empty(m, 256, sub, dtype=torch.float32, device=disp.device)
    for j in range(m):
        cw[j] = kmeans(disp[:, j * sub:(j + 1) * sub].contiguous(), 256, iters,
                       derive_seed(seed, f"pq{j}"))
    return cw


def norm_terms(c, nbr, alphas) -> torch.Tensor:
    """Per-group constants that turn scores into anchor distances
    (index.py:173-192), float64 then float32."""
    c64 = c.double()
    c_sq = (c64 * c64).sum(1)
    out = torch.empty(nbr.shape, dtype=torch.float32, device=c.device)
    nbr = nbr.long()
    for s in range(0, c.shape[0], 1 << 14):
        e = min(c.shape[0], s + (1 << 14))
        a = alphas[s:e].double()[:, None, None]
        cc = c64[s:e, None, :]
        ss = c64[nbr[s:e]]
        t = cc + a * (ss - cc)
        t_sq = (t * t).sum(-1)
        out[s:e] = (t_sq - (1.0 - a[:, :, 0]) * c_sq[s:e, None] - a[:, :, 0] * c_sq[nbr[s:e]]).float()
    return out


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
    fast: bool = False          # kept for cache keys of older workloads (unused)
    alpha_rows: int = 4_000_000   # learn rows the alpha fit reads
    pq_rows: int = 1_000_000      # learn rows the PQ k-means reads

    def learn_rows(self) -> int:
        return self.n_learn or max(100_000, 32 * self.k)


def train_model(data: SynthSpec, spec: BuildSpec, means, device, log=print) -> Model:
    """Coarse k-means, neighbour lists, alphas, PQ codebooks and the constant
    quantizer on the held-out learn stream (index.py:214-312)."""
    t0 = time.perf_counter()
    learn = synth_rows(data, "learn", 0, spec.learn_rows(), means, device)
    k, l = spec.k, spec.l
    cent = kmeans(learn, k, spec.kmeans_iters, derive_seed(spec.seed, "kmeans"))
    log(f"[build] kmeans K={k} on {learn.shape[0]} learn rows: {time.perf_counter()-t0:.1f}s")
    lr, _ = assign_nearest(learn, cent)
    if spec.grouping:
        nbr = neighbor_centroids(cent, l)
        na = min(learn.shape[0], spec.alpha_rows)
        alphas = learn_alphas(learn[:na], lr[:na], cent, nbr, k)
    else:
        nbr = None
        alphas = torch.zeros(k, dtype=torch.float32, device=device)
    log(f"[build] neighbours + alphas: {time.perf_counter()-t0:.1f}s")
    # group picks of the learn rows (KE with a placeholder codebook), then
    # the PQ codebooks on their displacements (index.py:213-246)
    d = cent.shape[1]
    tmp = Model(cent, nbr if nbr is not None else torch.zeros(k, 1, dtype=torch.int32, device=device),
                alphas, torch.zeros(spec.m, 256, d // spec.m, device=device), 0.0, 0.0,
                spec.grouping, l)
    lp, _, _, _ = encode_rows(learn, lr, tmp, want_bytes=False)
    np_ = min(learn.shape[0], spec.pq_rows)
    disp = learn[:np_] - anchors_of(cent, nbr, alphas, lr[:np_], lp[:np_])
    cw = pq_train(disp, spec.m, spec.pq_iters, derive_seed(spec.seed, "pq"))
    del disp
    # constant quantizer from the learn rows' own constants (grouping.py:132-145):
    # percentile bounds rounded through float32
    md = Model(cent, tmp.nbr, alphas, cw, 0.0, 0.0, spec.grouping, l)
    _, _, _, lconst = encode_rows(learn, lr, md, want_consts=True, want_bytes=False)
    qlo, qhi = (float(np.float32(v)) for v in np.percentile(lconst.cpu().numpy(), [0.1, 99.9]))
    lo_, hi_ = min(qlo, qhi), max(qlo, qhi)
    log(f"[build] grouping + PQ(M={spec.m}) trained: {time.perf_counter()-t0:.1f}s")
    del learn, lconst
    return Model(cent, tmp.nbr, alphas, cw, lo_, hi_, spec.grouping, l)


class GroundTruth:
    """Running exact top-t (float64 distance, id) per query over base row
    blocks (datasets.py:34-61), through the certified probe."""

    BLOCK = 1 << 20

    def __init__(self, queries: torch.Tensor, t: int = 10):
        self.q = queries.contiguous()
        self.t = t
        nq = queries.shape[0]
        self.d = torch.full((nq, t), float("inf"), dtype=torch.float64, device=queries.device)
        self.i = torch.full((nq, t), -1, dtype=torch.int64, device=queries.device)

    def update(self, x: torch.Tensor, first_id: int):
        for s in range(0, x.shape[0], self.BLOCK):
            xs = x[s:s + self.BLOCK]
            kk = min(self.t, xs.shape[0])
            ids, dd = knn_exact(self.q, xs, kk)
            d = torch.cat([self.d, dd], 1)
            i = torch.cat([self.i, ids.long() + (first_id + s)], 1)
            d, i = lexsort_rows(d, i)
            self.d, self.i = d[:, : self.t].contiguous(), i[:, : self.t].contiguous()

    def result(self) -> np.ndarray:
        return self.i.to(torch.int32).cpu().numpy()


def build_synthetic(data: SynthSpec, spec: BuildSpec, n_queries: int, gt_t: int = 10,
                    device="cuda", log=print, rows_on_device: bool = False):
    """Generate, train, encode and lay out a grouped index on the GPU.

    Returns (IndexArrays, queries (nq, d) f32 numpy, gt (nq, gt_t) i32).
    With rows_on_device the row arrays (point_ids, codes, const_bytes) stay
    torch CUDA tensors (1B-row indexes never visit the host); otherwise every
    array is numpy.
    """
    t0 = time.perf_counter()
    means = cluster_means(data, device)
    queries = synth_rows(data, "query", 0, n_queries, means, device)
    md = train_model(data, spec, means, device, log)
    k, l = spec.k, spec.l
    groups = l if spec.grouping else 1

    n = spec.n
    key = torch.empty(n, dtype=torch.int32, device=device)
    codes = torch.empty(n, spec.m, dtype=torch.uint8, device=device)
    cbytes = torch.empty(n, dtype=torch.uint8, device=device)
    gt = GroundTruth(queries, gt_t)
    x = None
    for s in range(0, n, ENCODE_ROWS):
        e = min(n, s + ENCODE_ROWS)
        x = synth_rows(data, "base", s, e - s, means, device,
                       out=x[: e - s] if x is not None and x.shape[0] >= e - s else None)
        r, _ = assign_nearest(x, md.cent)
        p, cd, cb, _ = encode_rows(x, r, md)
        key[s:e] = r * groups + p.int()
        codes[s:e] = cd
        cbytes[s:e] = cb
        gt.update(x, s)
        if n >= 8 * ENCODE_ROWS and (s // ENCODE_ROWS) % 8 == 7:
            torch.cuda.synchronize()
            log(f"[build]   {e} rows encoded: {time.perf_counter()-t0:.1f}s")
    del x
    torch.cuda.synchronize()
    log(f"[build] {n} base rows assigned/encoded + ground truth: {time.perf_counter()-t0:.1f}s")

    # (region, group, id) layout (index.py:326-337): a stable sort by key
    order = torch.sort(key, stable=True).indices
    gsize = torch.bincount(key.long(), minlength=k * groups).reshape(k, groups).int()
    del key
    offs = torch.zeros(k + 1, dtype=torch.int64, device=device)
    offs[1:] = torch.cumsum(gsize.sum(1).long(), 0)
    pids = order.int()
    codes_s = codes[order]
    del codes
    cb_s = cbytes[order]
    del cbytes, order
    torch.cuda.synchronize()
    log(f"[build] layout done: {time.perf_counter()-t0:.1f}s")

    def rowarr(t):
        return t if rows_on_device else t.cpu().numpy()

    arr = IndexArrays(
        centroids=md.cent.cpu().numpy(),
        alphas=md.alphas.cpu().numpy(),
        neighbor_ids=md.nbr.cpu().numpy() if spec.grouping else None,
        norm_terms=norm_terms(md.cent, md.nbr, md.alphas).cpu().numpy() if spec.grouping else None,
        group_sizes=gsize.cpu().numpy(),
        region_offsets=offs.cpu().numpy(),
        point_ids=rowarr(pids),
        codes=rowarr(codes_s),
        const_bytes=rowarr(cb_s),
        codewords=md.cw.cpu().numpy(),
        rotation=None,
        const_lo=md.lo,
        const_hi=md.hi,
        grouping=spec.grouping,
    )
    return arr, queries.cpu().numpy(), gt.result()
