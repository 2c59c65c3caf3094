"""Drop-in query API: the surface of `givf.search` on the B200 path.

Same names, argument meaning, defaults and error behaviour as
/root/reference/pkg/src/givf/search.py:
  SearchParams (23-30), SearchStats (33-39), SearchResult (42-63),
  search (93-163), decomposed_distance (166-183), recall_at_r (186-201),
  SweepRow / sweep (204-249), write_sweep_csv (252-262),
  verify_results (265-278).
Added: `search_batch(index, queries, params, k=None)`.

Every query runs through the sm_100a kernels behind the C ABI
(include/givf_b200.h).  The region probe is exact (the reference's
ef_search == K ranking); `ef_search` is validated and otherwise unused.
"""

from __future__ import annotations

import ctypes
import struct
import time
from dataclasses import dataclass
from hashlib import blake2b

import numpy as np

from . import _native
from .device_index import DeviceIndex, device_index


@dataclass(frozen=True)
class SearchParams:
    nprobe: int = 32
    tau: float = 1.0
    candidates: int = 10_000
    ef_search: int = 128
    rerank: bool = True
    prune: bool = True


@dataclass
class SearchStats:
    regions_visited: int = 0
    subregions_visited: int = 0
    subregions_pruned: int = 0
    codes_scanned: int = 0
    wall_time_s: float = 0.0


@dataclass
class SearchResult:
    ids: np.ndarray  # (r,) int32
    distances: np.ndarray  # (r,) float32
    stats: SearchStats

    def signature(self) -> str:
        """Content hash of everything except wall time (search.py:48-63)."""
        h = blake2b(digest_size=16)
        h.update(np.ascontiguousarray(self.ids, dtype="<i4").tobytes())
        h.update(np.ascontiguousarray(self.distances, dtype="<f4").tobytes())
        s = self.stats
        h.update(struct.pack("<4q", s.regions_visited, s.subregions_visited,
                             s.subregions_pruned, s.codes_scanned))
        return h.hexdigest()


def _cparams(p: SearchParams) -> _native.SearchParamsC:
    cand = int(p.candidates)
    cand = min(cand, (1 << 62)) if cand > 0 else cand
    return _native.SearchParamsC(
        nprobe=int(p.nprobe), tau=float(p.tau), candidates=cand,
        ef_search=int(p.ef_search), rerank=1 if p.rerank else 0, prune=1 if p.prune else 0,
    )


def _check_query_dim(dev: DeviceIndex, q: np.ndarray) -> None:
    if q.shape[-1] != dev.dim:
        raise ValueError(f"query dim {q.shape[-1]} != index dim {dev.dim}")


def _vp(a) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def search_batch(index, queries, params: SearchParams, k: int | None = None, device: int = 0,
                 out=None):
    """Batched search.

    k=None: one `SearchResult` per query with the reference's full semantics
    (every scanned code, reranked or in scan order).
    k=int:  (ids (B, k) int32 padded -1, dists (B, k) float32 padded +inf,
    stats (B, 4) int64) -- row b is the first k entries of search()'s
    reranked list.  `queries` may be a numpy array or a CUDA torch tensor;
    with a tensor the outputs are CUDA tensors on the current stream.
    `out=(ids, dists, stats)` reuses caller-owned (e.g. pinned) arrays.
    """
    dev = device_index(index, device)
    lib = _native.load()
    cp = _cparams(params)
    if _is_torch_cuda(queries):
        return _search_batch_torch(dev, queries, cp, params, k, out)
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
    if q.ndim == 1:
        q = q[None, :]
    _check_query_dim(dev, q)
    b = q.shape[0]
    if k is not None and out is not None:
        ids, dists, stats = out
        _check_out(ids, dists, stats, b, int(k))
        _native.check(lib.givf_search_topk(dev.handle, _vp(q), b, ctypes.byref(cp), int(k),
                                           _vp(ids), _vp(dists), _vp(stats), None))
        return ids, dists, stats
    stats = np.zeros((b, 4), np.int64)
    if k is not None:
        ids = np.empty((b, int(k)), np.int32)
        dists = np.empty((b, int(k)), np.float32)
        _native.check(lib.givf_search_topk(dev.handle, _vp(q), b, ctypes.byref(cp), int(k),
                                           _vp(ids), _vp(dists), _vp(stats), None))
        return ids, dists, stats
    cap = max(1, min(int(params.candidates), dev.n_local))
    ids = np.empty((b, cap), np.int32)
    dists = np.empty((b, cap), np.float32)
    t0 = time.perf_counter()
    _native.check(lib.givf_search_full(dev.handle, _vp(q), b, ctypes.byref(cp), cap,
                                       _vp(ids), _vp(dists), _vp(stats), None))
    wall = (time.perf_counter() - t0) / max(b, 1)
    out = []
    for i in range(b):
        n = int(stats[i, 3])
        out.append(SearchResult(
            ids=ids[i, :n].copy(), distances=dists[i, :n].copy(),
            stats=SearchStats(int(stats[i, 0]), int(stats[i, 1]), int(stats[i, 2]), n, wall)))
    return out


def _check_out(ids, dists, stats, b, k, device=None):
    """Caller-owned outputs: right dtype, shape, C-contiguous, writable, and
    (torch) on the index's device -- the kernels write them raw."""
    want = ((ids, "ids", (b, k), "int32"), (dists, "dists", (b, k), "float32"),
            (stats, "stats", (b, 4), "int64"))
    for a, name, shape, dt in want:
        if tuple(a.shape) != shape:
            raise ValueError(f"out {name}: shape {tuple(a.shape)} != {shape}")
        if str(a.dtype).replace("torch.", "") != dt:
            raise ValueError(f"out {name}: dtype {a.dtype} != {dt}")
        if hasattr(a, "is_contiguous"):
            if not a.is_contiguous():
                raise ValueError(f"out {name}: not contiguous")
            if device is not None and a.is_cuda and a.device.index != device:
                raise ValueError(f"out {name}: on cuda:{a.device.index}, index on cuda:{device}")
        else:
            if not a.flags.c_contiguous or not a.flags.writeable:
                raise ValueError(f"out {name}: not C-contiguous and writable")


def _is_torch_cuda(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch") and getattr(x, "is_cuda", False)


def _search_batch_torch(dev, queries, cp, params, k, out=None):
    import torch

    if k is None:
        raise ValueError("torch input needs k (device top-k mode)")
    q = queries.contiguous().to(torch.float32)
    if q.dim() == 1:
        q = q[None, :]
    if q.shape[-1] != dev.dim:
        raise ValueError(f"query dim {q.shape[-1]} != index dim {dev.dim}")
    b = q.shape[0]
    if q.device.index != dev.device:
        raise ValueError(f"queries on cuda:{q.device.index}, index on cuda:{dev.device}")
    if out is not None:
        ids, dists, stats = out
        _check_out(ids, dists, stats, b, int(k), dev.device)
    else:
        ids = torch.empty((b, int(k)), dtype=torch.int32, device=q.device)
        dists = torch.empty((b, int(k)), dtype=torch.float32, device=q.device)
        stats = torch.empty((b, 4), dtype=torch.int64, device=q.device)
    stream = torch.cuda.current_stream(q.device).cuda_stream
    _native.check(_native.load().givf_search_topk(
        dev.handle, ctypes.c_void_p(q.data_ptr()), b, ctypes.byref(cp), int(k),
        ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(dists.data_ptr()),
        ctypes.c_void_p(stats.data_ptr()), ctypes.c_void_p(stream)))
    return ids, dists, stats


def search(index, query, params: SearchParams) -> SearchResult:
    """Run one query; returns SearchResult with ids/distances/stats.

    With rerank=True results are sorted by (estimated distance, id) and
    distances hold the per-point estimates.  With rerank=False points stay in
    scan order and each carries its group's anchor distance instead.
    """
    dev = device_index(index)
    q = np.asarray(query, dtype=np.float32).reshape(-1)
    _check_query_dim(dev, q)
    t0 = time.perf_counter()
    res = search_batch(dev, q[None, :], params)[0]
    res.stats.wall_time_s = time.perf_counter() - t0
    return res


def probe(index, queries, nprobe: int, device: int = 0):
    """Exact region ranking (search.py:77-90 at ef_search == K):
    region ids (B, nprobe) int32 and float64 qc2 (B, nprobe)."""
    dev = device_index(index, device)
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
    if q.ndim == 1:
        q = q[None, :]
    _check_query_dim(dev, q)
    b = q.shape[0]
    regions = np.empty((b, int(nprobe)), np.int32)
    qc2 = np.empty((b, int(nprobe)), np.float64)
    _native.check(_native.load().givf_probe(dev.handle, _vp(q), b, int(nprobe), _vp(regions),
                                           _vp(qc2), None))
    return regions, qc2


def probe_scores(index, queries, device: int = 0):
    """Approximate region scores |c|^2 - 2 q.c from the probe GEMM (tensor
    cores unless GIVF_PROBE=simt) and their error-bound scale."""
    dev = device_index(index, device)
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
    if q.ndim == 1:
        q = q[None, :]
    _check_query_dim(dev, q)
    out = np.empty((q.shape[0], dev.k), np.float32)
    eps = ctypes.c_float(0.0)
    _native.check(_native.load().givf_probe_scores(dev.handle, _vp(q), q.shape[0], _vp(out),
                                                  ctypes.byref(eps), None))
    return out, float(eps.value)


def plan_capacity(index, params: SearchParams, device: int = 0) -> int:
    """Records per query givf_plan needs: min(ceil(tau * P * L), candidates)."""
    dev = device_index(index, device)
    cap = ctypes.c_int64(0)
    _native.check(_native.load().givf_plan_capacity(dev.handle, ctypes.byref(_cparams(params)),
                                                    ctypes.byref(cap)))
    return int(cap.value)


def plan_batch(index, queries, params: SearchParams, device: int = 0):
    """The planning half of search() (search.py:77-139) for a share of the
    queries, in the global form the list-sharded layout exchanges (SURVEY
    §8e): CUDA tensors items (B, cap, 4) int32 = givf_plan_item records
    (group, len, base as two words), nitems (B,) int32, stats (B, 4) int64."""
    import torch

    dev = device_index(index, device)
    cp = _cparams(params)
    cap = plan_capacity(dev, params)
    if _is_torch_cuda(queries):
        q = queries.contiguous().to(torch.float32)
        qp = ctypes.c_void_p(q.data_ptr())
    else:
        q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
        qp = _vp(q)
    if q.ndim == 1:
        q = q[None, :]
    if q.shape[-1] != dev.dim:
        raise ValueError(f"query dim {q.shape[-1]} != index dim {dev.dim}")
    b = q.shape[0]
    cuda = torch.device("cuda", dev.device)
    items = torch.empty((b, cap, 4), dtype=torch.int32, device=cuda)
    nitems = torch.empty((b,), dtype=torch.int32, device=cuda)
    stats = torch.empty((b, 4), dtype=torch.int64, device=cuda)
    stream = torch.cuda.current_stream(cuda).cuda_stream
    _native.check(_native.load().givf_plan(
        dev.handle, qp, b, ctypes.byref(cp), cap, ctypes.c_void_p(items.data_ptr()),
        ctypes.c_void_p(nitems.data_ptr()), ctypes.c_void_p(stats.data_ptr()),
        ctypes.c_void_p(stream)))
    return items, nitems, stats


def compact_plans(items, nitems):
    """(B, cap, 4) padded plans -> CSR: offsets (B + 1,) int64, flat (T, 4)."""
    import torch

    cap = items.shape[1]
    mask = torch.arange(cap, device=items.device)[None, :] < nitems[:, None].to(torch.int64)
    flat = items[mask].contiguous()
    offsets = torch.zeros(items.shape[0] + 1, dtype=torch.int64, device=items.device)
    offsets[1:] = torch.cumsum(nitems.to(torch.int64), 0)
    return offsets, flat


def search_planned(index, queries, params: SearchParams, offsets, items, k: int,
                   device: int = 0):
    """Top-k from plans made by plan_batch on any rank (search.py:138-158),
    scanning the rows this (shard) index holds: CUDA tensors ids (B, k),
    dists (B, k).  offsets / items: the CSR of compact_plans, on the device."""
    import torch

    dev = device_index(index, device)
    cp = _cparams(params)
    if _is_torch_cuda(queries):
        q = queries.contiguous().to(torch.float32)
        qp = ctypes.c_void_p(q.data_ptr())
    else:
        q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
        qp = _vp(q)
    b = q.shape[0]
    cuda = torch.device("cuda", dev.device)
    ids = torch.empty((b, int(k)), dtype=torch.int32, device=cuda)
    dists = torch.empty((b, int(k)), dtype=torch.float32, device=cuda)
    stream = torch.cuda.current_stream(cuda).cuda_stream
    _native.check(_native.load().givf_search_planned(
        dev.handle, qp, b, ctypes.byref(cp), ctypes.c_void_p(offsets.data_ptr()),
        ctypes.c_void_p(items.data_ptr()), int(k), ctypes.c_void_p(ids.data_ptr()),
        ctypes.c_void_p(dists.data_ptr()), ctypes.c_void_p(stream)))
    return ids, dists


def decomposed_distance(query, centroid, neighbor, alpha, code, tables, const_term):
    """Scalar float64 evaluation of the expanded distance form for one point
    (search.py:166-183); `tables` is an inner-product lookup table object with
    `.entries` (M, 256) and `.mode`."""
    if tables.mode != "inner":
        raise ValueError("decomposed_distance needs an inner-product table")
    q = np.asarray(query, dtype=np.float64)
    c = np.asarray(centroid, dtype=np.float64)
    s = np.asarray(neighbor, dtype=np.float64)
    a = float(alpha)
    m = tables.entries.shape[0]
    ip = float(tables.entries[np.arange(m), np.asarray(code)].sum(dtype=np.float64))
    return (1.0 - a) * float(((q - c) ** 2).sum()) + a * float(((q - s) ** 2).sum()) \
        - 2.0 * ip + float(const_term)


def recall_at_r(results, truth, r):
    """Fraction of queries whose true nearest neighbor appears in the top r
    (search.py:186-201).  results: SearchResults, id arrays or an (B, k) array."""
    truth = np.asarray(truth)
    if truth.ndim == 2:
        truth = truth[:, 0]
    if len(results) != truth.shape[0]:
        raise ValueError("results/truth length mismatch")
    hits = 0
    for res, t in zip(results, truth):
        ids = getattr(res, "ids", res)
        hits += int(np.any(np.asarray(ids)[:r] == t))
    return hits / max(len(results), 1)


@dataclass
class SweepRow:
    nprobe: int
    tau: float
    candidates: int
    r: int
    recall: float
    latency_ms: float
    codes_scanned: float


def sweep(index, queries, truth, grid, r_values=(1, 10, 100), latency_runs=1, batched=False):
    """One SweepRow per (params, r) (search.py:215-249).

    Default (batched=False) keeps the reference's semantics: every query is
    its own search() call, latency_ms is the mean over queries of each
    query's median wall time over latency_runs repeats (0 when latency_runs
    == 0, so runs compare byte for byte).  batched=True runs each grid point
    as one batch on the device and reports the batch wall time per query
    (a throughput figure, not the reference's per-query latency)."""
    queries = np.asarray(queries, dtype=np.float32)
    rows = []
    for params in grid:
        reps = max(1, latency_runs)
        if batched:
            times = []
            for _ in range(reps):
                t0 = time.perf_counter()
                results = search_batch(index, queries, params)
                times.append((time.perf_counter() - t0) / max(len(queries), 1))
            latency_ms = float(np.median(times)) * 1e3 if latency_runs > 0 else 0.0
        else:
            results, lat = [], []
            for qi in range(queries.shape[0]):
                t = np.empty(reps, dtype=np.float64)
                for j in range(reps):
                    res = search(index, queries[qi], params)
                    t[j] = res.stats.wall_time_s
                results.append(res)
                lat.append(float(np.median(t)))
            latency_ms = float(np.mean(lat)) * 1e3 if latency_runs > 0 else 0.0
        codes = float(np.mean([r.stats.codes_scanned for r in results])) if results else 0.0
        for r in r_values:
            rows.append(SweepRow(nprobe=params.nprobe, tau=params.tau,
                                 candidates=params.candidates, r=r,
                                 recall=recall_at_r(results, truth, r),
                                 latency_ms=latency_ms, codes_scanned=codes))
    return rows


def write_sweep_csv(rows, path):
    lines = ["nprobe,tau,candidates,R,recall,latency_ms,codes_scanned"]
    for row in rows:
        lines.append(
            f"{row.nprobe},{row.tau:g},{row.candidates},{row.r},"
            f"{row.recall:.6f},{row.latency_ms:.4f},{row.codes_scanned:.1f}"
        )
    data = "\n".join(lines) + "\n"
    with open(path, "w", encoding="utf-8") as f:
        f.write(data)
    return data


def verify_results(results):
    """Sanity checks on a batch of results; raises InvariantError on failure."""
    from .errors import InvariantError

    for i, res in enumerate(results):
        ids = res.ids
        if ids.shape[0] != np.unique(ids).shape[0]:
            raise InvariantError(f"query {i}: duplicate ids in results")
        d = res.distances
        if d.shape[0] > 1 and np.any(np.diff(d) < 0):
            raise InvariantError(f"query {i}: distances not sorted")
        if res.stats.codes_scanned != ids.shape[0]:
            raise InvariantError(f"query {i}: codes_scanned != result length")
    return True
