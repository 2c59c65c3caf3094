"""Device-resident grouped index (the read-only input of every kernel).

`IndexArrays` is the flat host form of the reference `GroupedIndex`
(/root/reference/pkg/src/givf/index.py:48-85); `DeviceIndex` uploads it once
through `givf_index_create` and owns the device copy.  A multi-GPU layout
 gives every device a `shard` of each (region, group) slice while
the GLOBAL group-size table is replicated, so each shard walks the same
candidate budget and needs no communication before its scan.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass
class IndexArrays:
    """Flat arrays of a GroupedIndex (index.py:48-62)."""

    centroids: np.ndarray            # (K, d) f32
    alphas: np.ndarray               # (K,) f32
    neighbor_ids: np.ndarray | None  # (K, L) i32
    norm_terms: np.ndarray | None    # (K, L) f32
    group_sizes: np.ndarray          # (K, G) i32
    region_offsets: np.ndarray       # (K+1,) i64
    point_ids: np.ndarray            # (n,) i32
    codes: np.ndarray                # (n, M) u8
    const_bytes: np.ndarray          # (n,) u8
    codewords: np.ndarray            # (M, 256, d/M) f32
    rotation: np.ndarray | None      # (d, d) f32
    const_lo: float
    const_hi: float
    grouping: bool
    meta: object = None              # storage.FileMeta when read from a .givf file

    def to_host(self) -> "IndexArrays":
        """A copy whose arrays are all numpy (row arrays may be CUDA tensors
        after a device-resident build)."""
        import dataclasses

        def h(a):
            return a.cpu().numpy() if hasattr(a, "cpu") and not isinstance(a, np.ndarray) else a

        return dataclasses.replace(self, point_ids=h(self.point_ids), codes=h(self.codes),
                                   const_bytes=h(self.const_bytes))

    @property
    def k(self) -> int:
        return int(self.centroids.shape[0])

    @property
    def dim(self) -> int:
        return int(self.centroids.shape[1])

    @property
    def n(self) -> int:
        return int(self.point_ids.shape[0])

    @property
    def m(self) -> int:
        return int(self.codewords.shape[0])

    @property
    def groups_per_region(self) -> int:
        return int(self.group_sizes.shape[1])

    @classmethod
    def from_any(cls, index) -> "IndexArrays":
        """Adapt a reference GroupedIndex, an IndexArrays or any object with
        the same flat attribute names."""
        if isinstance(index, cls):
            return index
        if hasattr(index, "centroids"):
            g = bool(index.grouping)
            return cls(
                centroids=_f32(index.centroids), alphas=_f32(index.alphas),
                neighbor_ids=_i32(index.neighbor_ids) if g else None,
                norm_terms=_f32(index.norm_terms) if g else None,
                group_sizes=_i32(index.group_sizes), region_offsets=_i64(index.region_offsets),
                point_ids=_i32(index.point_ids), codes=_u8(index.codes),
                const_bytes=_u8(index.const_bytes), codewords=_f32(index.codewords),
                rotation=None if index.rotation is None else _f32(index.rotation),
                const_lo=float(index.const_lo), const_hi=float(index.const_hi), grouping=g,
            )
        g = bool(index.params.grouping)
        k = index.coarse.centroids.shape[0]
        return cls(
            centroids=_f32(index.coarse.centroids), alphas=_f32(index.alphas),
            neighbor_ids=_i32(index.neighbor_ids) if g else None,
            norm_terms=_f32(index.norm_terms) if g else None,
            group_sizes=_i32(np.asarray(index.group_sizes).reshape(k, -1)),
            region_offsets=_i64(index.region_offsets), point_ids=_i32(index.point_ids),
            codes=_u8(index.codes), const_bytes=_u8(index.const_bytes),
            codewords=_f32(index.pq.codewords),
            rotation=None if index.pq.rotation is None else _f32(index.pq.rotation),
            const_lo=float(index.const_quant.lo), const_hi=float(index.const_quant.hi),
            grouping=g,
        )


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(a.data_ptr())  # CUDA tensor (device-resident row arrays)


def _is_torch(a):
    return a is not None and not isinstance(a, np.ndarray) and hasattr(a, "data_ptr")


def _rows(a, dtype):
    """Row arrays: numpy (converted) or CUDA tensors (checked, kept)."""
    if _is_torch(a):
        import torch

        want = {np.int32: torch.int32, np.uint8: torch.uint8}[dtype]
        if a.dtype != want or not a.is_contiguous():
            a = a.to(want).contiguous()
        return a
    return np.ascontiguousarray(a, dtype=dtype)


def shard_rows(arr: IndexArrays, g: int, shards: int):
    """Rows of shard g: slice [floor(g*s/G), floor((g+1)*s/G)) of every
    (region, group) segment of size s, in stored (ascending id) order."""
    if _is_torch(arr.codes):
        return _shard_rows_torch(arr, g, shards)
    sizes = arr.group_sizes.astype(np.int64)
    lo = (g * sizes) // shards
    hi = ((g + 1) * sizes) // shards
    starts = arr.region_offsets[:-1, None] + (np.cumsum(sizes, axis=1) - sizes)
    cnt = (hi - lo).ravel()
    first = (starts + lo).ravel()
    seg = np.repeat(np.arange(cnt.shape[0]), cnt)
    offs = np.cumsum(cnt) - cnt
    rows = first[seg] + (np.arange(seg.shape[0]) - offs[seg])
    return rows, lo.astype(np.int32), (hi - lo).astype(np.int32)


def _shard_rows_torch(arr: IndexArrays, g: int, shards: int):
    """shard_rows on the device (row arrays held as CUDA tensors)."""
    import torch

    dev = arr.codes.device
    sizes = torch.from_numpy(arr.group_sizes.astype(np.int64)).to(dev)
    lo = (g * sizes) // shards
    hi = ((g + 1) * sizes) // shards
    offs = torch.from_numpy(np.ascontiguousarray(arr.region_offsets[:-1])).to(dev)
    starts = offs[:, None] + (torch.cumsum(sizes, 1) - sizes)
    cnt = (hi - lo).reshape(-1)
    first = (starts + lo).reshape(-1)
    seg = torch.repeat_interleave(torch.arange(cnt.shape[0], device=dev), cnt)
    ends = torch.cumsum(cnt, 0)
    rows = first[seg] + (torch.arange(seg.shape[0], device=dev) - (ends - cnt)[seg])
    return rows, lo.int().cpu().numpy(), (hi - lo).int().cpu().numpy()


class DeviceIndex:
    """A GroupedIndex (or one shard of it) resident on one GPU."""

    def __init__(self, index, device: int = 0, shard: tuple[int, int] | None = None):
        lib = _native.load()
        arr = IndexArrays.from_any(index)
        self.arrays = arr
        self.device = int(device)
        self.shard = shard
        k, d = arr.centroids.shape
        gsz = arr.group_sizes
        if shard is not None and shard[1] > 1:
            g, ns = shard
            rows, lo, cnt = shard_rows(arr, g, ns)
            offs = np.zeros(k + 1, np.int64)
            np.cumsum(cnt.sum(axis=1, dtype=np.int64), out=offs[1:])
            pids, codes, cbytes = arr.point_ids[rows], arr.codes[rows], arr.const_bytes[rows]
            local_sizes, local_lo = _i32(cnt), _i32(lo)
        else:
            offs, pids, codes, cbytes = arr.region_offsets, arr.point_ids, arr.codes, arr.const_bytes
            local_sizes = local_lo = None
        offs, pids, codes, cbytes = _i64(offs), _rows(pids, np.int32), _rows(codes, np.uint8), _rows(cbytes, np.uint8)
        keep = [arr.centroids, arr.alphas, arr.neighbor_ids, arr.norm_terms, gsz, offs,
                local_sizes, local_lo, pids, codes, cbytes, arr.codewords, arr.rotation]
        desc = _native.IndexDesc(
            k=k, dim=d, groups=gsz.shape[1], m=arr.codewords.shape[0],
            grouping=1 if arr.grouping else 0, n=int(pids.shape[0]),
            centroids=_ptr(arr.centroids), alphas=_ptr(arr.alphas),
            neighbor_ids=_ptr(arr.neighbor_ids), norm_terms=_ptr(arr.norm_terms),
            group_sizes=_ptr(gsz), region_offsets=_ptr(offs),
            local_sizes=_ptr(local_sizes), local_lo=_ptr(local_lo),
            point_ids=_ptr(pids), codes=_ptr(codes), const_bytes=_ptr(cbytes),
            codewords=_ptr(arr.codewords), rotation=_ptr(arr.rotation),
            const_lo=arr.const_lo, const_hi=arr.const_hi,
        )
        h = ctypes.c_void_p()
        _native.check(lib.givf_index_create(ctypes.byref(desc), self.device, ctypes.byref(h)))
        del keep
        self._h = h
        self.n_local = int(pids.shape[0])
        self.k, self.dim = int(k), int(d)
        self.n = arr.n

    @property
    def handle(self):
        return self._h

    def device_bytes(self) -> int:
        return int(_native.load().givf_index_device_bytes(self._h))

    def fallback_counts(self) -> dict:
        """Queries that left the fast path so far (probe re-check / planner)."""
        out = np.zeros(16, np.int64)
        _native.check(_native.load().givf_index_counters(self._h, out.ctypes.data, 16))
        return {"probe": int(out[0]), "plan": int(out[1])}

    def probe_retries(self) -> int:
        """Queries the fused probe re-ran with its guaranteed threshold (their
        sampled threshold missed; the retry keeps them off the exhaustive path)."""
        out = np.zeros(16, np.int64)
        _native.check(_native.load().givf_index_counters(self._h, out.ctypes.data, 16))
        return int(out[8])

    def plan_retries(self) -> int:
        """Queries the approximate planner re-ran with a 2048-entry certified
        window (their first window overflowed)."""
        out = np.zeros(16, np.int64)
        _native.check(_native.load().givf_index_counters(self._h, out.ctypes.data, 16))
        return int(out[9])

    def plan_fallback_reasons(self) -> dict:
        """Approximate-planner fallbacks split by the check that failed."""
        out = np.zeros(8, np.int64)
        _native.check(_native.load().givf_index_counters(self._h, out.ctypes.data, 8))
        names = ("ties", "window_overflow", "crossing_before_window", "crossing_off_center",
                 "walk_not_ended", "too_many_groups")
        return {n: int(v) for n, v in zip(names, out[2:8])}

    def close(self):
        if getattr(self, "_h", None):
            _native.load().givf_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_index(index, device: int = 0) -> DeviceIndex:
    """Device copy of `index`, built once and cached on the object."""
    if isinstance(index, DeviceIndex):
        return index
    cached = getattr(index, "_givf_b200_device", None)
    if cached is not None and cached.device == device and cached._h:
        return cached
    dev = DeviceIndex(index, device=device)
    try:
        object.__setattr__(index, "_givf_b200_device", dev)
    except (AttributeError, TypeError):
        pass
    return dev
