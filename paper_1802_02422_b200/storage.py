"""`.givf` index files: the reference's single-file format, read and written
without materialising Python objects per region.

Layout (storage.py:1-28 of the reference, version 1, little-endian): magic,
header (version, flags, dim, k, m, l, dataset hash, build seed, const lo/hi),
centroids, optional rotation, PQ codewords, the proximity graph, then per
region `u32 size, f32 alpha, [l u32 neighbor ids, l f32 norm terms, l u32
group sizes]` followed by `size` records `(u32 id, m u8 code, u8 const)`,
and a blake2b-8 checksum of everything before it.

`load_index` (reference storage.py:162-281) memory-maps the file, checks the
checksum in streaming chunks and lifts every section with numpy views; the
result is an `IndexArrays` ready for `DeviceIndex` (one upload).  The graph
is kept as raw bytes (the B200 path probes exactly and never walks it) so
that `save_index` (reference storage.py:114-127) writes a loaded index back
byte for byte.  Errors are the reference's classes and messages.
"""

from __future__ import annotations

import hashlib
import os
import struct
from dataclasses import dataclass

import numpy as np

from .device_index import IndexArrays
from .errors import BadMagicError, ChecksumError, StorageError, VersionError

MAGIC = b"GIVF"
_HEADER = struct.Struct("<II4I2Q2f")  # after the magic (storage.py:39)
_U64_MASK = (1 << 64) - 1
_CHUNK = 1 << 26


@dataclass
class FileMeta:
    """Header fields and the graph section that IndexArrays does not carry."""

    version: int
    l: int
    dataset_hash: int
    build_seed: int
    rotation: bool
    graph: bytes  # raw graph section (entry point, max links, per-node layers)


def _record_dtype(m):
    return np.dtype([("id", "<u4"), ("code", "u1", (m,)), ("const", "u1")])


def _digest(buf) -> bytes:
    h = hashlib.blake2b(digest_size=8)
    for o in range(0, len(buf), _CHUNK):
        h.update(memoryview(buf[o:o + _CHUNK]))
    return h.digest()


class _Cursor:
    def __init__(self, buf):
        self.buf = buf
        self.o = 0

    def need(self, count):
        if self.o + count > len(self.buf):
            raise StorageError(f"index file truncated: need {count} bytes at offset {self.o}")

    def u32(self):
        self.need(4)
        v = int.from_bytes(bytes(self.buf[self.o:self.o + 4]), "little")
        self.o += 4
        return v

    def array(self, dtype, count):
        dtype = np.dtype(dtype)
        self.need(dtype.itemsize * count)
        out = np.frombuffer(self.buf, dtype=dtype, count=count, offset=self.o)
        self.o += dtype.itemsize * count
        return out


def load_index(path, verify: bool = True) -> IndexArrays:
    """Read a .givf file into flat arrays (reference storage.py:162-281)."""
    raw = np.memmap(os.fspath(path), dtype=np.uint8, mode="r")
    if raw.size < len(MAGIC) + _HEADER.size + 8:
        raise StorageError(f"index file too short ({raw.size} bytes)")
    if bytes(raw[:4]) != MAGIC:
        raise BadMagicError(f"not an index file (magic {bytes(raw[:4])!r})")
    if verify and _digest(raw[:-8]) != bytes(raw[-8:]):
        raise ChecksumError("index file checksum mismatch")
    cur = _Cursor(raw[:-8])
    cur.o = 4
    cur.need(_HEADER.size)
    (version, flags, dim, k, m, l, dataset_hash, build_seed, lo, hi) = _HEADER.unpack(
        bytes(raw[4:4 + _HEADER.size]))
    cur.o += _HEADER.size
    if version != 1:
        raise VersionError(f"unsupported index version {version}")
    grouping = bool(flags & 1)
    rotation_flag = bool(flags & 2)
    if dim <= 0 or k <= 0 or m <= 0 or dim % m != 0:
        raise StorageError(f"corrupt header: dim={dim} k={k} m={m}")
    if grouping and not 0 < l < k:
        raise StorageError(f"corrupt header: l={l} out of range for k={k}")

    centroids = cur.array("<f4", k * dim).reshape(k, dim).copy()
    rotation = cur.array("<f4", dim * dim).reshape(dim, dim).copy() if rotation_flag else None
    codewords = cur.array("<f4", m * 256 * (dim // m)).reshape(m, 256, dim // m).copy()

    # graph: validated like the reference, kept raw
    g0 = cur.o
    entry_point = cur.u32()
    max_links = cur.u32()
    if entry_point >= k or max_links < 2:
        raise StorageError("corrupt graph header")
    spans = []
    for i in range(k):
        layer_count = cur.u32()
        if layer_count < 1:
            raise StorageError(f"corrupt graph: node {i} has no layers")
        for _ in range(layer_count):
            degree = cur.u32()
            cur.need(4 * degree)
            if degree:
                spans.append((cur.o, degree))
            cur.o += 4 * degree
    if spans:
        starts = np.fromiter((s for s, _ in spans), np.int64, len(spans))
        degs = np.fromiter((d for _, d in spans), np.int64, len(spans))
        idx = np.repeat(starts, degs) + 4 * (np.arange(int(degs.sum()))
                                             - np.repeat(np.cumsum(degs) - degs, degs))
        words = raw[idx[:, None] + np.arange(4)].copy().view("<u4").ravel()
        if int(words.max()) >= k:
            raise StorageError("corrupt graph: neighbor id out of range")
    graph = bytes(raw[g0:cur.o])

    groups = l if grouping else 1
    hsz = 8 + (12 * l if grouping else 0)
    rec = _record_dtype(m)
    heads = np.empty(k, np.int64)
    sizes = np.empty(k, np.int64)
    for r in range(k):  # one u32 per region; records are skipped, not parsed
        heads[r] = cur.o
        size = cur.u32()
        sizes[r] = size
        cur.o += hsz - 4
        cur.need(rec.itemsize * size)
        cur.o += rec.itemsize * size
    if cur.o != len(cur.buf):
        raise StorageError(f"{len(cur.buf) - cur.o} unexpected trailing bytes")

    def field(off, count, dt):  # (k, count) values at heads + off
        idx = heads[:, None] + off + 4 * np.arange(count)
        return raw[idx[..., None] + np.arange(4)].copy().view(dt).reshape(k, count)

    alphas = field(4, 1, "<f4").ravel().copy()
    if grouping:
        neighbor_ids = field(8, l, "<u4").astype(np.int32)
        norm_terms = field(8 + 4 * l, l, "<f4").copy()
        group_sizes = field(8 + 8 * l, l, "<u4").astype(np.int32)
        bad = np.nonzero(group_sizes.sum(axis=1, dtype=np.int64) != sizes)[0]
        if bad.size:
            raise StorageError(f"corrupt region {int(bad[0])}: group sizes do not add up")
        if int(neighbor_ids.max(initial=0)) >= k:
            raise StorageError("corrupt region header: neighbor id out of range")
    else:
        neighbor_ids = norm_terms = None
        group_sizes = sizes.astype(np.int32).reshape(k, 1)
    region_offsets = np.zeros(k + 1, np.int64)
    np.cumsum(sizes, out=region_offsets[1:])
    n = int(region_offsets[-1])
    point_ids = np.empty(n, np.int32)
    codes = np.empty((n, m), np.uint8)
    const_bytes = np.empty(n, np.uint8)
    for r in np.nonzero(sizes)[0]:
        a, b = int(region_offsets[r]), int(region_offsets[r + 1])
        recs = np.frombuffer(raw, dtype=rec, count=b - a, offset=int(heads[r]) + hsz)
        point_ids[a:b] = recs["id"]
        codes[a:b] = recs["code"]
        const_bytes[a:b] = recs["const"]
    arr = IndexArrays(
        centroids=centroids, alphas=alphas, neighbor_ids=neighbor_ids, norm_terms=norm_terms,
        group_sizes=group_sizes, region_offsets=region_offsets, point_ids=point_ids,
        codes=codes, const_bytes=const_bytes, codewords=codewords, rotation=rotation,
        const_lo=float(lo), const_hi=float(hi), grouping=grouping,
        meta=FileMeta(version=version, l=l, dataset_hash=dataset_hash,
                      build_seed=build_seed, rotation=rotation_flag, graph=graph),
    )
    return arr


def _graph_bytes(index, k, allow_no_graph=False) -> bytes:
    meta = getattr(index, "meta", None)
    if isinstance(meta, FileMeta):
        return meta.graph
    g = getattr(index, "graph", None)
    if g is not None:  # a reference GroupedIndex: the reference writer's walk
        parts = [struct.pack("<II", int(g.entry_point), int(g.max_links))]
        for i in range(k):
            layer_count = int(g.levels[i]) + 1
            parts.append(struct.pack("<I", layer_count))
            for layer in range(layer_count):
                lay = g.layers[layer]
                row = lay.adjacency[lay.local_of[i]]
                row = row[row >= 0]
                parts.append(struct.pack("<I", row.size))
                parts.append(row.astype("<u4").tobytes())
        return b"".join(parts)
    # GPU-built index (no graph): a valid one-layer graph without edges.  The
    # reference's search_graph would then return only the entry point (one
    # probed region whatever nprobe says), so it is written only on request.
    if not allow_no_graph:
        raise ValueError("index has no proximity graph: the reference could load the file but "
                         "its graph probe would visit one region; pass allow_no_graph=True to "
                         "write an edgeless graph (for this package's loader)")
    return struct.pack("<II", 0, 2) + struct.pack("<II", 1, 0) * k


def save_index(index, path, *, l=None, dataset_hash=0, build_seed=0,
               allow_no_graph=False) -> int:
    """Write `index` (IndexArrays from load_index / the builder, or a
    reference GroupedIndex) as a .givf file; returns the bytes written.
    An index without a proximity graph (GPU-built) needs allow_no_graph=True:
    the file then carries an edgeless graph that the reference's own search
    cannot probe with (see _graph_bytes)."""
    arr = IndexArrays.from_any(index)
    meta = getattr(index, "meta", None)
    params = getattr(index, "params", None)
    k, dim, m = arr.k, arr.dim, arr.m
    if isinstance(meta, FileMeta):
        version, l_hdr, dh, seed = meta.version, meta.l, meta.dataset_hash, meta.build_seed
    elif params is not None:
        version, l_hdr, dh, seed = params.version, params.l, params.dataset_hash, params.seed
    else:
        version, dh, seed = 1, dataset_hash, build_seed
        l_hdr = l if l is not None else (arr.groups_per_region if arr.grouping else 0)
    flags = (1 if arr.grouping else 0) | (2 if arr.rotation is not None else 0)
    path = os.fspath(path)
    tmp = path + ".tmp"
    h = hashlib.blake2b(digest_size=8)
    with open(tmp, "wb") as f:
        def w(b):
            h.update(b)
            f.write(b)

        w(MAGIC)
        w(_HEADER.pack(version, flags, dim, k, m, l_hdr, dh & _U64_MASK, seed & _U64_MASK,
                       float(arr.const_lo), float(arr.const_hi)))
        w(np.ascontiguousarray(arr.centroids, "<f4").tobytes())
        if arr.rotation is not None:
            w(np.ascontiguousarray(arr.rotation, "<f4").tobytes())
        w(np.ascontiguousarray(arr.codewords, "<f4").tobytes())
        w(_graph_bytes(index, k, allow_no_graph))
        recs = np.zeros(arr.n, _record_dtype(m))
        recs["id"] = arr.point_ids
        recs["code"] = arr.codes
        recs["const"] = arr.const_bytes
        offs = arr.region_offsets
        for r in range(k):
            a, b = int(offs[r]), int(offs[r + 1])
            head = [struct.pack("<If", b - a, float(arr.alphas[r]))]
            if arr.grouping:
                head.append(arr.neighbor_ids[r].astype("<u4").tobytes())
                head.append(arr.norm_terms[r].astype("<f4").tobytes())
                head.append(arr.group_sizes[r].astype("<u4").tobytes())
            w(b"".join(head))
            w(recs[a:b].tobytes())
        f.write(h.digest())
        size = f.tell()
    os.replace(tmp, path)
    return size
