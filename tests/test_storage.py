"""`.givf` reader / writer against files written by the reference's own
save_index (tests/golden/make_golden.py: fixture_givf) -- reference
storage.py:114-281 and its tests (pkg/tests/test_storage.py)."""

import os

import numpy as np
import pytest

from golden_io import load
from paper_1802_02422_b200.device_index import IndexArrays
from paper_1802_02422_b200.errors import (BadMagicError, ChecksumError, StorageError,
                                          VersionError)
from paper_1802_02422_b200.storage import _digest, load_index, save_index

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NAMES = ["small_grouped", "small_flat"]


def _path(name):
    return os.path.join(GOLDEN, f"{name}.givf")


@pytest.mark.parametrize("name", NAMES)
def test_load_matches_reference_arrays(name):
    arr = load_index(_path(name))
    g = load(name)
    want = g.index
    assert arr.grouping == want.grouping
    for f in ("centroids", "alphas", "group_sizes", "region_offsets", "point_ids", "codes",
              "const_bytes", "codewords"):
        np.testing.assert_array_equal(getattr(arr, f), getattr(want, f), err_msg=f)
    if arr.grouping:
        np.testing.assert_array_equal(arr.neighbor_ids, want.neighbor_ids)
        np.testing.assert_array_equal(arr.norm_terms, want.norm_terms)
    assert (arr.const_lo, arr.const_hi) == (np.float32(want.const_lo), np.float32(want.const_hi))


@pytest.mark.parametrize("name", NAMES)
def test_save_reproduces_reference_bytes(name, tmp_path):
    arr = load_index(_path(name))
    out = tmp_path / "x.givf"
    size = save_index(arr, out)
    ref = open(_path(name), "rb").read()
    assert size == len(ref)
    assert out.read_bytes() == ref


def test_roundtrip_without_graph(tmp_path):
    arr = load_index(_path("small_grouped"))
    bare = IndexArrays(**{f: getattr(arr, f) for f in (
        "centroids", "alphas", "neighbor_ids", "norm_terms", "group_sizes", "region_offsets",
        "point_ids", "codes", "const_bytes", "codewords", "rotation", "const_lo", "const_hi",
        "grouping")})
    out = tmp_path / "bare.givf"
    with pytest.raises(ValueError, match="allow_no_graph"):
        save_index(bare, out)
    save_index(bare, out, allow_no_graph=True)
    back = load_index(out)
    for f in ("centroids", "alphas", "neighbor_ids", "norm_terms", "group_sizes",
              "region_offsets", "point_ids", "codes", "const_bytes", "codewords"):
        np.testing.assert_array_equal(getattr(back, f), getattr(bare, f), err_msg=f)


def _rewrite(tmp_path, mutate, fix_checksum=True):
    raw = bytearray(open(_path("small_grouped"), "rb").read())
    mutate(raw)
    if fix_checksum:
        raw[-8:] = _digest(np.frombuffer(bytes(raw[:-8]), np.uint8))
    p = tmp_path / "bad.givf"
    p.write_bytes(bytes(raw))
    return p


def test_errors(tmp_path):
    def magic(raw):
        raw[0:4] = b"XXXX"

    with pytest.raises(BadMagicError, match="not an index file"):
        load_index(_rewrite(tmp_path, magic))

    def flip(raw):
        raw[200] ^= 1

    with pytest.raises(ChecksumError, match="checksum mismatch"):
        load_index(_rewrite(tmp_path, flip, fix_checksum=False))

    def version(raw):
        raw[4:8] = (2).to_bytes(4, "little")

    with pytest.raises(VersionError, match="unsupported index version 2"):
        load_index(_rewrite(tmp_path, version))

    def truncate(raw):
        del raw[-100:-8]

    with pytest.raises(StorageError, match="truncated"):
        load_index(_rewrite(tmp_path, truncate))

    short = tmp_path / "short.givf"
    short.write_bytes(b"GIVF")
    with pytest.raises(StorageError, match="too short"):
        load_index(short)

    assert issubclass(ChecksumError, StorageError)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_search_from_file(name):
    """The file path end to end: .givf -> DeviceIndex -> search == reference."""
    from golden_io import exact_runs
    from paper_1802_02422_b200 import SearchParams, search_batch
    from parity import assert_ranked_equal

    arr = load_index(_path(name))
    g = load(name)
    for run in exact_runs(g):
        p = SearchParams(**vars(run.params))
        for i, r in enumerate(search_batch(arr, g.queries, p)):
            want_ids, want_d = run.results[i]
            s = r.stats
            assert [s.regions_visited, s.subregions_visited, s.subregions_pruned,
                    s.codes_scanned] == list(run.stats[i])
            if run.params.rerank:
                assert_ranked_equal(r.ids, r.distances, want_ids, want_d)
            else:
                np.testing.assert_array_equal(r.ids, want_ids)
