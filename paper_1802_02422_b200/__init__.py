"""B200-native search path for the grouped inverted index of arXiv 1802.02422.

Drop-in for the query API of the reference package `givf`
(/root/reference/pkg/src/givf/search.py): `search`, `SearchParams`,
`SearchResult`, `sweep`, `recall_at_r`, ... plus `search_batch`.  The work
runs in hand-written sm_100a kernels behind a C ABI (include/givf_b200.h);
there is no CPU fallback.
"""

import importlib

__version__ = "0.1.0"

_EXPORTS = {
    "SearchParams": ".query",
    "SearchStats": ".query",
    "SearchResult": ".query",
    "search": ".query",
    "search_batch": ".query",
    "probe": ".query",
    "decomposed_distance": ".query",
    "recall_at_r": ".query",
    "sweep": ".query",
    "SweepRow": ".query",
    "write_sweep_csv": ".query",
    "verify_results": ".query",
    "IndexArrays": ".device_index",
    "DeviceIndex": ".device_index",
    "device_index": ".device_index",
    "ShardedIndex": ".sharded",
    "GivfError": ".errors",
    "InvariantError": ".errors",
    "StorageError": ".errors",
    "load_index": ".storage",
    "save_index": ".storage",
}

__all__ = sorted(_EXPORTS) + ["__version__"]


def __getattr__(name):
    if name in _EXPORTS:
        value = getattr(importlib.import_module(_EXPORTS[name], __name__), name)
        globals()[name] = value
        return value
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def __dir__():
    return __all__
