"""Run the reference's own search tests against the CUDA path.

Needs a machine that has BOTH the reference tree and a B200 (this round's GPU
boxes do not carry /root/reference, and reference sources are not copied into
this repo, so the driver's runs use tests/test_reference_scenarios.py
instead).  The overlay is a pytest plugin: before collection it imports the
reference package and rebinds `givf.search.search` to this package's
`search`, which accepts the reference's GroupedIndex as is
(device_index.IndexArrays.from_any); the reference's test modules then import
the rebound function.

    python tools/run_reference_suite.py [--reference /root/reference]
        [-- extra pytest args]

Default selection: pkg/tests/test_search.py and the acceptance scenarios 06,
07 and 08 (test_acceptance.py).
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class Overlay:
    def __init__(self):
        self.calls = 0

    def pytest_configure(self, config):
        import givf.search as ref_search

        import paper_1802_02422_b200 as ours

        overlay = self

        def search(index, query, params):
            overlay.calls += 1
            p = ours.SearchParams(nprobe=params.nprobe, tau=params.tau, candidates=params.candidates,
                                  ef_search=params.ef_search, rerank=params.rerank, prune=params.prune)
            r = ours.search(index, query, p)
            stats = ref_search.SearchStats(
                regions_visited=r.stats.regions_visited, subregions_visited=r.stats.subregions_visited,
                subregions_pruned=r.stats.subregions_pruned, codes_scanned=r.stats.codes_scanned,
                wall_time_s=r.stats.wall_time_s)
            return ref_search.SearchResult(ids=r.ids, distances=r.distances, stats=stats)

        ref_search.search = search

    def pytest_terminal_summary(self, terminalreporter):
        terminalreporter.write_line(f"overlay: {self.calls} search() calls served by libgivf_b200.so")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference")
    ap.add_argument("rest", nargs="*")
    args = ap.parse_args()
    src = os.path.join(args.reference, "pkg", "src")
    tests = os.path.join(args.reference, "pkg", "tests")
    if not os.path.isdir(src):
        sys.exit(f"no reference tree at {args.reference}")
    sys.path[:0] = [ROOT, src, tests]
    import pytest
    import torch

    if not torch.cuda.is_available():
        sys.exit("no CUDA device: the overlay has no CPU path")
    sel = args.rest or [os.path.join(tests, "test_search.py"),
                        os.path.join(tests, "test_acceptance.py"), "-k",
                        "test_search or scenario_06 or scenario_07 or scenario_08 or 06 or 07 or 08"]
    sys.exit(pytest.main(["-q", "-p", "no:cacheprovider", f"--rootdir={tests}"] + sel, plugins=[Overlay()]))


if __name__ == "__main__":
    main()
