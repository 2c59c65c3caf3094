"""Parity rules of the north star (BASELINE.json): candidate ids and stats
bit-exact, distances within 1e-4 relative, ranked ids equal except inside
runs of near-ties (the reference's own acceptance-08 rule,
test_acceptance.py:350-357)."""

import numpy as np

RTOL = 1e-4  # north_star: "Distances must agree within 1e-4 relative"


def tie_safe_mask(want_d):
    want_d = np.asarray(want_d, np.float64)
    tol = RTOL * (1.0 + np.abs(want_d))
    tied = np.diff(want_d) <= tol[:-1]
    safe = np.ones(want_d.shape[0], dtype=bool)
    safe[:-1] &= ~tied
    safe[1:] &= ~tied
    return safe


def assert_ranked_equal(got_ids, got_d, want_ids, want_d, exact_set=True):
    got_ids, want_ids = np.asarray(got_ids), np.asarray(want_ids)
    assert got_ids.shape == want_ids.shape, (got_ids.shape, want_ids.shape)
    if exact_set:
        assert np.array_equal(np.sort(got_ids), np.sort(want_ids)), "candidate id sets differ"
    np.testing.assert_allclose(np.asarray(got_d, np.float64), np.asarray(want_d, np.float64),
                               rtol=RTOL, atol=RTOL)
    safe = tie_safe_mask(want_d)
    assert np.array_equal(got_ids[safe], want_ids[safe]), "ranked ids differ outside ties"


def assert_topk_equal(got_ids, got_d, want_ids, want_d):
    """Top-k prefix: the last tie run may be cut differently at position k."""
    got_ids, want_ids = np.asarray(got_ids), np.asarray(want_ids)
    valid = want_ids >= 0
    assert np.array_equal(got_ids >= 0, valid)
    np.testing.assert_allclose(np.asarray(got_d, np.float64)[valid],
                               np.asarray(want_d, np.float64)[valid], rtol=RTOL, atol=RTOL)
    safe = tie_safe_mask(np.asarray(want_d)[valid])
    assert np.array_equal(got_ids[valid][safe], want_ids[valid][safe])
