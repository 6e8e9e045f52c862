"""Shared rank-parity check for the BASELINE-size tests (test infrastructure)."""

from __future__ import annotations

import numpy as np


def rank_parity(got_ids, ref_ids, ref_score_of, tol):
    """The north star's dense/binary rank contract: the GPU list equals the
    reference's list as a set, and in order, except where the two entries involved are near-tied
    under the REFERENCE's own scores (|ds| <= tol; ties resolve by id in both).

    ``ref_score_of`` maps an id to the reference's score (an array indexed by id, or a dict).
    Returns (swaps, boundary) — positions whose ids differ, ids in one list but not the other —
    so the tests can print them. Raises AssertionError with the first violation."""
    got = [int(i) for i in got_ids]
    ref = [int(i) for i in ref_ids]
    assert len(got) == len(ref), f"length {len(got)} != {len(ref)}"
    if got == ref:
        return 0, 0
    last = float(ref_score_of[ref[-1]])
    extra = set(got) ^ set(ref)
    for i in extra:
        d = abs(float(ref_score_of[i]) - last)
        assert d <= tol, f"id {i} in only one list, {d:.3g} from the k-th reference score (tol {tol:.3g})"
    swaps = 0
    for pos, (a, b) in enumerate(zip(got, ref)):
        if a != b:
            swaps += 1
            d = abs(float(ref_score_of[a]) - float(ref_score_of[b]))
            assert d <= tol, f"position {pos}: got id {a}, reference id {b}, scores {d:.3g} apart (tol {tol:.3g})"
    return swaps, len(extra) // 2
