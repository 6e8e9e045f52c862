"""Randomised sweep of the rank path through the C ABI: repository kind, size (including sizes
around the top-k candidate cap and not multiples of any vector width), dimension, k (0, 1, near n,
> n, past the 8192-candidate layout), id mode (none / shuffled / with an id base via from_device),
score distribution (continuous / heavy ties / all equal), and host vs device calls. Every list
must be the oracle's top_k (ranker.py:97-143) of the GPU's own scores, and PQ scores must be
bit-identical to the oracle (pq.py:248-276)."""

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    kind = ["dense", "pq", "binary"][seed % 3]
    n = int(rng.choice([1, 2, 7, 33, 1000, 4097, 8191, 8193, 20_011, 65_537, 300_007]))
    k = int(rng.choice([0, 1, 5, 100, 1000, 8192, 9000, n, n + 3]))
    dist = ["cont", "ties", "const"][rng.integers(3)]
    ids = None
    if rng.random() < 0.5:
        ids = rng.permutation(3 * n + 5)[:n].astype(np.int64)
    return rng, kind, n, k, dist, ids


@pytest.mark.parametrize("seed", range(72))
def test_random_rank(otf, seed):
    rng, kind, n, k, dist, ids = _case(seed)
    if kind == "dense":
        d = int(rng.choice([3, 32, 128, 200, 2048]))
        x = rng.standard_normal((n, d)).astype(np.float32)
        if dist == "ties":
            x = np.round(x)
        elif dist == "const":
            x[:] = 1.0
        repo = otf.Repository.dense(otf.FeatureStore(x, ids=ids))
        w = rng.standard_normal(d)
    elif kind == "pq":
        m = int(rng.choice([4, 8, 16]))
        q = int(rng.choice([2, 8]))
        kc = int(rng.choice([16, 256]))
        cents = rng.standard_normal((m, kc, q)).astype(np.float32)
        if dist == "ties":
            cents = np.round(cents)
        elif dist == "const":
            cents[:] = 0.5
        codes = rng.integers(0, kc, (n, m), dtype=np.uint8)
        repo = otf.Repository.quantized(otf.PQCodebook(cents), codes, ids=ids)
        w = rng.standard_normal(m * q)
        ref = O.score_pq(w, cents, codes)
    else:
        bits = int(rng.choice([13, 64, 1024, 2048]))
        codes = rng.integers(0, 256, (n, (bits + 7) // 8), dtype=np.uint8)
        if dist == "const":
            codes[:] = 0xFF
        codec = otf.BinaryCodec(otf.TightFrame(np.eye(bits, 128 if bits >= 128 else bits)),
                                np.zeros(128 if bits >= 128 else bits, np.float32))
        repo = otf.Repository.binary(codec, codes, ids=ids)
        w = np.round(rng.standard_normal(bits)) if dist == "ties" else rng.standard_normal(bits)
    s = repo.score(w)
    if kind == "pq":
        assert s.tobytes() == ref.tobytes()
    r = repo.rank(otf.LinearModel(w, 1, 1), k)
    o_ids, o_sc, _ = O.top_k(s, k, ids)
    np.testing.assert_array_equal(r.ids, o_ids)
    np.testing.assert_array_equal(r.scores, np.asarray(o_sc, np.float64))


@pytest.mark.parametrize("seed", range(12))
def test_random_rank_many(otf, seed):
    """score_many / rank_many: random sizes (partial 128-row tiles, odd n), dims (multiples of
    32), classifier counts (1..130: several 64-classifier groups), k (0, > n)."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([129, 1000, 4097, 20_001]))
    d = int(rng.choice([32, 96, 512]))
    c = int(rng.choice([1, 7, 64, 65, 130]))
    k = int(rng.choice([0, 1, 100, n + 1]))
    x = rng.standard_normal((n, d)).astype(np.float32)
    W = rng.standard_normal((c, d))
    ids = rng.permutation(2 * n)[:n].astype(np.int64) if seed % 2 else None
    repo = otf.Repository.dense(otf.FeatureStore(x, ids=ids))
    S = repo.score_many(list(W))
    ex = (x.astype(np.float64) @ W.astype(np.float32).astype(np.float64).T).T
    mag = np.abs(W.astype(np.float32).astype(np.float64)) @ np.abs(x.astype(np.float64)).T
    assert np.all(np.abs(S - ex) <= 2.0 ** -20 * mag + np.spacing(np.abs(S)) + 1e-30)
    lists = repo.rank_many([otf.LinearModel(w, 1, 1) for w in W], k)
    for i in range(c):
        o_ids, o_sc, _ = O.top_k(S[i], k, ids)
        np.testing.assert_array_equal(lists[i].ids, o_ids)
        np.testing.assert_array_equal(lists[i].scores, np.asarray(o_sc, np.float64))


@pytest.mark.parametrize("seed", range(12))
def test_random_pq_encode(otf, seed):
    """pq_encode: random block counts, centroid counts (<= 256, not multiples of 8), sub-dims (the
    tensor-core form for Q = 8, the FFMA form otherwise) and scales; codes equal the float64
    oracle's except at rounding-level near-ties."""
    rng = np.random.default_rng(2000 + seed)
    m = int(rng.choice([1, 3, 16]))
    k = int(rng.choice([1, 5, 100, 256]))
    q = int(rng.choice([4, 8, 8, 16]))
    n = int(rng.choice([1, 31, 1000, 5003]))
    scale = float(10.0 ** rng.integers(-3, 4))
    cents = (rng.standard_normal((m, k, q)) * scale).astype(np.float32)
    vecs = (rng.standard_normal((n, m * q)) * scale).astype(np.float32)
    ref, _ = O.pq_encode(cents, vecs)
    gpu = otf.pq_encode(otf.PQCodebook(cents), vecs)
    for i, b in np.argwhere(gpu != ref):  # a differing code must be a rounding-level near-tie
        x = vecs[i, b * q:(b + 1) * q].astype(np.float64)
        c = cents[b].astype(np.float64)
        dist = (c * c).sum(1) - 2.0 * (c @ x)
        a, r = dist[int(gpu[i, b])], dist[int(ref[i, b])]
        assert abs(a - r) <= 1e-12 * max(1.0, abs(a), abs(r)), (i, b, a, r)
