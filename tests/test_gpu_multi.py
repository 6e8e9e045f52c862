"""Many classifiers at once (C5b) on the tcgen05 tensor cores, through the C ABI.

Bar: every classifier's scores stay within the reference tolerance of its own score_dense
(ranker.py:63-69; 1e-6 * ||w|| * ||x||) and within the documented error of the split products
of the exact dot (FP16 form, the default: x1 w1 + x1 w2 + x2 w1 in kind::f16; TF32 form:
x_hi w_hi + x_hi w_lo + x_lo w_hi in kind::tf32 — both <= 2^-20 of sum |x_j w_j| with the
float32 accumulation); rank_many equals the oracle's exact top_k of those scores; a row's scores
do not depend on its position (128-row tiles, padding rows, permutations).
"""

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


def exact(x, W):
    return x.astype(np.float64) @ W.astype(np.float32).astype(np.float64).T


@pytest.fixture(params=["fp16", "tf32"])
def form(request, monkeypatch):
    """Both operand forms of otf_multi.cu (OTF_MULTI_TF32=1 selects the TF32x3 kernel)."""
    if request.param == "tf32":
        monkeypatch.setenv("OTF_MULTI_TF32", "1")
    else:
        monkeypatch.delenv("OTF_MULTI_TF32", raising=False)
    return request.param


@pytest.mark.parametrize("n,d,c", [(1000, 128, 7), (129, 32, 1), (4096, 256, 64), (777, 4096, 3), (300, 2048, 70)])
def test_score_many_matches_dense(otf, form, n, d, c):
    rng = np.random.default_rng(n + d + c)
    x = rng.standard_normal((n, d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    W = rng.standard_normal((c, d))
    repo = otf.Repository.dense(otf.FeatureStore(x))
    S = repo.score_many(list(W))
    assert S.shape == (c, n) and S.dtype == np.float32
    ex = exact(x, W).T
    mag = np.abs(W.astype(np.float32).astype(np.float64)) @ np.abs(x.astype(np.float64)).T
    # TF32 x3: dropped lo*lo and TF32 truncation of the lo parts (<= 2^-21 relative per product);
    # FP16: dropped x2*w2 and the float16 rounding of x2, w2 (<= 3 * 2^-22); float32 accumulation
    # restarted every 128 K values (measured max 2^-22 of mag, numpy's own float32 sgemm: 2^-22.3)
    assert np.all(np.abs(S - ex) <= 2.0 ** -20 * mag + np.spacing(np.abs(S)) + 1e-30)
    for i in range(min(c, 5)):
        ref = O.score_dense(W[i], x)
        assert np.max(np.abs(S[i].astype(np.float64) - ref)) <= 1e-6 * np.linalg.norm(W[i]) * 1.0001


def test_score_many_position_independent(otf):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1500, 512)).astype(np.float32)
    W = rng.standard_normal((16, 512))
    S = otf.Repository.dense(otf.FeatureStore(x)).score_many(list(W))
    perm = rng.permutation(1500)
    S2 = otf.Repository.dense(otf.FeatureStore(x[perm])).score_many(list(W))
    np.testing.assert_array_equal(S2, S[:, perm])


def test_rank_many_exact_topk(otf):
    rng = np.random.default_rng(9)
    n, d, c, k = 20_000, 256, 12, 300
    x = rng.standard_normal((n, d)).astype(np.float32)
    ids = rng.permutation(3 * n)[:n].astype(np.int64)
    W = rng.standard_normal((c, d))
    repo = otf.Repository.dense(otf.FeatureStore(x, ids=ids))
    S = repo.score_many(list(W))
    lists = repo.rank_many([otf.LinearModel(w, 1, 3) for w in W], k)
    assert len(lists) == c
    for i in range(c):
        o_ids, o_sc, _ = O.top_k(S[i], k, ids)
        np.testing.assert_array_equal(lists[i].ids, o_ids)
        np.testing.assert_array_equal(lists[i].scores, o_sc)
        assert lists[i].model_version == 3


@pytest.mark.parametrize("case", ["huge", "tiny", "inf_row", "classifier_range"])
def test_score_many_data_scales(otf, case):
    """The FP16 form scales X by 2^ex (max |x| 2^ex in [2^14, 2^15), one pass per repository) and
    each classifier by its own 2^ew; extreme data magnitudes and non-finite data use the TF32 form.
    Finite rows stay within the bound either way."""
    rng = np.random.default_rng({"huge": 1, "tiny": 2, "inf_row": 3, "classifier_range": 4}[case])
    n, d, c = 700, 256, 9
    x = rng.standard_normal((n, d)).astype(np.float32)
    W = rng.standard_normal((c, d))
    if case == "huge":
        x *= np.float32(1e12)
    elif case == "tiny":
        x *= np.float32(1e-25)  # 2^ex out of the FP16 form's range -> TF32 form
    elif case == "inf_row":
        x[17, 3] = np.inf
    else:
        W *= 10.0 ** np.arange(-12, 15, 3)[:, None]
    repo = otf.Repository.dense(otf.FeatureStore(x))
    S = repo.score_many(list(W))
    ok = np.isfinite(x).all(axis=1)
    ex = exact(x[ok], W).T
    mag = np.abs(W.astype(np.float32).astype(np.float64)) @ np.abs(x[ok].astype(np.float64)).T
    assert np.all(np.abs(S[:, ok] - ex) <= 2.0 ** -20 * mag + np.spacing(np.abs(S[:, ok])) + 1e-30)
    if case == "inf_row":
        assert not np.all(np.isfinite(S[:, 17]))


@pytest.mark.parametrize("scale", [1e7, 1e-7, 30.0])
def test_score_many_mixed_row_magnitudes(otf, scale):
    """Normalised rows plus one outlier row (x 1e7: every other row is 1e-7 of the largest
    element; x 1e-7: one tiny row). The FP16 form's absolute error floor (~max|X| 2^-39.5 per
    element) would break the per-row reference tolerance, so the repository must pick the TF32
    form; a mild spread (x 30) keeps the FP16 form. Every row stays within 1e-6 |w| |x_row|."""
    rng = np.random.default_rng(int(scale * 1000) % 977)
    n, d, c = 2000, 512, 8
    x = rng.standard_normal((n, d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    x[123] *= np.float32(scale)
    W = rng.standard_normal((c, d))
    S = otf.Repository.dense(otf.FeatureStore(x)).score_many(list(W))
    ex = exact(x, W).T
    xn = np.linalg.norm(x.astype(np.float64), axis=1)
    for i in range(c):
        tol = 1e-6 * np.linalg.norm(W[i]) * xn
        err = np.abs(S[i].astype(np.float64) - ex[i])
        assert np.all(err <= 0.25 * tol + np.spacing(np.abs(S[i]))), (i, float(np.max(err / tol)))


def test_multi_errors(otf):
    repo = otf.Repository.dense(otf.FeatureStore(np.ones((10, 30), np.float32)))
    with pytest.raises(otf.ConfigError):
        repo.score_many([np.ones(30)])  # dim % 32 != 0
    repo2 = otf.Repository.dense(otf.FeatureStore(np.ones((10, 64), np.float32)))
    with pytest.raises(otf.ConfigError):
        repo2.score_many([np.ones(32)])


@pytest.mark.parametrize("n,d,c", [(1000, 128, 7), (300, 2048, 64)])
def test_single_cta_path_matches_pair_path(otf, monkeypatch, form, n, d, c):
    """The CTA-pair kernel (default) and the single-CTA kernel (inputs of one 128-row tile, forced
    here with OTF_MULTI_SINGLE) both meet the TF32x3 bound and agree with each other."""
    rng = np.random.default_rng(n * 7 + c)
    x = rng.standard_normal((n, d)).astype(np.float32)
    W = rng.standard_normal((c, d))
    repo = otf.Repository.dense(otf.FeatureStore(x))
    S_pair = repo.score_many(list(W))
    monkeypatch.setenv("OTF_MULTI_SINGLE", "1")
    S_single = repo.score_many(list(W))
    monkeypatch.delenv("OTF_MULTI_SINGLE")
    ex = exact(x, W).T
    mag = np.abs(W.astype(np.float32).astype(np.float64)) @ np.abs(x.astype(np.float64)).T
    for S in (S_pair, S_single):
        assert np.all(np.abs(S - ex) <= 2.0 ** -20 * mag + np.spacing(np.abs(S)) + 1e-30)
    assert np.all(np.abs(S_pair - S_single) <= 2.0 ** -19 * mag + 2 * np.spacing(np.abs(S_pair)) + 1e-30)


@pytest.mark.parametrize("n,d,c,k", [(50_000, 64, 64, 1000), (3000, 32, 40, 3000), (9000, 96, 5, 8500),
                                     (4000, 64, 70, 50), (600, 32, 130, 17),
                                     # larger segments (several gather passes per thread)
                                     (70_001, 32, 16, 500), (140_000, 64, 64, 2000)])
def test_rank_many_segmented_topk(otf, n, d, c, k):
    """rank_many selects all classifiers of a group in one segmented cooperative launch (two or
    more SMs per classifier); lists equal the oracle's top_k of the scores, including heavy ties
    (zero and constant classifiers -> the radix-select path), k > the 8192-candidate cap, k == n,
    and groups too large for one launch (per-classifier fallback; > 64 classifiers = 2 groups)."""
    rng = np.random.default_rng(n + c + k)
    x = np.round(rng.standard_normal((n, d)) * 4).astype(np.float32) / 4  # many exact ties
    ids = rng.permutation(4 * n)[:n].astype(np.int64)
    W = rng.standard_normal((c, d))
    W[0] = 0.0                 # all scores 0: one giant tie
    W[c // 2] = np.round(W[c // 2])
    repo = otf.Repository.dense(otf.FeatureStore(x, ids=ids))
    S = repo.score_many(list(W))
    lists = repo.rank_many([otf.LinearModel(w, 1, 1) for w in W], k)
    for i in range(c):
        o_ids, o_sc, _ = O.top_k(S[i], k, ids)
        np.testing.assert_array_equal(lists[i].ids, o_ids)
        np.testing.assert_array_equal(lists[i].scores, o_sc)
    # the single-classifier ranking of the same repository is unaffected (separate workspace)
    r1 = repo.rank(otf.LinearModel(W[1], 1, 1), k)
    assert len(r1.ids) == min(k, n)


@pytest.mark.parametrize("n,c", [(1001, 3), (5003, 64), (2, 5)])
def test_rank_many_unaligned_segments(otf, n, c):
    """Classifier-major score rows start at c * n floats: n not a multiple of 4 leaves them
    unaligned for the top-k's vector loads (they fall back to scalar loads)."""
    rng = np.random.default_rng(n + c)
    x = rng.standard_normal((n, 64)).astype(np.float32)
    W = rng.standard_normal((c, 64))
    repo = otf.Repository.dense(otf.FeatureStore(x))
    S = repo.score_many(list(W))
    k = min(n, 50)
    lists = repo.rank_many([otf.LinearModel(w, 1, 1) for w in W], k)
    for i in range(c):
        o_ids, o_sc, _ = O.top_k(S[i], k)
        np.testing.assert_array_equal(lists[i].ids, o_ids)
        np.testing.assert_array_equal(lists[i].scores, o_sc)


@pytest.mark.parametrize("n,c,k", [(1_100_003, 64, 1000), (1_048_576, 9, 1), (2_000_000, 33, 700)])
def test_rank_many_sampled_threshold(otf, n, c, k):
    """Segments of >= 1M rows take the sampled-threshold selection (topk_seg_cut_kernel: a sample
    per classifier, one emission pass, rank by counting): lists equal the oracle's top_k of the
    scores, with a zero classifier (every row reaches T -> that segment's exact radix select), a
    tie-heavy one, shuffled (and, for odd c, negative) ids and unaligned segment starts; a following k beyond the plan (the
    histogram path, same workspace) is unaffected."""
    rng = np.random.default_rng(n + c + k)
    x = np.round(rng.standard_normal((n, 64)) * 8).astype(np.float32) / 8
    ids = rng.permutation(2 * n)[:n].astype(np.int64) - (n if c % 2 else 0)  # (negative ids: the signed tie order)
    W = rng.standard_normal((c, 64))
    W[0] = 0.0
    W[c // 2] = np.round(W[c // 2])
    if c % 2:  # a duck-typed store (FeatureStore itself rejects negative ids, as the reference's does)
        store = type("Store", (), {"data": x, "ids": ids})()
        repo = otf.Repository.dense(store)
    else:
        repo = otf.Repository.dense(otf.FeatureStore(x, ids=ids))
    S = repo.score_many(list(W))
    for kk in (k, 3000):
        lists = repo.rank_many([otf.LinearModel(w, 1, 1) for w in W], kk)
        for i in range(c):
            o_ids, o_sc, _ = O.top_k(S[i], kk, ids)
            np.testing.assert_array_equal(lists[i].ids, o_ids)
            np.testing.assert_array_equal(lists[i].scores, o_sc)
