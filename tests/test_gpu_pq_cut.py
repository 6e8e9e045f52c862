"""PQ cut path (pq_build_lut_kernel -> pq_rank_cut_kernel): large repositories,
M == 16. The scan emits only the rows that can reach a sampled threshold; the selection ranks
them or falls back to an exact select over every row. Every case must stay bit-identical to the
reference's arithmetic (oracle: build_score_lut + score_codes + top_k, pq.py:248-276,
ranker.py:97-143), on the fast path and on both fallbacks. Each test checks which branch ran
through otf_repo_cut_fallbacks."""

import ctypes as C

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu

N = 10_000_000  # the cut path applies for k <= ~1100 at this size (148 SMs)


def fallbacks(otf, repo):
    v = C.c_int64()
    otf._lib.check(otf._lib.load().otf_repo_cut_fallbacks(repo.handle, C.byref(v)))
    return v.value


def check(otf, repo, w, cents, codes, k, ids=None):
    r = repo.rank(otf.LinearModel(w, 1, 1), k)
    ref = O.score_pq(w, cents, codes)
    o_ids, o_sc, _ = O.top_k(ref, k, ids)
    np.testing.assert_array_equal(r.ids, o_ids)
    assert r.scores.tobytes() == np.asarray(o_sc, np.float64).tobytes()
    return r


@pytest.fixture(scope="module")
def data():
    rng = np.random.default_rng(77)
    cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
    codes = rng.integers(0, 256, (N, 16), dtype=np.uint8)
    return cents, codes


@pytest.mark.parametrize("k", [1, 37, 1000, 1050])
def test_cut_path_bit_exact(otf, data, k):
    cents, codes = data
    repo = otf.Repository.quantized(otf.PQCodebook(cents), codes)
    w = np.random.default_rng(k).standard_normal(128)
    f0 = fallbacks(otf, repo)
    check(otf, repo, w, cents, codes, k)
    check(otf, repo, w, cents, codes, k)  # repeatable: the cut workspace is clean after a query
    assert fallbacks(otf, repo) == f0  # the sampled threshold held


def test_cut_path_shuffled_ids_and_graph(otf, data):
    cents, codes = data
    ids = np.random.default_rng(3).permutation(2 * N)[:N].astype(np.int64) - N  # negative ids too
    repo = otf.Repository.quantized(otf.PQCodebook(cents), codes, ids=ids)
    w = np.random.default_rng(5).standard_normal(128) * 1e-3
    check(otf, repo, w, cents, codes, 1000, ids)
    assert fallbacks(otf, repo) == 0


def test_cut_fallback_all_tied(otf, data):
    """w = 0: every score is 0.0, every row reaches the threshold -> overflow -> exact select;
    ties break toward the smallest ids."""
    cents, codes = data
    repo = otf.Repository.quantized(otf.PQCodebook(cents), codes)
    r = check(otf, repo, np.zeros(128), cents, codes, 1000)
    assert list(r.ids) == list(range(1000))
    assert fallbacks(otf, repo) == 1


def test_cut_fallback_threshold_too_high(otf, data):
    """Adversarial layout: one sampled row per sample CTA (the first of its chunk) holds the best codes,
    so the sampled threshold sits in the top bin, which ~150 rows reach: fewer than k -> the
    selection must fall back and still return the exact top-k."""
    cents, codes0 = data
    codes = codes0.copy()
    w = np.random.default_rng(9).standard_normal(128)
    lut = O.build_score_lut(w, cents)
    best = np.argmax(lut, axis=1).astype(np.uint8)
    g = 148
    chunk = 512 * 4 * 2  # kCutChunkRows (otf_pq.cu: kCutScanThreads x kCutRows x kCutBatches)
    nchunks = -(-N // chunk)
    sampled = np.arange(g) * nchunks // g * chunk  # the first row of every CTA's first chunk (its sample)
    codes[sampled] = best
    repo = otf.Repository.quantized(otf.PQCodebook(cents), codes)
    f0 = fallbacks(otf, repo)
    check(otf, repo, w, cents, codes, 1000)
    # on a GPU with 148 SMs the sampled rows are exactly these, so the fallback must have run
    import torch

    if torch.cuda.get_device_properties(0).multi_processor_count == g:
        assert fallbacks(otf, repo) == f0 + 1


def test_cut_then_small_repository_paths_agree(otf, data):
    """The same rows ranked through the cut path (N rows) and through the bins path (a 1M-row
    prefix is below the cut threshold size) agree with the oracle on both."""
    cents, codes = data
    w = np.random.default_rng(11).standard_normal(128)
    small = codes[:1_000_000]
    repo_s = otf.Repository.quantized(otf.PQCodebook(cents), small)
    check(otf, repo_s, w, cents, small, 1000)
    assert fallbacks(otf, repo_s) == 0  # the bins path never touches the cut counters
