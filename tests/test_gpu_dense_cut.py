"""Dense cut path (dense_rank_cut): one cooperative kernel scores every row, samples a
threshold, emits only the rows that reach it and ranks those — or falls back to an exact radix
select over every row's score. The ranked list must be exactly the top-k (score desc, id asc,
ranker.py:97-143) of the SAME float32 scores the scoring kernel gives (`Repository.score`, one
shared per-row reduction), on the fast path and on the fallbacks; each test checks which branch
ran through otf_repo_cut_fallbacks. (Parity of those scores with the reference's sgemv is
tests/test_gpu_parity.py and tests/test_baseline_sizes.py.)"""

import ctypes as C

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


def fallbacks(otf, repo):
    v = C.c_int64()
    otf._lib.check(otf._lib.load().otf_repo_cut_fallbacks(repo.handle, C.byref(v)))
    return v.value


def rows(n, d, seed):
    x = np.random.default_rng(seed).standard_normal((n, d), dtype=np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x


def check(otf, repo, w, k, ids=None):
    model = otf.LinearModel(w, 1, 1)
    r = repo.rank(model, k)
    s = np.asarray(repo.score(model), np.float32)
    o_ids, o_sc, _ = O.top_k(s, k, ids)
    np.testing.assert_array_equal(r.ids, o_ids)
    assert r.scores.tobytes() == np.asarray(o_sc, np.float64).tobytes()
    return r


D, N, R = 256, 600_000, 4


@pytest.fixture(scope="module")
def c1_rows():
    return rows(N, D, 5)


@pytest.mark.parametrize("k", [1, 100, 1000, 1200])
def test_cut_path(otf, c1_rows, k):
    repo = otf.Repository.dense(c1_rows)
    w = np.random.default_rng(k).standard_normal(D)
    f0 = fallbacks(otf, repo)
    check(otf, repo, w, k)
    check(otf, repo, w, k)  # repeatable: the candidate counter is clean after a query
    assert fallbacks(otf, repo) == f0  # the sampled threshold held


@pytest.mark.parametrize("d,n", [(512, 200_000), (1024, 120_000), (2048, 100_000),
                                 (4096, 60_000)])
def test_cut_every_fast_width(otf, d, n):
    x = rows(n, d, d)
    repo = otf.Repository.dense(x)
    w = np.random.default_rng(d).standard_normal(d)
    check(otf, repo, w, 1000)
    check(otf, repo, w, 7)
    assert fallbacks(otf, repo) == 0


def test_cut_ids_negative_and_duplicate(otf, c1_rows):
    """Caller ids (shuffled, negative, some duplicated): ties in (score, id) resolve by row."""
    n = len(c1_rows)
    ids = np.random.default_rng(3).permutation(2 * n)[:n].astype(np.int64) - n
    ids[1::1000] = ids[0::1000][: len(ids[1::1000])]  # duplicate ids on some neighbouring rows
    x = c1_rows.copy()
    x[1::1000] = x[0::1000][: len(x[1::1000])]  # ... with identical rows (same score, same id)
    class Store:  # duck-typed store (the reference's ranker reads .data and .ids)
        data, ids = None, None

    st = Store()
    st.data, st.ids = x, ids
    repo = otf.Repository.dense(st)
    w = np.random.default_rng(4).standard_normal(D)
    r = check(otf, repo, w, 1000, ids)
    assert len(r.ids) == 1000


def test_cut_fallback_all_tied(otf, c1_rows):
    """w = 0: every score is 0.0, every row reaches T -> overflow -> exact select, smallest ids."""
    repo = otf.Repository.dense(c1_rows)
    f0 = fallbacks(otf, repo)
    r = check(otf, repo, np.zeros(D), 1000)
    assert list(r.ids) == list(range(1000))
    assert fallbacks(otf, repo) == f0 + 1


def test_cut_fallback_threshold_too_high(otf, c1_rows):
    """Adversarial layout: the first row of every warp's sample group scores far
    above the rest, so T lands among those ~2 400 planted rows and only ~r of them reach it:
    fewer than k -> the selection falls back and still returns the exact top-k."""
    import torch

    x = c1_rows.copy()
    n = len(x)
    w = np.random.default_rng(9).standard_normal(D)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nwarp = 2 * sms * 8
    gps = (-(-n // R)) // nwarp  # sample stride in R-row groups (dense_rank_cut)
    first = np.arange(nwarp) * gps * R
    first = first[first < n]
    x[first] = (w / np.linalg.norm(w)).astype(np.float32) * np.linspace(1.0, 0.9, len(first))[:, None].astype(np.float32)
    repo = otf.Repository.dense(x)
    f0 = fallbacks(otf, repo)
    check(otf, repo, w, 1000)
    if sms == 148:
        assert fallbacks(otf, repo) == f0 + 1


def test_cut_device_graph_and_large_k_agree(otf, c1_rows):
    """The device-memory graph replay (live ranker path) and a k beyond the cut's candidate cap
    (score kernel + top-k kernel) give the same list prefix."""
    import torch

    repo = otf.Repository.dense(c1_rows)
    w = np.random.default_rng(21).standard_normal(D)
    lib = otf._lib.load()
    dev = torch.device("cuda", 0)
    w_dev = torch.as_tensor(w, device=dev)
    k = 1000
    o_ids = torch.empty(k, dtype=torch.int64, device=dev)
    o_sc = torch.empty(k, dtype=torch.float64, device=dev)
    o_rows = torch.empty(k, dtype=torch.int64, device=dev)
    sp = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    for _ in range(3):
        otf._lib.check(lib.otf_repo_rank_graph(repo.handle, otf._lib.tptr(w_dev), k, otf._lib.tptr(o_ids),
                                               otf._lib.tptr(o_sc), otf._lib.tptr(o_rows), sp))
    torch.cuda.synchronize(dev)
    big = repo.rank(otf.LinearModel(w, 1, 1), 3000)  # no cut (2 k + 128 > cap / 2)
    np.testing.assert_array_equal(o_ids.cpu().numpy(), big.ids[:k])
    np.testing.assert_array_equal(o_rows.cpu().numpy(), big.ids[:k])
    assert o_sc.cpu().numpy().tobytes() == big.scores[:k].tobytes()
