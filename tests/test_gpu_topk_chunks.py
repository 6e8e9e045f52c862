"""Top-k through the chunk maxima (otf_topk.cu phase C'): repositories above ~4.8M rows, where the
gather reads the per-chunk maximum bins the scoring kernel wrote and scans only the chunks that
can hold a candidate. The selection must stay exactly the oracle's top_k (ranker.py:97-143) of
the GPU's own scores: heavy ties at the threshold bin spread over many chunks, a partial last
chunk, ids in shuffled order, k up to the 8192-candidate cap and beyond (radix-select fallback),
and all three chunk sizes (dense d=128: 32 rows — the two-kernel path for k beyond the fused
selection's cap, the fused dense_rank_cut below it —, binary 2048-bit: 32, PQ-16: 128).
"""

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu

N = 5_000_037  # > 32 x the top-k grid's threads, and not a multiple of any chunk size


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _check(repo, model, k, ids=None):
    s = repo.score(model.weights)
    r = repo.rank(model, k)
    o_ids, o_sc, _ = O.top_k(s, k, ids)
    np.testing.assert_array_equal(r.ids, o_ids)
    np.testing.assert_array_equal(r.scores, np.asarray(o_sc, np.float64))
    r2 = repo.rank(model, k)  # repeatable bit for bit
    assert r2.ids.tobytes() == r.ids.tobytes() and r2.scores.tobytes() == r.scores.tobytes()


@pytest.mark.parametrize("k", [1, 1000, 7000])
def test_dense_d128_chunks(otf, torch_cuda, k):
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(k)
    x = torch.randn((N, 128), device="cuda", generator=g)
    x = torch.round(x * 2) / 2  # coarse values: many exact score ties across chunks
    repo = otf.Repository.from_device("dense", x.data_ptr(), N, 128)
    w = np.round(np.random.default_rng(k).standard_normal(128))
    _check(repo, otf.LinearModel(w, 1, 1), k)


def test_dense_d128_chunks_shuffled_ids(otf, torch_cuda):
    torch = torch_cuda
    n = N
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((n, 128), device="cuda", generator=g)
    ids = np.random.default_rng(6).permutation(3 * n)[:n].astype(np.int64)
    repo = otf.Repository.from_device("dense", x.data_ptr(), n, 128, ids=ids)
    w = np.random.default_rng(7).standard_normal(128)
    _check(repo, otf.LinearModel(w, 1, 1), 2000, ids)


@pytest.mark.parametrize("k", [1000, 9000])
def test_binary_2048_chunks(otf, torch_cuda, k):
    torch = torch_cuda
    codes = torch.empty((N, 256), dtype=torch.uint8, device="cuda")
    codes.random_(0, 256, generator=torch.Generator(device="cuda").manual_seed(k))
    repo = otf.Repository.from_device("binary", codes.data_ptr(), N, 2048)
    w = np.where(np.random.default_rng(k).random(2048) < 0.5, -1.0, 1.0)  # integer scores: ties
    _check(repo, otf.LinearModel(w, 1, 1), k)


@pytest.mark.parametrize("k", [1000, 8192])
def test_pq16_chunks(otf, torch_cuda, k):
    torch = torch_cuda
    codes = torch.randint(0, 256, (N, 16), dtype=torch.uint8, device="cuda",
                          generator=torch.Generator(device="cuda").manual_seed(k))
    rng = np.random.default_rng(k)
    cents = (rng.integers(-4, 5, (16, 256, 8)) / 4.0).astype(np.float32)  # few distinct sums: ties
    w = np.zeros(128)
    w[::8] = 1.0
    repo = otf.Repository.from_device("pq", codes.data_ptr(), N, 16, codebook=otf.PQCodebook(cents))
    _check(repo, otf.LinearModel(w, 1, 1), k)
