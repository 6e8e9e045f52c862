"""The repository's cached CUDA graphs of rank (host-memory otf_repo_rank and otf_repo_rank_graph):
every replay must equal the oracle's top_k (ranker.py:97-143) while k changes, the top-k
workspace grows past the 8192-candidate layout (the graphs are keyed by every pointer they
touch), and host / device calls interleave."""

import ctypes as C

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["dense", "pq"])
def test_graph_cache_interleaved_k(otf, kind):
    torch = pytest.importorskip("torch")
    from paper_1407_4764_b200 import _lib

    rng = np.random.default_rng(3)
    n = 120_000
    if kind == "dense":
        x = rng.standard_normal((n, 64)).astype(np.float32)
        repo = otf.Repository.dense(otf.FeatureStore(x))
        w = rng.standard_normal(64)
    else:
        cents = rng.standard_normal((16, 256, 8)).astype(np.float32)
        repo = otf.Repository.quantized(otf.PQCodebook(cents), rng.integers(0, 256, (n, 16), dtype=np.uint8))
        w = rng.standard_normal(128)
    s = repo.score(w)
    lib = _lib.load()
    w_dev = torch.as_tensor(w, device="cuda")
    for k in [100, 20_000, 100, 50, 30_000, 9000, 100, 1]:
        r = repo.rank(otf.LinearModel(w, 1, 1), k)  # host memory: graph replay
        o_ids, o_sc, _ = O.top_k(s, k)
        np.testing.assert_array_equal(r.ids, o_ids)
        np.testing.assert_array_equal(r.scores, np.asarray(o_sc, np.float64))
        ids = torch.empty(k, dtype=torch.int64, device="cuda")
        sc = torch.empty(k, dtype=torch.float64, device="cuda")
        rows = torch.empty(k, dtype=torch.int64, device="cuda")
        st = torch.cuda.current_stream()
        _lib.check(lib.otf_repo_rank_graph(repo.handle, _lib.tptr(w_dev), k, _lib.tptr(ids), _lib.tptr(sc),
                                           _lib.tptr(rows), C.c_void_p(st.cuda_stream)))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ids.cpu().numpy(), o_ids)
        np.testing.assert_array_equal(sc.cpu().numpy(), np.asarray(o_sc, np.float64))
