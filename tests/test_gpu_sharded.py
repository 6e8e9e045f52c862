"""The multi-GPU ranking path's device pieces on one GPU: several shards (separate repository
handles with global ids) -> GpuShardBackend.local_topk (padded) -> concatenation (what all_gather
produces) -> GpuShardBackend.merge_topk. The merged list must be bit-identical to ranking the
whole repository at once, for any number of shards, including shards smaller than k."""

import numpy as np
import pytest

import otf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,k,shards,kind", [(50_000, 128, 1000, 2, "rand"), (20_000, 256, 300, 8, "rand"),
                                               (3000, 64, 1000, 8, "ties"), (999, 32, 999, 3, "rand")])
def test_shards_merge_equals_single(otf, n, d, k, shards, kind):
    torch = pytest.importorskip("torch")
    from paper_1407_4764_b200.distributed import GpuShardBackend, shard_bounds

    rng = np.random.default_rng(n + shards)
    x = rng.standard_normal((n, d)).astype(np.float32)
    if kind == "ties":
        x = np.round(x)
    ids = rng.permutation(2 * n)[:n].astype(np.int64)
    w = rng.standard_normal(d)
    full = otf.Repository.dense(otf.FeatureStore(x, ids=ids)).rank(otf.LinearModel(w, 1), k)
    w_dev = torch.as_tensor(w, device="cuda")
    parts = []
    for r in range(shards):
        a, b = shard_bounds(n, shards, r)
        local = otf.Repository.dense(otf.FeatureStore(x[a:b], ids=ids[a:b]))
        be = GpuShardBackend(local, a)
        sc, i, rows = be.local_topk(w_dev, min(k, n))
        parts.append((sc.clone(), i.clone(), rows.clone()))
    sc = torch.cat([p[0] for p in parts])
    i = torch.cat([p[1] for p in parts])
    rows = torch.cat([p[2] for p in parts])
    m_sc, m_ids, m_rows = be.merge_topk(sc, i, rows, min(k, n))
    np.testing.assert_array_equal(m_ids.cpu().numpy(), full.ids)
    np.testing.assert_array_equal(m_sc.cpu().numpy(), full.scores)
    # global rows point back at the right ids
    np.testing.assert_array_equal(ids[m_rows.cpu().numpy()], full.ids)
