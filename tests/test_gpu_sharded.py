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


@pytest.mark.parametrize("n,d,k,offset", [(20_000, 128, 1000, 0), (700, 64, 1000, 5_000_000), (4096, 32, 1, 3)])
def test_native_nccl_group_single_rank(otf, n, d, k, offset):
    """The library's own NCCL group (otf_group_*: ncclBroadcast of w, local top-k, ncclAllGather,
    exact merge) on a one-rank communicator equals Repository.rank; rows come back global
    (row_offset added), shards smaller than k are padded and never selected. Multi-rank runs
    need one process per GPU (the driver's scaling run); the merge logic is the same
    top-k kernel the gloo-tested ShardedRepository uses."""
    torch = pytest.importorskip("torch")
    from paper_1407_4764_b200.distributed import NcclShardGroup

    rng = np.random.default_rng(n + k)
    x = rng.standard_normal((n, d)).astype(np.float32)
    ids = rng.permutation(3 * n)[:n].astype(np.int64)
    w = rng.standard_normal(d)
    repo = otf.Repository.dense(otf.FeatureStore(x, ids=ids))
    ref = repo.rank(otf.LinearModel(w, 1), k)
    g = NcclShardGroup(repo, NcclShardGroup.unique_id(), 1, 0, row_offset=offset, total_rows=n)
    got = g.rank(otf.LinearModel(w, 1), k)
    np.testing.assert_array_equal(got.ids, ref.ids)
    np.testing.assert_array_equal(got.scores, ref.scores)
    sc, i, rows = g.rank_device(torch.as_tensor(w, device="cuda"), k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(i.cpu().numpy(), ref.ids)
    np.testing.assert_array_equal(sc.cpu().numpy(), ref.scores)
    pos = {int(v): j for j, v in enumerate(ids)}
    np.testing.assert_array_equal(rows.cpu().numpy(), [pos[int(v)] + offset for v in ref.ids])
    g.close()
